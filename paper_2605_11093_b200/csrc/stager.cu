// stager.cu — staging engine: drains published ring regions to a pinned
// host ring and pages them out (exporter.py:1-303 restated for a real GPU).
//
//   thresholds_met      exporter.py:166-178  ANY of entries / bytes / age
//   drain_once          exporter.py:182-228  ready descriptors that fit one
//                                            pinned buffer, one batched D2H
//   complete_transfer   exporter.py:230-233  release regions after the copy
//   stage_to_pageable   exporter.py:237-249  buffer back to the pool first
//   run_threaded shape  wallclock.py:136-181 drain + stage threads, bounded
//                                            hand-off queue (STAGE_QUEUE_SLOTS)
//
// Two D2H engines (north star): TF_STAGE_COPY_ENGINE issues one
// cudaMemcpyAsync per contiguous run of ring bytes on a private non-blocking
// stream fenced by events; TF_STAGE_MAPPED launches a small kernel that
// stores into the mapped pinned buffer from the SMs.
#include <cuda_runtime.h>
#include <pthread.h>
#include <sched.h>
#include <sys/mman.h>
#include <sys/syscall.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <functional>
#include <map>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "ring2_internal.h"


#define CUDA_TRY(expr)                                                      \
  do {                                                                      \
    cudaError_t _e = (expr);                                                \
    if (_e != cudaSuccess) {                                                \
      tf_set_error("%s: %s (%s:%d)", #expr, cudaGetErrorString(_e),         \
                   __FILE__, __LINE__);                                     \
      return TF_ERR_CUDA;                                                   \
    }                                                                       \
  } while (0)

namespace {

// ---------------------------------------------------------------------------
// mapped-store D2H kernel: SM stores into pinned host memory over PCIe
// ---------------------------------------------------------------------------
constexpr int kMapMaxEntries = 48;
struct MapCopyArgs {
  int n;
  const uint8_t* src[kMapMaxEntries];
  uint8_t* dst[kMapMaxEntries];
  uint64_t len[kMapMaxEntries];
  uint64_t prefix[kMapMaxEntries + 1];  // byte prefix over entries
};

__global__ void __launch_bounds__(256) mapped_copy_kernel(MapCopyArgs a) {
  // Each CTA walks its share of the batch in 16-B words where both sides
  // are aligned, bytes otherwise.
  const uint64_t total = a.prefix[a.n];
  const uint64_t per = (total + gridDim.x - 1) / gridDim.x;
  uint64_t b0 = min(total, (uint64_t)blockIdx.x * per);
  const uint64_t b1 = min(total, b0 + per);
  int e = 0;
  while (e < a.n && a.prefix[e + 1] <= b0) ++e;
  while (b0 < b1 && e < a.n) {
    const uint64_t seg_end = min(b1, a.prefix[e + 1]);
    const uint64_t o0 = b0 - a.prefix[e], o1 = seg_end - a.prefix[e];
    const uint8_t* s = a.src[e];
    uint8_t* d = a.dst[e];
    const bool vec = (((uintptr_t)(s + o0) | (uintptr_t)(d + o0)) & 15) == 0;
    uint64_t o = o0;
    if (vec) {
      const uint64_t nw = (o1 - o0) / 16;
      const uint4* s4 = reinterpret_cast<const uint4*>(s + o0);
      uint4* d4 = reinterpret_cast<uint4*>(d + o0);
      for (uint64_t w = threadIdx.x; w < nw; w += blockDim.x) {
        uint4 v;
        asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(s4 + w));
        d4[w] = v;
      }
      o = o0 + nw * 16;
    }
    for (uint64_t k = o + threadIdx.x; k < o1; k += blockDim.x) d[k] = s[k];
    b0 = seg_end;
    ++e;
  }
}

// ---------------------------------------------------------------------------
// helpers
// ---------------------------------------------------------------------------
std::vector<int> parse_cpulist(const char* s) {
  std::vector<int> out;
  while (*s) {
    char* end;
    long a = strtol(s, &end, 10);
    if (end == s) break;
    long b = a;
    s = end;
    if (*s == '-') {
      b = strtol(s + 1, &end, 10);
      s = end;
    }
    for (long c = a; c <= b; ++c) out.push_back((int)c);
    if (*s == ',') ++s;
    else if (*s == '\n') break;
  }
  return out;
}

// CPUs local to the GPU's PCIe root (NUMA placement of staging threads)
std::vector<int> gpu_local_cpus(int device) {
  std::vector<int> cpus;
  char bus[64] = {0};
  if (cudaDeviceGetPCIBusId(bus, sizeof(bus), device) != cudaSuccess) {
    cudaGetLastError();
    return cpus;
  }
  for (char* p = bus; *p; ++p) *p = (char)tolower(*p);
  char path[256];
  snprintf(path, sizeof(path), "/sys/bus/pci/devices/%s/local_cpulist", bus);
  FILE* f = fopen(path, "r");
  if (!f) return cpus;
  char buf[4096] = {0};
  if (fgets(buf, sizeof(buf), f)) cpus = parse_cpulist(buf);
  fclose(f);
  // keep only CPUs we are allowed to run on
  cpu_set_t allowed;
  if (sched_getaffinity(0, sizeof(allowed), &allowed) == 0) {
    std::vector<int> ok;
    for (int c : cpus)
      if (c < CPU_SETSIZE && CPU_ISSET(c, &allowed)) ok.push_back(c);
    cpus = ok;
  }
  return cpus;
}

void bind_thread(const std::vector<int>& cpus) {
  if (cpus.empty()) return;
  cpu_set_t set;
  CPU_ZERO(&set);
  for (int c : cpus) CPU_SET(c, &set);
  pthread_setaffinity_np(pthread_self(), sizeof(set), &set);
}

inline void cpu_relax() {
#if defined(__x86_64__)
  __builtin_ia32_pause();
#endif
}

// Persistent workers for the pinned -> pageable copy of large batches.
class CopyPool {
 public:
  void start(int n, const std::vector<int>& cpus) {
    stop_ = false;
    for (int i = 0; i < n; ++i)
      th_.emplace_back([this, cpus] {
        bind_thread(cpus);
        loop();
      });
  }
  void stop() {
    {
      std::lock_guard<std::mutex> g(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : th_) t.join();
    th_.clear();
  }
  // parallel memcpy; the caller thread takes one share
  void copy(uint8_t* dst, const uint8_t* src, uint64_t n) {
    const uint64_t min_chunk = 4ull << 20;
    size_t parts = th_.size() + 1;
    if (n < 2 * min_chunk || th_.empty()) {
      memcpy(dst, src, n);
      return;
    }
    parts = std::min<size_t>(parts, (size_t)(n / min_chunk));
    uint64_t per = ((n + parts - 1) / parts + 4095) & ~uint64_t(4095);
    std::atomic<int> left{0};
    {
      std::lock_guard<std::mutex> g(mu_);
      for (size_t p = 1; p < parts; ++p) {
        uint64_t a = p * per;
        if (a >= n) break;
        uint64_t b = std::min(n, a + per);
        left.fetch_add(1);
        jobs_.push_back([=, &left] {
          memcpy(dst + a, src + a, b - a);
          left.fetch_sub(1, std::memory_order_release);
        });
      }
    }
    cv_.notify_all();
    memcpy(dst, src, std::min(n, per));
    while (left.load(std::memory_order_acquire) > 0) cpu_relax();
  }

 private:
  void loop() {
    for (;;) {
      std::function<void()> job;
      {
        std::unique_lock<std::mutex> g(mu_);
        cv_.wait(g, [&] { return stop_ || !jobs_.empty(); });
        if (stop_ && jobs_.empty()) return;
        job = std::move(jobs_.front());
        jobs_.pop_front();
      }
      job();
    }
  }
  std::vector<std::thread> th_;
  std::mutex mu_;
  std::condition_variable cv_;
  std::deque<std::function<void()>> jobs_;
  bool stop_ = false;
};

}  // namespace

// ---------------------------------------------------------------------------
// stager state
// ---------------------------------------------------------------------------
struct Batch {
  uint64_t id = 0;
  uint32_t buf = 0;
  // a split (oversize) capture: its chunks' pool buffers in order (buf is
  // the first); empty for an ordinary batch
  std::vector<uint32_t> chunk_bufs;
  uint32_t reason = 0;
  std::vector<tf_descriptor> descs;
  std::vector<uint64_t> starts;
  uint64_t bytes = 0;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  bool transferred = false;  // D2H known complete
  bool released = false;     // payload regions released
  double transfer_s = 0;
};

struct tf_stager {
  tf_ring* ring = nullptr;
  tf_drain_config cfg{};
  int device = 0;
  cudaStream_t stream = nullptr;
  std::vector<uint8_t*> bufs;
  std::vector<uint32_t> free_bufs;
  std::vector<cudaEvent_t> event_pool;
  std::mutex mu;  // stager state
  std::condition_variable cv;
  std::map<uint64_t, Batch*> batches;
  uint64_t next_id = 1;
  std::deque<double> pending_times;  // note_publish (exporter.py:158-164)
  tf_stager_stats stats{};
  uint64_t pageable_in_flight = 0;
  int sm_count = 148;
  std::vector<int> cpus;
  // background engine
  std::atomic<bool> running{false};
  std::atomic<bool> stop_req{false};
  std::atomic<int> flush_req{0};
  std::thread drain_th, completion_th, stage_th;
  std::atomic<bool> drain_done{false}, completion_done{false};
  std::deque<Batch*> inflight;
  std::deque<Batch*> to_stage;
  std::deque<tf_paged_batch> out_q;
  std::vector<uint8_t*> paged_pool;
  // page-out buffers of split (oversize) captures, kept for reuse: a fresh
  // allocation of hundreds of MiB pays its page faults inside the copy
  std::multimap<uint64_t, uint8_t*> oversize_pool;   // capacity -> buffer
  std::map<uint8_t*, uint64_t> oversize_cap;         // buffer -> capacity
  uint32_t outstanding_paged = 0;
  uint64_t outstanding_handoff = 0;  // pinned buffers held by the consumer
  uint64_t max_split_bufs = 0;       // most chunk buffers one split capture took
  uint64_t pageable_budget = 0;      // paged-out bytes the stage thread may run ahead by
  std::atomic<int> bg_error{0};
  std::atomic<uint32_t> completion_phase{0}, stage_phase{0};  // diagnostics
  std::string bg_errmsg;
  CopyPool copy_pool;
};

static cudaEvent_t take_event(tf_stager* st) {
  if (!st->event_pool.empty()) {
    cudaEvent_t e = st->event_pool.back();
    st->event_pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreateWithFlags(&e, cudaEventBlockingSync);
  return e;
}

static void note_transient(tf_stager* st) {  // exporter.py:251-254
  uint64_t pinned = uint64_t(st->bufs.size() - st->free_bufs.size()) * st->cfg.staging_buffer_size;
  uint64_t t = pinned + st->pageable_in_flight;
  if (t > st->stats.max_transient_bytes) st->stats.max_transient_bytes = t;
  st->stats.pageable_bytes_in_flight = st->pageable_in_flight;
}

extern "C" int tf_stager_create(tf_ring* ring, const tf_drain_config* cfg, tf_stager** out) {
  if (!ring || !cfg || !out) return TF_ERR_VALUE;
  // exporter.py:45-51
  if (cfg->min_ready_entries == 0 || cfg->min_ready_bytes == 0) {
    tf_set_error("ready thresholds must be positive");
    return TF_ERR_CONFIG;
  }
  if (!(cfg->max_wait > 0)) { tf_set_error("max_wait must be positive"); return TF_ERR_CONFIG; }
  if (cfg->staging_buffer_size == 0 || cfg->staging_buffer_count == 0) {
    tf_set_error("staging pool sizing must be positive");
    return TF_ERR_CONFIG;
  }
  if (cfg->mode > TF_STAGE_MAPPED) { tf_set_error("unknown staging mode"); return TF_ERR_CONFIG; }
  tf_stager* st = new tf_stager();
  st->ring = ring;
  st->cfg = *cfg;
  if (!st->cfg.stage_queue_slots) st->cfg.stage_queue_slots = 16;  // exporter.py:32
  st->pageable_budget = uint64_t(32) << 30;
  if (const char* e = getenv("TF_PAGEABLE_BUDGET_MIB")) st->pageable_budget = strtoull(e, nullptr, 10) << 20;
  st->device = ring->device;
  if (cudaSetDevice(st->device) != cudaSuccess) {
    delete st;
    tf_set_error("cudaSetDevice failed");
    return TF_ERR_CUDA;
  }
  cudaDeviceGetAttribute(&st->sm_count, cudaDevAttrMultiProcessorCount, st->device);
  {  // load the staging kernel now, not lazily at its first launch (ring2.cu preload_kernels)
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, mapped_copy_kernel);
    cudaGetLastError();
  }
  st->cpus = gpu_local_cpus(st->device);
  if (cfg->numa_node == -2) st->cpus.clear();  // explicit opt-out
  // allocate the pinned pool from a thread bound near the GPU (first touch)
  int rc = TF_OK;
  std::thread alloc([&] {
    bind_thread(st->cpus);
    cudaSetDevice(st->device);
    for (uint64_t i = 0; i < cfg->staging_buffer_count; ++i) {
      uint8_t* p = nullptr;
      cudaError_t e = cudaHostAlloc((void**)&p, cfg->staging_buffer_size,
                                    cudaHostAllocMapped | cudaHostAllocPortable);
      if (e != cudaSuccess) {
        tf_set_error("pinned staging allocation failed: %s", cudaGetErrorString(e));
        cudaGetLastError();
        rc = TF_ERR_ALLOCATION;
        return;
      }
      memset(p, 0, cfg->staging_buffer_size);
      st->bufs.push_back(p);
    }
    if (cudaStreamCreateWithFlags(&st->stream, cudaStreamNonBlocking) != cudaSuccess) rc = TF_ERR_CUDA;
  });
  alloc.join();
  if (rc) {
    for (auto p : st->bufs) cudaFreeHost(p);
    delete st;
    return rc;
  }
  for (uint32_t i = (uint32_t)st->bufs.size(); i > 0; --i) st->free_bufs.push_back(i - 1);
  *out = st;
  return TF_OK;
}

static void free_paged_batch(tf_stager* st, tf_paged_batch* b, bool to_pool);

extern "C" int tf_stager_stop(tf_stager* st);

extern "C" int tf_stager_destroy(tf_stager* st) {
  if (!st) return TF_OK;
  tf_stager_stop(st);
  cudaSetDevice(st->device);
  if (st->stream) cudaStreamSynchronize(st->stream);
  for (auto& kv : st->batches) {
    Batch* b = kv.second;
    if (b->ev0) cudaEventDestroy(b->ev0);
    if (b->ev1) cudaEventDestroy(b->ev1);
    delete b;
  }
  for (auto& pb : st->out_q) free_paged_batch(st, &pb, false);
  for (auto e : st->event_pool) cudaEventDestroy(e);
  for (auto p : st->bufs) cudaFreeHost(p);
  for (auto p : st->paged_pool) free(p);
  for (auto& kv : st->oversize_pool) free(kv.second);
  if (st->stream) cudaStreamDestroy(st->stream);
  delete st;
  return TF_OK;
}

// ---------------------------------------------------------------------------
// thresholds (exporter.py:166-178)
// ---------------------------------------------------------------------------
static uint32_t reason_for(tf_stager* st, uint64_t entries, uint64_t bytes,
                           double oldest_age) {
  if (entries == 0) return TF_REASON_NONE;
  if (entries >= st->cfg.min_ready_entries) return TF_REASON_ENTRIES;
  if (bytes >= st->cfg.min_ready_bytes) return TF_REASON_BYTES;
  if (oldest_age >= 0 && oldest_age >= st->cfg.max_wait - 1e-12) return TF_REASON_TIMEOUT;
  return TF_REASON_NONE;
}

static void ready_summary(tf_stager* st, std::vector<tf_descriptor>& tmp, uint32_t* n, uint64_t* bytes) {
  tmp.resize(st->ring->cfg.meta_slots);
  tf_ring_peek_ready(st->ring, (uint32_t)tmp.size(), tmp.data(), n);
  uint64_t b = 0;
  for (uint32_t i = 0; i < *n; ++i) b += tmp[i].payload_len;
  *bytes = b;
}

// Pool buffers the next batch needs: 1, or ceil(len / buffer) for an
// oversize head capture when splitting is enabled.
static uint64_t bufs_needed(const tf_stager* st, const tf_descriptor* head) {
  const uint64_t cap = st->cfg.staging_buffer_size;
  if (!st->cfg.split_oversize || head->payload_len <= cap) return 1;
  return (head->payload_len + cap - 1) / cap;
}

extern "C" int tf_stager_note_publish(tf_stager* st, double now) {
  if (!st) return TF_ERR_VALUE;
  std::lock_guard<std::mutex> g(st->mu);
  st->pending_times.push_back(now);
  return TF_OK;
}

extern "C" int tf_stager_thresholds_met(tf_stager* st, double now, uint32_t* reason) {
  if (!st || !reason) return TF_ERR_VALUE;
  std::vector<tf_descriptor> tmp;
  uint32_t n;
  uint64_t bytes;
  ready_summary(st, tmp, &n, &bytes);
  std::lock_guard<std::mutex> g(st->mu);
  double age = st->pending_times.empty() ? -1.0 : now - st->pending_times.front();
  *reason = reason_for(st, n, bytes, age);
  return TF_OK;
}

// ---------------------------------------------------------------------------
// drain (exporter.py:182-228)
// ---------------------------------------------------------------------------
// Caller holds st->mu. Takes ready descriptors (in order) that fit one
// buffer, polls them, and enqueues the D2H. *out == nullptr if nothing ready.
static int issue_batch(tf_stager* st, uint32_t reason, Batch** out) {
  *out = nullptr;
  std::vector<tf_descriptor> ready(st->ring->cfg.meta_slots);
  uint32_t n = 0;
  int rc = tf_ring_peek_ready(st->ring, (uint32_t)ready.size(), ready.data(), &n);
  if (rc) return rc;
  if (n == 0) return TF_OK;
  if (st->free_bufs.empty()) {
    tf_set_error("all staging buffers are in flight");
    return TF_ERR_STAGING_EXHAUSTED;
  }
  const uint64_t cap = st->cfg.staging_buffer_size;
  uint32_t take = 0;
  uint64_t used = 0;
  std::vector<uint64_t> starts;
  std::vector<uint32_t> chunk_bufs;
  if (ready[0].payload_len > cap) {
    // exporter.py:197-202: the reference rejects a capture no buffer can
    // hold; with split_oversize it is staged alone, in buffer-sized chunks
    const uint64_t k = bufs_needed(st, &ready[0]);
    if (!st->cfg.split_oversize || k > st->bufs.size()) {
      tf_set_error("capture of %llu bytes exceeds the staging buffer (%llu bytes)%s",
                   (unsigned long long)ready[0].payload_len, (unsigned long long)cap,
                   st->cfg.split_oversize ? " x the whole pool" : "");
      return TF_ERR_CONFIG;
    }
    if (st->free_bufs.size() < k) {
      tf_set_error("a split capture needs %llu staging buffers, %zu free",
                   (unsigned long long)k, st->free_bufs.size());
      return TF_ERR_STAGING_EXHAUSTED;
    }
    st->max_split_bufs = std::max<uint64_t>(st->max_split_bufs, k);
    for (uint64_t c = 0; c < k; ++c) {
      chunk_bufs.push_back(st->free_bufs.back());
      st->free_bufs.pop_back();
    }
    starts.push_back(0);
    used = ready[0].payload_len;
    take = 1;
  } else {
    for (uint32_t i = 0; i < n; ++i) {
      if (used + ready[i].payload_len > cap) break;
      starts.push_back(used);
      used += ready[i].payload_len;
      ++take;
    }
  }
  uint32_t b;
  if (chunk_bufs.empty()) {
    b = st->free_bufs.back();
    st->free_bufs.pop_back();
  } else {
    b = chunk_bufs[0];
  }
  st->stats.pool_checkouts += chunk_bufs.empty() ? 1 : chunk_bufs.size();
  uint64_t in_use = st->bufs.size() - st->free_bufs.size();
  if (in_use > st->stats.pool_max_in_use) st->stats.pool_max_in_use = in_use;

  std::vector<tf_descriptor> got(take);
  uint32_t polled = 0;
  rc = tf_ring_poll_ready(st->ring, take, got.data(), &polled);
  if (rc || polled != take) {
    if (chunk_bufs.empty()) st->free_bufs.push_back(b);
    for (uint32_t c : chunk_bufs) st->free_bufs.push_back(c);
    if (!rc) {
      tf_set_error("ready window shrank under the drain");
      rc = TF_ERR_PROTOCOL;
    }
    return rc;
  }
  Batch* bt = new Batch();
  bt->id = st->next_id++;
  bt->buf = b;
  bt->chunk_bufs = chunk_bufs;
  bt->reason = reason;
  bt->descs = got;
  bt->starts = starts;
  bt->bytes = used;
  bt->ev0 = take_event(st);
  bt->ev1 = take_event(st);
  cudaSetDevice(st->device);
  cudaEventRecord(bt->ev0, st->stream);
  uint8_t* host = st->bufs[b];
  const uint8_t* payload = st->ring->payload;
  if (!chunk_bufs.empty()) {
    // one oversize capture: chunk c of its (contiguous) ring region into
    // pool buffer chunk_bufs[c]
    const uint64_t src = got[0].payload_offset, len = got[0].payload_len;
    if (st->cfg.mode == TF_STAGE_COPY_ENGINE) {
      for (size_t c = 0; c < chunk_bufs.size(); ++c) {
        const uint64_t a = c * cap, l = std::min(cap, len - a);
        cudaError_t e = cudaMemcpyAsync(st->bufs[chunk_bufs[c]], payload + src + a, l,
                                        cudaMemcpyDeviceToHost, st->stream);
        if (e != cudaSuccess) {
          tf_set_error("D2H issue failed: %s", cudaGetErrorString(e));
          return TF_ERR_CUDA;
        }
      }
    } else {
      size_t c = 0;
      while (c < chunk_bufs.size()) {
        MapCopyArgs a;
        a.n = 0;
        a.prefix[0] = 0;
        uint64_t bytes = 0;
        for (; c < chunk_bufs.size() && a.n < kMapMaxEntries; ++c) {
          const uint64_t o = c * cap, l = std::min(cap, len - o);
          a.src[a.n] = payload + src + o;
          a.dst[a.n] = st->bufs[chunk_bufs[c]];
          a.len[a.n] = l;
          bytes += l;
          a.prefix[a.n + 1] = bytes;
          ++a.n;
        }
        int ctas = st->cfg.mapped_ctas ? (int)st->cfg.mapped_ctas : 32;
        ctas = (int)std::max<uint64_t>(1, std::min<uint64_t>((uint64_t)ctas, (bytes + 65535) / 65536));
        mapped_copy_kernel<<<ctas, 256, 0, st->stream>>>(a);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) {
          tf_set_error("mapped copy launch failed: %s", cudaGetErrorString(e));
          return TF_ERR_CUDA;
        }
      }
    }
  } else if (st->cfg.mode == TF_STAGE_COPY_ENGINE) {
    // merge runs that are adjacent in the ring and in the buffer
    uint32_t i = 0;
    while (i < take) {
      uint64_t src = got[i].payload_offset, dst = starts[i], len = got[i].payload_len;
      uint32_t j = i + 1;
      while (j < take && got[j - 1].payload_len % TF_COPY_UNIT == 0 &&
             got[j].payload_offset == src + len && got[j].skip_before == 0) {
        len += got[j].payload_len;
        ++j;
      }
      cudaError_t e = cudaMemcpyAsync(host + dst, payload + src, len, cudaMemcpyDeviceToHost, st->stream);
      if (e != cudaSuccess) {
        tf_set_error("D2H issue failed: %s", cudaGetErrorString(e));
        return TF_ERR_CUDA;
      }
      i = j;
    }
  } else {
    uint32_t i = 0;
    while (i < take) {
      MapCopyArgs a;
      a.n = 0;
      a.prefix[0] = 0;
      uint64_t bytes = 0;
      while (i < take && a.n < kMapMaxEntries) {
        a.src[a.n] = payload + got[i].payload_offset;
        a.dst[a.n] = host + starts[i];
        a.len[a.n] = got[i].payload_len;
        bytes += got[i].payload_len;
        a.prefix[a.n + 1] = bytes;
        ++a.n;
        ++i;
      }
      int ctas = st->cfg.mapped_ctas ? (int)st->cfg.mapped_ctas : 32;
      ctas = (int)std::max<uint64_t>(1, std::min<uint64_t>((uint64_t)ctas, (bytes + 65535) / 65536));
      mapped_copy_kernel<<<ctas, 256, 0, st->stream>>>(a);
      cudaError_t e = cudaGetLastError();
      if (e != cudaSuccess) {
        tf_set_error("mapped copy launch failed: %s", cudaGetErrorString(e));
        return TF_ERR_CUDA;
      }
    }
  }
  // Free the regions for the device producer as soon as the copy is done:
  // a stream-ordered write of the release cursor right behind the D2H, so
  // the capture kernel sees space without a host round trip.
  int wrc = tf_internal_write_u64(st->stream, &st->ring->dcons->L,
                                  tf_internal_l_after_all(st->ring));
  if (wrc) return wrc;
  cudaEventRecord(bt->ev1, st->stream);
  st->batches[bt->id] = bt;
  st->stats.batches_drained += 1;
  st->stats.entries_drained += take;
  st->stats.bytes_drained += used;
  if (st->stats.first_drain_time == 0) st->stats.first_drain_time = tf_monotonic();
  *out = bt;
  return TF_OK;
}

extern "C" int tf_stager_drain_once(tf_stager* st, double now, int flush, tf_batch_info* out) {
  if (!st || !out) return TF_ERR_VALUE;
  if (st->running) { tf_set_error("background engine running"); return TF_ERR_PROTOCOL; }
  memset(out, 0, sizeof(*out));
  uint32_t reason = TF_REASON_FLUSH;
  if (!flush) {
    int rc = tf_stager_thresholds_met(st, now, &reason);
    if (rc) return rc;
  }
  if (reason == TF_REASON_NONE) return TF_OK;
  std::lock_guard<std::mutex> g(st->mu);
  Batch* b = nullptr;
  int rc = issue_batch(st, reason, &b);
  if (rc) return rc;
  if (!b) return TF_OK;
  size_t k = std::min(st->pending_times.size(), b->descs.size());
  st->pending_times.erase(st->pending_times.begin(), st->pending_times.begin() + k);
  out->batch_id = b->id;
  out->n_entries = (uint32_t)b->descs.size();
  out->buffer_index = b->buf;
  out->bytes_total = b->bytes;
  out->reason = reason;
  return TF_OK;
}

static Batch* find_batch(tf_stager* st, uint64_t id) {
  auto it = st->batches.find(id);
  if (it == st->batches.end()) {
    tf_set_error("unknown batch %llu", (unsigned long long)id);
    return nullptr;
  }
  return it->second;
}

extern "C" int tf_stager_batch_entries(tf_stager* st, uint64_t id, tf_descriptor* descs,
                                       uint64_t* starts, uint32_t max_entries) {
  if (!st) return TF_ERR_VALUE;
  std::lock_guard<std::mutex> g(st->mu);
  Batch* b = find_batch(st, id);
  if (!b) return TF_ERR_VALUE;
  for (uint32_t i = 0; i < b->descs.size() && i < max_entries; ++i) {
    if (descs) descs[i] = b->descs[i];
    if (starts) starts[i] = b->starts[i];
  }
  return TF_OK;
}

static int wait_transfer(tf_stager* st, Batch* b) {
  if (b->transferred) return TF_OK;
  cudaSetDevice(st->device);
  CUDA_TRY(cudaEventSynchronize(b->ev1));
  float ms = 0;
  cudaEventElapsedTime(&ms, b->ev0, b->ev1);
  b->transfer_s = ms * 1e-3;
  st->stats.transfer_seconds += b->transfer_s;
  b->transferred = true;
  return TF_OK;
}

extern "C" int tf_stager_batch_buffer(tf_stager* st, uint64_t id, void** host_ptr) {
  if (!st || !host_ptr) return TF_ERR_VALUE;
  std::lock_guard<std::mutex> g(st->mu);
  Batch* b = find_batch(st, id);
  if (!b) return TF_ERR_VALUE;
  if (!b->chunk_bufs.empty()) {
    tf_set_error("a split capture has no single staging buffer; use stage_to_pageable");
    return TF_ERR_PROTOCOL;
  }
  int rc = wait_transfer(st, b);
  if (rc) return rc;
  *host_ptr = st->bufs[b->buf];
  return TF_OK;
}

extern "C" int tf_stager_transfer_seconds(tf_stager* st, uint64_t id, double* seconds) {
  if (!st || !seconds) return TF_ERR_VALUE;
  std::lock_guard<std::mutex> g(st->mu);
  Batch* b = find_batch(st, id);
  if (!b) return TF_ERR_VALUE;
  int rc = wait_transfer(st, b);
  *seconds = b->transfer_s;
  return rc;
}

static int release_batch(tf_stager* st, Batch* b) {
  if (b->released) return TF_OK;
  for (auto& d : b->descs) {
    int rc = tf_internal_release(st->ring, d.payload_offset, tf_round_up16(d.payload_len), false);
    if (rc) return rc;
  }
  b->released = true;
  st->stats.last_release_time = tf_monotonic();
  return TF_OK;
}

extern "C" int tf_stager_complete_transfer(tf_stager* st, uint64_t id, double* seconds) {
  if (!st) return TF_ERR_VALUE;
  std::lock_guard<std::mutex> g(st->mu);
  Batch* b = find_batch(st, id);
  if (!b) return TF_ERR_VALUE;
  int rc = wait_transfer(st, b);
  if (rc) return rc;
  rc = release_batch(st, b);
  if (seconds) *seconds = b->transfer_s;
  return rc;
}

static void retire_batch(tf_stager* st, Batch* b, bool return_buffer = true) {
  if (!b->chunk_bufs.empty()) {
    for (uint32_t c : b->chunk_bufs) st->free_bufs.push_back(c);
  } else if (return_buffer) {
    st->free_bufs.push_back(b->buf);
  }
  st->event_pool.push_back(b->ev0);
  st->event_pool.push_back(b->ev1);
  st->batches.erase(b->id);
  delete b;
}

// The batch's bytes from its pinned buffer(s) into dst (bytes long).
static void gather_chunks(tf_stager* st, Batch* b, uint8_t* dst, bool parallel) {
  const uint64_t cap = st->cfg.staging_buffer_size;
  if (b->chunk_bufs.empty()) {
    if (parallel) st->copy_pool.copy(dst, st->bufs[b->buf], b->bytes);
    else memcpy(dst, st->bufs[b->buf], b->bytes);
    return;
  }
  for (size_t c = 0; c < b->chunk_bufs.size(); ++c) {
    const uint64_t a = c * cap, l = std::min(cap, b->bytes - a);
    if (parallel) st->copy_pool.copy(dst + a, st->bufs[b->chunk_bufs[c]], l);
    else memcpy(dst + a, st->bufs[b->chunk_bufs[c]], l);
  }
}

extern "C" int tf_stager_stage_to_pageable(tf_stager* st, uint64_t id, void* dst, uint64_t cap) {
  if (!st) return TF_ERR_VALUE;
  std::lock_guard<std::mutex> g(st->mu);
  Batch* b = find_batch(st, id);
  if (!b) return TF_ERR_VALUE;
  if (cap < b->bytes || (b->bytes && !dst)) { tf_set_error("pageable destination too small"); return TF_ERR_VALUE; }
  int rc = wait_transfer(st, b);
  if (rc) return rc;
  if (b->bytes) gather_chunks(st, b, (uint8_t*)dst, false);
  st->pageable_in_flight += b->bytes;
  st->stats.batches_staged += 1;
  retire_batch(st, b);  // buffer returns to the pool before anything downstream
  note_transient(st);
  st->cv.notify_all();
  return TF_OK;
}

extern "C" int tf_stager_note_sunk(tf_stager* st, uint64_t bytes) {
  if (!st) return TF_ERR_VALUE;
  std::lock_guard<std::mutex> g(st->mu);
  st->pageable_in_flight -= std::min(bytes, st->pageable_in_flight);
  st->stats.pageable_bytes_in_flight = st->pageable_in_flight;
  return TF_OK;
}

extern "C" int tf_stager_stats_get(tf_stager* st, tf_stager_stats* out) {
  if (!st || !out) return TF_ERR_VALUE;
  std::lock_guard<std::mutex> g(st->mu);
  *out = st->stats;
  out->pool_total = st->bufs.size();
  out->pool_free = st->free_bufs.size();
  out->inflight_batches = st->inflight.size();
  out->to_stage_batches = st->to_stage.size();
  out->out_q_batches = st->out_q.size();
  out->outstanding_paged = st->outstanding_paged;
  out->completion_phase = st->completion_phase.load();
  out->stage_phase = st->stage_phase.load();
  return TF_OK;
}

extern "C" int tf_stager_error(tf_stager* st) { return st ? st->bg_error.load() : TF_ERR_VALUE; }

extern "C" int tf_stager_stream(tf_stager* st, void** stream) {
  if (!st || !stream) return TF_ERR_VALUE;
  *stream = (void*)st->stream;
  return TF_OK;
}

// Placement evidence for replicas: the CPUs the staging
// threads are bound to (the GPU's PCIe-local CPUs) and the NUMA node that
// holds the pinned pool's first page (move_pages in query mode).
extern "C" int tf_stager_placement(tf_stager* st, int32_t* cpus, uint32_t max_cpus,
                                   uint32_t* n_cpus, int32_t* pool_node) {
  if (!st) return TF_ERR_VALUE;
  if (n_cpus) *n_cpus = (uint32_t)st->cpus.size();
  if (cpus)
    for (uint32_t i = 0; i < max_cpus && i < st->cpus.size(); ++i) cpus[i] = st->cpus[i];
  if (pool_node) {
    *pool_node = -1;
    if (!st->bufs.empty()) {
      void* page = st->bufs[0];
      int status = -1;
      if (syscall(SYS_move_pages, 0, 1UL, &page, nullptr, &status, 0) == 0 && status >= 0)
        *pool_node = status;
    }
  }
  return TF_OK;
}

// ---------------------------------------------------------------------------
// background engine (wallclock.py:136-181 shape, real threads, no GIL)
// ---------------------------------------------------------------------------
static void set_bg_error(tf_stager* st, int rc) {
  int z = 0;
  if (st->bg_error.compare_exchange_strong(z, rc)) st->bg_errmsg = tf_last_error();
  st->cv.notify_all();
}

// A page-out buffer for a split capture of `bytes` (caller holds st->mu):
// the smallest cached one that fits, else a new 2 MiB-aligned allocation
// advised for transparent huge pages.
static uint8_t* oversize_alloc(tf_stager* st, uint64_t bytes) {
  auto it = st->oversize_pool.lower_bound(bytes);
  if (it != st->oversize_pool.end()) {
    uint8_t* p = it->second;
    st->oversize_pool.erase(it);
    return p;
  }
  const uint64_t huge = uint64_t(2) << 20;
  const uint64_t cap = (bytes + huge - 1) & ~(huge - 1);
  uint8_t* p = (uint8_t*)aligned_alloc(huge, cap);
  if (!p) return nullptr;
  madvise(p, cap, MADV_HUGEPAGE);
  st->oversize_cap[p] = cap;
  return p;
}

// Back to the cache (at most kOversizeCached buffers), else freed.
constexpr size_t kOversizeCached = 4;
static void oversize_free(tf_stager* st, uint8_t* p) {
  auto c = st->oversize_cap.find(p);
  if (c == st->oversize_cap.end()) { free(p); return; }
  if (st->oversize_pool.size() < kOversizeCached) {
    st->oversize_pool.emplace(c->second, p);
    return;
  }
  st->oversize_cap.erase(c);
  free(p);
}

static uint8_t* paged_alloc(tf_stager* st) {  // caller holds st->mu
  if (!st->paged_pool.empty()) {
    uint8_t* p = st->paged_pool.back();
    st->paged_pool.pop_back();
    return p;
  }
  uint8_t* p = (uint8_t*)aligned_alloc(4096, (st->cfg.staging_buffer_size + 4095) & ~uint64_t(4095));
  if (p) memset(p, 0, st->cfg.staging_buffer_size);  // fault pages in once
  return p;
}

static void free_paged_batch(tf_stager* st, tf_paged_batch* b, bool to_pool) {
  if (b->pinned_buffer >= 0) {
    // zero-copy hand-off: the pinned staging buffer goes back to the pool
    st->free_bufs.push_back((uint32_t)b->pinned_buffer);
    if (st->outstanding_handoff) st->outstanding_handoff -= 1;
    st->cv.notify_all();
  } else if (b->payload) {
    if (b->oversize) oversize_free(st, (uint8_t*)b->payload);
    else if (to_pool) st->paged_pool.push_back((uint8_t*)b->payload);
    else free(b->payload);
  }
  b->pinned_buffer = -1;
  free(b->descs);
  free(b->starts);
  b->payload = nullptr;
  b->descs = nullptr;
  b->starts = nullptr;
}

static void drain_loop(tf_stager* st) {
  bind_thread(st->cpus);
  RelaxedCaptureMode relaxed;  // ring2_internal.h
  cudaSetDevice(st->device);
  std::vector<tf_descriptor> tmp;
  std::deque<double> seen;  // observation times of ready entries (max_wait)
  int idle = 0;
  // Only host-memory polling and D2H issue here: no CUDA query calls in the
  // spin (they contend with the inference thread's launches in the driver).
  while (!st->stop_req.load()) {
    bool did = false;
    uint32_t n = 0;
    uint64_t bytes = 0;
    ready_summary(st, tmp, &n, &bytes);
    double now = tf_monotonic();
    while (seen.size() < n) seen.push_back(now);
    uint32_t reason = st->flush_req.load() ? (n ? TF_REASON_FLUSH : TF_REASON_NONE)
                                           : reason_for(st, n, bytes, seen.empty() ? -1.0 : now - seen.front());
    if (reason != TF_REASON_NONE) {
      std::unique_lock<std::mutex> g(st->mu);
      if (st->free_bufs.size() < (n ? std::min<uint64_t>(bufs_needed(st, &tmp[0]), st->bufs.size()) : 1)) {
        st->stats.staging_exhausted_waits += 1;
        st->cv.wait_for(g, std::chrono::microseconds(200));
      } else {
        Batch* b = nullptr;
        int rc = issue_batch(st, reason, &b);
        if (rc) {
          g.unlock();
          set_bg_error(st, rc);
          break;
        }
        if (b) {
          size_t k = std::min(seen.size(), b->descs.size());
          seen.erase(seen.begin(), seen.begin() + k);
          st->inflight.push_back(b);
          st->cv.notify_all();
          did = true;
        }
      }
    }
    if (did) {
      idle = 0;
    } else if (++idle < 2000) {
      cpu_relax();
    } else {
      std::this_thread::sleep_for(std::chrono::microseconds(20));
    }
  }
  st->drain_done = true;
  st->cv.notify_all();
}

// Completion: block on the oldest D2H (blocking-sync event, the thread
// sleeps in the driver), then release its regions and hand it to staging.
static void completion_loop(tf_stager* st) {
  bind_thread(st->cpus);
  RelaxedCaptureMode relaxed;  // ring2_internal.h
  cudaSetDevice(st->device);
  for (;;) {
    Batch* b = nullptr;
    {
      std::unique_lock<std::mutex> g(st->mu);
      st->cv.wait(g, [&] { return !st->inflight.empty() || st->drain_done.load() || st->bg_error; });
      if (st->inflight.empty()) break;
      b = st->inflight.front();
    }
    st->completion_phase = 1;
    cudaError_t e = cudaEventSynchronize(b->ev1);
    st->completion_phase = 2;
    std::unique_lock<std::mutex> g(st->mu);
    if (e != cudaSuccess) {
      tf_set_error("D2H failed: %s", cudaGetErrorString(e));
      g.unlock();
      set_bg_error(st, TF_ERR_CUDA);
      break;
    }
    int rc = wait_transfer(st, b);
    if (!rc) rc = release_batch(st, b);
    if (rc) {
      g.unlock();
      set_bg_error(st, rc);
      break;
    }
    st->inflight.pop_front();
    st->to_stage.push_back(b);
    st->completion_phase = 0;
    st->cv.notify_all();
  }
  st->completion_done = true;
  st->cv.notify_all();
}

static void stage_loop(tf_stager* st) {
  bind_thread(st->cpus);
  RelaxedCaptureMode relaxed;  // ring2_internal.h
  for (;;) {
    Batch* b = nullptr;
    uint8_t* dst = nullptr;
    bool handoff_ok = false;
    {
      std::unique_lock<std::mutex> g(st->mu);
      st->cv.wait(g, [&] { return !st->to_stage.empty() || st->completion_done.load() || st->bg_error; });
      if (st->to_stage.empty()) return;
      b = st->to_stage.front();
      st->to_stage.pop_front();
      if (st->cfg.page_out == TF_PAGE_OUT_DISCARD) {
        // D2H-only measurement: the bytes have landed in the pinned host
        // ring; hand the buffer straight back.
        st->stats.batches_staged += 1;
        retire_batch(st, b);
        st->cv.notify_all();
        continue;
      }
      // Hand-off keeps a pinned buffer out of the pool until the consumer
      // frees the batch. The consumer may be Python (needs the GIL), and the
      // inference thread may block on the device holding the GIL while the
      // device waits for ring space (completeness): buffers the consumer
      // holds must never starve the drain. So a batch is handed off only
      // while at least half the pool stays with the engine; otherwise it is
      // copied out, and its buffer returns at once.
      // (and never into the buffers the largest split capture seen so far
      // needs at once: a split capture waits for all of its chunks' buffers)
      handoff_ok = st->cfg.page_out == TF_PAGE_OUT_HANDOFF &&
                   2 * (st->outstanding_handoff + 1) <= st->bufs.size() &&
                   st->outstanding_handoff + 1 + st->max_split_bufs <= st->bufs.size();
      if ((st->cfg.page_out == TF_PAGE_OUT_COPY || !handoff_ok) && b->chunk_bufs.empty())
        dst = paged_alloc(st);
      if (handoff_ok && b->chunk_bufs.empty()) st->outstanding_handoff += 1;
    }
    // a split capture is paged out into one contiguous allocation of its
    // own (the sink needs its payload in one piece), whatever the mode
    const bool split = !b->chunk_bufs.empty();
    st->stage_phase = 1;
    if (split) {
      {
        std::lock_guard<std::mutex> g(st->mu);
        dst = oversize_alloc(st, b->bytes);
      }
      if (!dst) {
        tf_set_error("pageable allocation of a split capture (%llu bytes) failed",
                     (unsigned long long)b->bytes);
        set_bg_error(st, TF_ERR_ALLOCATION);
        return;
      }
    }
    const bool handoff = handoff_ok && !split;
    if (!handoff && !dst) {
      tf_set_error("pageable allocation failed");
      set_bg_error(st, TF_ERR_ALLOCATION);
      return;
    }
    // pinned -> pageable (exporter.py:237-249), NUMA-local, parallel; or
    // zero-copy hand-off of the pinned buffer itself
    st->stage_phase = 2;
    if (!handoff) gather_chunks(st, b, dst, true);
    tf_paged_batch pb;
    memset(&pb, 0, sizeof(pb));
    pb.pinned_buffer = handoff ? (int32_t)b->buf : -1;
    pb.oversize = split ? 1u : 0u;
    if (handoff) dst = st->bufs[b->buf];
    pb.batch_id = b->id;
    pb.n_entries = (uint32_t)b->descs.size();
    pb.reason = b->reason;
    pb.bytes_total = b->bytes;
    pb.payload = dst;
    pb.descs = (tf_descriptor*)malloc(sizeof(tf_descriptor) * std::max<size_t>(1, b->descs.size()));
    pb.starts = (uint64_t*)malloc(sizeof(uint64_t) * std::max<size_t>(1, b->starts.size()));
    memcpy(pb.descs, b->descs.data(), sizeof(tf_descriptor) * b->descs.size());
    memcpy(pb.starts, b->starts.data(), sizeof(uint64_t) * b->starts.size());
    {
      std::unique_lock<std::mutex> g(st->mu);
      st->pageable_in_flight += b->bytes;
      st->stats.batches_staged += 1;
      retire_batch(st, b, !handoff);  // copy mode: buffer back before the hand-off
      note_transient(st);
      st->cv.notify_all();
      st->stage_phase = 3;
      // The queue bound (exporter.py:32) applies while the paged-out bytes
      // stay under the budget; past it the stage thread runs ahead of the
      // consumer into pageable memory. A Python consumer can be starved of
      // the GIL by an inference thread blocked in a CUDA call while the
      // device waits for ring space; the ring must still drain then.
      st->cv.wait(g, [&] {
        return st->out_q.size() < st->cfg.stage_queue_slots ||
               st->pageable_in_flight <= st->pageable_budget || st->stop_req;
      });
      st->stage_phase = 0;
      st->out_q.push_back(pb);
      st->cv.notify_all();
    }
  }
}

extern "C" int tf_stager_start(tf_stager* st) {
  if (!st) return TF_ERR_VALUE;
  if (st->running) return TF_OK;
  {
    std::lock_guard<std::mutex> g(st->mu);
    if (!st->batches.empty()) {
      tf_set_error("synchronous batches still outstanding");
      return TF_ERR_PROTOCOL;
    }
  }
  st->stop_req = false;
  st->bg_error = 0;
  unsigned nthreads = st->cfg.stage_threads ? st->cfg.stage_threads : 3;
  st->copy_pool.start((int)nthreads, st->cpus);
  st->running = true;
  st->drain_done = false;
  st->completion_done = false;
  st->drain_th = std::thread(drain_loop, st);
  st->completion_th = std::thread(completion_loop, st);
  st->stage_th = std::thread(stage_loop, st);
  return TF_OK;
}

extern "C" int tf_stager_stop(tf_stager* st) {
  if (!st) return TF_ERR_VALUE;
  if (!st->running) return TF_OK;
  st->stop_req = true;
  st->cv.notify_all();
  if (st->drain_th.joinable()) st->drain_th.join();
  st->cv.notify_all();
  if (st->completion_th.joinable()) st->completion_th.join();
  st->cv.notify_all();
  if (st->stage_th.joinable()) st->stage_th.join();
  st->copy_pool.stop();
  st->running = false;
  return st->bg_error.load();
}

extern "C" int tf_stager_flush(tf_stager* st, double timeout_s) {
  if (!st) return TF_ERR_VALUE;
  if (!st->running) { tf_set_error("background engine not running"); return TF_ERR_PROTOCOL; }
  st->flush_req.fetch_add(1);
  double t0 = tf_monotonic();
  int rc = TF_OK;
  for (;;) {
    if (st->bg_error) { rc = st->bg_error; break; }
    uint64_t ready = 0;
    tf_ring_ready_entries(st->ring, &ready);
    bool empty_regions;
    {
      std::lock_guard<std::mutex> g(st->ring->mu);
      empty_regions = st->ring->regions.empty();
    }
    bool idle;
    {
      std::lock_guard<std::mutex> g(st->mu);
      idle = st->inflight.empty();
    }
    if (ready == 0 && idle && empty_regions) break;
    if (tf_monotonic() - t0 > timeout_s) {
      tf_set_error("flush did not finish within %.1fs", timeout_s);
      rc = TF_ERR_TIMEOUT;
      break;
    }
    std::this_thread::sleep_for(std::chrono::microseconds(50));
  }
  st->flush_req.fetch_sub(1);
  return rc;
}

extern "C" int tf_stager_next(tf_stager* st, double timeout_s, tf_paged_batch* out) {
  if (!st || !out) return TF_ERR_VALUE;
  std::unique_lock<std::mutex> g(st->mu);
  bool ok = st->cv.wait_for(g, std::chrono::duration<double>(timeout_s), [&] {
    return !st->out_q.empty() || st->bg_error || (!st->running && st->to_stage.empty());
  });
  if (!st->out_q.empty()) {
    *out = st->out_q.front();
    st->out_q.pop_front();
    st->outstanding_paged += 1;
    st->cv.notify_all();
    return TF_OK;
  }
  if (st->bg_error) return st->bg_error;
  memset(out, 0, sizeof(*out));
  return ok ? TF_ERR_EMPTY : TF_ERR_TIMEOUT;
}

extern "C" int tf_stager_free_paged(tf_stager* st, tf_paged_batch* b) {
  if (!st || !b) return TF_ERR_VALUE;
  std::lock_guard<std::mutex> g(st->mu);
  st->pageable_in_flight -= std::min(b->bytes_total, st->pageable_in_flight);
  st->stats.pageable_bytes_in_flight = st->pageable_in_flight;
  if (st->outstanding_paged) st->outstanding_paged -= 1;
  free_paged_batch(st, b, st->paged_pool.size() < st->cfg.stage_queue_slots + 4);
  return TF_OK;
}

extern "C" void tf_free_host(void* p) { free(p); }

// ---------------------------------------------------------------------------
// measurement: pinned D2H bandwidth of the link this ring drains over
// ---------------------------------------------------------------------------
extern "C" int tf_measure_d2h(int device, uint64_t nbytes, int reps, double* gbps) {
  if (!gbps || nbytes == 0) return TF_ERR_VALUE;
  CUDA_TRY(cudaSetDevice(device));
  void* d = nullptr;
  void* h = nullptr;
  CUDA_TRY(cudaMalloc(&d, nbytes));
  if (cudaHostAlloc(&h, nbytes, cudaHostAllocPortable) != cudaSuccess) {
    cudaFree(d);
    tf_set_error("pinned alloc failed");
    return TF_ERR_ALLOCATION;
  }
  memset(h, 0, nbytes);
  cudaMemset(d, 1, nbytes);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  double best = 0;
  for (int i = 0; i < std::max(1, reps); ++i) {
    cudaEventRecord(a, s);
    cudaMemcpyAsync(h, d, nbytes, cudaMemcpyDeviceToHost, s);
    cudaEventRecord(b, s);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    if (ms > 0) best = std::max(best, double(nbytes) / (ms * 1e-3) / 1e9);
  }
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaStreamDestroy(s);
  cudaFreeHost(h);
  cudaFree(d);
  *gbps = best;
  return TF_OK;
}
