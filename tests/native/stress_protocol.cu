// Protocol stress driver for the sanitizers (test infrastructure, not product
// code). It drives the C ABI exactly as the Python host does — capture
// launches on an inference stream, the native staging engine (drain,
// completion and page-out threads) draining concurrently, and a consumer
// thread taking paged batches — and checks every payload byte.
//
// Each capture i first runs a fill kernel that writes a hash pattern of i
// into the source rows and a hash-chosen keep vector, then captures with
// TF_FULL_WAIT into a deliberately small ring, so wrap-around, dead-skips,
// empty-ring resets and device-side backpressure waits all happen. The
// consumer regenerates the expected kept rows on the host and compares.
//
//   stress_protocol [captures] [rings]
//
// rings > 1 runs independent ring pairs (one producer stream + stager +
// consumer each) concurrently in one process: the multi-replica layout of
// SURVEY §8(e) on one device.
//
// Builds (scripts/sanitize.sh): plain -G-free -lineinfo for compute-sanitizer
// (memcheck / racecheck / synccheck), and -fsanitize=thread on the host code
// (library + driver) for ThreadSanitizer.
#include <cuda_runtime.h>

#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

#include "../../include/ring2.h"

extern "C" int tf_stager_free_paged(tf_stager* st, tf_paged_batch* b);

#define CK(x)                                                                  \
  do {                                                                         \
    cudaError_t e_ = (x);                                                      \
    if (e_ != cudaSuccess) {                                                   \
      fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
      exit(3);                                                                 \
    }                                                                          \
  } while (0)
#define TK(x)                                                                  \
  do {                                                                         \
    int r_ = (x);                                                              \
    if (r_ != TF_OK) {                                                         \
      fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, tf_status_name(r_), \
              tf_last_error());                                                \
      exit(4);                                                                 \
    }                                                                          \
  } while (0)

__host__ __device__ inline uint32_t mix32(uint64_t x) {
  x ^= x >> 33;
  x *= 0xff51afd7ed558ccdull;
  x ^= x >> 33;
  x *= 0xc4ceb9fe1a85ec53ull;
  x ^= x >> 33;
  return uint32_t(x);
}
__host__ __device__ inline uint8_t pattern(uint64_t cap, uint64_t pos) {
  return uint8_t(mix32((cap << 40) ^ pos) >> 11);
}

struct Shape {
  int64_t outer, mid, row_bytes;
  bool per_outer;
};

// capture i's shape: a mix of request keeps and token-row keeps, rows of
// 16-B multiples and odd widths (the byte/tail paths), 3 B .. 1.5 MiB
static Shape shape_of(uint64_t i) {
  const uint32_t h = mix32(i * 7919 + 1);
  Shape s;
  s.outer = 1 + h % 16;
  s.mid = 1 + (h >> 4) % 24;
  const int64_t rb[] = {16, 48, 256, 1024, 2048, 4096, 17, 3, 130, 4000};
  s.row_bytes = rb[(h >> 10) % 10];
  s.per_outer = (h >> 14) & 1;
  return s;
}
__host__ __device__ inline bool kept(uint64_t cap, int64_t unit) {
  return (mix32(cap * 31 + uint64_t(unit) * 977 + 5) % 4) != 0;  // ~75 %
}

__global__ void fill(uint8_t* src, int64_t bytes, uint8_t* keep, int64_t units, uint64_t cap) {
  for (int64_t p = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; p < bytes;
       p += int64_t(gridDim.x) * blockDim.x)
    src[p] = pattern(cap, p);
  for (int64_t u = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; u < units;
       u += int64_t(gridDim.x) * blockDim.x)
    keep[u] = kept(cap, u) ? 1 : 0;
}

struct Replica {
  int idx;
  tf_ring* ring = nullptr;
  tf_stager* st = nullptr;
  cudaStream_t s{};
  uint8_t* src = nullptr;
  uint8_t* keep = nullptr;
  uint32_t* step = nullptr;
  std::atomic<uint64_t> checked_bytes{0}, records{0}, errors{0};
  uint64_t expected_records = 0;
};

static std::vector<uint8_t> expected(uint64_t cap, const Shape& s) {
  std::vector<uint8_t> out;
  const int64_t units = s.per_outer ? s.outer : s.outer * s.mid;
  const int64_t rpu = s.per_outer ? s.mid : 1;
  for (int64_t u = 0; u < units; ++u) {
    if (!kept(cap, u)) continue;
    for (int64_t r = u * rpu; r < (u + 1) * rpu; ++r)
      for (int64_t b = 0; b < s.row_bytes; ++b)
        out.push_back(pattern(cap, uint64_t(r * s.row_bytes + b)));
  }
  return out;
}

static void consumer(Replica* R, uint64_t n_caps) {
  // capture_seq is the ring's 1-based launch counter; captures that keep
  // nothing publish nothing but still take a sequence number
  uint64_t got = 0;
  while (got < R->expected_records) {
    tf_paged_batch b;
    int rc = tf_stager_next(R->st, 30.0, &b);
    if (rc == TF_ERR_TIMEOUT || rc == TF_ERR_EMPTY) {
      fprintf(stderr, "replica %d: timeout with %llu/%llu records\n", R->idx,
              (unsigned long long)got, (unsigned long long)R->expected_records);
      R->errors++;
      return;
    }
    TK(rc);
    for (uint32_t e = 0; e < b.n_entries; ++e) {
      const tf_descriptor& d = b.descs[e];
      const uint64_t cap = d.step_seq;  // the driver's capture index
      if (cap >= n_caps) { R->errors++; continue; }
      const std::vector<uint8_t> want = expected(cap, shape_of(cap));
      const uint8_t* p = static_cast<const uint8_t*>(b.payload) + b.starts[e];
      if (d.payload_len != want.size() || memcmp(p, want.data(), want.size()) != 0) {
        if (R->errors.load() < 5)
          fprintf(stderr, "replica %d: capture %llu mismatch (len %llu want %zu)\n", R->idx,
                  (unsigned long long)cap, (unsigned long long)d.payload_len, want.size());
        R->errors++;
      }
      R->checked_bytes += d.payload_len;
      ++got;
    }
    R->records += b.n_entries;
    TK(tf_stager_free_paged(R->st, &b));
  }
}

static bool g_sealed = false;  // argv[3]: TF_CAP_SEALED captures + seals

static void producer(Replica* R, uint64_t n_caps) {
  for (uint64_t i = 0; i < n_caps; ++i) {
    const Shape s = shape_of(i);
    const int64_t bytes = s.outer * s.mid * s.row_bytes;
    const int64_t units = s.per_outer ? s.outer : s.outer * s.mid;
    fill<<<64, 256, 0, R->s>>>(R->src, bytes, R->keep, units, i);
    CK(cudaGetLastError());
    tf_capture_args a;
    memset(&a, 0, sizeof(a));
    a.src = R->src;
    a.outer = s.outer;
    a.mid = s.mid;
    a.row_bytes = s.row_bytes;
    a.stride_outer = s.mid * s.row_bytes;
    a.stride_mid = s.row_bytes;
    a.keep = R->keep;
    a.step_seq = uint32_t(i);
    a.hook_id = uint32_t(i % 7);
    a.op = TF_OP_COPY;
    a.flags = TF_FULL_WAIT | (s.per_outer ? TF_CAP_KEEP_PER_OUTER : 0u) |
              (g_sealed ? TF_CAP_SEALED : 0u);
    TK(tf_capture(R->ring, R->s, &a));
    if (i % 64 == 63) {  // bound the fill backlog
      if (g_sealed) TK(tf_ring_seal(R->ring, R->s));
      CK(cudaStreamSynchronize(R->s));
    }
  }
  if (g_sealed) TK(tf_ring_seal(R->ring, R->s));
  CK(cudaStreamSynchronize(R->s));
}

int main(int argc, char** argv) {
  const uint64_t n_caps = argc > 1 ? strtoull(argv[1], nullptr, 10) : 1500;
  const int n_rings = argc > 2 ? atoi(argv[2]) : 1;
  g_sealed = argc > 3 && atoi(argv[3]) != 0;
  CK(cudaSetDevice(0));
  std::vector<Replica*> reps;
  for (int k = 0; k < n_rings; ++k) {
    Replica* R = new Replica();
    R->idx = k;
    tf_ring_config rc;
    memset(&rc, 0, sizeof(rc));
    rc.payload_capacity = 4u << 20;  // small: forces wrap, skips and waits
    rc.meta_slots = 48;
    rc.high_watermark = 1.0;
    rc.wait_timeout_ns = 20000000000ull;
    TK(tf_ring_create(&rc, 0, &R->ring));
    tf_drain_config dc;
    memset(&dc, 0, sizeof(dc));
    dc.min_ready_entries = 4;
    dc.min_ready_bytes = 256 << 10;
    dc.max_wait = 1e-4;
    dc.staging_buffer_size = 2u << 20;
    dc.staging_buffer_count = 4;
    dc.mode = TF_STAGE_COPY_ENGINE;
    dc.numa_node = -1;
    dc.page_out = TF_PAGE_OUT_HANDOFF;
    TK(tf_stager_create(R->ring, &dc, &R->st));
    CK(cudaStreamCreateWithFlags(&R->s, cudaStreamNonBlocking));
    CK(cudaMalloc(&R->src, 2u << 20));
    CK(cudaMalloc(&R->keep, 1024));
    for (uint64_t i = 0; i < n_caps; ++i)
      R->expected_records += expected(i, shape_of(i)).empty() ? 0 : 1;
    TK(tf_stager_start(R->st));
    reps.push_back(R);
  }
  std::vector<std::thread> th;
  for (Replica* R : reps) {
    th.emplace_back(consumer, R, n_caps);
    th.emplace_back(producer, R, n_caps);
  }
  for (auto& t : th) t.join();
  int bad = 0;
  for (Replica* R : reps) {
    TK(tf_stager_flush(R->st, 30.0));
    tf_ring_state s;
    TK(tf_ring_get_state(R->ring, &s));
    printf("{\"replica\": %d, \"captures\": %llu, \"records\": %llu, \"expected\": %llu, "
           "\"bytes_checked\": %llu, \"errors\": %llu, \"stall_events\": %llu, "
           "\"dead_created\": %llu, \"occupancy_end\": %llu, \"device_errors\": %llu}\n",
           R->idx, (unsigned long long)n_caps, (unsigned long long)R->records.load(),
           (unsigned long long)R->expected_records, (unsigned long long)R->checked_bytes.load(),
           (unsigned long long)R->errors.load(), (unsigned long long)s.stall_events,
           (unsigned long long)s.dead_created, (unsigned long long)s.occupancy,
           (unsigned long long)s.device_errors);
    bad |= R->errors.load() != 0 || R->records.load() != R->expected_records ||
           s.device_errors != 0 || s.occupancy != 0;
    TK(tf_stager_stop(R->st));
    TK(tf_stager_destroy(R->st));
    TK(tf_ring_destroy(R->ring));
  }
  printf(bad ? "STRESS FAIL\n" : "STRESS OK\n");
  return bad;
}
