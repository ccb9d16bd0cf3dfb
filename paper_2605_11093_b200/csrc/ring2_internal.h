// ring2_internal.h — memory layout of one ring pair (not part of the ABI).
//
//   payload ring     cudaMalloc            written by capture kernels, read by
//                                          the staging D2H
//   meta ring        cudaHostAlloc mapped  64-B descriptors; device posts the
//                                          words (no fence) with a checksum,
//                                          host polls and verifies
//   DevConsumer      cudaMalloc            host-owned release/meta cursors as
//                                          the device sees them; written by
//                                          stream-ordered cuStreamWriteValue64
//                                          (after each D2H, on its stream), so
//                                          the capture kernel never reads host
//                                          memory across a busy PCIe link
//   DevCtl           cudaMalloc            allocator state, counters,
//                                          per-launch CTA handshake, last
//                                          result; snapshotted by a D2H copy
//                                          on the ring's control stream
//
// The only host-memory traffic of a capture kernel is the one coalesced
// 64-byte descriptor store of its last CTA.
#pragma once
#include <stdint.h>

#include <deque>
#include <map>
#include <mutex>

#include <cuda_runtime.h>

#include "ring2_core.h"

// Host threads of the consumer side (staging threads) make stream-
// synchronising calls on their own private streams. Under another thread's
// global-mode CUDA graph capture (torch.cuda.graph's default) those calls
// would invalidate the capture, so these threads run in relaxed capture
// mode: nothing they touch is being captured.
struct RelaxedCaptureMode {
  cudaStreamCaptureMode prev = cudaStreamCaptureModeRelaxed;
  RelaxedCaptureMode() { cudaThreadExchangeStreamCaptureMode(&prev); }
  ~RelaxedCaptureMode() { cudaThreadExchangeStreamCaptureMode(&prev); }
  RelaxedCaptureMode(const RelaxedCaptureMode&) = delete;
  RelaxedCaptureMode& operator=(const RelaxedCaptureMode&) = delete;
};

struct alignas(128) DevConsumer {
  uint64_t L;          // virtual release cursor (ring2_core.h)
  uint64_t pad0[15];
  uint64_t meta_tail;  // descriptors consumed
  uint64_t pad1[15];
};

// Producer snapshot for the capture kernel's fast path: the allocator
// state, meta head and capture sequence after the last producer operation,
// the consumer cursors as that operation's final thread read them, and the
// (used, head, tail) derived from them. Every kernel that moves the producer
// state rewrites all replicas before it exits, so the words are stable for
// the whole next launch: each CTA reads its replica (spreading the reads of
// hundreds of CTAs over several L2 lines), runs the allocator on the same
// inputs and reaches the same offset with no cross-CTA handshake. L only
// grows, so a snapshot L is conservative (it never hands out live bytes).
struct alignas(128) ProdSnap {
  uint64_t V, reset_mark, reset_credit, meta_head;
  uint64_t L, meta_tail, capture_seq, L_phys;  // L_phys = L % capacity
  uint64_t used, head, tail, pad1[5];
};
constexpr int kSnapReplicas = 8;
constexpr int kMaxFlagCtas = 512;   // completion bytes per meta slot

struct alignas(128) DevCtl {
  // allocator (producer role)
  tf_pstate p;
  uint64_t meta_head;
  // counters
  uint64_t bytes_reserved, dead_created, captures, drops, drop_bytes;
  uint64_t stall_events, stall_ns, errors, capture_seq;
  // per-launch handshake between the CTAs of one capture kernel; launches
  // on one producer stream are serialised, the last CTA re-arms these.
  uint32_t arrive, done, plan_flag, plan_status;
  uint32_t readers, pad_r;  // fast-path CTAs that have read the snapshot (this launch)
  uint64_t plan_off, plan_skip, plan_len, plan_bytes, plan_rows, plan_seq;
  uint32_t plan_kind, pad0;

  // device-side timing of capture kernels (globaltimer, ns)
  uint64_t k_t0, kernel_ns, last_kernel_ns;
  uint64_t pad1;
  // result of the most recent launch (device memory; the host copies the
  // whole block on a side stream when it needs a snapshot)
  tf_capture_result res;
  ProdSnap snap[kSnapReplicas];
};

struct HostRegion {
  uint64_t off, len, skip;
  uint32_t kind;
  // descriptor polled by the consumer: only a leading run of polled regions
  // may be handed back to the device allocator ahead of its release
  bool polled = false;
  // reservation order: a device capture's capture_seq, or for a host
  // reservation the device capture count when it was made (it follows
  // capture `seq` and precedes capture seq+1); device regions become known
  // only when polled and are inserted at their reservation position
  bool host = false;
  uint64_t seq = 0;
};

struct tf_ring {
  int device = 0;
  tf_ring_config cfg{};
  uint8_t* payload = nullptr;     // device
  uint8_t* meta = nullptr;        // host pinned mapped (device alias == same VA)
  // per meta slot, one completion byte per capture CTA (host pinned mapped):
  // fast-path captures post their descriptor early and every CTA sets its
  // byte after its payload stores; the host takes the slot once all are set
  uint8_t* done_flags = nullptr;
  DevConsumer* dcons = nullptr;   // device
  DevCtl* ctl = nullptr;          // device
  uint64_t* seal_host = nullptr;  // pinned, host-mapped: descriptors below it are complete
  DevCtl* ctl_host = nullptr;     // pinned, host-mapped snapshot target
  DevCtl* ctl_host_dev = nullptr; // its device alias (snapshot kernel)
  void* snap_stream = nullptr;    // high-priority stream of the snapshot kernel
  void* ctrl_stream = nullptr;    // cudaStream_t for consumer-cursor updates
  // consumer-role state (host)
  std::mutex mu;
  uint64_t L = 0, meta_tail = 0, consumed = 0;
  uint64_t bytes_released = 0, dead_reclaimed = 0;
  std::deque<HostRegion> regions;               // reservation order
  std::map<uint64_t, HostRegion> host_reserved; // tf_ring_reserve'd, unpublished
};

// cross-TU helpers (ring2.cu)
int tf_internal_poll(tf_ring* r, uint32_t max_entries, tf_descriptor* out,
                     uint32_t* n, bool consume);
// release without pushing L to the device (the staging stream already
// wrote it behind the D2H)
int tf_internal_release(tf_ring* r, uint64_t offset, uint64_t length, bool push);
// L after releasing every region currently queued on the host
uint64_t tf_internal_l_after_all(tf_ring* r);
// stream-ordered write of one u64 into device memory
int tf_internal_write_u64(void* stream, uint64_t* dev_addr, uint64_t value);
void tf_set_error(const char* fmt, ...);

// descriptor checksum (word 7): the host accepts a slot only when the
// words it read hash to it, so publication needs no system-scope fence
TF_HD uint64_t tf_desc_mix(uint64_t h, uint64_t v) {
  h ^= v + 0x9E3779B97F4A7C15ull + (h << 6) + (h >> 2);
  h ^= h >> 31;
  h *= 0xBF58476D1CE4E5B9ull;
  h ^= h >> 29;
  return h;
}
TF_HD uint64_t tf_desc_checksum(const uint64_t* w) {
  uint64_t h = 0x5EED2605ull;
  for (int i = 0; i < 7; ++i) h = tf_desc_mix(h, w[i]);
  return h | 1ull;  // never 0 (a zeroed slot never verifies)
}
