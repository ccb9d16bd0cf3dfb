// ring2_internal.h — memory layout of one ring pair (not part of the ABI).
//
//   payload ring     cudaMalloc            device-written by capture kernels,
//                                          read by the staging D2H
//   meta ring        cudaHostAlloc mapped  64-B descriptors; device writes
//                                          body then ready_seq, host polls
//   ConsumerShared   cudaHostAlloc mapped  host-owned release/meta cursors the
//                                          device reads when it reserves
//   ProducerMirror   cudaHostAlloc mapped  device-owned cursors mirrored for
//                                          host snapshots (state/would_fit)
//   DevCtl           cudaMalloc            device-owned allocator state,
//                                          counters and per-launch handshake
#pragma once
#include <stdint.h>

#include <deque>
#include <map>
#include <mutex>

#include "ring2_core.h"

struct alignas(64) ConsumerShared {
  uint64_t L;          // virtual release cursor (ring2_core.h)
  uint64_t meta_tail;  // descriptors consumed
  uint64_t pad[6];
};

struct alignas(64) ProducerMirror {
  uint64_t V, reset_mark, reset_credit, meta_head;
  uint64_t bytes_reserved, dead_created, captures, drops;
  uint64_t drop_bytes, stall_events, stall_ns, errors;
  uint64_t capture_seq, pad[3];
};

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
  uint64_t plan_off, plan_skip, plan_len, plan_bytes, plan_rows, plan_seq;
  uint32_t plan_kind, pad0;
  uint64_t pad1[4];
};

struct HostRegion {
  uint64_t off, len, skip;
  uint32_t kind;
};

struct tf_ring {
  int device = 0;
  tf_ring_config cfg{};
  uint8_t* payload = nullptr;     // device
  uint8_t* meta = nullptr;        // host pinned mapped (device alias == same VA)
  ConsumerShared* cons = nullptr; // host pinned mapped
  ProducerMirror* mirror = nullptr;
  tf_capture_result* result = nullptr;
  DevCtl* ctl = nullptr;          // device
  void* own_stream = nullptr;     // cudaStream_t used when the caller passes NULL
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
void tf_set_error(const char* fmt, ...);
