// ring2_core.h — allocator and producer-state arithmetic shared verbatim by
// the device producer (capture kernels) and the host shadow (policy replay,
// state snapshots). One copy of the rules, so the device reserves exactly
// what the host predicts (SURVEY §3.5 invariant).
#pragma once
#include <stdint.h>

#if defined(__CUDACC__)
#define TF_HD __host__ __device__ __forceinline__
#else
#define TF_HD static inline
#endif

#include "../../include/ring2.h"

// rings.py:63-64 round_up_to_copy_unit
TF_HD uint64_t tf_round_up16(uint64_t n) { return (n + 15u) & ~(uint64_t)15; }

// rings.py:166-193 _plan_reservation. Returns 1 and (offset, dead) when the
// request fits, else 0. Rules in order: full; empty -> offset 0; wrapped
// (head <= tail) -> only the gap; else end space; else dead-skip to 0 iff
// the skipped tail end plus the request fit and length <= tail.
TF_HD int tf_plan(uint64_t head, uint64_t tail, uint64_t used, uint64_t cap,
                  uint64_t len, uint64_t* off, uint64_t* dead) {
  if (used + len > cap) return 0;
  if (used == 0) { *off = 0; *dead = 0; return 1; }
  if (head <= tail && !(head == tail && used == cap)) {
    if (len <= tail - head) { *off = head; *dead = 0; return 1; }
    return 0;
  }
  uint64_t end_space = cap - head;
  if (len <= end_space) { *off = head; *dead = 0; return 1; }
  if (used + end_space + len <= cap && len <= tail) {
    *off = 0; *dead = end_space; return 1;
  }
  return 0;
}

// Producer-owned state. The reference keeps (head, tail, used) in one
// object (rings.py:216-218); on a GPU the producer (device) and consumer
// (host) must not write each other's words, so ownership is split:
//   V            device: virtual reserve cursor; every reservation consumes
//                virtual bytes [V, V+skip+len) and physical = virtual % cap.
//                A dead-skip fills exactly to the end of the buffer, so the
//                mapping survives wraparound.
//   L            host:   virtual release cursor (advanced by skip+reserved_len
//                at each in-order release, rings.py:408-431).
//   reset_mark/credit    the empty-ring reset (rings.py:178-181, 309-310)
//                restarts placement at offset 0 without occupying the skipped
//                bytes; until the host releases past it (L moves off
//                reset_mark) those `credit` bytes are not occupancy and the
//                reference's tail is 0.
typedef struct tf_pstate {
  uint64_t V;
  uint64_t reset_mark;
  uint64_t reset_credit;
} tf_pstate;

#define TF_NO_MARK 0xFFFFFFFFFFFFFFFFull

TF_HD uint64_t tf_credit(const tf_pstate* p, uint64_t L) {
  return L == p->reset_mark ? p->reset_credit : 0;
}
// rings.py:237-239 occupancy (live + dead bytes)
TF_HD uint64_t tf_used(const tf_pstate* p, uint64_t L) {
  return p->V - L - tf_credit(p, L);
}
TF_HD uint64_t tf_head(const tf_pstate* p, uint64_t cap) { return p->V % cap; }
TF_HD uint64_t tf_tail(const tf_pstate* p, uint64_t L, uint64_t cap) {
  return (L + tf_credit(p, L)) % cap;
}

// rings.py:286-319 reserve_payload as a state transition on (pstate, L).
// `skip` is the number of virtual bytes consumed before the region and
// `kind` says whether they were a dead region or an empty-ring reset.
// tf_reserve with (used, head, tail) of (p, L) already derived, so a caller
// holding them precomputed skips the 64-bit modulo arithmetic.
TF_HD int tf_reserve_derived(tf_pstate* p, uint64_t L, uint64_t cap, uint64_t len,
                             uint64_t used, uint64_t head, uint64_t tail,
                             uint64_t* off, uint64_t* skip, uint32_t* kind) {
  uint64_t o = 0, d = 0;
  if (!tf_plan(head, tail, used, cap, len, &o, &d)) return 0;
  if (used == 0) {
    // empty: V == L here (a pending credit implies used > 0)
    uint64_t s = head ? cap - head : 0;
    p->reset_mark = L;
    p->reset_credit = s;
    *skip = s;
    *kind = s ? TF_DESC_EMPTY_RESET : 0u;
    p->V += s + len;
  } else if (d) {
    *skip = d;
    *kind = TF_DESC_DEAD_SKIP;
    p->V += d + len;
  } else {
    *skip = 0;
    *kind = 0;
    p->V += len;
  }
  *off = o;
  return 1;
}

TF_HD int tf_reserve(tf_pstate* p, uint64_t L, uint64_t cap, uint64_t len,
                     uint64_t* off, uint64_t* skip, uint32_t* kind) {
  return tf_reserve_derived(p, L, cap, len, tf_used(p, L), tf_head(p, cap),
                            tf_tail(p, L, cap), off, skip, kind);
}
