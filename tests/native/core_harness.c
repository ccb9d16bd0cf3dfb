/* Test harness: exposes the product allocator (ring2_core.h, the code the
 * capture kernel runs on the device) to Python on the CPU, so its
 * split-ownership state machine can be replayed against the oracle. */
#include "../../paper_2605_11093_b200/csrc/ring2_core.h"

int core_reserve(tf_pstate* p, uint64_t L, uint64_t cap, uint64_t len,
                 uint64_t* off, uint64_t* skip, uint32_t* kind) {
  return tf_reserve(p, L, cap, len, off, skip, kind);
}
uint64_t core_used(const tf_pstate* p, uint64_t L) { return tf_used(p, L); }
uint64_t core_tail(const tf_pstate* p, uint64_t L, uint64_t cap) { return tf_tail(p, L, cap); }
uint64_t core_head(const tf_pstate* p, uint64_t cap) { return tf_head(p, cap); }
