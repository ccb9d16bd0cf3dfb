// ring2.cu — device Ring^2: allocator, capture kernels, publish protocol,
// and the host consumer role. sm_100a only.
//
// Reference behaviour restated here (tapflow, pure Python):
//   capture()         hooks.py:281-324   -> capture_kernel (one launch)
//   _gather_compact   hooks.py:266-278   -> ordered compaction + 128-bit copy
//   reserve_payload   rings.py:286-319   -> leader CTA, tf_reserve (ring2_core.h)
//   publish           rings.py:321-353   -> last CTA: one coalesced 64-B post
//   poll_ready        rings.py:380-406   -> tf_ring_poll_ready (host)
//   release_payload   rings.py:408-431   -> tf_ring_release_payload (host)
//
// Placement rule learned on the box: while the staging D2H saturates PCIe,
// anything a kernel on the inference stream does with host memory (reads,
// system fences, scattered stores) waits behind that traffic. The capture
// kernel therefore reads only device memory and posts exactly one 64-byte
// descriptor (checksummed, no fence) to the mapped meta ring.
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_fp8.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <mutex>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <time.h>

#include "ring2_internal.h"

// ---------------------------------------------------------------------------
// errors
// ---------------------------------------------------------------------------
static thread_local std::string g_err;

void tf_set_error(const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
}

#define CUDA_TRY(expr)                                                     \
  do {                                                                     \
    cudaError_t _e = (expr);                                               \
    if (_e != cudaSuccess) {                                               \
      tf_set_error("%s: %s (%s:%d)", #expr, cudaGetErrorString(_e),        \
                   __FILE__, __LINE__);                                    \
      return TF_ERR_CUDA;                                                  \
    }                                                                      \
  } while (0)

extern "C" int tf_abi_version(void) { return TF_ABI_VERSION; }
extern "C" const char* tf_last_error(void) { return g_err.c_str(); }
extern "C" const char* tf_status_name(int s) {
  switch (s) {
    case TF_OK: return "ok";
    case TF_ERR_CONFIG: return "ConfigError";
    case TF_ERR_ALLOCATION: return "AllocationError";
    case TF_ERR_PAYLOAD_RING_FULL: return "PayloadRingFull";
    case TF_ERR_META_RING_FULL: return "MetaRingFull";
    case TF_ERR_OUT_OF_ORDER_RELEASE: return "OutOfOrderRelease";
    case TF_ERR_PROTOCOL: return "ProtocolError";
    case TF_ERR_META_MISMATCH: return "MetaMismatch";
    case TF_ERR_POLICY_UNDERESTIMATE: return "PolicyUnderestimate";
    case TF_ERR_STAGING_EXHAUSTED: return "StagingExhausted";
    case TF_ERR_HOOK_DISABLED: return "HookDisabled";
    case TF_ERR_VALUE: return "ValueError";
    case TF_ERR_CUDA: return "CudaError";
    case TF_ERR_TIMEOUT: return "Timeout";
    case TF_ERR_EMPTY: return "Empty";
  }
  return "unknown";
}
extern "C" int tf_device_count(int* out) {
  CUDA_TRY(cudaGetDeviceCount(out));
  return TF_OK;
}
extern "C" double tf_monotonic(void) {
  timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return double(ts.tv_sec) + 1e-9 * double(ts.tv_nsec);
}

extern "C" int tf_plan_reservation(uint64_t head, uint64_t tail, uint64_t used,
                                   uint64_t capacity, uint64_t length,
                                   uint64_t* offset, uint64_t* dead) {
  uint64_t o = 0, d = 0;
  int ok = tf_plan(head, tail, used, capacity, length, &o, &d);
  if (offset) *offset = o;
  if (dead) *dead = d;
  return ok;
}

// ---------------------------------------------------------------------------
// PTX memory-model helpers
// ---------------------------------------------------------------------------
namespace {

__device__ __forceinline__ uint64_t ld_relaxed_gpu(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t ld_relaxed_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_gpu(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__host__ __device__ __forceinline__ int64_t imin64(int64_t a, int64_t b) { return a < b ? a : b; }
__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Phase tracing of the capture kernel (experiment builds only, -DTF_TRACE):
// thread 0 of every CTA keeps its entry / offset-known / copy-done times in
// registers and stores them (plain stores, no contention) into a per-launch
// slot chosen by the capture sequence; the last CTA adds its publish time.
#ifdef TF_TRACE
constexpr int kTrLaunches = 64, kTrCtas = 1024;
__device__ unsigned long long g_stamp[kTrLaunches][kTrCtas][6];
__device__ unsigned long long g_pub[kTrLaunches][2];  // publish time, grid size
#endif

// streaming loads: source activations are read exactly once
template <int VW> struct VecT;
template <> struct VecT<16> { using T = uint4; };
template <> struct VecT<8> { using T = uint2; };
template <> struct VecT<4> { using T = uint32_t; };
template <> struct VecT<2> { using T = uint16_t; };
template <> struct VecT<1> { using T = uint8_t; };

template <int VW>
__device__ __forceinline__ typename VecT<VW>::T ld_stream(const uint8_t* p) {
  using T = typename VecT<VW>::T;
  if constexpr (VW == 16) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    return r;
  } else {
    return __ldg(reinterpret_cast<const T*>(p));
  }
}
template <int VW>
// evict-first ring stores: A/B on B200 (profiles/r02/stcs_ab/) 32 MiB
// 13.15 -> 12.80 us, 112 MiB 40.27 -> 39.64 us, model overhead unchanged
#ifndef TF_ST_CS
#define TF_ST_CS 1
#endif
__device__ __forceinline__ void st_vec(uint8_t* p, typename VecT<VW>::T v) {
  if constexpr (VW == 16 && TF_ST_CS) {
    // ring payload is read once, by the staging copy: stream it through L2
    // (evict-first) so it does not push the model's working set out
    asm volatile("st.global.cs.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y),
                 "r"(v.z), "r"(v.w)
                 : "memory");
  } else {
    *reinterpret_cast<typename VecT<VW>::T*>(p) = v;
  }
}

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kTableMax = 2048;
#ifndef TF_UNROLL
#define TF_UNROLL 8
#endif
constexpr int kUnroll = TF_UNROLL;
constexpr int kSeg = 32 * kUnroll;  // vector words per warp segment
#ifndef TF_SMEM_SPEC
#define TF_SMEM_SPEC 2
#endif
// COPY with 16-B words: segments 2..(1+kSmemSpec) of each warp are also
// fetched before the plan, into shared memory with cp.async
constexpr int kSmemSpec = TF_SMEM_SPEC;
constexpr int kSpecSmemBytes = kSmemSpec * 8 /*warps*/ * kSeg * 16;
#ifndef TF_CTAS_PER_SM
#define TF_CTAS_PER_SM 2
#endif
constexpr int kCtasPerSm = TF_CTAS_PER_SM;
// TF_CONTROLLER_CTA=1 (default): one extra CTA posts the descriptor and,
// after every copy CTA has counted itself into `readers` (a fire-and-forget
// reduction), commits the producer state while the copy CTAs copy.
// TF_CONTROLLER_CTA=0 (experiment build "noctl"): no extra CTA; each copy
// CTA counts itself with an atomic whose old value it inspects after its
// copy, and the last CTA to have read the snapshot commits. Measured slower
// on B200 (scripts/exp_fixed.cu variants 15 vs 39: the returning atomic's
// round trip lands on the critical path; 2.23 vs 2.87 us per 128 KiB launch).
#ifndef TF_CONTROLLER_CTA
#define TF_CONTROLLER_CTA 1
#endif
constexpr int kCtl = TF_CONTROLLER_CTA;

// ---------------------------------------------------------------------------
// element conversions (bit-exact with oracle/cast_oracle.c)
// ---------------------------------------------------------------------------
template <int DT> struct Elem;
template <> struct Elem<TF_F32> { static constexpr int W = 4; };
template <> struct Elem<TF_F16> { static constexpr int W = 2; };
template <> struct Elem<TF_BF16> { static constexpr int W = 2; };
template <> struct Elem<TF_F8E4M3> { static constexpr int W = 1; };
template <> struct Elem<TF_F8E5M2> { static constexpr int W = 1; };

template <int DT>
__device__ __forceinline__ float load_elem(const uint8_t* p) {
  if constexpr (DT == TF_F32) return *reinterpret_cast<const float*>(p);
  if constexpr (DT == TF_F16) return __half2float(*reinterpret_cast<const __half*>(p));
  if constexpr (DT == TF_BF16) return __bfloat162float(*reinterpret_cast<const __nv_bfloat16*>(p));
  return 0.f;
}
__device__ __forceinline__ float bits_to_f(int dt, uint32_t bits) {
  if (dt == TF_F16) { __half_raw h; h.x = (unsigned short)bits; return __half2float(__half(h)); }
  __nv_bfloat16_raw b; b.x = (unsigned short)bits; return __bfloat162float(__nv_bfloat16(b));
}
template <int DT>
__device__ __forceinline__ void store_elem(uint8_t* p, float v) {
  if constexpr (DT == TF_F32) *reinterpret_cast<float*>(p) = v;
  if constexpr (DT == TF_F16) *reinterpret_cast<__half*>(p) = __float2half_rn(v);
  if constexpr (DT == TF_BF16) *reinterpret_cast<__nv_bfloat16*>(p) = __float2bfloat16_rn(v);
  if constexpr (DT == TF_F8E4M3) {
    *reinterpret_cast<__nv_fp8_storage_t*>(p) =
        __nv_cvt_float_to_fp8(v, __NV_SATFINITE, __NV_E4M3);
  }
  if constexpr (DT == TF_F8E5M2) {
    *reinterpret_cast<__nv_fp8_storage_t*>(p) =
        __nv_cvt_float_to_fp8(v, __NV_SATFINITE, __NV_E5M2);
  }
}

// 8 input elements -> 8 floats (vector path, 16/32-byte aligned)
template <int DT>
__device__ __forceinline__ void load8(const uint8_t* p, float* f) {
  if constexpr (DT == TF_F32) {
    uint4 a = ld_stream<16>(p), b = ld_stream<16>(p + 16);
    f[0] = __uint_as_float(a.x); f[1] = __uint_as_float(a.y);
    f[2] = __uint_as_float(a.z); f[3] = __uint_as_float(a.w);
    f[4] = __uint_as_float(b.x); f[5] = __uint_as_float(b.y);
    f[6] = __uint_as_float(b.z); f[7] = __uint_as_float(b.w);
  } else {
    uint4 a = ld_stream<16>(p);
    uint32_t w[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      f[2 * i] = bits_to_f(DT, w[i] & 0xFFFFu);
      f[2 * i + 1] = bits_to_f(DT, w[i] >> 16);
    }
  }
}
// the same, from 16-B words already in registers (f32: two words)
template <int DT>
__device__ __forceinline__ void cvt8(const uint4* r, float* f) {
  if constexpr (DT == TF_F32) {
    f[0] = __uint_as_float(r[0].x); f[1] = __uint_as_float(r[0].y);
    f[2] = __uint_as_float(r[0].z); f[3] = __uint_as_float(r[0].w);
    f[4] = __uint_as_float(r[1].x); f[5] = __uint_as_float(r[1].y);
    f[6] = __uint_as_float(r[1].z); f[7] = __uint_as_float(r[1].w);
  } else {
    const uint32_t w[4] = {r[0].x, r[0].y, r[0].z, r[0].w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      f[2 * i] = bits_to_f(DT, w[i] & 0xFFFFu);
      f[2 * i + 1] = bits_to_f(DT, w[i] >> 16);
    }
  }
}
template <int DT>
__device__ __forceinline__ void store8(uint8_t* p, const float* f) {
  if constexpr (DT == TF_F32) {
    uint4 a = make_uint4(__float_as_uint(f[0]), __float_as_uint(f[1]),
                         __float_as_uint(f[2]), __float_as_uint(f[3]));
    uint4 b = make_uint4(__float_as_uint(f[4]), __float_as_uint(f[5]),
                         __float_as_uint(f[6]), __float_as_uint(f[7]));
    *reinterpret_cast<uint4*>(p) = a;
    *reinterpret_cast<uint4*>(p + 16) = b;
  } else if constexpr (DT == TF_F16 || DT == TF_BF16) {
    uint32_t w[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      unsigned short lo, hi;
      if constexpr (DT == TF_F16) {
        lo = __half_as_ushort(__float2half_rn(f[2 * i]));
        hi = __half_as_ushort(__float2half_rn(f[2 * i + 1]));
      } else {
        lo = __bfloat16_as_ushort(__float2bfloat16_rn(f[2 * i]));
        hi = __bfloat16_as_ushort(__float2bfloat16_rn(f[2 * i + 1]));
      }
      w[i] = uint32_t(lo) | (uint32_t(hi) << 16);
    }
    *reinterpret_cast<uint4*>(p) = make_uint4(w[0], w[1], w[2], w[3]);
  } else {
    // fp8: cvt.rn.satfinite.{e4m3,e5m2}x2.f32 packs (hi, lo)
    uint32_t w[2];
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      uint16_t a, b;
      if constexpr (DT == TF_F8E4M3) {
        asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(a) : "f"(f[4 * i + 1]), "f"(f[4 * i]));
        asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(b) : "f"(f[4 * i + 3]), "f"(f[4 * i + 2]));
      } else {
        asm("cvt.rn.satfinite.e5m2x2.f32 %0, %1, %2;" : "=h"(a) : "f"(f[4 * i + 1]), "f"(f[4 * i]));
        asm("cvt.rn.satfinite.e5m2x2.f32 %0, %1, %2;" : "=h"(b) : "f"(f[4 * i + 3]), "f"(f[4 * i + 2]));
      }
      w[i] = uint32_t(a) | (uint32_t(b) << 16);
    }
    *reinterpret_cast<uint2*>(p) = make_uint2(w[0], w[1]);
  }
}

// ---------------------------------------------------------------------------
// capture kernel
// ---------------------------------------------------------------------------
// Division by a launch-constant divisor as a multiply-high and a shift
// (the divisors -- segments per row, rows per keep unit, rows per outer
// index, copy CTAs -- are known on the host at launch; ncu attributed ~25 %
// of a decode-size capture's instructions to the divider). q = n / d for
// n < 2^31: mul = ceil(2^p / d) with p = 31 + ceil(log2 d), q = umulhi(n, mul)
// >> (p - 32); d == 1 is mul == 0.
struct FastDiv {
  uint32_t d, mul, shr;
};

struct CapParams {
  const uint8_t* src;
  int64_t outer, mid, row_bytes, s_outer, s_mid;
  const uint8_t* keep;
  const uint32_t* step_ptr;
  uint32_t step_imm, hook_id, flags, reduce_op;
  int64_t units, rpu;         // keep units and rows per unit
  int64_t out_row_bytes;
  int64_t row_elems;          // elements per row (cast/reduce)
  int64_t words_per_row;      // vector words (copy) / groups (cast) per row
  int keep_vec;               // keep[] is 16-B aligned
  // ring
  uint8_t* payload;
  uint64_t cap;
  uint64_t slots;
  uint8_t* meta;              // mapped host memory (descriptors only)
  const DevConsumer* dcons;
  DevCtl* ctl;
  uint64_t timeout_ns;
  uint8_t* done_flags;        // mapped host memory, kMaxFlagCtas per slot
  // launch-constant divisors (set_fastdiv); fd_ok: every dividend < 2^31
  FastDiv fd_spr, fd_rpu, fd_mid, fd_cg;
  uint32_t fd_ok;
  uint64_t* seal;             // mapped host word: descriptors below it are complete
};

enum { MODE_COPY = 0, MODE_CAST = 1, MODE_REDUCE = 2 };

// producer snapshot values (ring2_internal.h ProdSnap)
struct SnapVals {
  tf_pstate p;
  uint64_t mh, cseq, L, mt, L_phys, used, head, tail;
};

struct CapShared {
  uint32_t warp_sums[kWarps];
  uint32_t total;
  uint32_t status;
  uint64_t off;
  uint32_t is_last;
  uint32_t publish;
  uint32_t fast, fast_kind;   // fast-path plan (identical in every CTA)
  uint64_t fast_skip, fast_mh, fast_seq;
  tf_pstate fast_p;
  uint64_t old_L, old_L_phys, old_head;  // snapshot inputs of the fast plan
  uint64_t slot_idx;                      // meta slot of a published capture
  uint32_t flagmode;                      // completion via per-CTA flags
  SnapVals next;                          // last CTA: the next snapshot
  uint64_t desc[8];
  uint64_t* slot;
  uint32_t table[kTableMax];
};

__device__ __forceinline__ uint32_t count_nonzero_bytes(uint32_t w) {
  uint32_t nz = (((w & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | w) & 0x80808080u;
  return __popc(nz);
}
__device__ __forceinline__ uint32_t count_nonzero16(uint4 g) {
  return count_nonzero_bytes(g.x) + count_nonzero_bytes(g.y) + count_nonzero_bytes(g.z) +
         count_nonzero_bytes(g.w);
}

// keep[u, min(u+16, u1)) as 16 bytes (zero past u1): one 16-B load when the
// vector is aligned and the group is whole, else 16 independent predicated
// byte loads (issued together, one memory latency).
__device__ __forceinline__ uint4 load_keep16(const uint8_t* keep, int64_t u, int64_t u1, int vec) {
  if (vec && u + 16 <= u1) return *reinterpret_cast<const uint4*>(keep + u);
  uint32_t w[4] = {0u, 0u, 0u, 0u};
#pragma unroll
  for (int k = 0; k < 16; ++k)
    if (u + k < u1) w[k >> 2] |= uint32_t(keep[u + k] != 0) << (8 * (k & 3));
  return make_uint4(w[0], w[1], w[2], w[3]);
}

// Block-wide exclusive scan of one u32 per thread; returns the exclusive
// prefix, writes the total to sh.total.
template <int NWARPS = kWarps>
__device__ __forceinline__ uint32_t block_exclusive_scan(uint32_t v, CapShared& sh) {
  constexpr int kWarps = NWARPS;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    uint32_t y = __shfl_up_sync(0xffffffffu, x, d);
    if (lane >= d) x += y;
  }
  if (lane == 31) sh.warp_sums[warp] = x;
  __syncthreads();
  if (warp == 0) {
    uint32_t s = lane < kWarps ? sh.warp_sums[lane] : 0u;
    uint32_t t = s;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      uint32_t y = __shfl_up_sync(0xffffffffu, t, d);
      if (lane >= d) t += y;
    }
    if (lane < kWarps) sh.warp_sums[lane] = t - s;  // exclusive warp offsets
    if (lane == kWarps - 1) sh.total = t;
  }
  __syncthreads();
  return sh.warp_sums[warp] + x - v;
}

// Leader: reservation against the device view of the consumer cursors
// (rings.py:286-319; hooks.py:313-315: meta availability first, then payload).
__device__ void leader_reserve(const CapParams& P, uint64_t bytes, uint64_t rows) {
  DevCtl* c = P.ctl;
  const uint32_t mode = P.flags & TF_FULL_MASK;
  uint64_t len = tf_round_up16(bytes);
  c->captures += 1;
  uint64_t seq = ++c->capture_seq;
  c->plan_seq = seq;
  c->plan_bytes = bytes;
  c->plan_rows = rows;
  c->plan_len = len;
  c->plan_skip = 0;
  c->plan_kind = 0;
  if (len > P.cap) {  // rings.py:297-298 ValueError
    c->plan_status = TF_ERR_VALUE;
    c->errors |= TF_DEVERR_TOO_LARGE;
    c->drops += 1;
    c->drop_bytes += bytes;
    return;
  }
  uint64_t t0 = 0;
  bool stalled = false;
  for (;;) {
    uint64_t L = ld_relaxed_gpu(&P.dcons->L);
    uint64_t mtail = ld_relaxed_gpu(&P.dcons->meta_tail);
    bool meta_ok = (c->meta_head - mtail) < P.slots;
    uint32_t status = TF_ERR_META_RING_FULL;
    if (meta_ok) {
      tf_pstate p = c->p;
      uint64_t off, skip;
      uint32_t kind;
      if (tf_reserve(&p, L, P.cap, len, &off, &skip, &kind)) {
        c->p = p;
        c->plan_off = off;
        c->plan_skip = skip;
        c->plan_kind = kind;
        c->bytes_reserved += len;
        if (kind & TF_DESC_DEAD_SKIP) c->dead_created += skip;
        c->plan_status = TF_OK;
        if (stalled) c->stall_ns += globaltimer() - t0;
        return;
      }
      status = TF_ERR_PAYLOAD_RING_FULL;
    }
    if (mode == TF_FULL_WAIT) {  // completeness: stall in-step (simulator.py:384-393)
      uint64_t now = globaltimer();
      if (!stalled) {
        stalled = true;
        t0 = now;
        c->stall_events += 1;
        // every earlier capture on this stream has finished (this grid is
        // past griddepcontrol.wait): seal their descriptors, or a
        // TF_CAP_SEALED predecessor would wait for a post this capture
        // cannot make until the consumer frees its space
        if (P.seal)
          asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(P.seal), "l"(c->meta_head)
                       : "memory");
      } else if (now - t0 > P.timeout_ns) {
        c->stall_ns += now - t0;
        c->errors |= TF_DEVERR_TIMEOUT;
        c->drops += 1;
        c->drop_bytes += bytes;
        c->plan_status = TF_ERR_TIMEOUT;
        return;
      }
      __nanosleep(1000);
      continue;
    }
    if (mode == TF_FULL_DROP) {
      c->drops += 1;
      c->drop_bytes += bytes;
      c->errors |= TF_DEVERR_UNDERESTIMATE;
    }
    c->plan_status = status;
    return;
  }
}

__device__ __forceinline__ ulonglong2 ld_cg_v2(const uint64_t* p) {
  ulonglong2 v;
  asm volatile("ld.global.cg.v2.u64 {%0,%1}, [%2];" : "=l"(v.x), "=l"(v.y) : "l"(p));
  return v;
}

// Rewrite the snapshot replicas (ring2_internal.h ProdSnap); lanes
// [0, nlanes) of the caller's group share the work.
__device__ __forceinline__ void write_snap(DevCtl* c, const SnapVals& v, int lane, int nlanes) {
  for (int r = lane; r < kSnapReplicas; r += nlanes) {
    ProdSnap* q = &c->snap[r];
    q->V = v.p.V;
    q->reset_mark = v.p.reset_mark;
    q->reset_credit = v.p.reset_credit;
    q->meta_head = v.mh;
    q->L = v.L;
    q->meta_tail = v.mt;
    q->capture_seq = v.cseq;
    q->L_phys = v.L_phys;
    q->used = v.used;
    q->head = v.head;
    q->tail = v.tail;
  }
}

// Single thread, after any slow-path producer operation: snapshot the
// canonical state and the live consumer cursors (full 64-bit arithmetic).
__device__ void write_snap_ctl(const CapParams& P) {
  DevCtl* c = P.ctl;
  SnapVals v;
  v.p = c->p;
  v.mh = c->meta_head;
  v.cseq = c->capture_seq;
  v.L = ld_relaxed_gpu(&P.dcons->L);
  v.mt = ld_relaxed_gpu(&P.dcons->meta_tail);
  v.L_phys = v.L % P.cap;
  v.used = tf_used(&v.p, v.L);
  v.head = tf_head(&v.p, P.cap);
  v.tail = tf_tail(&v.p, v.L, P.cap);
  write_snap(c, v, 0, 1);
}

// x mod m through the 32-bit unit when both fit
__device__ __forceinline__ uint64_t umod64(uint64_t x, uint64_t m) {
  if ((x | m) >> 32 == 0) return (uint32_t)x % (uint32_t)m;
  return x % m;
}

__device__ __forceinline__ uint32_t atom_add_relaxed_gpu(uint32_t* p, uint32_t v) {
  uint32_t old;
  asm volatile("atom.add.relaxed.gpu.global.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ uint32_t atom_add_acqrel_gpu(uint32_t* p, uint32_t v) {
  uint32_t old;
  asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

struct SnapRegs {  // a={V,mark} b={credit,mh} l={L,mt} e={cseq,L_phys} u={used,head} t={tail,-}
  ulonglong2 a, b, l, e, u, t;
};
__device__ __forceinline__ void snap_load(const CapParams& P, SnapRegs& r) {
  const ProdSnap* q = &P.ctl->snap[blockIdx.x % kSnapReplicas];
  r.a = ld_cg_v2(&q->V);
  r.b = ld_cg_v2(&q->reset_credit);
  r.l = ld_cg_v2(&q->L);
  r.e = ld_cg_v2(&q->capture_seq);
  r.u = ld_cg_v2(&q->used);
  r.t = ld_cg_v2(&q->tail);
}
__device__ __forceinline__ bool fast_plan(const CapParams& P, const SnapRegs& r, uint64_t bytes,
                                          CapShared& sh) {
  const uint64_t len = tf_round_up16(bytes);
  if (len > P.cap) return false;
  const uint64_t mh = r.b.y, mt = r.l.y;
  if (mh - mt >= P.slots) return false;
  tf_pstate p;
  p.V = r.a.x;
  p.reset_mark = r.a.y;
  p.reset_credit = r.b.x;
  uint64_t off, skip;
  uint32_t kind;
  if (!tf_reserve_derived(&p, r.l.x, P.cap, len, r.u.x, r.u.y, r.t.x, &off, &skip, &kind))
    return false;
  sh.fast_p = p;
  sh.off = off;
  sh.fast_skip = skip;
  sh.fast_kind = kind;
  sh.fast_mh = mh;
  sh.fast_seq = r.e.x + 1;
  sh.old_L = r.l.x;
  sh.old_L_phys = r.e.y;
  sh.old_head = r.u.y;
  return true;
}

__device__ __forceinline__ void cpa16(uint32_t smem, const void* g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem), "l"(g) : "memory");
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cpa_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// Fast path, thread 0 of the publishing CTA: the 64-B descriptor of this
// capture. With completion flags (n_ctas > 0) it is posted as soon as the
// plan is known; the host takes the slot only when all n_ctas CTAs have set
// their completion byte.
__device__ void fast_desc(const CapParams& P, CapShared& sh, uint64_t bytes, uint64_t rows,
                          uint32_t step, uint32_t n_ctas, uint32_t pending) {
  tf_descriptor d;
  d.payload_offset = sh.off;
  d.payload_len = bytes;
  d.hook_id = P.hook_id;
  d.step_seq = step;
  d.ready_seq = TF_READY_SENTINEL;
  d.skip_before = sh.fast_skip;
  d.flags = sh.fast_kind | (n_ctas << TF_DESC_CTA_SHIFT) | pending;
  d.n_rows = (uint32_t)rows;
  d.capture_seq = sh.fast_seq;
  d.checksum = 0;
  uint64_t mh = sh.fast_mh;
  sh.publish = 0;
  if (!(P.flags & TF_CAP_DEFER_PUBLISH)) {
    d.ready_seq = mh;
    d.checksum = tf_desc_checksum(reinterpret_cast<const uint64_t*>(&d));
    sh.slot_idx = umod64(mh, P.slots);
    sh.slot = reinterpret_cast<uint64_t*>(P.meta + sh.slot_idx * TF_DESCRIPTOR_SIZE);
    sh.publish = 1;
    mh += 1;
  }
  const uint64_t* w = reinterpret_cast<const uint64_t*>(&d);
  for (int i = 0; i < 8; ++i) sh.desc[i] = w[i];
  sh.next.mh = mh;
}

// Fast path, thread 0 of the committing CTA, after the capture's copy: the
// result record, the canonical state and the next snapshot (derived
// incrementally: skip + len <= cap and L - old_L <= cap, so one conditional
// subtraction replaces each 64-bit modulo).
__device__ void fast_state(const CapParams& P, CapShared& sh, uint64_t bytes, uint64_t rows,
                           uint64_t L, uint64_t mt, uint64_t k0) {
  DevCtl* c = P.ctl;
  const uint64_t len = tf_round_up16(bytes), seq = sh.fast_seq;
  const uint64_t mh = sh.next.mh;
  {
    const uint64_t cap = P.cap;
    SnapVals& v = sh.next;
    v.p = sh.fast_p;
    v.cseq = seq;
    v.mt = mt;
    if (L < sh.old_L) L = sh.old_L;
    v.L = L;
    uint64_t lp = sh.old_L_phys + (L - sh.old_L);
    if (L - sh.old_L > cap) lp = L % cap;
    else if (lp >= cap) lp -= cap;
    v.L_phys = lp;
    uint64_t h = sh.old_head + sh.fast_skip + len;
    if (h >= cap) h -= cap;
    v.head = h;
    const uint64_t credit = tf_credit(&v.p, L);
    v.used = v.p.V - L - credit;
    uint64_t t = lp + credit;
    if (t >= cap) t -= cap;
    v.tail = t;
  }
  c->p = sh.fast_p;
  c->meta_head = mh;
  c->capture_seq = seq;
  c->plan_seq = seq;
  c->plan_bytes = bytes;
  c->plan_rows = rows;
  c->plan_len = len;
  c->plan_off = sh.off;
  c->plan_skip = sh.fast_skip;
  c->plan_kind = sh.fast_kind;
  c->plan_status = TF_OK;
  tf_capture_result& r = c->res;
  r.capture_seq = seq;
  r.status = TF_OK;
  r.n_rows = (uint32_t)rows;
  r.payload_offset = sh.off;
  r.payload_len = bytes;
  r.skip_before = sh.fast_skip;
  const tf_descriptor* d = reinterpret_cast<const tf_descriptor*>(sh.desc);
  r.ready_seq = d->ready_seq;
  r.desc = *d;
  r.desc.flags &= (1u << TF_DESC_CTA_SHIFT) - 1u;
  atomicAdd((unsigned long long*)&c->captures, 1ull);
  atomicAdd((unsigned long long*)&c->bytes_reserved, (unsigned long long)len);
  if (sh.fast_kind & TF_DESC_DEAD_SKIP)
    atomicAdd((unsigned long long*)&c->dead_created, (unsigned long long)sh.fast_skip);
  const uint64_t dt = globaltimer() - k0;
  c->last_kernel_ns = dt;
  atomicAdd((unsigned long long*)&c->kernel_ns, (unsigned long long)dt);
}

__device__ __forceinline__ void fence_acq_rel_sys() {
  asm volatile("fence.acq_rel.sys;" ::: "memory");
}
__device__ __forceinline__ void st_relaxed_sys_u8(uint8_t* p, uint8_t v) {
  asm volatile("st.relaxed.sys.global.u8 [%0], %1;" ::"l"(p), "h"((unsigned short)v) : "memory");
}
__device__ __forceinline__ void red_add_gpu(uint32_t* p, uint32_t v) {
  asm volatile("red.relaxed.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Non-leader CTAs wait for the leader's plan with exponential backoff: under
// completeness the leader may wait milliseconds for ring space, and a tight
// poll of one L2 line by hundreds of CTAs taxes the memory system the
// staging copy engine is reading from.
__device__ __forceinline__ void wait_plan(DevCtl* c) {
  uint32_t ns = 32;
  while (ld_acquire_gpu(&c->plan_flag) == 0) {
    __nanosleep(ns);
    ns = ns < 2048 ? ns * 2 : ns;
  }
}

// Last CTA, thread 0: build the descriptor and the result record; the
// caller posts the descriptor with one coalesced warp store.
__device__ void last_cta_prepare(const CapParams& P, CapShared& sh) {
  DevCtl* c = P.ctl;
  const uint32_t status = c->plan_status;
  const uint64_t dt = globaltimer() - c->k_t0;
  c->last_kernel_ns = dt;
  c->kernel_ns += dt;
  tf_descriptor d;
  d.payload_offset = c->plan_off;
  d.payload_len = c->plan_bytes;
  d.hook_id = P.hook_id;
  d.step_seq = P.step_ptr ? *P.step_ptr : P.step_imm;
  d.ready_seq = TF_READY_SENTINEL;
  d.skip_before = c->plan_skip;
  d.flags = c->plan_kind;
  d.n_rows = (uint32_t)c->plan_rows;
  d.capture_seq = c->plan_seq;
  d.checksum = 0;
  sh.publish = 0;
  if (status == TF_OK && !(P.flags & TF_CAP_DEFER_PUBLISH)) {
    const uint64_t seq = c->meta_head;
    d.ready_seq = seq;
    d.checksum = tf_desc_checksum(reinterpret_cast<const uint64_t*>(&d));
    sh.slot = reinterpret_cast<uint64_t*>(P.meta + (seq % P.slots) * TF_DESCRIPTOR_SIZE);
    sh.publish = 1;
    c->meta_head = seq + 1;
  }
  const uint64_t* w = reinterpret_cast<const uint64_t*>(&d);
  for (int i = 0; i < 8; ++i) sh.desc[i] = w[i];
  tf_capture_result& r = c->res;
  r.capture_seq = c->plan_seq;
  r.status = status;
  r.n_rows = (uint32_t)c->plan_rows;
  r.payload_offset = status == TF_OK ? c->plan_off : 0;
  r.payload_len = status == TF_OK ? c->plan_bytes : 0;
  r.skip_before = c->plan_skip;
  r.ready_seq = d.ready_seq;
  r.desc = d;
}

// 64-bit quotient through the 32-bit divider when both operands fit (the
// usual case: rows, segments and items of one capture are < 2^32)
__device__ __forceinline__ int64_t qdiv(int64_t a, int64_t b) {
  if (((uint64_t)a | (uint64_t)b) >> 32 == 0) return (int64_t)((uint32_t)a / (uint32_t)b);
  return a / b;
}

// a / b where b is the divisor `f` was built for (fast path when P.fd_ok)
__device__ __forceinline__ int64_t fdiv(const CapParams& P, int64_t a, const FastDiv& f,
                                        int64_t b) {
  if (P.fd_ok) return f.mul ? int64_t(__umulhi(uint32_t(a), f.mul) >> f.shr) : a;
  return qdiv(a, b);
}

__device__ __forceinline__ const uint8_t* row_src(const CapParams& P, int64_t row) {
  int64_t o = fdiv(P, row, P.fd_mid, P.mid);
  int64_t m = row - o * P.mid;
  return P.src + o * P.s_outer + m * P.s_mid;
}

// SS: shared-memory speculative segments per warp (COPY/16). They only pay
// off once the grid is capped and warps own several segments; below that
// (captures up to ~4.6 MiB) the launch uses SS = 0 and no dynamic shared
// memory (decode-size captures 0.34 us faster, profiles/r02/ablation_*).
template <int MODE, int VW, int IN_DT, int OUT_DT, int SS = kSmemSpec>
__global__ void __launch_bounds__(kThreads, kCtasPerSm) capture_kernel(CapParams P) {
  __shared__ CapShared sh;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // Copy CTA cb of cg owns a share of the work. (Controller builds: CTA 0
  // owns none; it posts the descriptor and commits the producer state.)
  const int cb = int(blockIdx.x) - kCtl, cg = int(gridDim.x) - kCtl;
  extern __shared__ __align__(16) uint4 spec_smem[];  // COPY/16: kSpecSmemBytes
  const int64_t U = P.units;
  const uint64_t t_entry = tid == 0 ? globaltimer() : 0;
#ifdef TF_TRACE
  uint64_t t_plan = 0, t_scan = 0, t_fast = 0, t_table = 0;
#define TSTAMP(v) do { if (tid == 0) v = globaltimer(); } while (0)
#else
#define TSTAMP(v) ((void)0)
#endif

#ifndef TF_ABL
#define TF_ABL 0
#endif
  // experiment builds: TF_ABL bit 1 = no keep scan, bit 2 = no publish
  // epilogue, bit 4 = no snapshot (fixed offset 0), 8 = no descriptor post,
  // 16 = no snapshot rewrite, 32 = no state commit
  if (TF_ABL & 1) P.keep = nullptr;
  // PDL: let the next kernel on the stream get scheduled now; it still waits
  // for this grid's completion before touching memory. Then wait for the
  // previous kernel (it may have produced the source rows, and the previous
  // capture wrote the producer snapshot). No-ops without the launch attribute.
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
#ifdef TF_TRACE
  // phase stamps start when the CTA may touch memory (a PDL-launched CTA
  // can be resident long before that)
  const uint64_t t_go = tid == 0 ? globaltimer() : 0;
#endif
  // Issue the producer-snapshot and step loads first: their latency hides
  // behind the keep scan (step is consumed only by the publishing CTA).
  SnapRegs sr;
  uint32_t step = 0;
  uint64_t L_now = 0, mt_now = 0;  // consumer cursors for the next snapshot
  if (tid == 0 && !(TF_ABL & 4)) {
    snap_load(P, sr);
    step = P.step_ptr ? *P.step_ptr : P.step_imm;
    if (!kCtl) {  // only the committing CTA uses them; any older L is conservative
      L_now = ld_relaxed_gpu(&P.dcons->L);
      mt_now = ld_relaxed_gpu(&P.dcons->meta_tail);
    }
  }
  // The keep bytes of a small keep vector are loaded before the speculative
  // segment: memory requests leave the SM roughly in issue order, and the
  // plan (which waits on them) must not queue behind megabytes of reads.
  // <= 256 keep units (request keep, or the token rows of a decode step):
  // one byte per thread, ranks by warp ballots, the whole rank table in
  // shared memory
  const bool small = P.keep && U <= kThreads;
  // <= 32 keep units (a request keep, or the token rows of a small decode
  // step): every warp loads the same 32 keep bytes and ranks them with its
  // own ballot, so no block barrier is needed before the plan
  const bool tiny = small && U <= 32;
  const int kidx = tiny ? lane : tid;
  const uint32_t kbyte = (small && kidx < U) ? P.keep[kidx] : 0u;
  // COPY: speculatively load this warp's first segment of the
  // grid-interleaved order assuming every unit is kept (identity row map),
  // so the source read overlaps the keep/snapshot round trip; used only if
  // the keep scan confirms it.
  using CV = typename VecT<MODE == MODE_COPY ? VW : 16>::T;
  CV v[kUnroll];
  int64_t spec_s = -1;
  // rows shorter than a quarter warp segment (< 1 KiB of 16-B words) are
  // packed several per segment (below); that path loads after the plan, so
  // it takes no speculation (at 1 KiB rows the speculative unpacked path
  // measured faster: 16.6 vs 17.5 us for 16 MiB; at 256 B rows packing is
  // 2.3x faster)
  const bool packable = MODE == MODE_COPY && 4 * P.words_per_row < kSeg && !(TF_ABL & 512);
  if constexpr (MODE == MODE_COPY) {
    if (!(TF_ABL & 256) && !packable && (!P.keep || U <= kThreads)) {
      const int64_t spr0 = (P.words_per_row + kSeg - 1) / kSeg;
      const int64_t s0 = int64_t(cb) * kWarps + warp;
#ifndef TF_SPEC_WARP0
#define TF_SPEC_WARP0 1
#endif
      // (TF_SPEC_WARP0=0: warp 0, which runs the plan, skips the speculative
      // load so its memory queue stays empty; A/B builds)
      if (cb >= 0 && (TF_SPEC_WARP0 || warp != 0) && s0 < U * P.rpu * spr0) {
        const int64_t j0 = fdiv(P, s0, P.fd_spr, spr0);
        const int64_t k0 = (s0 - j0 * spr0) * kSeg;
        const int64_t k1 = imin64(k0 + kSeg, P.words_per_row);
        const uint8_t* src = row_src(P, j0);
#pragma unroll
        for (int i = 0; i < kUnroll; ++i) {
          int64_t k = k0 + lane + i * 32;
          if (k < k1) v[i] = ld_stream<VW>(src + k * VW);
        }
        spec_s = s0;
        if constexpr (VW == 16 && SS > 0) {
          // the warp's next segments of the grid-interleaved order, into its
          // shared-memory slots (each lane later reads back its own words)
          const int64_t sstep = int64_t(cg) * kWarps;
          const int64_t all = U * P.rpu * spr0;
#pragma unroll
          for (int t = 0; t < SS; ++t) {
            const int64_t sn = s0 + (t + 1) * sstep;
            if (sn < all) {
              const int64_t jn = fdiv(P, sn, P.fd_spr, spr0);
              const int64_t kn0 = (sn - jn * spr0) * kSeg;
              const int64_t kn1 = imin64(kn0 + kSeg, P.words_per_row);
              const uint8_t* srcn = row_src(P, jn);
              uint4* slot = spec_smem + (size_t(t) * kWarps + warp) * kSeg;
#pragma unroll
              for (int i = 0; i < kUnroll; ++i) {
                int64_t k = kn0 + lane + i * 32;
                if (k < kn1)
                  cpa16(static_cast<uint32_t>(__cvta_generic_to_shared(slot + lane + i * 32)),
                        srcn + k * 16);
              }
            }
          }
          cpa_commit();
        }
      }
    }
  }

  // ---- 1. ordered compaction: count kept units (batch order, no atomics) ----
  // Each thread owns a run of whole 16-unit groups; the first group stays
  // in registers for the rank table below (one keep load per thread in the
  // common case of <= 4096 units).
  int64_t u0 = 0, u1 = 0;
  uint32_t mycnt = 0, mybase = 0;
  uint4 g0 = make_uint4(0u, 0u, 0u, 0u);
  uint64_t K;
  // <= 32 keep units (request keep): one warp, one coalesced load, ranks by
  // ballot; the whole rank table is built here and indexed from rank 0
  bool prefix = !P.keep;  // kept units are exactly units [0, K): identity map
  if (tiny) {
    const uint32_t m = __ballot_sync(0xffffffffu, kbyte != 0);
    const uint32_t tot = __popc(m);
    if (warp == 0 && kbyte) sh.table[__popc(m & ((1u << lane) - 1u))] = uint32_t(lane);
    K = tot;
    prefix = m == (tot == 32 ? 0xffffffffu : (1u << tot) - 1u);  // kept units are [0, K)
    TSTAMP(t_scan);
  } else if (small) {
    const uint32_t m = __ballot_sync(0xffffffffu, kbyte != 0);
    if (lane == 0) sh.warp_sums[warp] = __popc(m);
    __syncthreads();
    uint32_t base = 0, tot = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
      const uint32_t c = sh.warp_sums[w];
      base += w < warp ? c : 0u;
      tot += c;
    }
    if (kbyte) sh.table[base + __popc(m & ((1u << lane) - 1u))] = (uint32_t)tid;
    K = tot;
    // a prefix of ones (e.g. a graph-padded token layout) keeps the identity
    // row map, so the speculative segments stay valid; the block-wide AND is
    // taken at the table barrier below (one barrier fewer on this path)
    prefix = tid >= U || ((kbyte != 0) == (uint32_t(tid) < tot));
    TSTAMP(t_scan);
  } else if (P.keep) {
    int64_t per = (U + kThreads - 1) / kThreads;
    per = (per + 15) & ~int64_t(15);
    u0 = imin64(int64_t(tid) * per, U);
    u1 = imin64(u0 + per, U);
    if (u0 < u1) {
      g0 = load_keep16(P.keep, u0, u1, P.keep_vec);
      mycnt = count_nonzero16(g0);
#pragma unroll 1
      for (int64_t u = u0 + 16; u < u1; u += 16)
        mycnt += count_nonzero16(load_keep16(P.keep, u, u1, P.keep_vec));
    }
    mybase = block_exclusive_scan(mycnt, sh);
    K = sh.total;
    TSTAMP(t_scan);
  } else {
    K = (uint64_t)U;
  }
  const uint64_t n_rows = K * (uint64_t)P.rpu;
  if (n_rows == 0) {  // hooks.py:309-311 nothing kept: identity, no descriptor
    if (blockIdx.x == 0 && tid == 0) {
      tf_capture_result& r = P.ctl->res;
      r.capture_seq = 0;
      r.status = TF_OK;
      r.n_rows = 0;
      r.payload_len = 0;
      r.ready_seq = TF_READY_SENTINEL;
    }
    return;
  }
  const uint64_t out_bytes = n_rows * (uint64_t)P.out_row_bytes;

  // ---- 2. reservation: fast path in every CTA, else leader election ----
  // (the leader's reservation runs while the others prefetch)
  bool leader = false, fast = false;
  uint32_t readers_before = 0;  // thread 0: CTAs that had read the snapshot before this one
  if (tid == 0) {
    if (TF_ABL & 4) {
      fast = true;
      sh.off = 0;
    } else {
      fast = fast_plan(P, sr, out_bytes, sh);
    }
    sh.fast = fast;
    TSTAMP(t_fast);
    if (fast) {
      sh.status = TF_OK;
      // completion flags: every CTA reports; CTA 0 posts the descriptor now
      sh.flagmode = cg <= kMaxFlagCtas && P.done_flags != nullptr;
      if (sh.flagmode) {
        // snapshot consumed (its values fed fast_plan above). The old value
        // is needed only after the copy, so the round trip is hidden.
        if (kCtl) red_add_gpu(&P.ctl->readers, 1u);
        else readers_before = atom_add_relaxed_gpu(&P.ctl->readers, 1u);
        sh.publish = !(P.flags & TF_CAP_DEFER_PUBLISH);  // every CTA reports
        sh.slot_idx = umod64(sh.fast_mh, P.slots);
      }
      // (every CTA builds it: whichever commits needs it; CTA 0 posts it)
      if (!kCtl || blockIdx.x == 0 || !sh.flagmode) {
        // sealed: completion follows from stream order (TF_CAP_SEALED), the
        // copy CTAs report nothing
        const bool sealed = sh.flagmode && (P.flags & TF_CAP_SEALED);
        fast_desc(P, sh, out_bytes, n_rows, step,
                  sh.flagmode && !sealed ? uint32_t(cg) : 0u, sealed ? TF_DESC_PENDING : 0u);
      }
    } else {
      sh.flagmode = 0;
      uint32_t t = atomicAdd(&P.ctl->arrive, 1u);
      leader = (t == 0);
      if (leader) {
        P.ctl->k_t0 = t_entry;
        leader_reserve(P, out_bytes, n_rows);
        __threadfence();
        st_release_gpu(&P.ctl->plan_flag, 1u);
      }
    }
  }

  // ---- 3. this CTA's slice of the output (independent of the offset) ----
  // packed: rows of < kSeg/4 words, rps whole rows per warp segment (only
  // with a global rank table, i.e. the grid-interleaved order)
  const bool packed = packable && (small || !P.keep);
  const int64_t rps = packed ? kSeg / P.words_per_row : 1;
  int64_t items, spr = 1;
  if constexpr (MODE == MODE_REDUCE) {
    items = (int64_t)n_rows;
  } else {
    spr = (P.words_per_row + kSeg - 1) / kSeg;
    items = packed ? qdiv((int64_t)n_rows + rps - 1, rps) : (int64_t)n_rows * spr;
  }
  const int64_t chunk = fdiv(P, items + cg - 1, P.fd_cg, cg);
  const int64_t i0 = cb < 0 ? items : imin64(int64_t(cb) * chunk, items);
  const int64_t i1 = imin64(i0 + chunk, items);
  const int64_t j_lo = fdiv(P, i0, P.fd_spr, spr);
  const int64_t r_lo = fdiv(P, j_lo, P.fd_rpu, P.rpu);
  const int64_t tbase = small ? 0 : r_lo;  // rank of sh.table[0]
  if (P.keep && !small && i0 < i1) {
    const int64_t r_hi = fdiv(P, fdiv(P, i1 - 1, P.fd_spr, spr), P.fd_rpu, P.rpu);
    // rank -> unit table for the ranks this CTA touches
    if ((int64_t)mybase <= r_hi && (int64_t)(mybase + mycnt) > r_lo) {
      int64_t rank = mybase;
      for (int64_t u = u0; u < u1 && rank <= r_hi; u += 16) {
        const uint4 g = u == u0 ? g0 : load_keep16(P.keep, u, u1, P.keep_vec);
        const uint32_t gw[4] = {g.x, g.y, g.z, g.w};
#pragma unroll
        for (int k = 0; k < 16; ++k) {
          if ((gw[k >> 2] >> (8 * (k & 3))) & 0xFFu) {
            if (rank >= r_lo && rank <= r_hi) sh.table[rank - r_lo] = (uint32_t)(u + k);
            ++rank;
          }
        }
      }
    }
  }
  prefix = __syncthreads_and(prefix) != 0;  // (uniform unless the ballot path ran)
  TSTAMP(t_table);
  if (sh.flagmode && blockIdx.x == 0 && sh.publish && warp == 0 && lane < 8)
    sh.slot[lane] = sh.desc[lane];  // early post; the host waits for the flags
  // Work order. With a global rank table (small keep, or no keep) the warps
  // of all CTAs walk the segments grid-interleaved, so at any moment the
  // active reads and writes cover one contiguous window of the source and
  // the ring (DRAM page locality, like a grid-stride copy); otherwise each
  // CTA walks its own contiguous slice [i0, i1) whose ranks its table holds.
  const bool inter = (small || !P.keep) && !(TF_ABL & 64);
  const int64_t s_end = inter ? items : i1;
  const int64_t s_first = cb < 0 ? s_end : inter ? int64_t(cb) * kWarps + warp : i0 + warp;
  const int64_t s_step = inter ? int64_t(cg) * kWarps : kWarps;

  // Controller, fast path: commit the allocator state, the result record and
  // the next snapshot as soon as every CTA has read the current snapshot,
  // while the copy CTAs copy; then leave (it owns no payload).
  if (kCtl && sh.flagmode && cb < 0) {
    if (tid == 0) {
      L_now = ld_relaxed_gpu(&P.dcons->L);
      mt_now = ld_relaxed_gpu(&P.dcons->meta_tail);
      uint32_t ns = 32;
      while (ld_acquire_gpu(&P.ctl->readers) < gridDim.x) {
        __nanosleep(ns);
        ns = ns < 256 ? ns * 2 : ns;
      }
      fast_state(P, sh, out_bytes, n_rows, L_now, mt_now, t_entry);
      P.ctl->readers = 0;  // every CTA has read: re-armed for the next launch
    }
    __syncthreads();
    if (warp == 1) write_snap(P.ctl, sh.next, lane, 32);  // next launch's snapshot
#ifdef TF_TRACE
    if (tid == 0) {
      const int slot = int(sh.fast_seq % kTrLaunches);
      g_pub[slot][0] = globaltimer();
      g_pub[slot][1] = gridDim.x;
    }
#endif
    return;
  }
  auto row_of = [&](int64_t j) -> int64_t {
    int64_t r = fdiv(P, j, P.fd_rpu, P.rpu);
    int64_t sub = j - r * P.rpu;
    int64_t unit = P.keep ? (int64_t)sh.table[r - tbase] : r;
    return unit * P.rpu + sub;
  };

  if constexpr (MODE == MODE_COPY) {
   if (packed) {
    // Short rows: segment s holds rows [s*rps, s*rps + rps) back to back,
    // so lanes stay busy and the ring stores stay one contiguous span
    // (COPY output rows are the source rows, packed). Each lane finds its
    // row and column with a 32-bit division by the row's word count.
    if (!sh.fast) {
      if (tid == 0) {
        if (!leader)
          wait_plan(P.ctl);
        sh.status = *((volatile uint32_t*)&P.ctl->plan_status);
        sh.off = *((volatile uint64_t*)&P.ctl->plan_off);
      }
      __syncthreads();
    }
    if (sh.status == TF_OK) {
      const uint32_t wpr = (uint32_t)P.words_per_row;
      uint8_t* dst_base = P.payload + sh.off;
      for (int64_t s = s_first; s < s_end; s += s_step) {
        const int64_t row0 = s * rps;
        const int64_t nw = imin64(rps, (int64_t)n_rows - row0) * (int64_t)wpr;
#pragma unroll
        for (int i = 0; i < kUnroll; ++i) {
          const uint32_t w = uint32_t(lane + i * 32);
          if (w < nw) {
            const uint32_t rr = w / wpr;
            v[i] = ld_stream<VW>(row_src(P, row_of(row0 + rr)) + int64_t(w - rr * wpr) * VW);
          }
        }
        uint8_t* dst = dst_base + row0 * P.out_row_bytes;
#pragma unroll
        for (int i = 0; i < kUnroll; ++i) {
          const uint32_t w = uint32_t(lane + i * 32);
          if (w < nw) st_vec<VW>(dst + int64_t(w) * VW, v[i]);
        }
      }
    }
   } else {
    const int64_t wpr = P.words_per_row;
    // first segment: the speculative load when every unit was kept, else
    // load it now (before the offset is known on the slow path)
    int64_t s = s_first;
    int64_t k0 = 0, k1 = 0, j = 0;
    if (s < s_end) {
      j = fdiv(P, s, P.fd_spr, spr);
      k0 = (s - j * spr) * kSeg;
      k1 = imin64(k0 + kSeg, wpr);
      if (!(spec_s == s && prefix)) {
        const uint8_t* src = row_src(P, row_of(j));
#pragma unroll
        for (int i = 0; i < kUnroll; ++i) {
          int64_t k = k0 + lane + i * 32;
          if (k < k1) v[i] = ld_stream<VW>(src + k * VW);
        }
      }
    }
    if (!sh.fast) {  // uniform: sh.fast was set before the table barrier
      if (tid == 0) {
        if (!leader)
          wait_plan(P.ctl);
        sh.status = *((volatile uint32_t*)&P.ctl->plan_status);
        sh.off = *((volatile uint64_t*)&P.ctl->plan_off);
      }
      __syncthreads();
    }
#ifdef TF_TRACE
    if (tid == 0) t_plan = globaltimer();
#endif
    // the shared-memory speculation holds iff the register one does (same
    // identity map, same interleaved order)
    const bool smem_ok = VW == 16 && SS > 0 && spec_s == s && prefix;
    if (sh.status == TF_OK && s < s_end) {
      uint8_t* dst_base = P.payload + sh.off;
      int it = 0;
      for (;;) {
        uint8_t* dst = dst_base + j * P.out_row_bytes;
#pragma unroll
        for (int i = 0; i < kUnroll; ++i) {
          int64_t k = k0 + lane + i * 32;
          if (k < k1) st_vec<VW>(dst + k * VW, v[i]);
        }
        s += s_step;
        ++it;
        if (s >= s_end) break;
        j = fdiv(P, s, P.fd_spr, spr);
        k0 = (s - j * spr) * kSeg;
        k1 = imin64(k0 + kSeg, wpr);
        if (smem_ok && it <= SS) {
          if constexpr (VW == 16 && SS > 0) {
            cpa_wait_all();
            const uint4* slot = spec_smem + (size_t(it - 1) * kWarps + warp) * kSeg;
#pragma unroll
            for (int i = 0; i < kUnroll; ++i) {
              int64_t k = k0 + lane + i * 32;
              if (k < k1) v[i] = slot[lane + i * 32];
            }
          }
        } else {
          const uint8_t* src = row_src(P, row_of(j));
#pragma unroll
          for (int i = 0; i < kUnroll; ++i) {
            int64_t k = k0 + lane + i * 32;
            if (k < k1) v[i] = ld_stream<VW>(src + k * VW);
          }
        }
      }
    }
    if constexpr (VW == 16 && SS > 0) cpa_wait_all();  // no copy left in flight
   }
  } else {
    if (tid == 0 && !fast) {
      if (!leader)
        wait_plan(P.ctl);
      sh.status = *((volatile uint32_t*)&P.ctl->plan_status);
      sh.off = *((volatile uint64_t*)&P.ctl->plan_off);
    }
    __syncthreads();
    if (sh.status == TF_OK && s_first < s_end) {
      uint8_t* dst_base = P.payload + sh.off;
      if constexpr (MODE == MODE_CAST) {
        // VW == 8: groups of 8 elements; VW == 1: single elements
        constexpr int WI = Elem<IN_DT>::W, WO = Elem<OUT_DT>::W;
        const int64_t wpr = P.words_per_row;
        for (int64_t s = s_first; s < s_end; s += s_step) {
          const int64_t j = fdiv(P, s, P.fd_spr, spr);
          const int64_t k0 = (s - j * spr) * kSeg;
          const int64_t k1 = imin64(k0 + kSeg, wpr);
          const uint8_t* src = row_src(P, row_of(j));
          uint8_t* dst = dst_base + j * P.out_row_bytes;
          if constexpr (VW == 8) {
            // the segment's loads all in flight before any conversion (as
            // the copy path: ~64 KiB of reads outstanding per SM)
            constexpr int NR = IN_DT == TF_F32 ? 2 : 1;  // 16-B words per 8 elements
            uint4 raw[kUnroll][NR];
#pragma unroll
            for (int i = 0; i < kUnroll; ++i) {
              int64_t k = k0 + lane + i * 32;
              if (k < k1) {
#pragma unroll
                for (int q = 0; q < NR; ++q) raw[i][q] = ld_stream<16>(src + k * 8 * WI + 16 * q);
              }
            }
#pragma unroll
            for (int i = 0; i < kUnroll; ++i) {
              int64_t k = k0 + lane + i * 32;
              if (k < k1) {
                float f[8];
                cvt8<IN_DT>(raw[i], f);
                store8<OUT_DT>(dst + k * 8 * WO, f);
              }
            }
          } else {
            for (int i = 0; i < kUnroll; ++i) {
              int64_t k = k0 + lane + i * 32;
              if (k < k1) store_elem<OUT_DT>(dst + k * WO, load_elem<IN_DT>(src + k * WI));
            }
          }
        }
      } else {
        // MODE_REDUCE: one warp per row, fp64 accumulation, f32 outputs
        constexpr int WI = Elem<IN_DT>::W;
        const int64_t H = P.row_elems;
        for (int64_t j = s_first; j < s_end; j += s_step) {
          const uint8_t* src = row_src(P, row_of(j));
          double sum = 0.0, sq = 0.0;
          float mn = __int_as_float(0x7f800000), mx = -__int_as_float(0x7f800000), amax = 0.f;
          if (VW == 8) {
            const int64_t G8 = H / 8;
            constexpr int NR = IN_DT == TF_F32 ? 2 : 1;
            constexpr int RU = IN_DT == TF_F32 ? kUnroll / 2 : kUnroll;  // loads in flight
            for (int64_t g0 = lane; g0 < G8; g0 += 32 * RU) {
              uint4 raw[RU][NR];
#pragma unroll
              for (int u = 0; u < RU; ++u) {
                const int64_t g = g0 + int64_t(u) * 32;
                if (g < G8) {
#pragma unroll
                  for (int q = 0; q < NR; ++q) raw[u][q] = ld_stream<16>(src + g * 8 * WI + 16 * q);
                }
              }
#pragma unroll
              for (int u = 0; u < RU; ++u) {
                if (g0 + int64_t(u) * 32 < G8) {
                  float f[8];
                  cvt8<IN_DT>(raw[u], f);
#pragma unroll
                  for (int e = 0; e < 8; ++e) {
                    sum += (double)f[e];
                    sq += (double)f[e] * (double)f[e];
                    mn = fminf(mn, f[e]);
                    mx = fmaxf(mx, f[e]);
                    amax = fmaxf(amax, fabsf(f[e]));
                  }
                }
              }
            }
          } else {
            for (int64_t e = lane; e < H; e += 32) {
              float x = load_elem<IN_DT>(src + e * WI);
              sum += (double)x;
              sq += (double)x * (double)x;
              mn = fminf(mn, x);
              mx = fmaxf(mx, x);
              amax = fmaxf(amax, fabsf(x));
            }
          }
#pragma unroll
          for (int d = 16; d > 0; d >>= 1) {
            sum += __shfl_xor_sync(0xffffffffu, sum, d);
            sq += __shfl_xor_sync(0xffffffffu, sq, d);
            mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, d));
            mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, d));
            amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, d));
          }
          if (lane == 0) {
            float* o = reinterpret_cast<float*>(dst_base + j * P.out_row_bytes);
            switch (P.reduce_op) {
              case TF_RED_MEAN: o[0] = (float)(sum / (double)H); break;
              case TF_RED_L2: o[0] = (float)sqrt(sq); break;
              case TF_RED_ABSMAX: o[0] = amax; break;
              case TF_RED_RMS: o[0] = (float)sqrt(sq / (double)H); break;
              default:
                o[0] = (float)(sum / (double)H);
                o[1] = (float)sqrt(sq);
                o[2] = mn;
                o[3] = mx;
            }
          }
        }
      }
    }
  }

  // ---- 4. completion ----
  if (TF_ABL & 2) return;
  __syncthreads();
  if (sh.flagmode) {
    // Fast path: each copy CTA orders its payload stores before its
    // completion byte (the host takes the descriptor the controller posted
    // once every byte is set). The controller committed the producer state
    // meanwhile. No last-CTA election, no round trip on the critical path.
    if (tid == 0) {
      if (sh.publish && cb >= 0 && !(P.flags & TF_CAP_SEALED)) {
#if TF_FLAG_FENCE_SYS
        fence_acq_rel_sys();
#else
        // gpu scope, as the last-CTA publish: the payload is in L2 before
        // the byte leaves, and the D2H copy engine reads through L2
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
#endif
        st_relaxed_sys_u8(P.done_flags + sh.slot_idx * kMaxFlagCtas + cb, 1);
      }
      if (!kCtl && readers_before == uint32_t(cg) - 1) {
        // the last CTA to read the snapshot: every CTA of this launch holds
        // its plan, so the producer state, the result record and the next
        // launch's snapshot can be written (the next launch reads them only
        // after this grid completes: stream order / griddepcontrol.wait)
        fast_state(P, sh, out_bytes, n_rows, L_now, mt_now, t_entry);
        P.ctl->readers = 0;
        write_snap(P.ctl, sh.next, 0, 1);
      }
    }
#ifdef TF_TRACE
    if (tid == 0 && blockIdx.x < kTrCtas) {
      const int slot = int(sh.fast_seq % kTrLaunches);
      g_stamp[slot][blockIdx.x][0] = t_go;
      g_stamp[slot][blockIdx.x][1] = t_plan;
      g_stamp[slot][blockIdx.x][2] = globaltimer();
      g_stamp[slot][blockIdx.x][3] = t_scan;
      g_stamp[slot][blockIdx.x][4] = t_fast;
      g_stamp[slot][blockIdx.x][5] = t_table;
    }
#endif
    return;
  }
  if (tid == 0) {
    // consumer cursors for the next snapshot, loaded while the fence and the
    // done count are in flight (any older L is conservative)
    L_now = ld_relaxed_gpu(&P.dcons->L);
    mt_now = ld_relaxed_gpu(&P.dcons->meta_tail);
#ifdef TF_TRACE
    {
      const int slot = sh.fast ? int(sh.fast_seq % kTrLaunches) : kTrLaunches - 1;
      if (blockIdx.x < kTrCtas) {
        g_stamp[slot][blockIdx.x][0] = t_go;
        g_stamp[slot][blockIdx.x][1] = t_plan;
        g_stamp[slot][blockIdx.x][2] = globaltimer();
        g_stamp[slot][blockIdx.x][3] = t_scan;
        g_stamp[slot][blockIdx.x][4] = t_fast;
        g_stamp[slot][blockIdx.x][5] = t_table;
      }
    }
#endif
    // release: the CTA's payload stores (ordered by the barrier above)
    // before the count; acquire: the last CTA sees every other CTA's
    uint32_t t = atom_add_acqrel_gpu(&P.ctl->done, 1u);
    sh.is_last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (sh.is_last) {
    if (tid == 0) {
      if (sh.fast) {
        if (!(TF_ABL & 32)) fast_state(P, sh, out_bytes, n_rows, L_now, mt_now, t_entry);
      } else {
        last_cta_prepare(P, sh);
        write_snap_ctl(P);
      }
    }
    __syncthreads();
    // one coalesced 64-byte post of the descriptor, no system fence: the
    // host verifies the checksum before it trusts the slot
    if (!(TF_ABL & 8) && sh.publish && warp == 0 && lane < 8) sh.slot[lane] = sh.desc[lane];
    if (!(TF_ABL & 16) && sh.fast && warp == 1)
      write_snap(P.ctl, sh.next, lane, 32);  // next launch's snapshot
    if (tid == 0) {  // re-arm the handshake for the next launch on this stream
      P.ctl->arrive = 0;
      P.ctl->done = 0;
      P.ctl->plan_flag = 0;  // visible to the next launch (kernel boundary)
#ifdef TF_TRACE
      const int slot = sh.fast ? int(sh.fast_seq % kTrLaunches) : kTrLaunches - 1;
      g_pub[slot][0] = globaltimer();
      g_pub[slot][1] = gridDim.x;
#endif
    }
  }
}

// Rejected copy-path variants (measured slower on B200) are
// compiled only into experiment builds (-DTF_COPY_VARIANTS).
#ifdef TF_COPY_VARIANTS
// ---------------------------------------------------------------------------
// TMA bulk-copy capture (COPY, 16-B aligned rows): global -> smem -> ring
// with cp.async.bulk. One CTA per SM, kTmaStages x 32 KiB stages. The
// loads of the first stages are issued before the reservation is known
// (the source read does not depend on the ring offset), so the leader's
// allocator round trip hides behind data already in flight.
// ---------------------------------------------------------------------------
constexpr int kTmaThreads = 128;
constexpr int kTmaWarps = kTmaThreads / 32;
constexpr int kTmaTile = 32 * 1024;
constexpr int kTmaStages = 6;
constexpr int kTmaSmem = kTmaTile * kTmaStages;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  uint32_t done = 0;
  do {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(phase)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ void bulk_load(void* smem_dst, const void* gsrc, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(smem_dst)),
      "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void bulk_store(void* gdst, const void* smem_src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(smem_u32(smem_src)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

__global__ void __launch_bounds__(kTmaThreads, 1) capture_tma_kernel(CapParams P) {
  extern __shared__ __align__(128) uint8_t tiles[];
  __shared__ CapShared sh;
  __shared__ __align__(8) uint64_t full[kTmaStages];
  const int tid = threadIdx.x;
  const int64_t U = P.units;
  const uint64_t t_entry = tid == 0 ? globaltimer() : 0;
  if (tid == 0) {
    for (int s = 0; s < kTmaStages; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }

  // ---- 1. ordered compaction (same as capture_kernel) ----
  int64_t u0 = 0, u1 = 0;
  uint32_t mycnt = 0, mybase = 0;
  uint64_t K;
  if (P.keep) {
    int64_t per = (U + kTmaThreads - 1) / kTmaThreads;
    if (P.keep_vec) per = (per + 15) & ~int64_t(15);
    u0 = imin64(int64_t(tid) * per, U);
    u1 = imin64(u0 + per, U);
    int64_t u = u0;
    if (P.keep_vec) {
      for (; u + 16 <= u1; u += 16) {
        uint4 k = *reinterpret_cast<const uint4*>(P.keep + u);
        mycnt += count_nonzero_bytes(k.x) + count_nonzero_bytes(k.y) +
                 count_nonzero_bytes(k.z) + count_nonzero_bytes(k.w);
      }
    }
    for (; u < u1; ++u) mycnt += P.keep[u] != 0;
    mybase = block_exclusive_scan<kTmaWarps>(mycnt, sh);
    K = sh.total;
  } else {
    K = (uint64_t)U;
  }
  const uint64_t n_rows = K * (uint64_t)P.rpu;
  if (n_rows == 0) {
    if (blockIdx.x == 0 && tid == 0) {
      tf_capture_result& r = P.ctl->res;
      r.capture_seq = 0;
      r.status = TF_OK;
      r.n_rows = 0;
      r.payload_len = 0;
      r.ready_seq = TF_READY_SENTINEL;
    }
    return;
  }
  const uint64_t row = (uint64_t)P.out_row_bytes;
  const uint64_t out_bytes = n_rows * row;

  // ---- 2. this CTA's byte range of the output and its rank table ----
  uint64_t per_cta = (out_bytes + gridDim.x - 1) / gridDim.x;
  per_cta = (per_cta + 15) & ~uint64_t(15);
  const uint64_t b0 = min(out_bytes, uint64_t(blockIdx.x) * per_cta);
  const uint64_t b1 = min(out_bytes, b0 + per_cta);
  const int64_t r_lo = int64_t(b0 / row) / P.rpu;
  if (P.keep && b0 < b1) {
    const int64_t r_hi = int64_t((b1 - 1) / row) / P.rpu;
    if ((int64_t)mybase <= r_hi && (int64_t)(mybase + mycnt) > r_lo) {
      int64_t rank = mybase;
      for (int64_t u = u0; u < u1 && rank <= r_hi; ++u) {
        if (P.keep[u]) {
          if (rank >= r_lo) sh.table[rank - r_lo] = (uint32_t)u;
          ++rank;
        }
      }
    }
  }
  __syncthreads();

  // ---- 3. one thread drives the bulk-copy pipeline ----
  if (tid == 0) {
    auto row_of = [&](int64_t j) -> int64_t {
      int64_t r = j / P.rpu;
      int64_t sub = j - r * P.rpu;
      int64_t unit = P.keep ? (int64_t)sh.table[r - r_lo] : r;
      return unit * P.rpu + sub;
    };
    const uint64_t span = b1 - b0;
    const int ntiles = int((span + kTmaTile - 1) / kTmaTile);
    auto issue = [&](int t) {
      const int st = t % kTmaStages;
      const uint64_t tb0 = b0 + uint64_t(t) * kTmaTile;
      const uint64_t tb1 = min(b1, tb0 + kTmaTile);
      mbar_expect_tx(&full[st], uint32_t(tb1 - tb0));
      uint8_t* sdst = tiles + st * kTmaTile;
      uint64_t cur = tb0;
      while (cur < tb1) {
        const uint64_t j = cur / row;
        const uint64_t off = cur - j * row;
        const uint64_t len = min(row - off, tb1 - cur);
        bulk_load(sdst + (cur - tb0), row_src(P, row_of((int64_t)j)) + off, uint32_t(len), &full[st]);
        cur += len;
      }
    };
    const int pre = ntiles < kTmaStages ? ntiles : kTmaStages;
    for (int t = 0; t < pre; ++t) issue(t);

    // election + reservation after the prefetch is in flight
    const uint32_t ticket = atomicAdd(&P.ctl->arrive, 1u);
    if (ticket == 0) {
      P.ctl->k_t0 = t_entry;
      leader_reserve(P, out_bytes, n_rows);
      __threadfence();
      st_release_gpu(&P.ctl->plan_flag, 1u);
    } else {
      wait_plan(P.ctl);
    }
    const uint32_t status = *((volatile uint32_t*)&P.ctl->plan_status);
    uint8_t* dst_base = P.payload + *((volatile uint64_t*)&P.ctl->plan_off);
    if (status != TF_OK) {
      // rejected: only drain the prefetches (smem must outlive them)
      for (int t = 0; t < pre; ++t) mbar_wait(&full[t], 0u);
    } else {
      for (int t = 0; t < ntiles; ++t) {
        const int st = t % kTmaStages;
        mbar_wait(&full[st], uint32_t((t / kTmaStages) & 1));
        const uint64_t tb0 = b0 + uint64_t(t) * kTmaTile;
        const uint64_t tb1 = min(b1, tb0 + kTmaTile);
        bulk_store(dst_base + tb0, tiles + st * kTmaTile, uint32_t(tb1 - tb0));
        bulk_commit();
        // refill the stage of tile t-1 once its store has read the smem
        const int nt = t - 1 + kTmaStages;
        if (t >= 1 && nt < ntiles) {
          bulk_wait_read<1>();
          issue(nt);
        }
      }
    }
    bulk_wait_all();  // every tile written before this CTA counts as done
    asm volatile("fence.proxy.async.global;" ::: "memory");
    __threadfence();
    sh.status = status;
  }
  __syncthreads();

  // ---- 4. the last CTA to retire publishes ----
  if (tid == 0) {
    uint32_t t = atomicAdd(&P.ctl->done, 1u);
    sh.is_last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (sh.is_last) {
    if (tid == 0) {
      __threadfence();
      last_cta_prepare(P, sh);
      write_snap_ctl(P);
    }
    __syncthreads();
    if (sh.publish && tid < 8) sh.slot[tid] = sh.desc[tid];
    if (tid == 0) {
      P.ctl->arrive = 0;
      P.ctl->done = 0;
      P.ctl->plan_flag = 0;  // visible to the next launch (kernel boundary)
    }
  }
}

// ---------------------------------------------------------------------------
// Shared-memory staged capture (COPY, 16-B aligned rows): every thread
// issues cp.async (LDGSTS) 16-B copies of the CTA's slice into a double
// buffer of 2 x 32 KiB, so up to 192 KiB per SM are in flight with few
// registers; the first chunk is requested before the reservation is
// known. Stores go smem -> ring with 128-bit STG, coalesced.
// ---------------------------------------------------------------------------
constexpr int kStgThreads = 256;
constexpr int kStgWarps = kStgThreads / 32;
constexpr int kStgChunk = 32 * 1024;
constexpr int kStgCtasPerSm = 3;

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc) {
  asm volatile("cp.async.cg.shared.global.L2::128B [%0], [%1], 16;" ::"r"(smem_u32(smem_dst)), "l"(gsrc)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

__global__ void __launch_bounds__(kStgThreads, kStgCtasPerSm) capture_stage_kernel(CapParams P) {
  extern __shared__ __align__(128) uint8_t sbuf[];  // 2 x kStgChunk
  __shared__ CapShared sh;
  const int tid = threadIdx.x;
  const int64_t U = P.units;
  const uint64_t t_entry = tid == 0 ? globaltimer() : 0;

  // ---- 1. ordered compaction ----
  int64_t u0 = 0, u1 = 0;
  uint32_t mycnt = 0, mybase = 0;
  uint64_t K;
  if (P.keep) {
    int64_t per = (U + kStgThreads - 1) / kStgThreads;
    if (P.keep_vec) per = (per + 15) & ~int64_t(15);
    u0 = imin64(int64_t(tid) * per, U);
    u1 = imin64(u0 + per, U);
    int64_t u = u0;
    if (P.keep_vec) {
      for (; u + 16 <= u1; u += 16) {
        uint4 k = *reinterpret_cast<const uint4*>(P.keep + u);
        mycnt += count_nonzero_bytes(k.x) + count_nonzero_bytes(k.y) +
                 count_nonzero_bytes(k.z) + count_nonzero_bytes(k.w);
      }
    }
    for (; u < u1; ++u) mycnt += P.keep[u] != 0;
    mybase = block_exclusive_scan<kStgWarps>(mycnt, sh);
    K = sh.total;
  } else {
    K = (uint64_t)U;
  }
  const uint64_t n_rows = K * (uint64_t)P.rpu;
  if (n_rows == 0) {
    if (blockIdx.x == 0 && tid == 0) {
      tf_capture_result& r = P.ctl->res;
      r.capture_seq = 0;
      r.status = TF_OK;
      r.n_rows = 0;
      r.payload_len = 0;
      r.ready_seq = TF_READY_SENTINEL;
    }
    return;
  }
  const uint32_t row_w = uint32_t(P.out_row_bytes / 16);  // 16-B words per row
  const uint64_t total_w = n_rows * row_w;

  // ---- 2. this CTA's word range and rank table ----
  const uint64_t per_cta = (total_w + gridDim.x - 1) / gridDim.x;
  const uint64_t w0 = min(total_w, uint64_t(blockIdx.x) * per_cta);
  const uint64_t w1 = min(total_w, w0 + per_cta);
  const int64_t r_lo = int64_t(w0 / row_w) / P.rpu;
  if (P.keep && w0 < w1) {
    const int64_t r_hi = int64_t((w1 - 1) / row_w) / P.rpu;
    if ((int64_t)mybase <= r_hi && (int64_t)(mybase + mycnt) > r_lo) {
      int64_t rank = mybase;
      for (int64_t u = u0; u < u1 && rank <= r_hi; ++u) {
        if (P.keep[u]) {
          if (rank >= r_lo) sh.table[rank - r_lo] = (uint32_t)u;
          ++rank;
        }
      }
    }
  }
  __syncthreads();
  auto src_word = [&](uint64_t w) -> const uint8_t* {
    const uint64_t j = w / row_w;
    const uint64_t k = w - j * row_w;
    const int64_t r = int64_t(j) / P.rpu;
    const int64_t sub = int64_t(j) - r * P.rpu;
    const int64_t unit = P.keep ? (int64_t)sh.table[r - r_lo] : r;
    return row_src(P, unit * P.rpu + sub) + k * 16;
  };
  constexpr uint32_t kChunkW = kStgChunk / 16;
  const uint32_t nchunks = uint32_t((w1 - w0 + kChunkW - 1) / kChunkW);
  auto load_chunk = [&](uint32_t c) {
    const uint64_t cw0 = w0 + uint64_t(c) * kChunkW;
    const uint64_t cw1 = min(w1, cw0 + kChunkW);
    uint8_t* buf = sbuf + (c & 1) * kStgChunk;
    for (uint64_t w = cw0 + tid; w < cw1; w += kStgThreads)
      cp_async16(buf + (w - cw0) * 16, src_word(w));
    cp_async_commit();
  };

  // ---- 3. prefetch chunk 0, then learn the offset ----
  if (nchunks > 0) load_chunk(0);
  if (tid == 0) {
    uint32_t t = atomicAdd(&P.ctl->arrive, 1u);
    if (t == 0) {
      P.ctl->k_t0 = t_entry;
      leader_reserve(P, total_w * 16, n_rows);
      __threadfence();
      st_release_gpu(&P.ctl->plan_flag, 1u);
    } else {
      wait_plan(P.ctl);
    }
    sh.status = *((volatile uint32_t*)&P.ctl->plan_status);
    sh.off = *((volatile uint64_t*)&P.ctl->plan_off);
  }
  __syncthreads();
  const bool ok = sh.status == TF_OK;
  uint8_t* dst_base = P.payload + sh.off;
  for (uint32_t c = 0; c < nchunks; ++c) {
    if (ok && c + 1 < nchunks) {
      load_chunk(c + 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();  // chunk c landed for every thread
    if (ok) {
      const uint64_t cw0 = w0 + uint64_t(c) * kChunkW;
      const uint64_t cw1 = min(w1, cw0 + kChunkW);
      const uint8_t* buf = sbuf + (c & 1) * kStgChunk;
#pragma unroll 4
      for (uint64_t w = cw0 + tid; w < cw1; w += kStgThreads) {
        uint4 v = *reinterpret_cast<const uint4*>(buf + (w - cw0) * 16);
        *reinterpret_cast<uint4*>(dst_base + w * 16) = v;
      }
    } else {
      break;  // rejected: chunk 0 drained above, nothing else was issued
    }
    __syncthreads();  // buffer (c & 1) is free for chunk c + 2
  }

  // ---- 4. the last CTA to retire publishes ----
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    uint32_t t = atomicAdd(&P.ctl->done, 1u);
    sh.is_last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (sh.is_last) {
    if (tid == 0) {
      __threadfence();
      last_cta_prepare(P, sh);
      write_snap_ctl(P);
    }
    __syncthreads();
    if (sh.publish && tid < 8) sh.slot[tid] = sh.desc[tid];
    if (tid == 0) {
      P.ctl->arrive = 0;
      P.ctl->done = 0;
      P.ctl->plan_flag = 0;  // visible to the next launch (kernel boundary)
    }
  }
}

#endif  // TF_COPY_VARIANTS

// Protocol-level producer ops (single thread): the same allocator and
// publish rules exposed one call at a time, for the reference's ring tests.
__global__ void reserve_kernel(CapParams P, uint64_t len) {
  DevCtl* c = P.ctl;
  uint64_t L = ld_relaxed_gpu(&P.dcons->L);
  tf_pstate p = c->p;
  uint64_t off = 0, skip = 0;
  uint32_t kind = 0;
  uint32_t status = TF_ERR_PAYLOAD_RING_FULL;
  if (tf_reserve(&p, L, P.cap, len, &off, &skip, &kind)) {
    c->p = p;
    c->bytes_reserved += len;
    if (kind & TF_DESC_DEAD_SKIP) c->dead_created += skip;
    status = TF_OK;
  }
  c->res.status = status;
  c->res.n_rows = kind;
  c->res.payload_offset = off;
  c->res.skip_before = skip;
  c->res.payload_len = len;
  c->res.capture_seq = c->capture_seq;  // device captures reserved before this one
  write_snap_ctl(P);
}

__global__ void publish_kernel(CapParams P, tf_descriptor d) {
  DevCtl* c = P.ctl;
  uint64_t mtail = ld_relaxed_gpu(&P.dcons->meta_tail);
  uint32_t status = TF_OK;
  uint64_t seq = TF_READY_SENTINEL;
  if (c->meta_head - mtail >= P.slots) {
    status = TF_ERR_META_RING_FULL;  // rings.py:327-330
  } else {
    uint64_t slot = c->meta_head % P.slots;
    uint64_t* w = reinterpret_cast<uint64_t*>(P.meta + slot * TF_DESCRIPTOR_SIZE);
    if (ld_relaxed_sys(w + 3) != TF_READY_SENTINEL) {
      status = TF_ERR_PROTOCOL;  // rings.py:334-335
      c->errors |= TF_DEVERR_PROTOCOL;
    } else {
      seq = c->meta_head;
      d.ready_seq = seq;
      uint64_t* s = reinterpret_cast<uint64_t*>(&d);
      d.checksum = tf_desc_checksum(s);
      for (int i = 0; i < 8; ++i)
        if (i != 3) st_relaxed_sys(w + i, s[i]);
      st_relaxed_sys(w + 3, seq);
      c->meta_head = seq + 1;
    }
  }
  c->res.ready_seq = seq;
  c->res.status = status;
  write_snap_ctl(P);
}

}  // namespace

// ---------------------------------------------------------------------------
// host: ring lifecycle
// ---------------------------------------------------------------------------
// CUDA loads kernels lazily (CUDA_MODULE_LOADING=LAZY by default): the first
// launch of a kernel loads it, and loading can wait on the device. A first
// launch made while a capture kernel waits on the device for the staging
// engine (the seal at the end of the first step, a snapshot) then deadlocks
// with it. So every kernel this library can launch is loaded when the first
// ring is created (querying a kernel's attributes loads it).
template <int MODE, int VW, int IN, int OUT, int SS = kSmemSpec>
static void touch() {
  cudaFuncAttributes a;
  cudaFuncGetAttributes(&a, capture_kernel<MODE, VW, IN, OUT, SS>);
}
template <int IN, int OUT>
static void touch_cast() {
  touch<MODE_CAST, 8, IN, OUT>();
  touch<MODE_CAST, 1, IN, OUT>();
}
template <int IN>
static void touch_in() {
  touch_cast<IN, TF_F32>();
  touch_cast<IN, TF_F16>();
  touch_cast<IN, TF_BF16>();
  touch_cast<IN, TF_F8E4M3>();
  touch_cast<IN, TF_F8E5M2>();
  touch<MODE_REDUCE, 8, IN, TF_F32>();
  touch<MODE_REDUCE, 1, IN, TF_F32>();
}
__global__ void seal_kernel(const DevCtl* c, uint64_t* host_word);
__global__ void snapshot_kernel(const uint64_t* __restrict__ src, uint64_t* dst, int words);
static void preload_kernels() {
#ifdef TF_NO_PRELOAD  // experiment builds only: reproduce the lazy-loading hang
  return;
#endif
  static std::once_flag once;
  std::call_once(once, [] {
    touch<MODE_COPY, 16, 0, 0>();
    touch<MODE_COPY, 16, 0, 0, 0>();
    touch<MODE_COPY, 8, 0, 0>();
    touch<MODE_COPY, 4, 0, 0>();
    touch<MODE_COPY, 2, 0, 0>();
    touch<MODE_COPY, 1, 0, 0>();
    touch_in<TF_F32>();
    touch_in<TF_F16>();
    touch_in<TF_BF16>();
    cudaFuncAttributes a;
    cudaFuncGetAttributes(&a, seal_kernel);
    cudaFuncGetAttributes(&a, snapshot_kernel);
    cudaFuncGetAttributes(&a, reserve_kernel);
    cudaFuncGetAttributes(&a, publish_kernel);
    cudaGetLastError();
  });
}

static int set_device(int dev) {
  CUDA_TRY(cudaSetDevice(dev));
  return TF_OK;
}

static CapParams base_params(tf_ring* r) {
  CapParams P;
  memset(&P, 0, sizeof(P));
  P.payload = r->payload;
  P.cap = r->cfg.payload_capacity;
  P.slots = r->cfg.meta_slots;
  P.meta = r->meta;
  P.dcons = r->dcons;
  P.ctl = r->ctl;
  P.done_flags = r->done_flags;
  P.seal = r->seal_host;
  P.timeout_ns = r->cfg.wait_timeout_ns ? r->cfg.wait_timeout_ns : 30000000000ull;
  return P;
}

// Copy the device control block to the pinned snapshot (control stream:
// never waits for the inference stream). Callers fence the producer first.
// Snapshot of the device control block for the host. A one-CTA kernel on a
// high-priority stream stores it into the host-mapped copy: a D2H memcpy
// would queue on the copy engine behind the staging engine's 128 MiB
// transfers (milliseconds per policy decision while PCIe is busy).
__global__ void snapshot_kernel(const uint64_t* __restrict__ src, uint64_t* dst, int words) {
  for (int i = threadIdx.x; i < words; i += blockDim.x)
    dst[i] = ld_relaxed_gpu(src + i);
}

// Runs after every earlier kernel on its stream has completed (launched
// without PDL): each descriptor below the committed meta head was posted by
// a finished capture, so all of them are complete.
__global__ void seal_kernel(const DevCtl* c, uint64_t* host_word) {
  const uint64_t mh = *reinterpret_cast<const volatile uint64_t*>(&c->meta_head);
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(host_word), "l"(mh) : "memory");
}

static int snapshot(tf_ring* r) {
  constexpr int words = int(sizeof(DevCtl) / 8);
  snapshot_kernel<<<1, 256, 0, (cudaStream_t)r->snap_stream>>>(
      reinterpret_cast<const uint64_t*>(r->ctl), reinterpret_cast<uint64_t*>(r->ctl_host_dev),
      words);
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaStreamSynchronize((cudaStream_t)r->snap_stream));
  return TF_OK;
}

extern "C" int tf_ring_create(const tf_ring_config* cfg, int device, tf_ring** out) {
  if (!cfg || !out) { tf_set_error("null argument"); return TF_ERR_VALUE; }
  // rings.py:75-85 RingConfig validation
  if (cfg->payload_capacity == 0) { tf_set_error("payload_capacity must be positive"); return TF_ERR_CONFIG; }
  if (cfg->payload_capacity % TF_COPY_UNIT) {
    tf_set_error("payload_capacity must be a multiple of 16 bytes");
    return TF_ERR_CONFIG;
  }
  if (cfg->meta_slots == 0) { tf_set_error("meta_slots must be positive"); return TF_ERR_CONFIG; }
  if (!(cfg->high_watermark > 0.0 && cfg->high_watermark <= 1.0)) {
    tf_set_error("high_watermark must be in (0, 1]");
    return TF_ERR_CONFIG;
  }
  int rc = set_device(device);
  if (rc) return rc;
  tf_ring* r = new tf_ring();
  r->device = device;
  r->cfg = *cfg;
  auto fail = [&](int code) {
    if (r->payload) cudaFree(r->payload);
    if (r->ctl) cudaFree(r->ctl);
    if (r->dcons) cudaFree(r->dcons);
    if (r->meta) cudaFreeHost(r->meta);
    if (r->done_flags) cudaFreeHost(r->done_flags);
    if (r->ctl_host) cudaFreeHost(r->ctl_host);
    if (r->seal_host) cudaFreeHost(r->seal_host);
    if (r->ctrl_stream) cudaStreamDestroy((cudaStream_t)r->ctrl_stream);
    delete r;
    return code;
  };
  cudaError_t e = cudaMalloc(&r->payload, cfg->payload_capacity);
  if (e != cudaSuccess) {
    tf_set_error("device arena cannot satisfy %llu bytes: %s",
                 (unsigned long long)cfg->payload_capacity, cudaGetErrorString(e));
    cudaGetLastError();
    return fail(TF_ERR_ALLOCATION);  // rings.py:155-160 AllocationError
  }
  size_t meta_bytes = size_t(cfg->meta_slots) * TF_DESCRIPTOR_SIZE;
  if (cudaHostAlloc((void**)&r->meta, meta_bytes, cudaHostAllocMapped | cudaHostAllocPortable) != cudaSuccess ||
      cudaHostAlloc((void**)&r->done_flags, size_t(cfg->meta_slots) * kMaxFlagCtas,
                    cudaHostAllocMapped | cudaHostAllocPortable) != cudaSuccess ||
      cudaHostAlloc((void**)&r->ctl_host, sizeof(DevCtl), cudaHostAllocPortable | cudaHostAllocMapped) != cudaSuccess ||
      cudaHostAlloc((void**)&r->seal_host, 64, cudaHostAllocPortable | cudaHostAllocMapped) != cudaSuccess) {
    tf_set_error("host arena allocation failed: %s", cudaGetErrorString(cudaGetLastError()));
    return fail(TF_ERR_ALLOCATION);
  }
  memset(r->seal_host, 0, 64);
  memset(r->meta, 0, meta_bytes);
  memset(r->done_flags, 0, size_t(cfg->meta_slots) * kMaxFlagCtas);
  for (uint32_t s = 0; s < cfg->meta_slots; ++s)  // rings.py:213-215
    reinterpret_cast<uint64_t*>(r->meta + size_t(s) * TF_DESCRIPTOR_SIZE)[3] = TF_READY_SENTINEL;
  if (cudaMalloc(&r->ctl, sizeof(DevCtl)) != cudaSuccess ||
      cudaMalloc(&r->dcons, sizeof(DevConsumer)) != cudaSuccess) {
    tf_set_error("device control block allocation failed");
    cudaGetLastError();
    return fail(TF_ERR_ALLOCATION);
  }
  memset(r->ctl_host, 0, sizeof(DevCtl));
  r->ctl_host->p.reset_mark = TF_NO_MARK;
  for (int i = 0; i < kSnapReplicas; ++i) r->ctl_host->snap[i].reset_mark = TF_NO_MARK;
  if (cudaMemcpy(r->ctl, r->ctl_host, sizeof(DevCtl), cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaMemset(r->dcons, 0, sizeof(DevConsumer)) != cudaSuccess ||
      cudaMemset(r->payload, 0, cfg->payload_capacity) != cudaSuccess) {
    tf_set_error("device init failed: %s", cudaGetErrorString(cudaGetLastError()));
    return fail(TF_ERR_CUDA);
  }
  cudaStream_t s;
  if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess) {
    tf_set_error("stream create failed");
    return fail(TF_ERR_CUDA);
  }
  r->ctrl_stream = s;
  int lo = 0, hi = 0;
  cudaDeviceGetStreamPriorityRange(&lo, &hi);
  if (cudaStreamCreateWithPriority(&s, cudaStreamNonBlocking, hi) != cudaSuccess ||
      cudaHostGetDevicePointer((void**)&r->ctl_host_dev, r->ctl_host, 0) != cudaSuccess) {
    tf_set_error("snapshot stream / mapping failed");
    return fail(TF_ERR_CUDA);
  }
  r->snap_stream = s;
  preload_kernels();
  if (kSmemSpec > 0 && kSpecSmemBytes > 48 * 1024 &&
      cudaFuncSetAttribute(capture_kernel<MODE_COPY, 16, 0, 0>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize,
                           kSpecSmemBytes) != cudaSuccess) {
    tf_set_error("shared-memory opt-in failed");
    return fail(TF_ERR_CUDA);
  }
  if (cudaDeviceSynchronize() != cudaSuccess) return fail(TF_ERR_CUDA);
  *out = r;
  return TF_OK;
}

extern "C" int tf_ring_destroy(tf_ring* r) {
  if (!r) return TF_OK;
  cudaSetDevice(r->device);
  cudaDeviceSynchronize();
  if (r->ctrl_stream) cudaStreamDestroy((cudaStream_t)r->ctrl_stream);
  if (r->snap_stream) cudaStreamDestroy((cudaStream_t)r->snap_stream);
  cudaFree(r->payload);
  cudaFree(r->ctl);
  cudaFree(r->dcons);
  cudaFreeHost(r->meta);
  cudaFreeHost(r->done_flags);
  cudaFreeHost(r->ctl_host);
  cudaFreeHost(r->seal_host);
  delete r;
  return TF_OK;
}

extern "C" int tf_ring_payload_ptr(tf_ring* r, void** p) {
  if (!r || !p) return TF_ERR_VALUE;
  *p = r->payload;
  return TF_OK;
}
extern "C" int tf_ring_meta_ptr(tf_ring* r, void** p) {
  if (!r || !p) return TF_ERR_VALUE;
  *p = r->meta;
  return TF_OK;
}

// ---------------------------------------------------------------------------
// host: capture launch
// ---------------------------------------------------------------------------
static int dtype_width(uint32_t dt) {
  switch (dt) {
    case TF_U8: case TF_I8: case TF_F8E4M3: case TF_F8E5M2: return 1;
    case TF_F16: case TF_BF16: return 2;
    case TF_F32: case TF_I32: return 4;
    case TF_F64: case TF_I64: return 8;
  }
  return 0;
}
static int reduce_k(uint32_t op) { return op == TF_RED_STATS ? 4 : 1; }

extern "C" int tf_capture_out_row_bytes(const tf_capture_args* a, int64_t* out) {
  if (!a || !out) return TF_ERR_VALUE;
  if (a->op == TF_OP_COPY) { *out = a->row_bytes; return TF_OK; }
  int wi = dtype_width(a->in_dtype);
  if (wi == 0 || a->row_bytes % wi) { tf_set_error("row_bytes not a multiple of the input width"); return TF_ERR_CONFIG; }
  int64_t elems = a->row_bytes / wi;
  if (a->op == TF_OP_CAST) {
    int wo = dtype_width(a->out_dtype);
    if (!wo) { tf_set_error("bad out dtype"); return TF_ERR_CONFIG; }
    *out = elems * wo;
    return TF_OK;
  }
  if (a->op == TF_OP_REDUCE) {
    if (a->reduce_op > TF_RED_STATS) { tf_set_error("bad reduce op"); return TF_ERR_CONFIG; }
    *out = int64_t(reduce_k(a->reduce_op)) * 4;
    return TF_OK;
  }
  tf_set_error("bad op");
  return TF_ERR_CONFIG;
}

// Programmatic dependent launch: a capture kernel may be scheduled while the
// kernel before it on the stream drains; it waits (griddepcontrol.wait) for
// that kernel's completion and memory before its first global access, so
// only launch latency and CTA start-up overlap. TF_PDL=0 disables.
static bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("TF_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

static FastDiv make_fastdiv(uint64_t d) {
  FastDiv f{uint32_t(d), 0u, 0u};
  if (d <= 1) return f;
  int l = 0;
  while ((uint64_t(1) << l) < d) ++l;  // ceil(log2 d)
  const int p = 31 + l;
  f.mul = uint32_t(((uint64_t(1) << p) + d - 1) / d);
  f.shr = uint32_t(p - 32);
  return f;
}

// The kernel's launch-constant divisors (its spr, rpu, mid and copy-CTA
// count) and whether every dividend it divides stays below 2^31.
template <int MODE>
static void set_fastdiv(CapParams& P, int grid) {
  const int64_t spr = MODE == MODE_REDUCE ? 1 : (P.words_per_row + kSeg - 1) / kSeg;
  const uint64_t rows = uint64_t(P.outer) * uint64_t(P.mid);
  const uint64_t lim = uint64_t(1) << 31;
  P.fd_ok = rows < lim && uint64_t(spr) < lim && rows * uint64_t(spr) + uint64_t(grid) < lim &&
            uint64_t(P.mid) < lim && uint64_t(P.rpu) < lim;
  P.fd_spr = make_fastdiv(uint64_t(spr));
  P.fd_rpu = make_fastdiv(uint64_t(P.rpu));
  P.fd_mid = make_fastdiv(uint64_t(P.mid));
  P.fd_cg = make_fastdiv(uint64_t(grid));
}

template <int MODE, int VW, int IN, int OUT, int SS = kSmemSpec>
static int launch(const CapParams& P0, int grid, cudaStream_t s) {
  CapParams P = P0;
  set_fastdiv<MODE>(P, grid);
  // (the >48 KiB opt-in is set once per device in tf_ring_create, outside
  // any stream capture)
  constexpr int smem = (MODE == MODE_COPY && VW == 16 && SS > 0) ? SS * 8 * kSeg * 16 : 0;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid + kCtl);  // (+ the controller CTA in controller builds)
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  cudaLaunchKernelEx(&cfg, capture_kernel<MODE, VW, IN, OUT, SS>, P);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    tf_set_error("capture launch: %s", cudaGetErrorString(e));
    return TF_ERR_CUDA;
  }
  return TF_OK;
}

static int pow2_align(uint64_t x) {
  if (x == 0) return 16;
  int a = 1;
  while (a < 16 && (x % (uint64_t)(a * 2)) == 0) a *= 2;
  return a;
}

template <int IN, int OUT>
static int launch_cast(const CapParams& P, bool vec, int grid, cudaStream_t s) {
  return vec ? launch<MODE_CAST, 8, IN, OUT>(P, grid, s) : launch<MODE_CAST, 1, IN, OUT>(P, grid, s);
}
template <int IN>
static int launch_cast_in(const CapParams& P, uint32_t out, bool vec, int grid, cudaStream_t s) {
  switch (out) {
    case TF_F32: return launch_cast<IN, TF_F32>(P, vec, grid, s);
    case TF_F16: return launch_cast<IN, TF_F16>(P, vec, grid, s);
    case TF_BF16: return launch_cast<IN, TF_BF16>(P, vec, grid, s);
    case TF_F8E4M3: return launch_cast<IN, TF_F8E4M3>(P, vec, grid, s);
    case TF_F8E5M2: return launch_cast<IN, TF_F8E5M2>(P, vec, grid, s);
  }
  tf_set_error("cast output dtype %u unsupported", out);
  return TF_ERR_CONFIG;
}
template <int IN>
static int launch_reduce(const CapParams& P, bool vec, int grid, cudaStream_t s) {
  return vec ? launch<MODE_REDUCE, 8, IN, TF_F32>(P, grid, s)
             : launch<MODE_REDUCE, 1, IN, TF_F32>(P, grid, s);
}

// SM count of the device (lazy, thread-safe: several producer threads may
// launch captures on different rings concurrently)
static std::atomic<int> g_sm_count{0};

// Grid sizing knobs (env, read once, thread-safe magic static)
struct GridKnobs {
  int chunk_kb, waves;
};
static const GridKnobs& grid_knobs() {
  static const GridKnobs k = [] {
    const char* e = getenv("TF_CAP_CHUNK_KB");
    const char* w = getenv("TF_CAP_WAVES");
    return GridKnobs{e ? std::max(1, atoi(e)) : 16, w ? std::max(1, atoi(w)) : 1};
  }();
  return k;
}

extern "C" int tf_capture(tf_ring* r, void* stream, const tf_capture_args* a) {
  if (!r || !a) { tf_set_error("null argument"); return TF_ERR_VALUE; }
  // TensorView validation, hooks.py:209-217
  if (a->outer <= 0 || a->mid <= 0 || a->row_bytes <= 0) {
    tf_set_error("view shape must be non-empty and positive");
    return TF_ERR_CONFIG;
  }
  if (!a->src) { tf_set_error("null source"); return TF_ERR_VALUE; }
  int64_t orb;
  int rc = tf_capture_out_row_bytes(a, &orb);
  if (rc) return rc;
  int rcd = set_device(r->device);
  if (rcd) return rcd;
  int sm_count = g_sm_count.load(std::memory_order_relaxed);
  if (!sm_count) {
    int n = 148;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, r->device);
    g_sm_count.store(n, std::memory_order_relaxed);
    sm_count = n;
  }
  CapParams P = base_params(r);
  P.src = (const uint8_t*)a->src;
  P.outer = a->outer;
  P.mid = a->mid;
  P.row_bytes = a->row_bytes;
  P.s_outer = a->stride_outer;
  P.s_mid = a->stride_mid;
  P.keep = a->keep;
  P.step_ptr = a->step_seq_ptr;
  P.step_imm = a->step_seq;
  P.hook_id = a->hook_id;
  P.flags = a->flags;
  P.reduce_op = a->reduce_op;
  const bool per_outer = (a->flags & TF_CAP_KEEP_PER_OUTER) != 0;
  P.units = per_outer ? a->outer : a->outer * a->mid;
  P.rpu = per_outer ? a->mid : 1;
  P.out_row_bytes = orb;
  P.keep_vec = ((uintptr_t)a->keep % 16) == 0;
  if ((a->flags & TF_FULL_MASK) > TF_FULL_DROP) { tf_set_error("bad full mode"); return TF_ERR_CONFIG; }
  // a sealed capture is completed by the next descriptor: with one meta
  // slot there is no next slot, so report per CTA instead
  if (r->cfg.meta_slots < 2) P.flags &= ~TF_CAP_SEALED;

  // alignment every source row start shares (pow2, capped at 16)
  int sal = pow2_align((uintptr_t)a->src);
  if (a->outer > 1) sal = std::min(sal, pow2_align((uint64_t)a->stride_outer));
  if (a->mid > 1) sal = std::min(sal, pow2_align((uint64_t)a->stride_mid));
  const int64_t total_rows = a->outer * a->mid;
  const uint64_t out_max = uint64_t(total_rows) * uint64_t(orb);
  // grid: one chunk (default 16 KiB) per CTA up to `waves` x kCtasPerSm
  // CTAs per SM. The leader of a slow-path launch is the first CTA to
  // arrive, so CTAs that become resident later never starve it.
  const int chunk_kb = grid_knobs().chunk_kb, waves = grid_knobs().waves;
  const uint64_t chunk = uint64_t(chunk_kb) << 10;
  // (- kCtl: a controller CTA must not push the grid past one resident wave)
  int grid_bytes = int(std::min<uint64_t>((out_max + chunk - 1) / chunk,
                                          uint64_t(sm_count) * kCtasPerSm * waves - kCtl));
  int grid_table = a->keep ? int((P.units + kTableMax - 5) / (kTableMax - 4)) : 1;
  int grid = std::max(1, std::max(grid_bytes, grid_table));
  if (a->max_ctas) grid = std::max(grid_table, std::min<int>(grid, (int)a->max_ctas));
  cudaStream_t s = (cudaStream_t)stream;  // NULL = legacy default stream (CUDA convention)

  if (a->op == TF_OP_COPY) {
    int vw = std::min<int>(sal, pow2_align((uint64_t)a->row_bytes));
    P.words_per_row = a->row_bytes / vw;
#ifdef TF_COPY_VARIANTS
    // 0 = LDG/STG warps (default: measured fastest on B200),
    // 1 = TMA bulk copies, 2 = cp.async smem staging (TF_COPY_PATH=tma|stage)
    static int copy_path = -1;
    if (copy_path < 0) {
      const char* e = getenv("TF_COPY_PATH");
      copy_path = (e && e[0] == 't') ? 1 : (e && e[0] == 's') ? 2 : 0;
    }
    if (vw == 16 && copy_path == 2) {
      static bool attr2 = false;
      if (!attr2) {
        CUDA_TRY(cudaFuncSetAttribute(capture_stage_kernel,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * kStgChunk));
        attr2 = true;
      }
      int g = int(std::min<uint64_t>((out_max + (16u << 10) - 1) / (16u << 10),
                                     uint64_t(sm_count) * kStgCtasPerSm));
      g = std::max(std::max(g, grid_table), 1);
      if (a->max_ctas) g = std::max(grid_table, std::min<int>(g, (int)a->max_ctas));
      capture_stage_kernel<<<g, kStgThreads, 2 * kStgChunk, s>>>(P);
      cudaError_t e = cudaGetLastError();
      if (e != cudaSuccess) {
        tf_set_error("capture launch: %s", cudaGetErrorString(e));
        return TF_ERR_CUDA;
      }
      return TF_OK;
    }
    if (vw == 16 && copy_path == 1) {
      static bool attr_set = false;
      if (!attr_set) {
        CUDA_TRY(cudaFuncSetAttribute(capture_tma_kernel,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, kTmaSmem));
        attr_set = true;
      }
      int g = int(std::min<uint64_t>((out_max + kTmaTile - 1) / kTmaTile, uint64_t(sm_count)));
      g = std::max(std::max(g, grid_table), 1);
      if (a->max_ctas) g = std::max(grid_table, std::min<int>(g, (int)a->max_ctas));
      capture_tma_kernel<<<g, kTmaThreads, kTmaSmem, s>>>(P);
      cudaError_t e = cudaGetLastError();
      if (e != cudaSuccess) {
        tf_set_error("capture launch: %s", cudaGetErrorString(e));
        return TF_ERR_CUDA;
      }
      return TF_OK;
    }
#endif
    switch (vw) {
      case 16:
        // below the grid cap every warp owns at most one segment: no
        // shared-memory speculation, no dynamic shared memory
        if (grid_bytes < int(uint64_t(sm_count) * kCtasPerSm * waves - kCtl))
          return launch<MODE_COPY, 16, 0, 0, 0>(P, grid, s);
        return launch<MODE_COPY, 16, 0, 0>(P, grid, s);
      case 8: return launch<MODE_COPY, 8, 0, 0>(P, grid, s);
      case 4: return launch<MODE_COPY, 4, 0, 0>(P, grid, s);
      case 2: return launch<MODE_COPY, 2, 0, 0>(P, grid, s);
      default: return launch<MODE_COPY, 1, 0, 0>(P, grid, s);
    }
  }
  const int wi = dtype_width(a->in_dtype);
  P.row_elems = a->row_bytes / wi;
  if (a->in_dtype != TF_F32 && a->in_dtype != TF_F16 && a->in_dtype != TF_BF16) {
    tf_set_error("cast/reduce input dtype must be f32, f16 or bf16");
    return TF_ERR_CONFIG;
  }
  // 8-element groups need 16-B aligned input groups
  const bool vec = (P.row_elems % 8 == 0) && sal >= 16 && ((uint64_t)(8 * wi) % 16 == 0);
  if (a->op == TF_OP_CAST) {
    P.words_per_row = vec ? P.row_elems / 8 : P.row_elems;
    switch (a->in_dtype) {
      case TF_F32: return launch_cast_in<TF_F32>(P, a->out_dtype, vec, grid, s);
      case TF_F16: return launch_cast_in<TF_F16>(P, a->out_dtype, vec, grid, s);
      default: return launch_cast_in<TF_BF16>(P, a->out_dtype, vec, grid, s);
    }
  }
  P.words_per_row = 1;
  // reduce: one warp per row; size the grid by rows
  {
    int64_t g = (total_rows + kWarps - 1) / kWarps;
    int gr = int(std::min<int64_t>(g, int64_t(sm_count) * kCtasPerSm));
    grid = std::max(std::max(gr, grid_table), 1);
  }
  switch (a->in_dtype) {
    case TF_F32: return launch_reduce<TF_F32>(P, vec, grid, s);
    case TF_F16: return launch_reduce<TF_F16>(P, vec, grid, s);
    default: return launch_reduce<TF_BF16>(P, vec, grid, s);
  }
}

extern "C" int tf_ring_last_result(tf_ring* r, tf_capture_result* out) {
  if (!r || !out) return TF_ERR_VALUE;
  int rc = set_device(r->device);
  if (rc) return rc;
  rc = snapshot(r);
  if (rc) return rc;
  *out = r->ctl_host->res;
  return TF_OK;
}

extern "C" int tf_ring_reserve(tf_ring* r, void* stream, uint64_t length,
                               uint64_t* offset, uint64_t* skip_before) {
  if (!r) return TF_ERR_VALUE;
  // rings.py:293-298
  if (length == 0) { tf_set_error("reservation length must be positive"); return TF_ERR_VALUE; }
  if (length % TF_COPY_UNIT) { tf_set_error("reservation length must be a copy-unit multiple"); return TF_ERR_VALUE; }
  if (length > r->cfg.payload_capacity) { tf_set_error("reservation exceeds payload capacity"); return TF_ERR_VALUE; }
  int rc = set_device(r->device);
  if (rc) return rc;
  cudaStream_t s = (cudaStream_t)stream;  // NULL = legacy default stream
  CUDA_TRY(cudaStreamSynchronize((cudaStream_t)r->ctrl_stream));
  CapParams P = base_params(r);
  reserve_kernel<<<1, 1, 0, s>>>(P, length);
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaStreamSynchronize(s));
  rc = snapshot(r);
  if (rc) return rc;
  const tf_capture_result& res = r->ctl_host->res;
  if (res.status != TF_OK) {
    tf_set_error("need %llu bytes", (unsigned long long)length);
    return TF_ERR_PAYLOAD_RING_FULL;
  }
  uint64_t off = res.payload_offset, skip = res.skip_before;
  {
    std::lock_guard<std::mutex> g(r->mu);
    HostRegion hr{off, length, skip, res.n_rows /* kind */, false, true, res.capture_seq};
    r->regions.push_back(hr);
    r->host_reserved[off] = hr;
  }
  if (offset) *offset = off;
  if (skip_before) *skip_before = skip;
  return TF_OK;
}

extern "C" int tf_ring_publish(tf_ring* r, void* stream, const tf_descriptor* d,
                               uint64_t* ready_seq) {
  if (!r || !d) return TF_ERR_VALUE;
  int rc = set_device(r->device);
  if (rc) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  tf_descriptor dd = *d;
  if (dd.capture_seq == 0) {
    // user-built descriptor for a tf_ring_reserve'd region: its region is
    // already in the host FIFO; carry the skip for completeness.
    std::lock_guard<std::mutex> g(r->mu);
    auto it = r->host_reserved.find(dd.payload_offset);
    if (it != r->host_reserved.end()) {
      dd.skip_before = it->second.skip;
      dd.flags = it->second.kind;
    }
    dd.flags |= TF_DESC_HOST_RESERVED;
  }
  CUDA_TRY(cudaStreamSynchronize((cudaStream_t)r->ctrl_stream));
  CapParams P = base_params(r);
  publish_kernel<<<1, 1, 0, s>>>(P, dd);
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaStreamSynchronize(s));
  rc = snapshot(r);
  if (rc) return rc;
  const tf_capture_result& res = r->ctl_host->res;
  if (res.status == TF_ERR_META_RING_FULL) {
    tf_set_error("all %u descriptor slots are in flight", r->cfg.meta_slots);
    return TF_ERR_META_RING_FULL;
  }
  if (res.status == TF_ERR_PROTOCOL) {
    tf_set_error("descriptor slot reused before consumption");
    return TF_ERR_PROTOCOL;
  }
  if (dd.capture_seq == 0) {
    std::lock_guard<std::mutex> g(r->mu);
    r->host_reserved.erase(dd.payload_offset);
  }
  if (ready_seq) *ready_seq = res.ready_seq;
  return TF_OK;
}

// ---------------------------------------------------------------------------
// host: consumer role
// ---------------------------------------------------------------------------
static inline uint64_t slot_ready(const tf_ring* r, uint64_t slot) {
  const uint64_t* p = reinterpret_cast<const uint64_t*>(r->meta + slot * TF_DESCRIPTOR_SIZE) + 3;
  return __atomic_load_n(p, __ATOMIC_ACQUIRE);
}

// Stream-ordered u64 write into device memory: cuStreamWriteValue64 via
// the driver entry point (the value rides in the command, no host buffer);
// a pinned-slot cudaMemcpyAsync if stream memory ops are unavailable.
typedef int (*write64_fn)(void*, unsigned long long, unsigned long long, unsigned int);
static std::atomic<write64_fn> g_write64{nullptr};
static std::atomic<int> g_write64_probe{0};  // double-checked: acquire/release
static std::mutex g_slot_mu;
static uint64_t* g_slots = nullptr;
static uint64_t g_slot_next = 0;
constexpr uint64_t kSlots = 1u << 16;

int tf_internal_write_u64(void* stream, uint64_t* dev_addr, uint64_t value) {
  if (!g_write64_probe.load(std::memory_order_acquire)) {
    std::lock_guard<std::mutex> g(g_slot_mu);
    if (!g_write64_probe.load(std::memory_order_relaxed)) {
      void* fn = nullptr;
      cudaDriverEntryPointQueryResult q;
      if (cudaGetDriverEntryPoint("cuStreamWriteValue64", &fn, cudaEnableDefault, &q) == cudaSuccess &&
          q == cudaDriverEntryPointSuccess && fn) {
        int dev = 0, ok = 0;
        cudaGetDevice(&dev);
        void* attr = nullptr;
        cudaDriverEntryPointQueryResult q2;
        if (cudaGetDriverEntryPoint("cuDeviceGetAttribute", &attr, cudaEnableDefault, &q2) == cudaSuccess && attr) {
          typedef int (*attr_fn)(int*, int, int);
          ((attr_fn)attr)(&ok, 122 /* CAN_USE_64_BIT_STREAM_MEM_OPS */, dev);
        }
        if (ok && !getenv("TF_NO_STREAM_MEMOPS"))
          g_write64.store((write64_fn)fn, std::memory_order_relaxed);
      }
      cudaGetLastError();
      g_write64_probe.store(1, std::memory_order_release);
    }
  }
  if (write64_fn w64 = g_write64.load(std::memory_order_relaxed)) {
    int rc = w64(stream, (unsigned long long)(uintptr_t)dev_addr, value, 0);
    if (rc != 0) {
      tf_set_error("cuStreamWriteValue64 failed (%d)", rc);
      return TF_ERR_CUDA;
    }
    return TF_OK;
  }
  uint64_t* slot;
  {
    std::lock_guard<std::mutex> g(g_slot_mu);
    if (!g_slots && cudaHostAlloc((void**)&g_slots, kSlots * 8, cudaHostAllocPortable) != cudaSuccess) {
      tf_set_error("pinned slot allocation failed");
      return TF_ERR_ALLOCATION;
    }
    slot = &g_slots[g_slot_next++ % kSlots];
  }
  *slot = value;
  CUDA_TRY(cudaMemcpyAsync(dev_addr, slot, 8, cudaMemcpyHostToDevice, (cudaStream_t)stream));
  return TF_OK;
}

static bool slot_verified(const uint8_t* raw, tf_descriptor* d) {
  uint64_t w[8];
  memcpy(w, raw, 64);
  if (w[3] == TF_READY_SENTINEL || tf_desc_checksum(w) != w[7]) return false;
  memcpy(d, w, 64);
  return true;
}

// A posted slot is complete when its checksum verifies and, for a capture
// posted before its copy finished, every CTA has set its completion byte.
// The CTA count is stripped from the flags handed out.
static bool slot_complete(const tf_ring* r, uint64_t slot, tf_descriptor* d) {
  if (!slot_verified(r->meta + slot * TF_DESCRIPTOR_SIZE, d)) return false;
  if (d->flags & TF_DESC_PENDING) {
    // TF_CAP_SEALED: complete once sealed, or once the next descriptor in
    // sequence was posted by a later capture (which started only after this
    // one finished: same stream, griddepcontrol.wait before its post)
    bool done = __atomic_load_n(r->seal_host, __ATOMIC_ACQUIRE) > d->ready_seq;
    if (!done) {
      tf_descriptor nd;
      const uint64_t ns = (slot + 1) % r->cfg.meta_slots;
      done = ns != slot && slot_verified(r->meta + ns * TF_DESCRIPTOR_SIZE, &nd) &&
             nd.ready_seq == d->ready_seq + 1 && !(nd.flags & TF_DESC_HOST_RESERVED);
    }
    if (!done) return false;
    d->flags &= ~TF_DESC_PENDING;
  }
  const uint32_t n = d->flags >> TF_DESC_CTA_SHIFT;
  if (n) {  // 8 completion bytes per load
    const uint8_t* f = r->done_flags + slot * kMaxFlagCtas;
    const uint64_t* w = reinterpret_cast<const uint64_t*>(f);
    uint32_t i = 0;
    for (; i + 8 <= n; i += 8)
      if (__atomic_load_n(w + i / 8, __ATOMIC_ACQUIRE) != 0x0101010101010101ull) return false;
    for (; i < n; ++i)
      if (__atomic_load_n(f + i, __ATOMIC_ACQUIRE) != 1) return false;
  }
  d->flags &= (1u << TF_DESC_CTA_SHIFT) - 1u;
  return true;
}

int tf_internal_poll(tf_ring* r, uint32_t max_entries, tf_descriptor* out,
                     uint32_t* n, bool consume) {
  uint32_t got = 0;
  const uint64_t slots = r->cfg.meta_slots;
  uint64_t tail = r->meta_tail;
  bool advanced = false;
  while (got < max_entries && got < slots) {
    uint64_t slot = tail % slots;
    uint64_t ready = slot_ready(r, slot);
    if (ready == TF_READY_SENTINEL) break;
    tf_descriptor d;
    // words may still be landing: accept only a slot whose checksum
    // verifies (and whose capture CTAs have all reported)
    if (!slot_complete(r, slot, &d)) break;
    if (consume) {
      if (d.ready_seq != r->consumed) {  // rings.py:397-401
        tf_set_error("descriptor sequence %llu out of order, expected %llu",
                     (unsigned long long)d.ready_seq, (unsigned long long)r->consumed);
        *n = got;
        return TF_ERR_PROTOCOL;
      }
      const uint32_t n_ctas = reinterpret_cast<const tf_descriptor*>(
          r->meta + slot * TF_DESCRIPTOR_SIZE)->flags >> TF_DESC_CTA_SHIFT;
      if (n_ctas) memset(r->done_flags + slot * kMaxFlagCtas, 0, n_ctas);
      uint64_t* rp = reinterpret_cast<uint64_t*>(r->meta + slot * TF_DESCRIPTOR_SIZE) + 3;
      __atomic_store_n(rp, TF_READY_SENTINEL, __ATOMIC_RELEASE);
      r->meta_tail = ++tail;
      r->consumed += 1;
      advanced = true;
      if (!(d.flags & TF_DESC_HOST_RESERVED)) {
        // before any host reservation made after this capture was reserved
        auto it = r->regions.end();
        while (it != r->regions.begin()) {
          auto prev = std::prev(it);
          if (prev->host && !prev->polled && prev->seq >= d.capture_seq) it = prev;
          else break;
        }
        r->regions.insert(it, HostRegion{d.payload_offset, tf_round_up16(d.payload_len),
                                         d.skip_before, d.flags, true, false, d.capture_seq});
      } else {
        for (HostRegion& h : r->regions)
          if (!h.polled && h.off == d.payload_offset) { h.polled = true; break; }
      }
    } else {
      ++tail;
    }
    if (out) out[got] = d;
    ++got;
  }
  *n = got;
  if (advanced)  // slots are free once consumed (rings.py:402-404)
    return tf_internal_write_u64(r->ctrl_stream, &r->dcons->meta_tail, r->meta_tail);
  return TF_OK;
}

extern "C" int tf_ring_ready_entries(tf_ring* r, uint64_t* n) {
  if (!r || !n) return TF_ERR_VALUE;
  std::lock_guard<std::mutex> g(r->mu);
  uint32_t k = 0;
  int rc = tf_internal_poll(r, r->cfg.meta_slots, nullptr, &k, false);
  *n = k;
  return rc;
}

extern "C" int tf_ring_ready_bytes(tf_ring* r, uint64_t* n) {
  if (!r || !n) return TF_ERR_VALUE;
  std::lock_guard<std::mutex> g(r->mu);
  uint64_t total = 0;
  const uint64_t slots = r->cfg.meta_slots;
  for (uint64_t i = 0; i < slots; ++i) {
    uint64_t slot = (r->meta_tail + i) % slots;
    tf_descriptor d;
    if (slot_ready(r, slot) == TF_READY_SENTINEL || !slot_complete(r, slot, &d))
      break;
    total += d.payload_len;
  }
  *n = total;
  return TF_OK;
}

extern "C" int tf_ring_peek_ready(tf_ring* r, uint32_t max_entries, tf_descriptor* out, uint32_t* n) {
  if (!r || !n) return TF_ERR_VALUE;
  std::lock_guard<std::mutex> g(r->mu);
  return tf_internal_poll(r, max_entries, out, n, false);
}

extern "C" int tf_ring_poll_ready(tf_ring* r, uint32_t max_entries, tf_descriptor* out, uint32_t* n) {
  if (!r || !n) return TF_ERR_VALUE;
  std::lock_guard<std::mutex> g(r->mu);
  return tf_internal_poll(r, max_entries, out, n, true);
}

int tf_internal_release(tf_ring* r, uint64_t offset, uint64_t length, bool push) {
  std::lock_guard<std::mutex> g(r->mu);
  if (r->regions.empty()) {  // rings.py:420-421
    tf_set_error("no outstanding reservation to release");
    return TF_ERR_OUT_OF_ORDER_RELEASE;
  }
  const HostRegion& h = r->regions.front();
  if (h.off != offset || h.len != length) {  // rings.py:423-427
    tf_set_error("release (%llu, %llu) does not match the oldest reservation (%llu, %llu)",
                 (unsigned long long)offset, (unsigned long long)length,
                 (unsigned long long)h.off, (unsigned long long)h.len);
    return TF_ERR_OUT_OF_ORDER_RELEASE;
  }
  if (h.kind & TF_DESC_DEAD_SKIP) r->dead_reclaimed += h.skip;  // :415-419
  r->L += h.skip + h.len;
  r->bytes_released += h.len;
  r->host_reserved.erase(h.off);
  r->regions.pop_front();
  if (push) return tf_internal_write_u64(r->ctrl_stream, &r->dcons->L, r->L);
  return TF_OK;
}

uint64_t tf_internal_l_after_all(tf_ring* r) {
  std::lock_guard<std::mutex> g(r->mu);
  uint64_t L = r->L;
  // stop at the first region whose descriptor the consumer has not taken:
  // a host-reserved region may still be waiting for its payload and publish
  for (const HostRegion& h : r->regions) {
    if (!h.polled) break;
    L += h.skip + h.len;
  }
  return L;
}

extern "C" int tf_ring_release_payload(tf_ring* r, uint64_t offset, uint64_t length) {
  if (!r) return TF_ERR_VALUE;
  return tf_internal_release(r, offset, length, true);
}

extern "C" int tf_ring_host_released(tf_ring* r, uint64_t* bytes_released, uint64_t* consumed) {
  if (!r) return TF_ERR_VALUE;
  std::lock_guard<std::mutex> g(r->mu);
  if (bytes_released) *bytes_released = r->bytes_released;  // reservations, no dead skips
  if (consumed) *consumed = r->consumed;
  return TF_OK;
}

extern "C" int tf_ring_seal(tf_ring* r, void* stream) {
  if (!r) return TF_ERR_VALUE;
  int rc = set_device(r->device);
  if (rc) return rc;
  seal_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(r->ctl, r->seal_host);
  CUDA_TRY(cudaGetLastError());
  return TF_OK;
}

extern "C" int tf_ring_sync_consumer(tf_ring* r) {
  if (!r) return TF_ERR_VALUE;
  int rc = set_device(r->device);
  if (rc) return rc;
  CUDA_TRY(cudaStreamSynchronize((cudaStream_t)r->ctrl_stream));
  return TF_OK;
}

// ---------------------------------------------------------------------------
// shared: snapshots (rings.py:241-276)
// ---------------------------------------------------------------------------
extern "C" int tf_ring_get_state(tf_ring* r, tf_ring_state* o) {
  if (!r || !o) return TF_ERR_VALUE;
  int rc = set_device(r->device);
  if (rc) return rc;
  rc = snapshot(r);
  if (rc) return rc;
  std::lock_guard<std::mutex> g(r->mu);
  const DevCtl* c = r->ctl_host;
  const uint64_t cap = r->cfg.payload_capacity;
  memset(o, 0, sizeof(*o));
  o->payload_head = tf_head(&c->p, cap);
  o->payload_tail = tf_tail(&c->p, r->L, cap);
  o->occupancy = tf_used(&c->p, r->L);
  o->payload_capacity = cap;
  o->meta_head = c->meta_head;
  o->meta_tail = r->meta_tail;
  o->meta_slots = r->cfg.meta_slots;
  o->high_watermark = r->cfg.high_watermark;
  o->bytes_reserved = c->bytes_reserved;
  o->bytes_released = r->bytes_released;
  o->dead_created = c->dead_created;
  o->dead_reclaimed = r->dead_reclaimed;
  o->descriptors_published = c->meta_head;
  o->descriptors_consumed = r->consumed;
  o->captures_launched = c->captures;
  o->drops = c->drops;
  o->drop_bytes = c->drop_bytes;
  o->stall_events = c->stall_events;
  o->stall_ns = c->stall_ns;
  o->device_errors = c->errors;
  o->kernel_ns = c->kernel_ns;
  o->last_kernel_ns = c->last_kernel_ns;
  return TF_OK;
}

extern "C" int tf_ring_free_meta_slots(tf_ring* r, uint64_t* n) {
  if (!r || !n) return TF_ERR_VALUE;
  int rc = set_device(r->device);
  if (rc) return rc;
  rc = snapshot(r);
  if (rc) return rc;
  std::lock_guard<std::mutex> g(r->mu);
  *n = r->cfg.meta_slots - (r->ctl_host->meta_head - r->meta_tail);
  return TF_OK;
}

// rings.py:256-276 would_fit: replay with a frozen consumer cursor.
extern "C" int tf_ring_would_fit(tf_ring* r, const uint64_t* lengths, uint32_t n,
                                 int64_t meta_entries, int* fits) {
  if (!r || !fits || (n && !lengths)) return TF_ERR_VALUE;
  for (uint32_t i = 0; i < n; ++i) {
    if (lengths[i] == 0 || lengths[i] % TF_COPY_UNIT) {
      tf_set_error("lengths must be positive copy-unit multiples");
      return TF_ERR_VALUE;
    }
  }
  int rc = set_device(r->device);
  if (rc) return rc;
  rc = snapshot(r);
  if (rc) return rc;
  std::lock_guard<std::mutex> g(r->mu);
  tf_pstate p = r->ctl_host->p;
  const uint64_t mh = r->ctl_host->meta_head;
  const uint64_t cap = r->cfg.payload_capacity;
  *fits = 0;
  for (uint32_t i = 0; i < n; ++i) {
    uint64_t off, skip;
    uint32_t kind;
    if (!tf_reserve(&p, r->L, cap, lengths[i], &off, &skip, &kind)) return TF_OK;
  }
  uint64_t entries = meta_entries < 0 ? n : (uint64_t)meta_entries;
  uint64_t free_slots = r->cfg.meta_slots - (mh - r->meta_tail);
  *fits = entries <= free_slots;
  return TF_OK;
}

#ifdef TF_TRACE
// experiment builds: copy out the per-launch stamps ([64][1024][6] entry,
// offset known, copy done, scan done, fast plan done, table done) and publish records ([64][2] time, grid)
extern "C" int tf_debug_trace(unsigned long long* stamps, unsigned long long* pub) {
  CUDA_TRY(cudaDeviceSynchronize());
  CUDA_TRY(cudaMemcpyFromSymbol(stamps, g_stamp, sizeof(g_stamp)));
  CUDA_TRY(cudaMemcpyFromSymbol(pub, g_pub, sizeof(g_pub)));
  return TF_OK;
}
#endif
