/*
 * cast_oracle.c — TEST INFRASTRUCTURE, not product code.
 *
 * CPU restatement of the north-star extensions that have no reference
 * implementation ("parity unpinned by reference tests;
 * pinned only by the builder's restatement"):
 *
 *   or_cast    element-wise conversion of captured rows, round-to-nearest-
 *              even; fp8 targets saturate to the largest finite value
 *              (the PTX cvt.rn.satfinite semantics). Written from the IEEE
 *              / OCP-FP8 definitions with integer bit manipulation, so it
 *              shares nothing with the CUDA intrinsics it checks.
 *   or_reduce  per-row (per-token) reductions in double precision:
 *              mean, l2 = sqrt(sum x^2), absmax, rms, stats = (mean, l2,
 *              min, max), results rounded to f32.
 *
 * dtype codes follow include/ring2.h tf_dtype.
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

enum { D_F16 = 2, D_BF16 = 3, D_F32 = 4, D_E4M3 = 8, D_E5M2 = 9 };

static float bits_f32(uint32_t u) { float f; memcpy(&f, &u, 4); return f; }
static uint32_t f32_bits(float f) { uint32_t u; memcpy(&u, &f, 4); return u; }

static float f16_to_f32(uint16_t h) {
  uint32_t sign = (uint32_t)(h & 0x8000u) << 16;
  uint32_t e = (h >> 10) & 0x1F, m = h & 0x3FF;
  if (e == 0) {
    float v = (float)m * 5.9604644775390625e-08f; /* 2^-24, exact */
    return sign ? -v : v;
  }
  if (e == 31) return bits_f32(sign | 0x7F800000u | (m << 13));
  return bits_f32(sign | ((e - 15 + 127) << 23) | (m << 13));
}

static float bf16_to_f32(uint16_t b) { return bits_f32((uint32_t)b << 16); }

static uint16_t f32_to_bf16(float f) {
  uint32_t u = f32_bits(f);
  if ((u & 0x7FFFFFFFu) > 0x7F800000u) return (uint16_t)((u >> 16) | 0x40);
  uint32_t lsb = (u >> 16) & 1u;
  return (uint16_t)((u + 0x7FFFu + lsb) >> 16);
}

static uint16_t f32_to_f16(float f) {
  uint32_t x = f32_bits(f);
  uint16_t sign = (uint16_t)((x >> 16) & 0x8000u);
  uint32_t ax = x & 0x7FFFFFFFu;
  if (ax > 0x7F800000u) return sign | 0x7E00u;
  if (ax >= 0x477FF000u) return sign | 0x7C00u;       /* >= 65520 -> inf */
  if (ax < 0x38800000u) {                              /* half subnormal */
    double q = (double)bits_f32(ax) * 16777216.0;      /* / 2^-24, exact */
    return sign | (uint16_t)rint(q);                   /* ties to even */
  }
  uint32_t e = (ax >> 23) - 127 + 15, m = ax & 0x7FFFFFu;
  uint32_t h = (e << 10) | (m >> 13), rem = m & 0x1FFFu;
  if (rem > 0x1000u || (rem == 0x1000u && (h & 1u))) h += 1;
  return sign | (uint16_t)h;
}

/* generic fp8 encode: ebits/mbits, bias, max finite code, subnormal scale */
static uint8_t f32_to_fp8(float f, int mbits, int bias, uint8_t maxcode,
                          uint8_t nancode, double maxval) {
  uint32_t x = f32_bits(f);
  uint8_t sign = (uint8_t)((x >> 24) & 0x80u);
  uint32_t ax = x & 0x7FFFFFFFu;
  if (ax > 0x7F800000u) return sign | nancode;
  double a = (double)bits_f32(ax);
  if (a >= maxval) return sign | maxcode;            /* satfinite */
  int E = (int)(ax >> 23) - 127;
  int emin = 1 - bias;
  if (E < emin) {                                    /* subnormal */
    double q = ldexp(a, -(emin - mbits));
    return sign | (uint8_t)rint(q);
  }
  uint32_t m = ax & 0x7FFFFFu;
  int drop = 23 - mbits;
  uint32_t keep = m >> drop, rem = m & ((1u << drop) - 1), half = 1u << (drop - 1);
  uint32_t code = ((uint32_t)(E + bias) << mbits) | keep;
  if (rem > half || (rem == half && (code & 1u))) code += 1;
  if (code > maxcode) code = maxcode;
  return sign | (uint8_t)code;
}

static float load_elem(const uint8_t* p, int dt) {
  uint16_t h;
  switch (dt) {
    case D_F32: { float f; memcpy(&f, p, 4); return f; }
    case D_F16: memcpy(&h, p, 2); return f16_to_f32(h);
    case D_BF16: memcpy(&h, p, 2); return bf16_to_f32(h);
  }
  return 0.f;
}

static int width(int dt) {
  switch (dt) {
    case D_F32: return 4;
    case D_F16: case D_BF16: return 2;
    case D_E4M3: case D_E5M2: return 1;
  }
  return 0;
}

/* Convert n elements; returns bytes written or -1 on a bad dtype. */
long or_cast(const uint8_t* src, long n, int in_dt, int out_dt, uint8_t* dst) {
  int wi = width(in_dt), wo = width(out_dt);
  if (!wi || !wo || in_dt == D_E4M3 || in_dt == D_E5M2) return -1;
  for (long i = 0; i < n; ++i) {
    float v = load_elem(src + i * wi, in_dt);
    uint8_t* o = dst + i * wo;
    uint16_t h;
    switch (out_dt) {
      case D_F32: memcpy(o, &v, 4); break;
      case D_F16: h = f32_to_f16(v); memcpy(o, &h, 2); break;
      case D_BF16: h = f32_to_bf16(v); memcpy(o, &h, 2); break;
      case D_E4M3: *o = f32_to_fp8(v, 3, 7, 0x7E, 0x7F, 448.0); break;
      case D_E5M2: *o = f32_to_fp8(v, 2, 15, 0x7B, 0x7F, 57344.0); break;
    }
  }
  return n * wo;
}

/* Decode one element of any supported dtype to f32 (for tests). */
float or_decode(const uint8_t* p, int dt) {
  if (dt == D_E4M3 || dt == D_E5M2) {
    int mbits = dt == D_E4M3 ? 3 : 2, bias = dt == D_E4M3 ? 7 : 15;
    uint8_t c = *p;
    int s = c >> 7, e = (c >> mbits) & ((1 << (7 - mbits)) - 1), m = c & ((1 << mbits) - 1);
    double v = e ? ldexp(1.0 + m / (double)(1 << mbits), e - bias)
                 : ldexp((double)m, 1 - bias - mbits);
    return (float)(s ? -v : v);
  }
  return load_elem(p, dt);
}

/* op: 0 mean, 1 l2, 2 absmax, 3 rms, 4 stats (4 outputs) */
long or_reduce(const uint8_t* src, long rows, long h, long row_stride,
               int in_dt, int op, float* dst) {
  int wi = width(in_dt);
  if (!wi || h <= 0) return -1;
  int k = op == 4 ? 4 : 1;
  for (long r = 0; r < rows; ++r) {
    const uint8_t* row = src + r * row_stride;
    double sum = 0, sq = 0;
    float mn = INFINITY, mx = -INFINITY, amax = 0.f;
    for (long i = 0; i < h; ++i) {
      float x = load_elem(row + i * wi, in_dt);
      sum += (double)x;
      sq += (double)x * (double)x;
      if (x < mn) mn = x;
      if (x > mx) mx = x;
      if (fabsf(x) > amax) amax = fabsf(x);
    }
    float* o = dst + r * k;
    switch (op) {
      case 0: o[0] = (float)(sum / (double)h); break;
      case 1: o[0] = (float)sqrt(sq); break;
      case 2: o[0] = amax; break;
      case 3: o[0] = (float)sqrt(sq / (double)h); break;
      default: o[0] = (float)(sum / (double)h); o[1] = (float)sqrt(sq); o[2] = mn; o[3] = mx;
    }
  }
  return rows * k * 4;
}
