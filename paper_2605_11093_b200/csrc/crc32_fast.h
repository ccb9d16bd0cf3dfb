// crc32_fast.h — zlib-compatible CRC-32 (ISO-HDLC, reflected 0xEDB88320)
// by carry-less multiplication folding (PCLMULQDQ), for the record
// checksums of the exporter's sinks (SRC/records.py crc32 = zlib.crc32).
//
// The bulk of a buffer is folded 64 bytes per step in four independent
// 128-bit lanes (x^(512±64) mod P constants), the lanes are folded into one,
// reduced to 64 and then 32 bits with a Barrett reduction; the sub-64-byte
// head/tail go through zlib. Same result as zlib's crc32() for every input
// (tests/test_native_sink.py compares them on random buffers and offsets).
// Falls back to zlib when the CPU lacks PCLMULQDQ.
#pragma once
#include <stddef.h>
#include <stdint.h>
#include <zlib.h>

#if defined(__x86_64__)
#include <immintrin.h>

namespace tfcrc {

__attribute__((target("pclmul,sse4.1"))) static inline __m128i fold16(__m128i a, __m128i next,
                                                                       __m128i k) {
  const __m128i h = _mm_clmulepi64_si128(a, k, 0x11);
  a = _mm_clmulepi64_si128(a, k, 0x00);
  return _mm_xor_si128(_mm_xor_si128(a, h), next);
}

// reflected-domain constants for P = 0x104C11DB7 (x^n mod P, bit-reflected)
//   k1 = x^(4*128+32) , k2 = x^(4*128-32)   fold 64 B
//   k3 = x^(128+32)   , k4 = x^(128-32)     fold 16 B
//   k5 = x^64                               64 -> 32 bit step
//   mu = floor(x^64 / P), poly = P          Barrett reduction
__attribute__((target("pclmul,sse4.1"))) static inline uint32_t fold_le(uint32_t crc,
                                                                        const uint8_t* p,
                                                                        size_t len) {
  // len >= 64 and a multiple of 16; crc in the un-inverted (kernel) domain
  const __m128i k1k2 = _mm_set_epi64x(0x1c6e41596ll, 0x154442bd4ll);
  const __m128i k3k4 = _mm_set_epi64x(0x0ccaa009ell, 0x1751997d0ll);
  const __m128i k5 = _mm_set_epi64x(0, 0x163cd6124ll);
  const __m128i mask32 = _mm_set_epi32(0, 0, 0, -1);
  const __m128i poly_mu = _mm_set_epi64x(0x1f7011641ll, 0x1db710641ll);
  __m128i x1 = _mm_loadu_si128(reinterpret_cast<const __m128i*>(p));
  __m128i x2 = _mm_loadu_si128(reinterpret_cast<const __m128i*>(p + 16));
  __m128i x3 = _mm_loadu_si128(reinterpret_cast<const __m128i*>(p + 32));
  __m128i x4 = _mm_loadu_si128(reinterpret_cast<const __m128i*>(p + 48));
  x1 = _mm_xor_si128(x1, _mm_cvtsi32_si128(int(crc)));
  p += 64;
  len -= 64;
  while (len >= 64) {
    __m128i h1 = _mm_clmulepi64_si128(x1, k1k2, 0x11);
    __m128i h2 = _mm_clmulepi64_si128(x2, k1k2, 0x11);
    __m128i h3 = _mm_clmulepi64_si128(x3, k1k2, 0x11);
    __m128i h4 = _mm_clmulepi64_si128(x4, k1k2, 0x11);
    x1 = _mm_clmulepi64_si128(x1, k1k2, 0x00);
    x2 = _mm_clmulepi64_si128(x2, k1k2, 0x00);
    x3 = _mm_clmulepi64_si128(x3, k1k2, 0x00);
    x4 = _mm_clmulepi64_si128(x4, k1k2, 0x00);
    x1 = _mm_xor_si128(_mm_xor_si128(x1, h1),
                       _mm_loadu_si128(reinterpret_cast<const __m128i*>(p)));
    x2 = _mm_xor_si128(_mm_xor_si128(x2, h2),
                       _mm_loadu_si128(reinterpret_cast<const __m128i*>(p + 16)));
    x3 = _mm_xor_si128(_mm_xor_si128(x3, h3),
                       _mm_loadu_si128(reinterpret_cast<const __m128i*>(p + 32)));
    x4 = _mm_xor_si128(_mm_xor_si128(x4, h4),
                       _mm_loadu_si128(reinterpret_cast<const __m128i*>(p + 48)));
    p += 64;
    len -= 64;
  }
  x1 = fold16(x1, x2, k3k4);
  x1 = fold16(x1, x3, k3k4);
  x1 = fold16(x1, x4, k3k4);
  while (len >= 16) {
    x1 = fold16(x1, _mm_loadu_si128(reinterpret_cast<const __m128i*>(p)), k3k4);
    p += 16;
    len -= 16;
  }
  // 128 -> 64 bits (appends 32 zero bits)
  __m128i t = _mm_clmulepi64_si128(k3k4, x1, 0x01);
  x1 = _mm_xor_si128(_mm_srli_si128(x1, 8), t);
  // 64 -> 32 bits
  __m128i x2b = _mm_srli_si128(x1, 4);
  x1 = _mm_and_si128(x1, mask32);
  x1 = _mm_clmulepi64_si128(x1, k5, 0x00);
  x1 = _mm_xor_si128(x1, x2b);
  // Barrett reduction
  __m128i x2c = x1;
  x1 = _mm_and_si128(x1, mask32);
  x1 = _mm_clmulepi64_si128(x1, poly_mu, 0x10);
  x1 = _mm_and_si128(x1, mask32);
  x1 = _mm_clmulepi64_si128(x1, poly_mu, 0x00);
  x1 = _mm_xor_si128(x1, x2c);
  return uint32_t(_mm_extract_epi32(x1, 1));
}

inline bool have_pclmul() {
  static const int ok = __builtin_cpu_supports("pclmul") && __builtin_cpu_supports("sse4.1");
  return ok;
}

}  // namespace tfcrc

// zlib.crc32(data, crc) semantics
inline uint32_t tf_crc32_fast(uint32_t crc, const uint8_t* p, size_t n) {
  if (n >= 128 && tfcrc::have_pclmul()) {
    const size_t bulk = n & ~size_t(15);
    crc = ~tfcrc::fold_le(~crc, p, bulk);
    p += bulk;
    n -= bulk;
  }
  while (n) {
    const uInt step = uInt(n < (1u << 30) ? n : (1u << 30));
    crc = uint32_t(crc32(crc, p, step));
    p += step;
    n -= step;
  }
  return crc;
}

#else
inline uint32_t tf_crc32_fast(uint32_t crc, const uint8_t* p, size_t n) {
  while (n) {
    const uInt step = uInt(n < (1u << 30) ? n : (1u << 30));
    crc = uint32_t(crc32(crc, p, step));
    p += step;
    n -= step;
  }
  return crc;
}
#endif
