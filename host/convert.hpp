// Host-side element conversions of the drop-in adapter (bfgpu_execute.cpp): float64 Eigen
// storage <-> bf16 / fp32 staging. The AVX2 forms are bit-for-bit the scalar ones
// (tests/cpp/selftest.cpp bfx_conversion_check).
#pragma once

#include <immintrin.h>

#include <cstdint>
#include <cstring>

namespace bfgpu {
namespace conv {

inline uint16_t to_bf16(float f) {
  uint32_t u;
  std::memcpy(&u, &f, 4);
  if ((u & 0x7fffffffu) > 0x7f800000u) return static_cast<uint16_t>((u >> 16) | 0x40u);  // NaN stays NaN
  u += 0x7fffu + ((u >> 16) & 1u);
  return static_cast<uint16_t>(u >> 16);
}

inline float from_bf16(uint16_t h) {
  const uint32_t u = static_cast<uint32_t>(h) << 16;
  float f;
  std::memcpy(&f, &u, 4);
  return f;
}

// 8 doubles -> 8 bf16: round to fp32 (as static_cast<float>), then to bf16 nearest-even, NaN
// kept quiet: the vector form of to_bf16(static_cast<float>(x)), bit for bit.
inline __m128i bf16x8_from_f64(const double* s) {
  const __m256 f = _mm256_set_m128(_mm256_cvtpd_ps(_mm256_loadu_pd(s + 4)), _mm256_cvtpd_ps(_mm256_loadu_pd(s)));
  const __m256i u = _mm256_castps_si256(f);
  const __m256i nan = _mm256_cmpgt_epi32(_mm256_and_si256(u, _mm256_set1_epi32(0x7fffffff)),
                                         _mm256_set1_epi32(0x7f800000));
  const __m256i lsb = _mm256_and_si256(_mm256_srli_epi32(u, 16), _mm256_set1_epi32(1));
  __m256i r = _mm256_add_epi32(u, _mm256_add_epi32(_mm256_set1_epi32(0x7fff), lsb));
  r = _mm256_blendv_epi8(r, _mm256_or_si256(u, _mm256_set1_epi32(0x00400000)), nan);
  r = _mm256_srli_epi32(r, 16);
  // pack within 128-bit lanes, then gather the two lanes' low halves
  const __m256i packed = _mm256_permute4x64_epi64(_mm256_packus_epi32(r, r), 0x08);
  return _mm256_castsi256_si128(packed);
}

// 8 bf16 -> 8 doubles (exact)
inline void f64x8_from_bf16(const uint16_t* s, double* d) {
  const __m256 f = _mm256_castsi256_ps(
      _mm256_slli_epi32(_mm256_cvtepu16_epi32(_mm_loadu_si128(reinterpret_cast<const __m128i*>(s))), 16));
  _mm256_storeu_pd(d, _mm256_cvtps_pd(_mm256_castps256_ps128(f)));
  _mm256_storeu_pd(d + 4, _mm256_cvtps_pd(_mm256_extractf128_ps(f, 1)));
}

}  // namespace conv
}  // namespace bfgpu
