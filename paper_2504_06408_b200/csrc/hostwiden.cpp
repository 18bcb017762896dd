// Host-side int32 -> int64 widening of downloaded column indices (the
// reference's index_t).  The destination is write-only, so AVX2 streaming
// stores skip the read-for-ownership of every output line: 12 instead of
// 20 bytes of host memory traffic per index, which is what bounds this copy
// while the DMA engine writes the next chunk into host memory.
#include <cstdint>
#include <immintrin.h>

namespace spg {

__attribute__((target("avx2"))) static void widen_avx2(const int32_t* in, int64_t* out, int64_t n) {
  int64_t e = 0;
  while (e < n && (reinterpret_cast<uintptr_t>(out + e) & 31)) {  // align the stores
    out[e] = in[e];
    ++e;
  }
  for (; e + 8 <= n; e += 8) {
    const __m256i x = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(in + e));
    _mm256_stream_si256(reinterpret_cast<__m256i*>(out + e), _mm256_cvtepi32_epi64(_mm256_castsi256_si128(x)));
    _mm256_stream_si256(reinterpret_cast<__m256i*>(out + e + 4), _mm256_cvtepi32_epi64(_mm256_extracti128_si256(x, 1)));
  }
  for (; e < n; ++e) out[e] = in[e];
  _mm_sfence();
}

void widen_i32_to_i64(const int32_t* in, int64_t* out, int64_t n) {
  static const bool avx2 = __builtin_cpu_supports("avx2");
  if (avx2) {
    widen_avx2(in, out, n);
    return;
  }
  for (int64_t e = 0; e < n; ++e) out[e] = in[e];
}

}  // namespace spg

namespace spg {

// int64 -> int32 narrowing of uploaded indices with the range check the
// device narrow kernel does ([0, bound)); returns false on a violation.
__attribute__((target("avx2"))) static bool narrow_avx2(const int64_t* in, int32_t* out, int64_t n, int64_t bound) {
  int64_t e = 0;
  bool ok = true;
  while (e < n && (reinterpret_cast<uintptr_t>(out + e) & 31)) {
    ok &= in[e] >= 0 && in[e] < bound;
    out[e] = (int32_t)in[e];
    ++e;
  }
  const __m256i lo_bad = _mm256_set1_epi64x(-1), hi_bad = _mm256_set1_epi64x(bound - 1);
  const __m256i pick = _mm256_setr_epi32(0, 2, 4, 6, 1, 3, 5, 7);
  __m256i bad = _mm256_setzero_si256();
  for (; e + 8 <= n; e += 8) {
    const __m256i a = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(in + e));
    const __m256i b = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(in + e + 4));
    bad = _mm256_or_si256(bad, _mm256_or_si256(_mm256_cmpgt_epi64(lo_bad, a), _mm256_cmpgt_epi64(a, hi_bad)));
    bad = _mm256_or_si256(bad, _mm256_or_si256(_mm256_cmpgt_epi64(lo_bad, b), _mm256_cmpgt_epi64(b, hi_bad)));
    const __m256i pa = _mm256_permutevar8x32_epi32(a, pick), pb = _mm256_permutevar8x32_epi32(b, pick);
    _mm256_stream_si256(reinterpret_cast<__m256i*>(out + e),
                        _mm256_inserti128_si256(pa, _mm256_castsi256_si128(pb), 1));
  }
  for (; e < n; ++e) {
    ok &= in[e] >= 0 && in[e] < bound;
    out[e] = (int32_t)in[e];
  }
  _mm_sfence();
  return ok && _mm256_testz_si256(bad, bad);
}

bool narrow_i64_to_i32(const int64_t* in, int32_t* out, int64_t n, int64_t bound) {
  static const bool avx2 = __builtin_cpu_supports("avx2");
  if (avx2) return narrow_avx2(in, out, n, bound);
  bool ok = true;
  for (int64_t e = 0; e < n; ++e) {
    ok &= in[e] >= 0 && in[e] < bound;
    out[e] = (int32_t)in[e];
  }
  return ok;
}

}  // namespace spg
