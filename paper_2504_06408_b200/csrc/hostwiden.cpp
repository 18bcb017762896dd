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
