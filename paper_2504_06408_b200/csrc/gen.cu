// Host-side workload generators (input plumbing for the BASELINE configs).
//
//  * generate_rmat — bit-identical restatement of the reference generator
//    (rmat.hpp:15-60): mt19937_64(seed), Graph500 quadrants (0.57, 0.19,
//    0.19, 0.05), no permutation, weight from_real(1 + u01) drawn after the
//    `scale` quadrant draws, then normalize_coo (formats.hpp:105-133): stable
//    row-major sort, duplicates folded with SR::add in input order, zeros
//    dropped.  The stable sort is an LSD radix sort over (row, col) keys.
//  * generate_er — counter-based Erdos-Renyi-style rows (SURVEY.md §8d
//    config 5): row i draws d columns col = h % n with
//    h = splitmix64(splitmix64(seed) + i*d + t); duplicates fold in t order.
//  * generate_stencil27 — 3D 27-point Laplacian on an N^3 grid, Dirichlet
//    boundary: diagonal from_real(26), off-diagonal from_real(-1) (config 4).
// Parity of generate_rmat against the reference is checked in
// tests/test_host.py through oracle/_ref.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <random>
#include <thread>
#include <vector>

#include "common.cuh"
#include "semiring.cuh"

namespace spg {
namespace {

SPG_HD uint64_t mix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

template <class T>
T* hmalloc(size_t n) {
  void* p = std::malloc(sizeof(T) * std::max<size_t>(n, 1));
  if (!p) fail(SPG_ERR_OOM, "host allocation failed");
  return static_cast<T*>(p);
}

// Stable LSD radix sort of `order` by keys[order[i]] (keys < 2^bits).
void stable_radix_order(const std::vector<uint64_t>& keys, int bits, std::vector<uint32_t>& order) {
  const size_t n = keys.size();
  std::vector<uint32_t> tmp(n);
  constexpr int kDigit = 11;
  constexpr int kBuckets = 1 << kDigit;
  for (int shift = 0; shift < bits; shift += kDigit) {
    std::vector<size_t> cnt(kBuckets + 1, 0);
    for (size_t i = 0; i < n; ++i) ++cnt[((keys[order[i]] >> shift) & (kBuckets - 1)) + 1];
    for (int b = 0; b < kBuckets; ++b) cnt[b + 1] += cnt[b];
    for (size_t i = 0; i < n; ++i) tmp[cnt[(keys[order[i]] >> shift) & (kBuckets - 1)]++] = order[i];
    order.swap(tmp);
  }
}

template <class SR>
void rmat(int scale, double edge_factor, uint64_t seed, int64_t* nrows, int64_t* nnz, int64_t** rows,
          int64_t** cols, void** vals) {
  using V = typename SR::value_type;
  if (scale < 1) fail(SPG_ERR_INVALID_RANGE, "rmat scale must be >= 1");
  if (scale > 31) fail(SPG_ERR_INVALID_RANGE, "rmat scale must be <= 31");
  if (edge_factor <= 0.0) fail(SPG_ERR_INVALID_RANGE, "rmat edge factor must be > 0");
  constexpr double kA = 0.57;
  constexpr double kB = 0.19;
  constexpr double kC = 0.19;
  const int64_t n = int64_t{1} << scale;
  const int64_t ne = static_cast<int64_t>(std::llround(edge_factor * static_cast<double>(n)));
  if (ne > (int64_t)UINT32_MAX) fail(SPG_ERR_INVALID_RANGE, "rmat: too many edges");
  std::mt19937_64 rng(seed);
  auto u01 = [&rng]() { return static_cast<double>(rng() >> 11) * 0x1.0p-53; };
  std::vector<uint64_t> keys(ne);
  std::vector<V> v(ne);
  for (int64_t e = 0; e < ne; ++e) {
    int64_t r = 0, c = 0;
    for (int level = 0; level < scale; ++level) {
      const double u = u01();
      r <<= 1;
      c <<= 1;
      if (u < kA) {
      } else if (u < kA + kB) {
        c |= 1;
      } else if (u < kA + kB + kC) {
        r |= 1;
      } else {
        r |= 1;
        c |= 1;
      }
    }
    keys[e] = ((uint64_t)r << scale) | (uint64_t)c;
    v[e] = SR::from_real(1.0 + u01());
  }
  std::vector<uint32_t> order(ne);
  for (int64_t e = 0; e < ne; ++e) order[e] = (uint32_t)e;
  stable_radix_order(keys, 2 * scale, order);
  // fold runs of equal keys in input order, drop zeros
  std::vector<int64_t> orow, ocol;
  std::vector<V> oval;
  orow.reserve(ne);
  ocol.reserve(ne);
  oval.reserve(ne);
  const uint64_t cmask = (uint64_t{1} << scale) - 1;
  for (int64_t i = 0; i < ne;) {
    const uint64_t k = keys[order[i]];
    V acc = v[order[i]];
    int64_t j = i + 1;
    for (; j < ne && keys[order[j]] == k; ++j) acc = SR::add(acc, v[order[j]]);
    if (!SR::is_zero(acc)) {
      orow.push_back((int64_t)(k >> scale));
      ocol.push_back((int64_t)(k & cmask));
      oval.push_back(acc);
    }
    i = j;
  }
  const size_t m = orow.size();
  *nrows = n;
  *nnz = (int64_t)m;
  *rows = hmalloc<int64_t>(m);
  *cols = hmalloc<int64_t>(m);
  V* ov = hmalloc<V>(m);
  std::memcpy(*rows, orow.data(), sizeof(int64_t) * m);
  std::memcpy(*cols, ocol.data(), sizeof(int64_t) * m);
  std::memcpy(ov, oval.data(), sizeof(V) * m);
  *vals = ov;
}

template <class SR>
void er(int64_t n, int d, uint64_t seed, int value_mode, int64_t r0, int64_t r1, int64_t c0, int64_t c1,
        int64_t* nnz, int64_t** rows, int64_t** cols, void** vals) {
  using V = typename SR::value_type;
  if (n < 1 || d < 1) fail(SPG_ERR_INVALID_RANGE, "er: need n >= 1 and d >= 1");
  if (r0 < 0 || r1 > n || r0 > r1 || c0 < 0 || c1 > n || c0 > c1) fail(SPG_ERR_INVALID_RANGE, "er: bad block");
  if (value_mode == 1 && sizeof(V) != 16) fail(SPG_ERR_ARG, "er: value_mode 1 needs a 16-byte value type");
  const uint64_t s = mix64(seed);
  const int T = std::max(1u, std::min(64u, std::thread::hardware_concurrency()));
  std::vector<std::vector<int64_t>> pr(T), pc(T);
  std::vector<std::vector<V>> pv(T);
  std::vector<std::thread> ts;
  for (int w = 0; w < T; ++w) {
    ts.emplace_back([&, w] {
      const int64_t lo = r0 + (r1 - r0) * w / T, hi = r0 + (r1 - r0) * (w + 1) / T;
      std::vector<std::pair<int64_t, V>> row(d);
      std::vector<int> idx(d);
      for (int64_t i = lo; i < hi; ++i) {
        for (int t = 0; t < d; ++t) {
          const uint64_t h = mix64(s + (uint64_t)i * (uint64_t)d + (uint64_t)t);
          const double u = static_cast<double>(mix64(h) >> 11) * 0x1.0p-53;
          V val;
          if (value_mode == 1) {
            struct { double w; uint64_t tag; } sv{0.5 + u, mix64(h ^ 0xd6e8feb86659fd93ULL)};
            std::memcpy(&val, &sv, sizeof(V));
          } else {
            val = SR::from_real(0.5 + u);
          }
          row[t] = {(int64_t)(h % (uint64_t)n), val};
          idx[t] = t;
        }
        std::stable_sort(idx.begin(), idx.end(), [&](int a, int b) { return row[a].first < row[b].first; });
        for (int a = 0; a < d;) {
          V acc = row[idx[a]].second;
          int b = a + 1;
          for (; b < d && row[idx[b]].first == row[idx[a]].first; ++b) acc = SR::add(acc, row[idx[b]].second);
          const int64_t col = row[idx[a]].first;
          if (!SR::is_zero(acc) && col >= c0 && col < c1) {
            pr[w].push_back(i);
            pc[w].push_back(col);
            pv[w].push_back(acc);
          }
          a = b;
        }
      }
    });
  }
  for (auto& t : ts) t.join();
  size_t m = 0;
  for (int w = 0; w < T; ++w) m += pr[w].size();
  *nnz = (int64_t)m;
  *rows = hmalloc<int64_t>(m);
  *cols = hmalloc<int64_t>(m);
  V* ov = hmalloc<V>(m);
  size_t o = 0;
  for (int w = 0; w < T; ++w) {
    std::memcpy(*rows + o, pr[w].data(), sizeof(int64_t) * pr[w].size());
    std::memcpy(*cols + o, pc[w].data(), sizeof(int64_t) * pc[w].size());
    std::memcpy(ov + o, pv[w].data(), sizeof(V) * pv[w].size());
    o += pr[w].size();
  }
  *vals = ov;
}

template <class SR>
void stencil27(int64_t N, int64_t r0, int64_t r1, int64_t c0, int64_t c1, int64_t* nrows, int64_t* nnz,
               int64_t** rows, int64_t** cols, void** vals) {
  using V = typename SR::value_type;
  if (N < 1) fail(SPG_ERR_INVALID_RANGE, "stencil27: N must be >= 1");
  const int64_t n = N * N * N;
  if (r0 < 0 || r1 > n || r0 > r1 || c0 < 0 || c1 > n || c0 > c1) fail(SPG_ERR_INVALID_RANGE, "stencil27: bad block");
  const V diag = SR::from_real(26.0), off = SR::from_real(-1.0);
  // rows are independent: threads take contiguous row ranges, then concatenate
  const int T = std::max(1u, std::min(64u, std::thread::hardware_concurrency()));
  std::vector<std::vector<int64_t>> pr(T), pc(T);
  std::vector<std::vector<V>> pv(T);
  std::vector<std::thread> ts;
  for (int w = 0; w < T; ++w) {
    ts.emplace_back([&, w] {
      const int64_t lo = r0 + (r1 - r0) * w / T, hi = r0 + (r1 - r0) * (w + 1) / T;
      for (int64_t i = lo; i < hi; ++i) {
        const int64_t x = i % N, y = (i / N) % N, z = i / (N * N);
        for (int dz = -1; dz <= 1; ++dz)
          for (int dy = -1; dy <= 1; ++dy)
            for (int dx = -1; dx <= 1; ++dx) {
              const int64_t zz = z + dz, yy = y + dy, xx = x + dx;
              if (zz < 0 || zz >= N || yy < 0 || yy >= N || xx < 0 || xx >= N) continue;
              const int64_t col = (zz * N + yy) * N + xx;
              if (col < c0 || col >= c1) continue;
              pr[w].push_back(i);
              pc[w].push_back(col);
              pv[w].push_back((dx == 0 && dy == 0 && dz == 0) ? diag : off);
            }
      }
    });
  }
  for (auto& t : ts) t.join();
  size_t m = 0;
  for (int w = 0; w < T; ++w) m += pr[w].size();
  int64_t* r = hmalloc<int64_t>(m);
  int64_t* c = hmalloc<int64_t>(m);
  V* v = hmalloc<V>(m);
  size_t o = 0;
  for (int w = 0; w < T; ++w) {
    std::memcpy(r + o, pr[w].data(), sizeof(int64_t) * pr[w].size());
    std::memcpy(c + o, pc[w].data(), sizeof(int64_t) * pc[w].size());
    std::memcpy(v + o, pv[w].data(), sizeof(V) * pv[w].size());
    o += pr[w].size();
  }
  *nrows = n;
  *nnz = (int64_t)m;
  *rows = r;
  *cols = c;
  *vals = v;
}

template <class F>
void with_builtin(int sr, F&& f) {
  switch (sr) {
    case SPG_SR_ARITHMETIC: f(Arithmetic{}); break;
    case SPG_SR_MINPLUS: f(MinPlus{}); break;
    case SPG_SR_BOOLEAN: f(Boolean{}); break;
    case SPG_SR_MINSELECT: f(MinSelect{}); break;
    case SPG_SR_TROPICAL_I32: f(TropicalI32{}); break;
    case SPG_SR_MAXTIMES: f(MaxTimes{}); break;
    default: fail(SPG_ERR_ARG, "unknown semiring id " + std::to_string(sr));
  }
}

}  // namespace

void gen_rmat(int sr, int scale, double ef, uint64_t seed, int64_t* nrows, int64_t* nnz, int64_t** rows,
              int64_t** cols, void** vals) {
  with_builtin(sr, [&](auto t) { rmat<decltype(t)>(scale, ef, seed, nrows, nnz, rows, cols, vals); });
}
void gen_er(int sr, int64_t n, int d, uint64_t seed, int mode, int64_t r0, int64_t r1, int64_t c0, int64_t c1,
            int64_t* nnz, int64_t** rows, int64_t** cols, void** vals) {
  with_builtin(sr, [&](auto t) { er<decltype(t)>(n, d, seed, mode, r0, r1, c0, c1, nnz, rows, cols, vals); });
}
void gen_stencil27(int sr, int64_t N, int64_t r0, int64_t r1, int64_t c0, int64_t c1, int64_t* nrows, int64_t* nnz,
                   int64_t** rows, int64_t** cols, void** vals) {
  with_builtin(sr, [&](auto t) { stencil27<decltype(t)>(N, r0, r1, c0, c1, nrows, nnz, rows, cols, vals); });
}

}  // namespace spg
