// TEST INFRASTRUCTURE — NOT PRODUCT CODE.
//
// CPU restatement of the reference's semiring algebra, used only by the
// parity oracle (oracle/spg_oracle.cpp).  Only tests/, __graft_entry__.smoke()
// and bench.py's cpu_baseline leg may load anything under oracle/.
//
// Each built-in follows /root/reference/proj/include/spsumma/semiring.hpp:
//   ArithmeticSemiring  :43-54   MinPlusSemiring :59-72
//   BooleanSemiring     :75-86   MinSelectSemiring :97-120
// Two semirings the reference lacks but BASELINE configs 2 and 5 need are
// restated here from SURVEY.md §8(a) row a2: TropicalI32 (min, saturating +
// over int32, zero = INT32_MAX) and MaxTimes (struct {double w; uint64 tag},
// add = max by (w, tag), mul = {w*w', tag ^ tag'}).
//
// Value byte encodings follow ValueCodec (serialize.hpp:29-76): little-endian
// fixed width; bool is one byte.
#pragma once
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>

namespace orc {

enum SrId : int {
  kArithmetic = 0,
  kMinPlus = 1,
  kBoolean = 2,
  kMinSelect = 3,
  kTropicalI32 = 4,
  kMaxTimes = 5,
};

struct MinSelectV {
  double weight;
  int64_t payload;
};
struct MaxTimesV {
  double w;
  uint64_t tag;
};

struct Arith {
  using V = double;
  static V zero() { return 0.0; }
  static V add(V a, V b) { return a + b; }
  static V mul(V a, V b) { return a * b; }
  static bool is_zero(V v) { return v == 0.0; }
  static bool eq(V a, V b) { return a == b; }
};

struct MinPlus {
  using V = double;
  static V zero() { return std::numeric_limits<double>::infinity(); }
  static V add(V a, V b) { return b < a ? b : a; }  // std::min(a, b) returns a on ties
  static V mul(V a, V b) { return a + b; }
  static bool is_zero(V v) { return v == zero(); }
  static bool eq(V a, V b) { return a == b; }
};

struct Boolean {
  using V = uint8_t;
  static V zero() { return 0; }
  static V add(V a, V b) { return (a || b) ? 1 : 0; }
  static V mul(V a, V b) { return (a && b) ? 1 : 0; }
  static bool is_zero(V v) { return v == 0; }
  static bool eq(V a, V b) { return (a != 0) == (b != 0); }
};

struct MinSelect {
  using V = MinSelectV;
  static constexpr int64_t kNeutral = -1;
  static V zero() { return {std::numeric_limits<double>::infinity(), std::numeric_limits<int64_t>::max()}; }
  static V add(const V& a, const V& b) {
    const V& p = (b.weight < a.weight || (b.weight == a.weight && b.payload < a.payload)) ? b : a;
    return std::isinf(p.weight) ? zero() : p;
  }
  static V mul(const V& a, const V& b) {
    const double w = a.weight + b.weight;
    if (std::isinf(w)) return zero();
    return {w, b.payload == kNeutral ? a.payload : b.payload};
  }
  static bool is_zero(const V& v) { return std::isinf(v.weight); }
  static bool eq(const V& a, const V& b) { return a.weight == b.weight && a.payload == b.payload; }
};

struct TropicalI32 {
  using V = int32_t;
  static V zero() { return std::numeric_limits<int32_t>::max(); }
  static V add(V a, V b) { return b < a ? b : a; }
  static V mul(V a, V b) {
    if (a == zero() || b == zero()) return zero();
    int64_t s = (int64_t)a + (int64_t)b;
    if (s >= (int64_t)zero()) return zero();
    if (s < (int64_t)std::numeric_limits<int32_t>::min()) return std::numeric_limits<int32_t>::min();
    return (V)s;
  }
  static bool is_zero(V v) { return v == zero(); }
  static bool eq(V a, V b) { return a == b; }
};

struct MaxTimes {
  using V = MaxTimesV;
  static V zero() { return {0.0, 0}; }
  static V add(const V& a, const V& b) {
    return (b.w > a.w || (b.w == a.w && b.tag > a.tag)) ? b : a;
  }
  static V mul(const V& a, const V& b) {
    const double w = a.w * b.w;
    if (w == 0.0) return zero();
    return {w, a.tag ^ b.tag};
  }
  static bool is_zero(const V& v) { return v.w == 0.0; }
  static bool eq(const V& a, const V& b) { return a.w == b.w && a.tag == b.tag; }
};

inline int value_size(int sr) {
  switch (sr) {
    case kArithmetic: case kMinPlus: return 8;
    case kBoolean: return 1;
    case kMinSelect: case kMaxTimes: return 16;
    case kTropicalI32: return 4;
  }
  return -1;
}

template <class SR>
inline int value_size_of() {
  return static_cast<int>(sizeof(typename SR::V));
}

// Dispatches a runtime semiring id to a template functor.
template <class F>
int with_sr(int sr, F&& f) {
  switch (sr) {
    case kArithmetic: return f(Arith{});
    case kMinPlus: return f(MinPlus{});
    case kBoolean: return f(Boolean{});
    case kMinSelect: return f(MinSelect{});
    case kTropicalI32: return f(TropicalI32{});
    case kMaxTimes: return f(MaxTimes{});
  }
  return -1;
}

// checksum.hpp:10-15
inline uint64_t splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

// FNV-1a over the ValueCodec little-endian bytes (checksum.hpp:25-29).
// The host is little-endian x86-64, so the in-memory bytes are the codec
// bytes for every value type used here.
inline uint64_t fnv1a(const void* p, int n) {
  const uint8_t* b = static_cast<const uint8_t*>(p);
  uint64_t v = 0xcbf29ce484222325ULL;
  for (int i = 0; i < n; ++i) v = (v ^ b[i]) * 0x100000001b3ULL;
  return v;
}

// One tuple's contribution (checksum.hpp:30-33).
inline uint64_t tuple_hash(int64_t row, int64_t col, uint64_t vhash) {
  uint64_t h = splitmix64((uint64_t)row);
  h ^= splitmix64((uint64_t)col + 0x9e3779b97f4a7c15ULL);
  h ^= vhash;
  return splitmix64(h);
}

// Dims seed (checksum.hpp:23-24).
inline uint64_t checksum_seed(int64_t nrows, int64_t ncols) {
  return splitmix64((uint64_t)nrows * 31 + (uint64_t)ncols);
}

}  // namespace orc
