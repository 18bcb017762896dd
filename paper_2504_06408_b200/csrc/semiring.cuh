// Semiring functors for the B200 SpGEMM engine.
//
// Each built-in restates a reference algebra with identical semantics
// (/root/reference/proj/include/spsumma/semiring.hpp):
//   Arithmetic  :43-54   MinPlus :59-72   Boolean :75-86   MinSelect :97-120
// plus the two BASELINE semirings the reference lacks:
//   TropicalI32 (config 2): (min, saturating +) over int32, zero = INT32_MAX
//   MaxTimes    (config 5): struct {double w; uint64 tag}, add = max by (w, tag),
//                           mul = {w * w', tag ^ tag'}; commutative.
//
// A semiring is a static policy type (the reference's SemiringLike concept):
//   value_type, add, mul, zero, one, is_zero, from_real, name,
//   is_commutative_mul
// all __host__ __device__ so they inline into the kernels (no virtual calls).
// Two optional members let a semiring pick a cheaper accumulate than the
// generic compare-and-swap loop:
//   acc_shared(V* p, V v)  - atomic  *p = add(*p, v)  on shared memory
//   acc_global(V* p, V v)  - same on global memory
// `has_acc` detects them; `spg::atomic_accumulate` falls back to a CAS loop
// of the value's width (4, 8 or 16 bytes; sm_90+ has native 128-bit CAS).
//
// Custom semirings: define a struct with the members above in your own .cu
// translation unit and instantiate the kernels with SPG_INSTANTIATE
// (spgemm_b200/instantiate.cuh).
#pragma once
#include <cstdint>
#include <cmath>

#ifndef SPG_HD
#define SPG_HD __host__ __device__ __forceinline__
#endif

namespace spg {

struct MinSelectV {
  double weight;
  int64_t payload;
};
struct __align__(16) MaxTimesV {
  double w;
  uint64_t tag;
};
// MinSelect needs 16-byte alignment for the 128-bit CAS.
struct __align__(16) MinSelectA {
  double weight;
  int64_t payload;
};

struct Arithmetic {
  using value_type = double;
  static constexpr const char* name = "arithmetic";
  static constexpr int id = 0;
  static constexpr bool is_commutative_mul = true;
  SPG_HD static value_type add(value_type a, value_type b) { return a + b; }
  SPG_HD static value_type mul(value_type a, value_type b) { return a * b; }
  SPG_HD static value_type zero() { return 0.0; }
  SPG_HD static value_type one() { return 1.0; }
  SPG_HD static bool is_zero(value_type v) { return v == 0.0; }
  SPG_HD static value_type from_real(double x) { return x; }
#ifdef __CUDACC__
  __device__ __forceinline__ static value_type acc_shared(value_type* p, value_type v) { return atomicAdd(p, v); }
  __device__ __forceinline__ static value_type acc_global(value_type* p, value_type v) { return atomicAdd(p, v); }
#endif
  // fp64 add has a native L2 reduction (RED.ADD.F64) but no shared-memory
  // one (a CAS loop): hash accumulators may keep their values in global memory
  static constexpr bool red_global = true;
};

struct MinPlus {
  using value_type = double;
  static constexpr const char* name = "minplus";
  static constexpr int id = 1;
  static constexpr bool is_commutative_mul = true;
  // std::min(a, b) keeps a on ties (semiring.hpp:64).
  SPG_HD static value_type add(value_type a, value_type b) { return b < a ? b : a; }
  SPG_HD static value_type mul(value_type a, value_type b) { return a + b; }
  SPG_HD static value_type zero() { return __builtin_huge_val(); }
  SPG_HD static value_type one() { return 0.0; }
  SPG_HD static bool is_zero(value_type v) { return v == __builtin_huge_val(); }
  SPG_HD static value_type from_real(double x) { return x; }
};

struct Boolean {
  using value_type = uint8_t;  // ValueCodec<bool>: one byte, 0 or 1
  static constexpr const char* name = "boolean";
  static constexpr int id = 2;
  static constexpr bool is_commutative_mul = true;
  SPG_HD static value_type add(value_type a, value_type b) { return (a | b) ? 1 : 0; }
  SPG_HD static value_type mul(value_type a, value_type b) { return (a && b) ? 1 : 0; }
  SPG_HD static value_type zero() { return 0; }
  SPG_HD static value_type one() { return 1; }
  SPG_HD static bool is_zero(value_type v) { return v == 0; }
  SPG_HD static value_type from_real(double x) { return x != 0.0 ? 1 : 0; }
  // pattern-only: the product of two non-zeros is one() and the fold is
  // idempotent, so C is the product's sparsity pattern with every value one()
  static constexpr bool pattern_only = true;
#ifdef __CUDACC__
  // OR with false is the identity and every writer of `true` writes the same
  // byte, so a plain store is a correct (race-free) accumulate.
  __device__ __forceinline__ static value_type acc_shared(value_type* p, value_type v) {
    const value_type old = *reinterpret_cast<volatile value_type*>(p);
    if (v && !old) *reinterpret_cast<volatile value_type*>(p) = 1;
    return old;
  }
  __device__ __forceinline__ static value_type acc_global(value_type* p, value_type v) {
    const value_type old = *reinterpret_cast<volatile value_type*>(p);
    if (v && !old) *reinterpret_cast<volatile value_type*>(p) = 1;
    return old;
  }
#endif
};

struct MinSelect {
  using value_type = MinSelectA;
  static constexpr const char* name = "minselect";
  static constexpr int id = 3;
  static constexpr bool is_commutative_mul = false;
  static constexpr int64_t neutral_payload = -1;
  SPG_HD static value_type zero() { return {__builtin_huge_val(), INT64_MAX}; }
  SPG_HD static value_type one() { return {0.0, neutral_payload}; }
  SPG_HD static bool is_zero(const value_type& v) { return isinf(v.weight); }
  SPG_HD static value_type add(const value_type& a, const value_type& b) {
    const bool pick_b = b.weight < a.weight || (b.weight == a.weight && b.payload < a.payload);
    const value_type p = pick_b ? b : a;
    return isinf(p.weight) ? zero() : p;
  }
  SPG_HD static value_type mul(const value_type& a, const value_type& b) {
    const double w = a.weight + b.weight;
    if (isinf(w)) return zero();
    return {w, b.payload == neutral_payload ? a.payload : b.payload};
  }
  SPG_HD static value_type from_real(double x) { return {x, 0}; }
};

struct TropicalI32 {
  using value_type = int32_t;
  static constexpr const char* name = "tropical_i32";
  static constexpr int id = 4;
  static constexpr bool is_commutative_mul = true;
  SPG_HD static value_type zero() { return INT32_MAX; }
  SPG_HD static value_type one() { return 0; }
  SPG_HD static bool is_zero(value_type v) { return v == INT32_MAX; }
  SPG_HD static value_type add(value_type a, value_type b) { return b < a ? b : a; }
  SPG_HD static value_type mul(value_type a, value_type b) {
    if (a == INT32_MAX || b == INT32_MAX) return INT32_MAX;
    const int64_t s = (int64_t)a + (int64_t)b;
    if (s >= (int64_t)INT32_MAX) return INT32_MAX;
    if (s < (int64_t)INT32_MIN) return INT32_MIN;
    return (value_type)s;
  }
  // Fixed point with 1/1024 resolution, round half away from zero.
  SPG_HD static value_type from_real(double x) {
    const double y = x * 1024.0;
    if (!(y < 2147483646.5)) return INT32_MAX;
    if (y < -2147483648.0) return INT32_MIN;
    return (value_type)llround(y);
  }
  // fast path (see has_mul_small): |a|, |b| < 2^29 => a + b neither saturates nor hits zero()
  SPG_HD static bool small(value_type v) { return v > -(1 << 29) && v < (1 << 29); }
  SPG_HD static value_type mul_small(value_type a, value_type b) { return a + b; }
  // add(cur, v) != cur: a fold may skip the atomic when v cannot change the slot
  SPG_HD static bool improves(value_type v, value_type cur) { return v < cur; }
#ifdef __CUDACC__
  __device__ __forceinline__ static value_type acc_shared(value_type* p, value_type v) { return atomicMin(p, v); }
  __device__ __forceinline__ static value_type acc_global(value_type* p, value_type v) { return atomicMin(p, v); }
#endif
};

struct MaxTimes {
  using value_type = MaxTimesV;
  static constexpr const char* name = "maxtimes";
  static constexpr int id = 5;
  static constexpr bool is_commutative_mul = true;
  SPG_HD static value_type zero() { return {0.0, 0}; }
  SPG_HD static value_type one() { return {1.0, 0}; }
  SPG_HD static bool is_zero(const value_type& v) { return v.w == 0.0; }
  SPG_HD static value_type add(const value_type& a, const value_type& b) {
    return (b.w > a.w || (b.w == a.w && b.tag > a.tag)) ? b : a;
  }
  SPG_HD static value_type mul(const value_type& a, const value_type& b) {
    const double w = a.w * b.w;
    if (w == 0.0) return zero();
    return {w, a.tag ^ b.tag};
  }
  SPG_HD static value_type from_real(double x) { return {x, 0}; }
};

// ---------------------------------------------------------------------------
// Accumulate traits
// ---------------------------------------------------------------------------
template <class SR, class = void>
struct has_acc {
  static constexpr bool value = false;
};
template <class SR>
struct has_acc<SR, decltype((void)SR::acc_shared((typename SR::value_type*)nullptr,
                                                 typename SR::value_type{}),
                            void())> {
  static constexpr bool value = true;
};

// Optional `improves(v, cur)` (idempotent, monotone adds such as min): true
// iff add(cur, v) != cur, so a fold may read the slot and skip the atomic
// when the product cannot change it (hub columns receive many products).
template <class SR, class = void>
struct has_improves {
  static constexpr bool value = false;
};
template <class SR>
struct has_improves<SR, decltype((void)SR::improves(typename SR::value_type{}, typename SR::value_type{}), void())> {
  static constexpr bool value = true;
};

// Optional `red_global`: acc_global is a native fire-and-forget L2 reduction
// that beats the shared-memory accumulate (fp64 +).
template <class SR, class = void>
struct has_red_global {
  static constexpr bool value = false;
};
template <class SR>
struct has_red_global<SR, decltype((void)SR::red_global, void())> {
  static constexpr bool value = SR::red_global;
};

// Optional `pattern_only` (Boolean): mul(a, b) == one() for non-zero a, b and
// add(one(), one()) == one(): C's values are all one(), only the pattern is
// computed (two column-only passes, bitmap_rank.cuh: br_pattern_kernel).
template <class SR, class = void>
struct is_pattern_only {
  static constexpr bool value = false;
};
template <class SR>
struct is_pattern_only<SR, decltype((void)SR::pattern_only, void())> {
  static constexpr bool value = SR::pattern_only;
};

// Optional fast multiply: a semiring may declare `small(v)` and
// `mul_small(a, b)`, promising mul_small(a, b) == mul(a, b) and
// !is_zero(mul(a, b)) whenever small(a) && small(b).  The bitmap-rank fold
// uses it for a batch whose left scalars and right-operand values are all
// small (checked per call / per batch), dropping the saturation and
// zero-product tests from the per-product work.
template <class SR, class = void>
struct has_mul_small {
  static constexpr bool value = false;
};
template <class SR>
struct has_mul_small<SR, decltype((void)SR::small(typename SR::value_type{}),
                                  (void)SR::mul_small(typename SR::value_type{}, typename SR::value_type{}), void())> {
  static constexpr bool value = true;
};

template <class V>
SPG_HD bool bits_equal(const V& a, const V& b) {
  const uint8_t* x = reinterpret_cast<const uint8_t*>(&a);
  const uint8_t* y = reinterpret_cast<const uint8_t*>(&b);
  bool eq = true;
#pragma unroll
  for (int i = 0; i < (int)sizeof(V); ++i) eq &= x[i] == y[i];
  return eq;
}

#ifdef __CUDACC__
template <class T, class V>
__device__ __forceinline__ T as_bits(const V& v) {
  static_assert(sizeof(T) == sizeof(V), "width");
  T t;
  memcpy(&t, &v, sizeof(V));
  return t;
}

// *p = add(*p, v), atomically; returns the previous value.  `kShared`
// selects the semiring's shared- or global-memory fast path when it has one;
// otherwise a CAS loop.
template <class SR, bool kShared>
__device__ __forceinline__ typename SR::value_type atomic_accumulate(typename SR::value_type* p,
                                                                     const typename SR::value_type& v) {
  using V = typename SR::value_type;
  if constexpr (has_acc<SR>::value) {
    if constexpr (kShared) return SR::acc_shared(p, v);
    else return SR::acc_global(p, v);
  } else if constexpr (sizeof(V) == 8) {
    unsigned long long* a = reinterpret_cast<unsigned long long*>(p);
    unsigned long long old = *reinterpret_cast<volatile unsigned long long*>(a);
    for (;;) {
      const V cur = as_bits<V>(old);
      const V nxt = SR::add(cur, v);
      const unsigned long long nb = as_bits<unsigned long long>(nxt);
      if (nb == old) return cur;
      const unsigned long long seen = atomicCAS(a, old, nb);
      if (seen == old) return cur;
      old = seen;
    }
  } else if constexpr (sizeof(V) == 4) {
    unsigned int* a = reinterpret_cast<unsigned int*>(p);
    unsigned int old = *reinterpret_cast<volatile unsigned int*>(a);
    for (;;) {
      const V cur = as_bits<V>(old);
      const V nxt = SR::add(cur, v);
      const unsigned int nb = as_bits<unsigned int>(nxt);
      if (nb == old) return cur;
      const unsigned int seen = atomicCAS(a, old, nb);
      if (seen == old) return cur;
      old = seen;
    }
  } else if constexpr (sizeof(V) == 16) {
    static_assert(alignof(V) >= 16, "16-byte semiring values need 16-byte alignment");
    struct __align__(16) U128 {
      unsigned long long lo, hi;
    };
    U128* a = reinterpret_cast<U128*>(p);
    U128 old;
    old.lo = reinterpret_cast<volatile unsigned long long*>(a)[0];
    old.hi = reinterpret_cast<volatile unsigned long long*>(a)[1];
    for (;;) {
      const V cur = as_bits<V>(old);
      const V nxt = SR::add(cur, v);
      const U128 nb = as_bits<U128>(nxt);
      if (nb.lo == old.lo && nb.hi == old.hi) return cur;
      const U128 seen = atomicCAS(a, old, nb);
      if (seen.lo == old.lo && seen.hi == old.hi) return cur;
      old = seen;
    }
  } else {
    static_assert(sizeof(V) == 0, "unsupported value width");
  }
}

template <class SR>
__device__ __forceinline__ bool is_zero_bits(const typename SR::value_type& v) {
  return bits_equal(v, SR::zero());
}
#endif

}  // namespace spg
