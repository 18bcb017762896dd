// A user-defined semiring built OUTSIDE the library, the way a reference
// user adds a SemiringLike type (semiring.hpp:28-40): the (max, min)
// "bottleneck path" semiring over int32 — the widest-path counterpart of the
// tropical (min, +) semiring.  Compiled into its own shared library against
// the repo headers (Makefile target tests/custom_sr/libmaxmin_sr.so) and
// registered at run time with spg_register_semiring(spg_user_maxmin_i32_ops()).
#include <climits>
#include <cmath>

#include "instantiate.cuh"

struct MaxMinI32 {
  using value_type = int32_t;
  static constexpr const char* name = "maxmin_i32";
  static constexpr bool is_commutative_mul = true;
  SPG_HD static value_type zero() { return INT32_MIN; }    // identity of max, absorbing for min
  SPG_HD static value_type one() { return INT32_MAX; }     // identity of min
  SPG_HD static bool is_zero(value_type v) { return v == INT32_MIN; }
  SPG_HD static value_type add(value_type a, value_type b) { return a > b ? a : b; }
  SPG_HD static value_type mul(value_type a, value_type b) { return a < b ? a : b; }
  SPG_HD static value_type from_real(double x) {
    const double y = std::round(x);
    return y >= 2147483647.0 ? INT32_MAX : y <= -2147483648.0 ? INT32_MIN : (value_type)y;
  }
  __device__ __forceinline__ static value_type acc_shared(value_type* p, value_type v) { return atomicMax(p, v); }
  __device__ __forceinline__ static value_type acc_global(value_type* p, value_type v) { return atomicMax(p, v); }
};

SPG_INSTANTIATE(MaxMinI32, spg_user_maxmin_i32_ops)
