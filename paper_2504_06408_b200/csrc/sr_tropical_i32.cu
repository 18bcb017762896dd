// Device pipeline instantiated for the tropical_i32 semiring (see instantiate.cuh).
#include "instantiate.cuh"
SPG_INSTANTIATE(spg::TropicalI32, spg_ops_tropical_i32)
