// Device pipeline instantiated for the boolean semiring (see instantiate.cuh).
#include "instantiate.cuh"
SPG_INSTANTIATE(spg::Boolean, spg_ops_boolean)
