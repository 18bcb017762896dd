// Device pipeline instantiated for the arithmetic semiring (see instantiate.cuh).
#include "instantiate.cuh"
SPG_INSTANTIATE(spg::Arithmetic, spg_ops_arithmetic)
