// Device pipeline instantiated for the minplus semiring (see instantiate.cuh).
#include "instantiate.cuh"
SPG_INSTANTIATE(spg::MinPlus, spg_ops_minplus)
