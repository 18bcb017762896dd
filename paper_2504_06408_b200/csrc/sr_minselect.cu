// Device pipeline instantiated for the minselect semiring (see instantiate.cuh).
#include "instantiate.cuh"
SPG_INSTANTIATE(spg::MinSelect, spg_ops_minselect)
