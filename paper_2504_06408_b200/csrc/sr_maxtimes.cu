// Device pipeline instantiated for the maxtimes semiring (see instantiate.cuh).
#include "instantiate.cuh"
SPG_INSTANTIATE(spg::MaxTimes, spg_ops_maxtimes)
