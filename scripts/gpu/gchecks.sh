# the GPU suite against the bounds-checked build (device traps on a violated invariant)
export SPG_LIB_PATH=variants/checks/libspgemm_b200.so
timeout 2400 python -m pytest tests -q -m gpu -k "not fullsize" -p no:cacheprovider 2>&1 | tail -4 | tee gpurun_out/r02_checked_build_gpu_tests.log
