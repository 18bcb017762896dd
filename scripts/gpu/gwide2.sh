export PYTHONFAULTHANDLER=1 CUDA_LAUNCH_BLOCKING=1
timeout 600 python -X faulthandler -m pytest "tests/test_gpu_local.py::test_wide_rows_sort_fallback_at_4m_columns" -x -s -v > gpurun_out/gwide2.log 2>&1; echo rc=$?
tail -40 gpurun_out/gwide2.log
