timeout 1200 python -m pytest tests/test_gpu_distribute.py tests/test_cpp_facade.py tests/test_custom_semiring.py tests/test_gpu_summa.py -x -q -m gpu > gpurun_out/gdist.log 2>&1
echo rc=$?; tail -15 gpurun_out/gdist.log
