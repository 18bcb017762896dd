set -x
nvidia-smi -L
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu2.log 2>&1; echo pytest_rc=$?
tail -30 gpurun_out/pytest_gpu2.log
