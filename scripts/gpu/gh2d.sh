timeout 900 python -m pytest tests/test_gpu_local.py -x -q -m gpu -k "large_upload or download or config4 or wide" > gpurun_out/gh2d.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/gh2d.log
bash scripts/gpu/gcfg.sh
