export PYTHONPATH=$PWD:$PWD/tests
timeout 300 python scripts/gpu/wide_repro.py > gpurun_out/wide3.log 2>&1; echo rc=$?; cat gpurun_out/wide3.log | tail -5
timeout 600 cuda-gdb -batch -ex "set pagination off" -ex "break exit" -ex "break _exit" -ex "break abort" -ex run -ex bt --args python scripts/gpu/wide_repro.py > gpurun_out/wide3_gdb.log 2>&1; echo gdb rc=$?
grep -v "^\[New Thread\|^\[Thread" gpurun_out/wide3_gdb.log | tail -40
