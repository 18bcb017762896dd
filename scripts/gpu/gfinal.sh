# full GPU suite + default bench line + smoke
timeout 2400 python -m pytest tests -x -q -m gpu > gpurun_out/gfinal_tests.log 2>&1; echo tests rc=$?; tail -4 gpurun_out/gfinal_tests.log
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.log; echo bench rc=$?
python -c "
import json; d=json.load(open('gpurun_out/bench_default.json')); print({k: d.get(k) for k in ('value','ms_per_step','parity','gpu_launches')}, d['roofline']['frac'], d['e2e'], d['clocks'])"
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
