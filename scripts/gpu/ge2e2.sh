for rep in 1 2; do
for f in 0.1 0.2 0.25 1.0; do
  SPG_D2H_GPU_WIDEN=$f timeout 600 python bench.py --steps 3 --warmup 3 --e2e-steps 6 --no-cpu-baseline --no-unpermuted > gpurun_out/e2e_$f.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/e2e_$f.json')); print('$f', round(d['e2e']['seconds'],4))"
done; done
