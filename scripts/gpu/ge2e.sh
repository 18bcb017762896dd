# e2e D2H split: share of index chunks widened on the GPU
for f in 0 0.2 0.35 0.5 1.0; do
  SPG_D2H_GPU_WIDEN=$f timeout 600 python bench.py --steps 3 --warmup 3 --e2e-steps 4 --no-cpu-baseline --no-unpermuted > gpurun_out/e2e_$f.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/e2e_$f.json')); print('$f', d['e2e']['seconds'], d['e2e']['value'], d['ms_per_step'])"
done
