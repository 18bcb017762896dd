nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw,utilization.gpu --format=csv
for r in 1 2 3; do
python bench.py --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/rep$r.json 2> gpurun_out/rep$r.err
python -c "import json;d=json.load(open('gpurun_out/rep$r.json'));print('rep$r', round(d['ms_per_step'],2), d['clocks'])"
done
