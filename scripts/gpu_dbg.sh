set -x
export SPG_COMM_TIMEOUT_S=60 SPG_DEBUG_HANG=100
for S in 14 16 18; do
timeout 150 python bench.py --summa --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline --scale $S > gpurun_out/d$S.json 2> gpurun_out/d$S.err; echo S=$S rc=$?
tail -c 600 gpurun_out/d$S.json; tail -25 gpurun_out/d$S.err
done
