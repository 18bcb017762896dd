for v in base $VARIANTS; do
  if [ "$v" = base ]; then unset SPG_LIB_PATH; else export SPG_LIB_PATH=variants/$v/libspgemm_b200.so; fi
  echo -n "$v "; timeout 300 python tools/local_probe.py rmat --scale 18 --sr tropical_i32 --permute --reps 4 2>/dev/null | grep -o '"ms_total": [0-9.]*' | tail -1
done
unset SPG_LIB_PATH
for m in 1024 4096; do echo -n "minf=$m "; SPG_BR_MINF=$m timeout 300 python tools/local_probe.py rmat --scale 18 --sr tropical_i32 --permute --reps 4 2>/dev/null | grep -o '"ms_total": [0-9.]*' | tail -1; done
