for v in base $VARIANTS; do
  if [ "$v" = base ]; then unset SPG_LIB_PATH; else export SPG_LIB_PATH=variants/$v/libspgemm_b200.so; fi
  for ws in 1 0; do
  echo -n "$v ws=$ws "; SPG_BR_WS=$ws timeout 300 python tools/local_probe.py rmat --scale 18 --sr tropical_i32 --permute --reps 4 2>/dev/null | grep -o '"ms_total": [0-9.]*' | tail -1
  done
done
