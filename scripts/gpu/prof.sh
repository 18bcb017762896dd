SPG_LIB_PATH=variants/prof/libspgemm_b200.so timeout 300 python tools/local_probe.py rmat --scale 18 --sr tropical_i32 --permute --reps 2 2>&1 | grep -E "br-prof|ms_total" | cut -c1-400
