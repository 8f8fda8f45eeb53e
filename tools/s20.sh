# k_esc_small capacity (build) x CTAs (option esc_small_grid)
for wl in dem10000 ens64 dem4000n2; do for i in 1 2; do
for v in "base 148" "c2048 444" "c1536 592" "c1024 888"; do set -- $v
  LEMGPU_LIB=tools/var_$1.so timeout -s KILL 200 python bench.py --workload $wl --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 0 --options "{\"esc_small_grid\": $2}" 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); k=d['roofline']['kernel_ms']; print('$wl $1 $2', round(d['ms_per_step'],4), round(k.get('escape:levels',0),4), d['details'].get('escaped_trees_last_step'))"
done; done; done
