timeout -s KILL 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -2
for wl in dem10000 dem1000 ens64 dem4000n2; do for i in 1 2; do for so in tools/var_base.so tools/var_new.so; do
  LEMGPU_LIB=$so timeout -s KILL 200 python bench.py --workload $wl --no-cpu-baseline --e2e-steps 0 --steps 30 2>/dev/null \
    | python -c "import json,sys; d=json.load(sys.stdin); print('$wl $so', round(d['ms_per_step'],4))"
done; done; done
