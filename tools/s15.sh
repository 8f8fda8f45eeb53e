# A/B tools/var_base.so vs tools/var_new.so on the large workloads, plus the GPU parity tests on the new build
LEMGPU_LIB=tools/var_new.so timeout -s KILL 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -1
for wl in dem10000 dem4000n2 ens64 dem1000fill dem1000mfd; do for so in tools/var_base.so tools/var_new.so tools/var_base.so tools/var_new.so; do
  LEMGPU_LIB=$so timeout -s KILL 200 python bench.py --workload $wl --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 0 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('$wl $so', round(d['ms_per_step'],4))"
done; done
