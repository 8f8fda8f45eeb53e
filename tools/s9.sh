LEMGPU_LIB=tools/var_new.so timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "host or dropin or cpp" -p no:cacheprovider 2>&1 | tail -1
for i in 1 2 3; do for so in tools/var_base.so tools/var_new.so; do
  LEMGPU_LIB=$so timeout -s KILL 200 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 8 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('$so', round(d['e2e']['ms_per_step'],3), round(d['e2e']['frac_of_copy_floor'],3))"
done; done
for so in tools/var_base.so tools/var_new.so; do
  LEMGPU_LIB=$so timeout -s KILL 200 python bench.py --workload ens64 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 4 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('ens64 $so', round(d['e2e']['ms_per_step'],3), round(d['e2e']['frac_of_copy_floor'],3))"
done
