# A/B of two builds on dem4000n2 (configs[2])
for i in 1 2 3; do for so in tools/var_base.so tools/var_new.so; do
  LEMGPU_LIB=$so timeout -s KILL 200 python bench.py --workload dem4000n2 --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 0 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('dem4000n2 $so', round(d['ms_per_step'],4))"
done; done
LEMGPU_LIB=tools/var_new.so timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_large.py -m gpu -q -x -k "n2 or general or schedules or nexp" -p no:cacheprovider 2>&1 | tail -1
