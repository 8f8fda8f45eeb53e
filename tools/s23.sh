LEMGPU_LIB=tools/var_new.so timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -1
for wl in dem1000 dem10000 dem4000n2; do for i in 1 2 3; do for so in tools/var_base.so tools/var_new.so; do
  LEMGPU_LIB=$so timeout -s KILL 200 python bench.py --workload $wl --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 0 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); k=d['roofline']['kernel_ms']; print('$wl $so', round(d['ms_per_step'],4), round(k.get('escape:levels',0),4))"
done; done; done
