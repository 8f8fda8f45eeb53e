timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "mfd" -p no:cacheprovider 2>&1 | tail -2
PROBE_STEPS=3 timeout -s KILL 300 python tools/mfd_probe.py 1000 10000
for i in 1 2; do for so in tools/var_base.so tools/var_new.so; do
  LEMGPU_LIB=$so timeout -s KILL 100 python bench.py --no-cpu-baseline --e2e-steps 0 --steps 30 2>/dev/null \
    | python -c "import json,sys; d=json.load(sys.stdin); k=d['roofline']['kernel_ms']; print('$so', round(d['ms_per_step'],4))"
done; done
