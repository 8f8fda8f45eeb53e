for so in tools/var_m*.so; do
  echo "== $so"
  LEMGPU_LIB=$so timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "mfd" -p no:cacheprovider 2>&1 | tail -1
  LEMGPU_LIB=$so PROBE_STEPS=3 timeout -s KILL 300 python tools/mfd_probe.py 1000 10000 | tail -2
done
