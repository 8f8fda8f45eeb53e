timeout -s KILL 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_large.py -m gpu -q -x -k "forest or filled or deep or schedules" -p no:cacheprovider 2>&1 | tail -1
for n in 1000 4000; do timeout -s KILL 300 python tools/forest_probe.py $n 3 2>/dev/null | sed -n 3p; done
