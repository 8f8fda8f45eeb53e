python tools/forest_probe.py 1000 3; python tools/forest_probe.py 4000 2
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "schedules or deep_plan or banded or random or filled" 2>&1 | tail -3
timeout -s KILL 900 python -m pytest tests/test_gpu_parity_large.py -q -x -p no:cacheprovider -k "filled" 2>&1 | tail -3
