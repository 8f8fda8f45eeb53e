timeout -s KILL 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "deep_plan or schedules_agree or filled or forest" -p no:cacheprovider 2>&1 | tail -3
timeout -s KILL 900 python -m pytest tests/test_gpu_parity_large.py -m gpu -q -x -k "filled" -p no:cacheprovider 2>&1 | tail -3
for n in 1000 4000; do timeout -s KILL 300 python tools/forest_probe.py $n 3 | head -4; timeout -s KILL 300 python tools/forest_probe.py $n 3 forest_seg=-1 | head -1; done
