timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "mfd" -p no:cacheprovider > gpurun_out/t_mfd.txt 2>&1
tail -3 gpurun_out/t_mfd.txt
PROBE_STEPS=3 timeout -s KILL 300 python tools/mfd_probe.py 1000 10000
