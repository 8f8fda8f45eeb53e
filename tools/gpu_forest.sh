# targeted GPU check of the escape paths + fill workloads (round-2 forest work)
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "schedules or deep_plan or banded or random or filled" > gpurun_out/forest_tests.txt 2>&1
timeout -s KILL 900 python -m pytest tests/test_gpu_parity_large.py -q -x -p no:cacheprovider -k "filled" >> gpurun_out/forest_tests.txt 2>&1
for wl in dem1000fill dem4000fill dem10000; do
  timeout -s KILL 400 python bench.py --workload $wl --no-cpu-baseline --e2e-steps 0 --steps 10 > gpurun_out/forest_$wl.json 2> gpurun_out/forest_$wl.err
  python -c "import json; d=json.load(open('gpurun_out/forest_$wl.json')); print('$wl', round(d['ms_per_step'],4), '%.3e' % d['value'], {k: round(v,4) for k,v in d['roofline']['kernel_ms'].items()})" >> gpurun_out/forest_summary.txt 2>&1 || tail -3 gpurun_out/forest_$wl.err >> gpurun_out/forest_summary.txt
done
