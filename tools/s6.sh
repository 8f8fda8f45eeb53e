timeout -s KILL 1800 python -m pytest tests -m gpu -q -rs -p no:cacheprovider > gpurun_out/gputest_r02d.txt 2>&1; tail -3 gpurun_out/gputest_r02d.txt
for wl in dem10000mfd dem1000mfd; do
timeout -s KILL 600 python bench.py --workload $wl > gpurun_out/bench_r02d_$wl.json 2> gpurun_out/bench_r02d_$wl.err
python -c "import json; d=json.load(open('gpurun_out/bench_r02d_$wl.json')); print('$wl', d['ms_per_step'], '%.3e'%d['value'], d['cpu_baseline']['value'], d['roofline']['frac'])"
done
