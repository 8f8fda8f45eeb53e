timeout -s KILL 1800 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -1
timeout -s KILL 200 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout -s KILL 400 python bench.py > gpurun_out/bench_r02k.json 2> gpurun_out/bench_r02k.err
timeout -s KILL 400 python bench.py --workload dem1000 > gpurun_out/bench_r02k_dem1000.json 2> /dev/null
python -c "import json; d=json.load(open('gpurun_out/bench_r02k.json')); print(d['ms_per_step'], d['value'], d['e2e']['value'], d['roofline']['frac'], d['clocks'])"
python -c "import json; d=json.load(open('gpurun_out/bench_r02k_dem1000.json')); print(d['ms_per_step'], d['value'], d['roofline']['frac'])"
