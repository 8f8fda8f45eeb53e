timeout -s KILL 400 python bench.py > gpurun_out/bench_r02l.json 2> gpurun_out/bench_r02l.err
timeout -s KILL 400 python bench.py --workload dem1000 > gpurun_out/bench_r02l_dem1000.json 2> gpurun_out/bench_r02l_dem1000.err
for f in bench_r02l bench_r02l_dem1000; do python -c "
import json; d=json.load(open('gpurun_out/$f.json')); print('$f', sorted(d.keys())); print(d['ms_per_step'], '%.4e'%d['value'], '%.4e'%d['e2e']['value'], d['roofline']['frac'], d['cpu_baseline']['value'], d['gpu_launches'], d['clocks'])" || tail -5 gpurun_out/$f.err; done
