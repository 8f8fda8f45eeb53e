# bench.py without per-step timing events in the timed region: every workload's line
for wl in dem10000 dem1000 dem4000n2 ens64 dem1000fill dem1000mfd; do
  timeout -s KILL 400 python bench.py --workload $wl --no-cpu-baseline > gpurun_out/b25_$wl.json 2> gpurun_out/b25_$wl.err
  python -c "import json; d=json.load(open('gpurun_out/b25_$wl.json')); r=d['roofline']; print('$wl', round(d['ms_per_step'],4), '%.3e'%d['value'], r['kernel'][:24], round(r['frac'],3), {k: round(v,4) for k,v in r['kernel_ms'].items()})" || tail -5 gpurun_out/b25_$wl.err
done
