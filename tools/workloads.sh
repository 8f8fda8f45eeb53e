#!/bin/bash
# Bench lines of every workload (device-resident value only), tagged $1 (default "wl").
tag=${1:-wl}
for wl in dem10000 dem1000 dem4000n2 dem1000fill dem4000fill ens64; do
  timeout -s KILL 400 python bench.py --workload $wl --no-cpu-baseline --e2e-steps 0 --steps 10 > gpurun_out/${tag}_$wl.json 2> gpurun_out/${tag}_$wl.err
  python -c "import json; d=json.load(open('gpurun_out/${tag}_$wl.json')); print('$wl', round(d['ms_per_step'],4), '%.3e' % d['value'], {k: round(v,4) for k,v in d['roofline']['kernel_ms'].items()}, d['config'].get('nlevels_last_step'))" || tail -3 gpurun_out/${tag}_$wl.err
done
