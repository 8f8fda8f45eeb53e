# bench lines (with the CPU baseline) of the given workloads, tagged $1
tag=$1; shift
for wl in "$@"; do
  timeout -s KILL 600 python bench.py --workload $wl --steps 10 --e2e-steps 2 > gpurun_out/${tag}_$wl.json 2> gpurun_out/${tag}_$wl.err
  python -c "import json; d=json.load(open('gpurun_out/${tag}_$wl.json')); c=d.get('cpu_baseline') or {}; print('$wl', round(d['ms_per_step'],4), '%.3e' % d['value'], 'e2e %.3e' % (d['e2e'] or {}).get('value',0), 'cpu %.3e' % (c.get('value') or 0), {k: round(v,4) for k,v in d['roofline']['kernel_ms'].items()}, 'frac', round(d['roofline']['frac'] or 0, 4))" || tail -3 gpurun_out/${tag}_$wl.err
done
