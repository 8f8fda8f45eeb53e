timeout -s KILL 300 python tools/mfd_probe.py 1000 4000 10000
LEMGPU_EAGER=1 timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launch_mfd1000.csv python bench.py --workload dem1000mfd --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
python - <<'PY'
import csv
rows=[r for r in csv.reader(l for l in open('gpurun_out/launch_mfd1000.csv') if l.startswith('"'))]
h=rows[0]; ix={k:i for i,k in enumerate(h)}
out=[(int(r[ix['ID']]), r[ix['Kernel Name']].split('(')[0][-40:], r[ix['Metric Value']]) for r in rows[1:]]
for o in out[-60:]: print(o)
PY
