LEMGPU_EAGER=1 timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launch_mfd10000.csv python bench.py --workload dem10000mfd --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
python - <<'PY'
import csv
rows=[r for r in csv.reader(l for l in open('gpurun_out/launch_mfd10000.csv') if l.startswith('"'))]
h=rows[0]; ix={k:i for i,k in enumerate(h)}
out=[(int(r[ix['ID']]), r[ix['Kernel Name']].split('(')[0][-40:], r[ix['Metric Value']]) for r in rows[1:]]
for o in out[-20:]: print(o)
PY
LEMGPU_EAGER=1 timeout -s KILL 300 ncu --set full --import-source on --clock-control none -k regex:k_mfd_tiles -s 9 -c 1 -o gpurun_out/ncu_mfd10000 python bench.py --workload dem10000mfd --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_mfd10000.log 2>&1
tail -2 gpurun_out/ncu_mfd10000.log
