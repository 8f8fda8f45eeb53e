LEMGPU_EAGER=1 timeout -s KILL 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -c 200 --csv --log-file gpurun_out/launch_mfdg.csv python bench.py --workload dem10000mfd --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
python - <<'PY'
import csv
rows=[r for r in csv.reader(l for l in open('gpurun_out/launch_mfdg.csv') if l.startswith('"'))]
h=rows[0]; ix={k:i for i,k in enumerate(h)}
d={}
for r in rows[1:]:
    d.setdefault(int(r[ix['ID']]),{})['name']=r[ix['Kernel Name']].split('(')[0][-30:]
    d[int(r[ix['ID']])][r[ix['Metric Name']]]=r[ix['Metric Value']]
ids=sorted(d); 
for i in ids[-22:]: print(i, d[i]['name'], d[i].get('gpu__time_duration.sum'), d[i].get('dram__bytes_read.sum'))
PY
