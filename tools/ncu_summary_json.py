"""profiles/ncu_summary_<tag>_<workload>.json from an ncu launch list (--metrics
gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv, eager
launches) of `bench.py --workload W --steps 2`: per kernel (short name) the
launches, cold ms and DRAM bytes per step over the last 2 timed steps; bench.py
reads `dram_bytes_per_step` of the dominant kernel(s) as its roofline `traffic`.
usage: ncu_summary_json.py launches.csv workload tag > profiles/ncu_summary_<tag>_<workload>.json"""
import csv, json, re, sys
from collections import OrderedDict, defaultdict

path, workload, tag = sys.argv[1], sys.argv[2], sys.argv[3]
steps = 2
rows = [r for r in csv.reader(l for l in open(path) if l.startswith('"'))]
ix = {h: i for i, h in enumerate(rows[0])}
launch = OrderedDict()
for r in rows[1:]:
    d = launch.setdefault(int(r[ix["ID"]]), {"name": re.sub(r"<.*", "", re.sub(r"^(void )?(lemgpu::)?", "", r[ix["Kernel Name"]]).split("(")[0]).strip()})
    scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0,
             "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(r[ix["Metric Unit"]], 1.0)
    d[r[ix["Metric Name"]]] = float(r[ix["Metric Value"]].replace(",", "")) * scale
ids = list(launch)
ends = [i for i in ids if launch[i]["name"] == "k_finalize"]
first = ends[-steps - 1] + 1 if len(ends) > steps else ids[0]
agg = defaultdict(lambda: {"launches": 0, "ms": 0.0, "dram": 0.0})
for i in ids:
    if first <= i <= ends[-1]:
        d = launch[i]
        a = agg[d["name"]]
        a["launches"] += 1
        a["ms"] += d.get("gpu__time_duration.sum", 0.0)
        a["dram"] += d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
tot = sum(a["ms"] for a in agg.values())
out = {"round": 2, "tag": tag, "workload": workload,
       "command": f"ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none "
                  f"(LEMGPU_EAGER=1) python bench.py --workload {workload} --steps 2; last {steps} timed steps "
                  "(cold, serialised launches: shares, not absolute times)",
       "source": path, "total_ms_cold_per_step": tot / steps, "kernels": {}}
for k, a in sorted(agg.items(), key=lambda kv: -kv[1]["ms"]):
    out["kernels"][k] = {"launches_per_step": a["launches"] / steps, "ms_cold": a["ms"] / steps,
                         "share": a["ms"] / tot if tot else None,
                         "dram_bytes_per_step": a["dram"] / steps,
                         "dram_bytes_per_launch": a["dram"] / max(a["launches"], 1)}
print(json.dumps(out, indent=1))
