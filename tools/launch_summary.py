"""Summarise an ncu launch list (--metrics gpu__time_duration.sum,dram__bytes_*; --csv)
per kernel over the last N timed steps: launches, total time share, DRAM bytes per launch.

usage: launch_summary.py launches.csv [steps] [> summary.json]"""
import csv, json, re, sys
from collections import OrderedDict, defaultdict

path = sys.argv[1]
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
rows = [r for r in csv.reader(l for l in open(path) if l.startswith('"'))]
hdr = rows[0]
ix = {h: i for i, h in enumerate(hdr)}
launch = OrderedDict()
for r in rows[1:]:
    k = int(r[ix["ID"]])
    name = r[ix["Kernel Name"]]
    short = re.sub(r"^(void )?lemgpu::", "", name).split("(")[0]
    d = launch.setdefault(k, {"name": short})
    d[r[ix["Metric Name"]]] = float(r[ix["Metric Value"]].replace(",", ""))
    d["unit_" + r[ix["Metric Name"]]] = r[ix["Metric Unit"]]
# the timed steps are the last `steps` k_finalize-terminated groups
ids = list(launch)
ends = [i for i in ids if launch[i]["name"] == "k_finalize"]
first = ends[-steps - 1] + 1 if len(ends) > steps else ids[0]
sel = [launch[i] for i in ids if i >= first and i <= ends[-1]]
agg = defaultdict(lambda: {"launches": 0, "ms": 0.0, "dram_bytes": 0.0})
for d in sel:
    t = d.get("gpu__time_duration.sum", 0.0)
    u = d.get("unit_gpu__time_duration.sum", "ns")
    ms = t * {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "nsecond": 1e-6, "ms": 1.0, "msecond": 1.0}.get(u, 1e-6)
    b = d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
    ub = d.get("unit_dram__bytes_read.sum", "byte")
    b *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(ub, 1)
    a = agg[d["name"]]
    a["launches"] += 1
    a["ms"] += ms
    a["dram_bytes"] += b
tot = sum(a["ms"] for a in agg.values())
out = {"source": path, "steps": steps, "total_ms_per_step": tot / steps, "kernels": {}}
for k, a in sorted(agg.items(), key=lambda kv: -kv[1]["ms"]):
    out["kernels"][k] = {"launches_per_step": a["launches"] / steps, "ms_per_step": a["ms"] / steps,
                         "share": a["ms"] / tot if tot else None,
                         "dram_bytes_per_launch": a["dram_bytes"] / max(a["launches"], 1)}
print(json.dumps(out, indent=1))
