"""Instructions executed per source-line range (ncu --page source --csv --print-source cuda,sass):
usage: ncu_phase_insts.py src.csv file.cuh name:a-b [name:a-b ...]"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
target = sys.argv[2]
ranges = [(n, int(r.split('-')[0]), int(r.split('-')[1])) for n, r in (x.split(':') for x in sys.argv[3:])]
per, cur, ie = {}, '?', None
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        cur = r[1].split('/')[-1]; continue
    if len(r) > 3 and r[0] == "Line No":
        ie = r.index("Instructions Executed"); continue
    if ie is None or len(r) <= ie or not r[0].isdigit():
        continue
    try:
        per[(cur, int(r[0]))] = per.get((cur, int(r[0])), 0) + int(r[ie])
    except ValueError:
        pass
tot = sum(per.values())
print("total warp instructions", tot)
for n, a, b in ranges:
    s = sum(v for (f, l), v in per.items() if f == target and a <= l <= b)
    print(f"{n:12s} {s:12d} {100 * s / tot:5.1f}%")
oth = {}
for (f, l), v in per.items():
    if f != target:
        oth[f] = oth.get(f, 0) + v
print("other files:", {k: f"{100 * v / tot:.1f}%" for k, v in oth.items()})
