"""Aggregate an ncu source page (cuda,sass csv) by file and line range.

usage: ncu_phases.py src.csv FILE:NAME:L0-L1 ...   (FILE is a basename suffix)"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
ranges = []
for spec in sys.argv[2:]:
    f, name, rg = spec.split(":")
    a, b = rg.split("-")
    ranges.append((f, name, int(a), int(b)))
cur = None; si = ie = ti = None
acc = {}
tot_s = tot_i = 0
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        cur = r[1].rsplit("/", 1)[-1]; continue
    if len(r) > 3 and r[0] == "Line No":
        si = r.index("Warp Stall Sampling (All Samples)"); ie = r.index("Instructions Executed")
        ti = r.index("Thread Instructions Executed"); continue
    if si is None or not r or not r[0]: continue
    try: ln = int(r[0]); s = int(r[si]); i = int(r[ie]); t = int(r[ti])
    except ValueError: continue
    tot_s += s; tot_i += i
    key = f"{cur}:other"
    for f, name, a, b in ranges:
        if cur.endswith(f) and a <= ln <= b: key = name; break
    v = acc.setdefault(key, [0, 0, 0]); v[0] += s; v[1] += i; v[2] += t
print(f"total samples {tot_s}  warp-inst {tot_i:.3e}")
for k, (s, i, t) in sorted(acc.items(), key=lambda kv: -kv[1][0]):
    print(f"{k:28s} samples {100*s/max(tot_s,1):5.1f}%  warp-inst {i:11d} ({100*i/max(tot_i,1):5.1f}%)  thr/warp-inst {t/max(i,1):5.1f}")
