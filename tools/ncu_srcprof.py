"""Summarise an ncu source page (cuda,sass csv) by CUDA source line."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
hdr = None; items = []; tot = 0
stall_cols = None
for r in rows:
    if len(r) > 3 and r[0] == "Line No":
        hdr = r; si = r.index("Warp Stall Sampling (All Samples)")
        ie = r.index("Instructions Executed")
        stall_cols = [i for i, h in enumerate(r) if h.startswith("stall_") and "Not Issued" not in h]
        continue
    if hdr is None or len(r) <= si: continue
    if r[0] and r[0] != "":
        try: v = int(r[si])
        except: continue
        tot += v
        st = sorted(((int(r[i]) if r[i].isdigit() else 0, hdr[i]) for i in stall_cols), reverse=True)[:3]
        items.append((v, r[0], r[1].strip()[:90], int(r[ie]) if r[ie].isdigit() else 0, st))
items.sort(reverse=True)
print("total samples", tot)
for v, l, s, ie, st in items[:top]:
    print(f"{v:7d} {100*v/max(tot,1):5.1f}% L{l:>4} inst={ie:>11} {s}  | " + ", ".join(f"{n[6:]}:{c}" for c, n in st if c))
