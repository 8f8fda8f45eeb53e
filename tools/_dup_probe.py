import sys, ctypes as C
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import numpy as np
import paper_1803_02977_b200 as lem
from paper_1803_02977_b200 import _abi
from _oracle import Oracle
w, h = int(sys.argv[1]), int(sys.argv[2])
o = Oracle.get()
e = o.terrain(w, h, 42)
ctx = lem.DeviceContext(w, h, lem.SimParams(), 8)
ctx.upload(e)
L = _abi.lib()
for s in range(3):
    e_before = e.copy()
    r = o.step(e, want_donor=False)
    try:
        ctx.step(1)
        err = None
    except Exception as ex:
        err = str(ex)
    lv = np.zeros(4, np.uint32)
    L.lemgpu_debug_copy(ctx._h, 1, lv.ctypes.data, 16)
    n = int(lv[1])
    order = np.zeros(w * h, np.uint32)
    L.lemgpu_debug_copy(ctx._h, 0, order.ctypes.data, order.nbytes)
    roots = order[:n]
    u, c = np.unique(roots, return_counts=True)
    isroot = r["rec"][roots] == 0xFFFFFFFF
    truth = np.nonzero(r["rec"] == 0xFFFFFFFF)[0]
    print(f"step {s} err={err} nesc={n} dups={int((c>1).sum())} nonroots={int((~isroot).sum())} true_roots={truth.size}", flush=True)
    if (c > 1).any():
        d = u[c > 1][:5]; print("dup cells", d, "x,y", d % w, d // w)
    if (~isroot).any():
        d = roots[~isroot][:5]; print("non-root cells", d, d % w, d // w)
    if err: break
