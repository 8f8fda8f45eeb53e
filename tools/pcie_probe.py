"""PCIe copy probe: 800 MB pinned H2D / D2H alone, concurrent, and banded
(29 bands, copies down trailing the copies up by one band), in place or on
separate host buffers.  Prints ms per variant (best of 3)."""
import torch

N = 10000 * 10000
nb = 29
dev = torch.device("cuda:0")
hin = torch.empty(N, dtype=torch.float64).pin_memory()
hout = torch.empty(N, dtype=torch.float64).pin_memory()
d0 = torch.empty(N, dtype=torch.float64, device=dev)
d1 = torch.empty(N, dtype=torch.float64, device=dev)
su, sd = torch.cuda.Stream(), torch.cuda.Stream()


def run(f):
    best = 1e9
    for _ in range(3):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        su.wait_event(e0)
        sd.wait_event(e0)
        f()
        torch.cuda.current_stream().wait_stream(su)
        torch.cuda.current_stream().wait_stream(sd)
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


def up():
    with torch.cuda.stream(su):
        d0.copy_(hin, non_blocking=True)


def down():
    with torch.cuda.stream(sd):
        hout.copy_(d1, non_blocking=True)


def both():
    up()
    down()


def banded(dst_host):
    def f():
        ev = []
        c = (N + nb - 1) // nb
        for b in range(nb):
            with torch.cuda.stream(su):
                d0[b * c:(b + 1) * c].copy_(hin[b * c:(b + 1) * c], non_blocking=True)
                e = torch.cuda.Event()
                e.record(su)
                ev.append(e)
        for b in range(nb):
            sd.wait_event(ev[b])
            with torch.cuda.stream(sd):
                dst_host[b * c:(b + 1) * c].copy_(d1[b * c:(b + 1) * c], non_blocking=True)
    return f


print("h2d alone      %.2f ms" % run(up))
print("d2h alone      %.2f ms" % run(down))
print("concurrent     %.2f ms" % run(both))
print("banded sep     %.2f ms" % run(banded(hout)))
print("banded inplace %.2f ms" % run(banded(hin)))
