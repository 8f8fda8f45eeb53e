"""Per-step cost of the kernel-timing events bench.py records around each graph launch."""
import sys, time, torch
sys.path.insert(0, '.')
from paper_1803_02977_b200 import lem
for N in (1000, 10000):
    ctx = lem.DeviceContext(N, N, lem.SimParams(), 8)
    ctx.generate_terrain([42])
    ext = torch.cuda.ExternalStream(ctx.stream_ptr(), device=torch.device('cuda', 0))
    for t in (False, True, False, True):
        for _ in range(5): ctx.step_async(1)
        ctx.sync()
        ctx.kernel_timing(t)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        K = 200 if N == 1000 else 20
        s.record(ext)
        for _ in range(K): ctx.step_async(1)
        e.record(ext)
        ctx.sync(); torch.cuda.synchronize()
        print(N, 'timing' if t else 'plain ', round(s.elapsed_time(e) / K, 5))
        ctx.kernel_timing(False)
    ctx.close()
