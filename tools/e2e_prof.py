"""lemgpu_step_host timing breakdown (host_profile) on 10000^2, pinned raster."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1803_02977_b200 import lem  # noqa: E402
N = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
bands = int(sys.argv[2]) if len(sys.argv) > 2 else 0
ctx = lem.DeviceContext(N, N, lem.SimParams(), 8, options={"host_profile": 1, "host_bands": bands})
ctx.generate_terrain([42])
h = torch.empty(N * N, dtype=torch.float64).pin_memory().numpy()
lem._abi.lib().lemgpu_download_elev(ctx.handle, h.ctypes.data)
for _ in range(6):
    ctx.step_host(h)
