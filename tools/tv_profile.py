"""Profile target for the TV prox kernels: one bsgd_tv_prox call (20 FGP iterations) on a
z-slab volume (default 512^3, 8 slabs: cfg4's layout).  The geometry is a tiny detector so
that context creation is cheap; the prox never touches it.

    ncu --metrics gpu__time_duration.sum python tools/tv_profile.py [nx ny nz bz]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_1903_11874_b200 as bs  # noqa: E402

nx, ny, nz, bz = (int(v) for v in (sys.argv[1:5] if len(sys.argv) >= 5 else (512, 512, 512, 8)))
calls = int(os.environ.get("TV_CALLS", "2"))
g = synth.Geometry(2, synth.circular("cone", 4, 360.0, 6.0 * nx, 4.0 * nx, 8, 8, 1.0, 1.0), 8, 8, (nx, ny, nz))
ctx = bs.Context.from_geometry(g, (1, 1, bz), 1)
x = torch.rand(nx * ny * nz, device="cuda")
for _ in range(calls):
    ctx.tv_prox(x, 0.05, 20)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
ctx.tv_prox(x, 0.05, 20)
e1.record()
torch.cuda.synchronize()
print(f"tv_prox {nx}x{ny}x{nz}: {e0.elapsed_time(e1):.2f} ms per call")
ctx.close()
