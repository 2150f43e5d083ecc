"""Per-ray FP comparison (library vs oracle) on one preset/block; prints the worst rays."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth
import paper_1903_11874_b200 as bs
from oracle.projector import Projector, BlockGrid
name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
j = int(sys.argv[2]) if len(sys.argv) > 2 else 0
p = synth.PRESETS[name]; g = p.geometry()
views = np.unique(np.linspace(0, g.n_views - 1, 48).round().astype(int))
ctx = bs.Context.from_geometry(g, p.blocks, p.M)
P = Projector(g, BlockGrid(g.dims, p.blocks))
x = np.random.default_rng(0).random(P.grid.bsize, dtype=np.float32)
proj = torch.full((g.n_rays,), -7.0, device="cuda")
ctx.forward(views, j, torch.from_numpy(x).cuda(), proj)
got = proj.cpu().numpy().astype(np.float64)
ref = P.fp(views, j, x.astype(np.float64))
rows = P.rows_of(views)
d = np.abs(got[rows] - ref[rows])
tol = 1e-5 * ref[rows] + 1e-7
bad = np.argsort(-d / tol)[:12]
print("projector", os.environ.get("BSGD_PROJECTOR", "2"), "max |d|/tol", (d / tol).max(), "n bad", (d > tol).sum())
for b in bad:
    r = rows[b]; view = r // (g.det_u * g.det_v); iu = r % g.det_u; iv = (r // g.det_u) % g.det_v
    print(f"view {view} iv {iv} iu {iu} got {got[r]:.6f} ref {ref[r]:.6f}")
