"""Debug helper: one fuzz case of tests/test_gpu_parity.py::test_operator_parity_fuzz, FP of
one block on the GPU vs the oracle, printing the worst rays."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth, paper_1903_11874_b200 as bs
from oracle.projector import BlockGrid, Projector

seed = int(sys.argv[1]); jsel = int(sys.argv[2]) if len(sys.argv) > 2 else None
rng = np.random.default_rng(1000 + seed)
beam = ["parallel", "fan", "cone"][seed % 3]
nx, ny = int(rng.integers(6, 33)), int(rng.integers(6, 33))
nz = 1 if beam == "fan" else int(rng.integers(2, 25))
nu = int(rng.integers(5, 48)); nv = 1 if beam == "fan" else int(rng.integers(2, 30))
nviews = int(rng.integers(3, 10)); arc = [180.0, 360.0, 90.0][int(rng.integers(0, 3))]
OP = float(rng.uniform(1.2, 4.0)) * max(nx, ny); OD = float(rng.uniform(0.5, 2.0)) * max(nx, ny)
pu, pv = float(rng.uniform(0.6, 2.5)), float(rng.uniform(0.6, 2.5))
vecs = synth.circular(beam, nviews, arc, OP, OD, nu, nv, pu, pv)
if seed % 4 == 3:
    vecs = np.concatenate([vecs, synth.circular(beam, 8, 360.0, OP, OD, nu, nv, pu, pv)[1:2]])
g = synth.Geometry(synth.BEAM_NAMES[beam], vecs, nu, nv, (nx, ny, nz))
div = lambda n: [d for d in range(1, n + 1) if n % d == 0]
blocks = tuple(int(rng.choice(div(n)[:3])) for n in (nx, ny, nz))
print(beam, g.dims, blocks, nu, nv, g.n_views)
ctx = bs.Context.from_geometry(g, blocks, 1)
P = Projector(g, BlockGrid(g.dims, blocks))
views = np.arange(g.n_views)
r2 = np.random.default_rng(seed)
for j in ([jsel] if jsel is not None else range(P.grid.N)):
    x = r2.random(P.grid.bsize, dtype=np.float32)
    proj = torch.zeros(g.n_rays, device="cuda")
    ctx.forward(views, j, torch.from_numpy(x).cuda(), proj)
    got = proj.cpu().numpy().astype(np.float64)
    ref = P.fp(views, j, x.astype(np.float64))
    d = np.abs(got - ref); tol = 1e-5 * ref + 1e-7 * x.max()
    bad = np.nonzero(d > tol)[0]
    if len(bad):
        print("block", j, P.grid.box(j), "bad rays", len(bad), "of", int((ref > 0).sum()))
        for q in bad[:6]:
            v, rem = divmod(q, nu * nv); iv, iu = divmod(rem, nu)
            print("  view", v, "iu", iu, "iv", iv, "got", got[q], "ref", ref[q])

if len(sys.argv) > 3:   # per-voxel lengths of one ray: view iu iv
    v, iu, iv = (int(t) for t in sys.argv[3].split(","))
    j = jsel
    q = (v * nv + iv) * nu + iu
    A = P.csr([v], j)
    row = q - v * nu * nv
    ref = dict(zip(A.indices[A.indptr[row]:A.indptr[row + 1]], A.data[A.indptr[row]:A.indptr[row + 1]]))
    print("oracle row", ref)
    for k in range(P.grid.bsize):
        x = np.zeros(P.grid.bsize, dtype=np.float32); x[k] = 1.0
        proj = torch.zeros(g.n_rays, device="cuda")
        ctx.forward(np.array([v]), j, torch.from_numpy(x).cuda(), proj)
        val = float(proj[q].item())
        if val != 0.0 or k in ref:
            print("  voxel", k, "gpu", val, "oracle", ref.get(k, 0.0))
    a_, b_ = P.ray(v, iu, iv)
    lo, hi = P.grid.box(j)
    print("ray a", a_, "b", b_, "box", lo, hi)
