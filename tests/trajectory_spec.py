"""Full-size trajectory fixtures: the run specifications and their seeded inputs (inputs
only — geometry, phantom, data, sampled voxel ids; none of the method's arithmetic).
Shared by the fixture generators under tests/golden/ (which run the ORACLE) and the GPU
tests (which run the CUDA path); neither side's numbers flow into the other."""
from __future__ import annotations

import numpy as np

import synth

# cfg4 (BASELINE.json configs[3]): BSGD-TV lambda = 0.1 + automatic step size, alpha M = 1,
# gamma N = 2; 40 epochs = Algo 3 decisions at k = 20, 30, 40 + the period-40 TV prox.
# mu0 = 0.5 / 3.59e5 (3.59e5 = the ones-vector Rayleigh lower bound of sigma_max^2, SURVEY
# App. A; the paper's mu is not transferable, reading A23).
CFG4 = dict(name="cfg4", blocks=(1, 1, 8), M=10, rows=1, cols=2, epochs=40, seed=5, row_seed=11,
            mu0=0.5 / 3.59e5, lam=0.1, n_sample=20000)

# cfg5 (configs[4]) at the Eq. 8 NodeNum = 1 schedule of BASELINE.md §3's cfg5 protocol:
# M = 10, N = 8, alpha M = 1, gamma N = 1, 20 epochs, plain BSGD (Algo 1); mu0 = 0.5 / 7.35e5
# (the cfg5 Rayleigh bound).
CFG5 = dict(name="cfg5", blocks=(1, 1, 8), M=10, rows=1, cols=1, epochs=20, seed=7, row_seed=13,
            mu0=0.5 / 7.35e5, n_sample=20000)


def inputs(spec, device="cpu"):
    """(geometry, y fp32, x_true fp32 volume [z][y][x]) of a preset, as synth makes them."""
    p = synth.PRESETS[spec["name"]]
    g = p.geometry()
    ells = synth.ellipsoids_world(p.phantom, g.dims)
    if device == "cpu":
        vol32 = synth.rasterise(ells, g.dims).astype(np.float32)
    else:   # the same values (identical fp64 operations), minutes faster at 1024^3
        vol32 = synth.rasterise_torch(ells, g.dims, device=device).cpu().numpy()
    y = synth.analytic_projection(g, ells, device=device).ravel()
    if p.noise is not None:
        kind, a, seed = p.noise
        y = synth.gaussian_noise_snr(y, a, seed) if kind == "gauss" else synth.poisson_noise(y, a, seed)
    return g, y.astype(np.float32), vol32


def checksums(y32):
    """Order-fixed fp64 sums that identify the data (1e-9 agreement expected across hosts:
    the generators' float64 reductions may differ in the last ulps)."""
    y = np.asarray(y32, dtype=np.float64)
    return dict(n=int(y.size), sum=float(np.sum(y)), sumsq=float(np.sum(y * y)),
                head=[float(v) for v in y[:4]], mid=float(y[y.size // 2]))


def sample_voxels(spec, n_vox):
    rng = np.random.default_rng(12345)
    return np.sort(rng.choice(n_vox, size=spec["n_sample"], replace=False))
