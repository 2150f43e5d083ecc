"""Convergence behaviour the paper reports, reproduced on synthetic data with the CUDA path
(SURVEY §8d "expected outcome" rows; no oracle involved -- data are the closed-form ellipse /
ellipsoid line integrals of synth, noise as in §8c A27 / P:506):

  cfg2  BSGD-IM vs BSGD-RAN (Fig. 18): 2D fan 256^2, 360 views, 4 x 4 blocks,
        M = 4, two half-detector tiles, alpha M = 1, gamma N = 2, Poisson noise (I0 = 2e3);
        GAP / GAP_0 = |y - A x_k| / |y| per epoch, median of 3 seeds.
  cfg3  BSGD (gamma N = 2) vs SAG (gamma N = N) vs mini-batch SGD (Eq. 4):
        3D cone 256^3, 360 views, 8 z-slabs, M = 5, 28.1 dB Gaussian noise; objective
        1/2 |y - A x|^2 against block multiplications (FP + BP block pairs).

    python tools/convergence.py [--epochs-cfg2 300] [--epochs-cfg3 60]
writes profiles/convergence_r01.json and prints a summary."""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
import paper_1903_11874_b200 as bs  # noqa: E402


def data(p, g, noise):
    ells = synth.ellipsoids_world(p.phantom, g.dims)
    y = synth.analytic_projection(g, ells).ravel()
    if noise[0] == "poisson":
        y = synth.poisson_noise(y, noise[1], noise[2])
    else:
        y = synth.gaussian_noise_snr(y, noise[1], noise[2])
    return y.astype(np.float32)


def run(p, g, y, epochs, omega, flags, aM, gN, seed):
    ctx = bs.Context.from_geometry(g, p.blocks, p.M, kind="random", row_seed=1, tiles=p.tiles)
    yd = torch.from_numpy(y).cuda()
    x = torch.zeros(ctx.owned_count * ctx.block_voxels, device="cuda")
    sig = ctx.power_iteration(30)
    res = ctx.run(yd, x, epochs=epochs, mu0=omega / sig, seed=seed, rows_per_epoch=aM, cols_per_epoch=gN,
                  flags=flags | bs.LOG_TRUE_OBJ)
    ctx.close()
    return res, sig


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--epochs-cfg2", type=int, default=300)
    ap.add_argument("--epochs-cfg3", type=int, default=60)
    a = ap.parse_args()
    out = {}
    # ---- cfg2: IM vs RAN (same M, same tiles, same seeds)
    p = synth.PRESETS["cfg2"]
    g = p.geometry()
    y = data(p, g, ("poisson", 2000.0, 7))
    y0 = float(np.linalg.norm(y))
    curves = {}
    for name, flags in [("IM", bs.IS), ("RAN", bs.IS | bs.IS_UNIFORM), ("full views", 0)]:
        gaps = []
        for seed in (1, 2, 3):
            res, sig = run(p, g, y, a.epochs_cfg2, 0.5, flags, 1, 2, seed)
            gaps.append(np.sqrt(2.0 * res.obj_true) / y0)
        curves[name] = np.median(np.array(gaps), axis=0)
    E = a.epochs_cfg2
    out["cfg2_im_vs_ran"] = {
        "what": "GAP/|y| per epoch, median of seeds 1-3; alpha M = 1, gamma N = 2, mu = 0.5/sigma_max^2; "
                "'full views' = Algo 1 without tiles (twice the FP/BP rows of IM / RAN)",
        "epochs": E,
        "at": {str(k): {n: float(c[k - 1]) for n, c in curves.items()} for k in (E // 4, E // 2, E)},
        "curves": {n: c.tolist() for n, c in curves.items()}}
    # ---- cfg3: BSGD vs SAG vs SGD per block multiplication
    p = synth.PRESETS["cfg3"]
    g = p.geometry()
    y = data(p, g, ("gauss", 28.1, 7))
    res3 = {}
    for name, flags, gN, omega in [("BSGD (gamma N = 2)", 0, 2, 0.5), ("SAG (gamma N = 8)", 0, 8, 0.5),
                                   ("SGD (Eq. 4)", bs.SGD, 8, 0.5)]:
        E3 = a.epochs_cfg3 if gN == 8 else 4 * a.epochs_cfg3
        r, sig = run(p, g, y, E3, omega, flags, 1, gN, 1)
        mult = np.arange(1, E3 + 1) * gN            # block multiplications (one row block per epoch)
        res3[name] = {"block_mult": mult.tolist(), "obj_true": r.obj_true.tolist()}
    out["cfg3_bsgd_sag_sgd"] = {
        "what": "1/2 |y - A x|^2 vs block multiplications (alpha M = 1 row block of 72 views per epoch), "
                "mu = 0.5/sigma_max^2, seed 1",
        "runs": res3}
    path = os.path.join(ROOT, "profiles", "convergence_r01.json")
    json.dump(out, open(path, "w"))
    print("cfg2 GAP/|y| (median of 3 seeds):")
    for k, row in out["cfg2_im_vs_ran"]["at"].items():
        print(f"  epoch {k}: " + ", ".join(f"{n} {v:.4f}" for n, v in row.items()))
    print("cfg3 objective at equal block multiplications:")
    for m in (16, 64, 8 * a.epochs_cfg3):
        row = []
        for n, rr in res3.items():
            bm = np.array(rr["block_mult"])
            i = int(np.searchsorted(bm, m))
            if i < len(bm):
                row.append(f"{n} {rr['obj_true'][i]:.4g}")
        print(f"  {m} block mult: " + ", ".join(row))


if __name__ == "__main__":
    main()
