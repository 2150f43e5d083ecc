"""Writes tests/golden/trajectory_cfg4.json: the fp64 ORACLE's trajectory of cfg4 at full
size (512^3, 720 x 512^2 cone beam, M = 10, N = 8 z-slabs) under its BASELINE.json
schedule: BSGD-TV (Algo 4; lambda = 0.1) with automatic step-size
tuning (Algo 3), alpha M = 1, gamma N = 2, 40 epochs, so that the run
contains Algo 3's decisions at k = 20, 30, 40 and the TV prox of period
round(1/(alpha gamma)) = 40 (reading A17).

Calls only oracle/ and synth/ (inputs).  Run once on a host with ~55 GB of RAM
(~15-25 min on 8 cores):  python tests/golden/gen_trajectory_cfg4.py
The GPU test (tests/test_gpu_trajectories.py) regenerates the same seeded inputs and checks
them against the checksums stored here before comparing."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import synth  # noqa: E402
from oracle import bsgd as ob  # noqa: E402
from oracle.projector import BlockGrid  # noqa: E402

import trajectory_spec as ts  # noqa: E402


def main():
    spec = ts.CFG4
    t0 = time.time()
    g, y, vol32 = ts.inputs(spec, device="cpu")
    grid = BlockGrid(g.dims, spec["blocks"])
    xt = grid.to_blocks(vol32.astype(np.float64))
    print(f"inputs {time.time() - t0:.1f} s", flush=True)
    prm = ob.Params(seed=spec["seed"], mu=float(np.float32(spec["mu0"])), rows_per_epoch=spec["rows"],
                    cols_per_epoch=spec["cols"], tv=True, lam=spec["lam"], tv_iters=20, auto_mu=True)
    o = ob.OracleBSGD(g, spec["blocks"], spec["M"], y.astype(np.float64), prm, row_kind="random",
                      row_seed=spec["row_seed"], x_true=xt)
    del xt
    for k in range(spec["epochs"]):
        t = time.time()
        rec = o.epoch()
        print(f"epoch {rec['k']}: rows {rec['rows']} cols {rec['cols']} mu {rec['mu']:.6g} "
              f"obj {rec['obj']:.9g} rmse {rec['rmse']:.9g}  {time.time() - t:.1f} s", flush=True)
    xs = o.x.ravel()
    idx = ts.sample_voxels(spec, xs.size)
    out = dict(
        spec={k: v for k, v in spec.items()},
        y_check=ts.checksums(y),
        log=[dict(k=r["k"], rows=r["rows"], cols=r["cols"], mu=r["mu"], obj=r["obj"], rmse=r["rmse"]) for r in o.log],
        x_sample_idx=idx.tolist(),
        x_sample=xs[idx].tolist(),
        x_absmax=float(np.max(np.abs(xs))),
        x_norm=float(np.linalg.norm(xs)),
        seconds=time.time() - t0,
    )
    path = os.path.join(ROOT, "tests", "golden", "trajectory_cfg4.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print("wrote", path, f"{time.time() - t0:.0f} s")


if __name__ == "__main__":
    main()
