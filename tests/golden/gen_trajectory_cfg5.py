"""Writes tests/golden/trajectory_cfg5.json: the fp64 ORACLE's trajectory of cfg5 at full
size (1024^3, 720 x 1024^2 cone beam, M = 10, N = 8 z-slabs) under the Eq. 8 NodeNum = 1
schedule of BASELINE.md §3's cfg5 protocol: Algo 1 with alpha M =
gamma N = 1, 20 epochs.  The dense oracle state would need ~130 GB, so the run uses
oracle.bsgd.OracleBSGDLean (the same Algo 1 with storage restricted to the touched (row
block, column block) pairs; pinned against the dense oracle in tests/test_oracle_bsgd.py),
with g-hat file-backed.

Calls only oracle/ and synth/ (inputs).  Needs ~40 GB of RAM, ~25 GB of scratch disk and
1.5-3 h on 8 cores (most of it the closed-form data):  python tests/golden/gen_trajectory_cfg5.py"""
import json
import os
import shutil
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from oracle import bsgd as ob  # noqa: E402
from oracle.projector import BlockGrid  # noqa: E402

import trajectory_spec as ts  # noqa: E402


def main():
    spec = ts.CFG5
    t0 = time.time()
    g, y, vol32 = ts.inputs(spec, device="cpu")
    grid = BlockGrid(g.dims, spec["blocks"])
    xt = grid.to_blocks(vol32)
    del vol32
    print(f"inputs {time.time() - t0:.1f} s", flush=True)
    prm = ob.Params(seed=spec["seed"], mu=float(np.float32(spec["mu0"])), rows_per_epoch=spec["rows"],
                    cols_per_epoch=spec["cols"])
    scratch = tempfile.mkdtemp(prefix="bsgd_cfg5_ghat_", dir=os.environ.get("BSGD_SCRATCH", "/tmp"))
    try:
        o = ob.OracleBSGDLean(g, spec["blocks"], spec["M"], y, prm, row_kind="random", row_seed=spec["row_seed"],
                              x_true32=xt, ghat_dir=scratch)
        for _ in range(spec["epochs"]):
            t = time.time()
            rec = o.epoch()
            print(f"epoch {rec['k']}: rows {rec['rows']} cols {rec['cols']} mu {rec['mu']:.6g} "
                  f"obj {rec['obj']:.9g} rmse {rec['rmse']:.9g}  {time.time() - t:.1f} s", flush=True)
        xs = o.x.ravel()
        idx = ts.sample_voxels(spec, xs.size)
        out = dict(
            spec={k: v for k, v in spec.items()},
            y_check=ts.checksums(y),
            log=[dict(k=r["k"], rows=r["rows"], cols=r["cols"], mu=r["mu"], obj=r["obj"], rmse=r["rmse"])
                 for r in o.log],
            x_sample_idx=idx.tolist(),
            x_sample=xs[idx].tolist(),
            x_absmax=float(np.max(np.abs(xs))),
            x_norm=float(np.linalg.norm(xs)),
            seconds=time.time() - t0,
        )
    finally:
        shutil.rmtree(scratch, ignore_errors=True)
    path = os.path.join(ROOT, "tests", "golden", "trajectory_cfg5.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print("wrote", path, f"{time.time() - t0:.0f} s")


if __name__ == "__main__":
    main()
