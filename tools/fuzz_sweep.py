"""One-off robustness sweep: tests/test_gpu_parity.py::test_operator_parity_fuzz over many
more seeds than the suite runs (FP/BP per ray / voxel vs the oracle on random beams, volumes,
block grids, detectors, orbits, IM rectangles, laminography), or of test_trajectory_fuzz
(random BSGD / IM / RAN / TV + auto-mu / SGD runs).
usage: python tools/fuzz_sweep.py A B [operator|trajectory]"""
import os
import sys
import traceback

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import paper_1903_11874_b200 as bs  # noqa: E402
import test_gpu_parity as t  # noqa: E402

a, b = int(sys.argv[1]), int(sys.argv[2])
which = sys.argv[3] if len(sys.argv) > 3 else "operator"
fn = t.test_operator_parity_fuzz if which == "operator" else t.test_trajectory_fuzz
bad = []
for seed in range(a, b):
    try:
        fn(bs, seed)
    except Exception:
        bad.append(seed)
        traceback.print_exc(limit=2)
print(f"{which} fuzz seeds {a}..{b - 1}: {b - a - len(bad)} passed, failed: {bad}")
