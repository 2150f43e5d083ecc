"""One-off robustness sweep: tests/test_gpu_parity.py::test_operator_parity_fuzz over many
more seeds than the suite runs (FP/BP per ray / voxel vs the oracle on random beams, volumes,
block grids, detectors, orbits, IM rectangles, laminography).  usage: python tools/fuzz_sweep.py A B"""
import os
import sys
import traceback

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import paper_1903_11874_b200 as bs  # noqa: E402
import test_gpu_parity as t  # noqa: E402

a, b = int(sys.argv[1]), int(sys.argv[2])
bad = []
for seed in range(a, b):
    try:
        t.test_operator_parity_fuzz.__wrapped__(bs, seed) if hasattr(t.test_operator_parity_fuzz, "__wrapped__") \
            else t.test_operator_parity_fuzz(bs, seed)
    except Exception:
        bad.append(seed)
        traceback.print_exc(limit=2)
print(f"fuzz seeds {a}..{b - 1}: {b - a - len(bad)} passed, failed: {bad}")
