"""CPU-side checks of the C-ABI library: it loads, exports every symbol that
include/bsgd.h declares, and its pure host functions (geometry, sampler,
partition, Eq. 8, ownership) agree bit-for-bit with the independent oracle /
synth implementations.  No device calls."""
import os
import re

import numpy as np
import pytest

import synth
from oracle import bsgd as ob

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def bs():
    import __graft_entry__
    __graft_entry__.build()       # compiles libbsgd.so if missing or stale
    import paper_1903_11874_b200 as m
    return m


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "bsgd.h")).read()
    return sorted(set(re.findall(r"\b(bsgd_[a-z0-9_]+)\s*\(", text)))


def test_exports_every_declared_symbol(bs):
    import subprocess
    out = subprocess.run(["nm", "-D", "--defined-only", bs.LIB_PATH], capture_output=True, text=True).stdout
    exported = {l.split()[-1] for l in out.splitlines() if " T " in l}
    want = set(declared_symbols())
    assert want, "header parse failed"
    assert want <= exported, want - exported
    assert bs.abi_version() == 4


def test_geometry_bit_exact(bs):
    for args in [("parallel", 90, 180.0, 0.0, 0.0, 95, 1, 1.0, 1.0),
                 ("fan", 360, 360.0, 400.0, 400.0, 367, 1, 2.0, 1.0),
                 ("cone", 720, 360.0, 6144.0, 4000.0, 1024, 1024, 1.5625, 1.5625),
                 ("cone", 7, 359.0, 10.0, 5.0, 3, 3, 0.3, 0.7)]:
        a = bs.geometry_circular(*args)
        b = synth.circular(*args)
        assert np.array_equal(a.view(np.uint64), b.view(np.uint64))
    v = bs.geometry_circular("parallel", 4, 360.0, 0, 0, 5, 1, 1.0, 1.0)
    assert v[1, 0] == 0.0 and v[1, 1] == -1.0 and v[2, 0] == 1.0   # exact quadrants


def test_sampler_bit_exact(bs):
    for seed in [0, 1, 12345, 2 ** 63 + 7]:
        for stream in [1, 2, 3]:
            for e in range(0, 300, 7):
                for n, m in [(10, 1), (8, 2), (8, 8), (5, 3), (1, 1)]:
                    assert bs.sample(seed, stream, e, n, m) == ob.select(seed, stream, e, n, m)
    # survey KATs: seed 1, epoch 0: rows (10 choose 1) -> [7]; cols (8 choose 2) epochs 0..4
    assert bs.sample(1, 1, 0, 10, 1) == [7]
    assert [bs.sample(1, 2, e, 8, 2) for e in range(5)] == [[2, 3], [3, 5], [4, 7], [2, 7], [5, 7]]


def test_stratified_sampler_bit_exact(bs):
    for seed in [0, 3, 2 ** 62 + 1]:
        for e in range(0, 200, 3):
            for n, m, S in [(8, 2, 2), (8, 8, 4), (8, 4, 4), (16, 4, 2), (6, 3, 3), (8, 2, 1)]:
                assert bs.sample_stratified(seed, e, n, m, S) == ob.select_stratified(seed, e, n, m, S)
    for bad in [(8, 3, 2), (8, 2, 3), (8, 2, 0)]:
        with pytest.raises(bs.BsgdError):
            bs.sample_stratified(1, 0, *bad)


def test_partition_and_eq8_bit_exact(bs):
    for kind in ["random", "contiguous", "interleaved"]:
        for nv, M, seed in [(360, 5, 1), (90, 4, 7), (720, 10, 3), (5, 5, 0)]:
            assert bs.view_partition(nv, M, kind, seed) == ob.view_partition(nv, M, kind, seed)
    for nodes in [1, 2, 4, 8, 16]:
        for M, N in [(20, 8), (5, 8), (4, 2), (10, 8), (1, 1)]:
            assert bs.eq8(nodes, M, N) == ob.eq8_counts(nodes, M, N)[:2]
    assert bs.owned_blocks(8, 4, 3) == (6, 2)


def test_invalid_arguments(bs):
    with pytest.raises(bs.BsgdError) as e:
        bs.view_partition(3, 4)
    assert e.value.code == 2
    with pytest.raises(bs.BsgdError) as e:
        bs.owned_blocks(8, 3, 0)
    assert e.value.code == 2
    with pytest.raises(bs.BsgdError):
        bs.sample(0, 1, 0, 3, 4)
    with pytest.raises(bs.BsgdError) as e:
        bs.geometry_circular("fan", 4, 360.0, -1.0, 1.0, 3, 1, 1.0, 1.0)
    assert e.value.code == 1
