"""Pins of the oracle's Siddon operator against things other than itself:
brute-force per-voxel clipping, closed-form chords, printed paper dimensions,
the adjoint identity, block additivity."""
import math

import numpy as np
import pytest

import synth
from oracle.projector import BlockGrid, Projector, lib, _p
import ctypes as C


def brute_force_row(a, b, dims):
    """Clip the ray against EVERY voxel box independently (no traversal).
    Half-open [lo, hi) emulated: an axis with b == 0 is inside iff lo <= a < hi."""
    nx, ny, nz = dims
    blen = math.sqrt(sum(v * v for v in b))
    out = {}
    for iz in range(nz):
        for iy in range(ny):
            for ix in range(nx):
                lo = (ix, iy, iz)
                t0, t1 = 0.0, 1.0
                ok = True
                for c in range(3):
                    if b[c] == 0.0:
                        if not (lo[c] <= a[c] < lo[c] + 1):
                            ok = False
                            break
                    else:
                        u0 = (lo[c] - a[c]) / b[c]
                        u1 = (lo[c] + 1 - a[c]) / b[c]
                        t0 = max(t0, min(u0, u1))
                        t1 = min(t1, max(u0, u1))
                if ok and t1 > t0:
                    out[(iz * ny + iy) * nx + ix] = (t1 - t0) * blen
    return out


def trace(a, b, lo, hi, cap=4096):
    idx = np.zeros(cap, dtype=np.int64)
    ln = np.zeros(cap)
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    lo = np.ascontiguousarray(lo, dtype=np.int32)
    hi = np.ascontiguousarray(hi, dtype=np.int32)
    n = lib().oracle_trace(_p(a, C.c_double), _p(b, C.c_double), _p(lo, C.c_int), _p(hi, C.c_int),
                           _p(idx, C.c_int64), _p(ln, C.c_double), cap)
    return dict(zip(idx[:n].tolist(), ln[:n].tolist()))


def _compare(a, b, dims, tol=1e-12):
    bf = {k: v for k, v in brute_force_row(a, b, dims).items() if v > 1e-12}
    tr = {k: v for k, v in trace(a, b, [0, 0, 0], list(dims)).items() if v > 1e-12}
    assert set(bf) == set(tr)
    for k in bf:
        assert abs(bf[k] - tr[k]) <= tol * max(1.0, bf[k])


@pytest.mark.parametrize("n", [4, 8])
def test_brute_force_2d(n):
    rng = np.random.default_rng(n)
    dims = (n, n, 1)
    for _ in range(200):
        ang = rng.uniform(0, 2 * math.pi)
        off = rng.uniform(-n, n)
        d = np.array([math.cos(ang), math.sin(ang), 0.0])
        perp = np.array([-d[1], d[0], 0.0])
        c = np.array([n / 2, n / 2, 0.5]) + off * perp
        _compare(c - 2 * n * d, 4 * n * d, dims)


@pytest.mark.parametrize("n", [4, 8])
def test_brute_force_3d(n):
    rng = np.random.default_rng(100 + n)
    dims = (n, n, n)
    for _ in range(60):
        d = rng.standard_normal(3)
        d /= np.linalg.norm(d)
        c = np.array([n / 2] * 3) + rng.uniform(-n / 2, n / 2, 3)
        _compare(c - 2 * n * d, 4 * n * d, dims)


def test_special_rays():
    # axis-aligned rays through a K=16 grid: 16 entries of length 1 (SPEC examples)
    n = 16
    for y in [0.0, 0.5, 7.0, 15.999]:
        tr = trace([-5.0, y, 0.5], [40.0, 0.0, 0.0], [0, 0, 0], [n, n, 1])
        assert len(tr) == n and all(abs(v - 1.0) < 1e-12 for v in tr.values())
    # a ray exactly on the plane y = 16 (upper face) misses (half-open)
    assert trace([-5.0, 16.0, 0.5], [40.0, 0.0, 0.0], [0, 0, 0], [n, n, 1]) == {}
    # ray lying on the interior plane y = 7 belongs to row 7 only
    tr = trace([-5.0, 7.0, 0.5], [40.0, 0.0, 0.0], [0, 0, 0], [n, n, 1])
    assert {k // n for k in tr} == {7}
    # 45° diagonal through voxel corners: n segments of sqrt(2) on the diagonal
    tr = {k: v for k, v in trace([-1.0, -1.0, 0.5], [n + 2.0, n + 2.0, 0.0], [0, 0, 0], [n, n, 1]).items()
          if v > 1e-12}
    assert sorted(tr) == [i * n + i for i in range(n)]
    assert all(abs(v - math.sqrt(2)) < 1e-12 for v in tr.values())
    # ray missing the grid -> empty row
    assert trace([-5.0, -3.0, 0.5], [40.0, 0.0, 0.0], [0, 0, 0], [n, n, 1]) == {}


def chord(a, b, lo, hi):
    """Closed-form chord length of the segment a + t b, t in [0,1], through a box."""
    t0, t1 = 0.0, 1.0
    for c in range(3):
        if b[c] == 0:
            if not (lo[c] <= a[c] < hi[c]):
                return 0.0
        else:
            u0, u1 = sorted(((lo[c] - a[c]) / b[c], (hi[c] - a[c]) / b[c]))
            t0, t1 = max(t0, u0), min(t1, u1)
    return max(0.0, t1 - t0) * float(np.linalg.norm(b))


def test_row_sums_equal_chords_cone():
    p = synth.scaled(synth.PRESETS["cfg3"], 16, n_views=12)
    g = p.geometry()
    P = Projector(g, BlockGrid(g.dims, (1, 1, 2)))
    ones = np.ones(P.grid.bsize)
    for j in range(2):
        lo, hi = P.grid.box(j)
        proj = P.fp(range(12), j, ones)
        for view in range(12):
            for iv in range(0, 16, 3):
                for iu in range(0, 16, 5):
                    a, b = P.ray(view, iu, iv)
                    ray = (view * 16 + iv) * 16 + iu
                    assert abs(proj[ray] - chord(a, b, lo, hi)) < 1e-11


def test_cfg1_half_open_kat():
    """cfg1 view 0 (theta = 0, parallel rays exactly on pixel planes y = k):
    exactly 64 of the 95 rays hit, each with 64 unit segments (brute force)."""
    g = synth.PRESETS["cfg1"].geometry()
    P = Projector(g, BlockGrid(g.dims, (1, 1, 1)))
    A = P.csr([0], 0)
    cnt = np.diff(A.indptr)
    assert (cnt > 0).sum() == 64
    assert set(cnt[cnt > 0]) == {64}
    assert np.allclose(A.data, 1.0, atol=1e-12)
    # brute force agrees on a few rays of view 0 and view 45 (90 degrees)
    for view, iu in [(0, 10), (0, 47), (0, 78), (45, 20), (45, 60)]:
        a, b = P.ray(view, iu, 0)
        bf = {k: v for k, v in brute_force_row(a, b, g.dims).items() if v > 1e-12}
        row = A if view == 0 else P.csr([view], 0)
        r = row.getrow(iu)
        got = {int(k): float(v) for k, v in zip(r.indices, r.data) if v > 1e-12}
        assert set(got) == set(bf)


def _paper_rows():
    rows = []
    with open(__file__.replace("test_oracle_siddon.py", "golden/paper_dims.txt")) as f:
        for line in f:
            if line.startswith("#") or not line.strip():
                continue
            t = line.split()
            rows.append(t)
    return rows


def _half_ulp(text):
    if "e" not in text:
        return 0.5
    mant, ex = text.split("e")
    dec = len(mant.split(".")[1]) if "." in mant else 0
    return 0.5 * 10.0 ** (int(ex) - dec)


def test_paper_dimensions():
    """Printed sizes of A: 1080 x 256, 32400 x 4096,
    Table 1, skull 9.4e7 x 1.7e7."""
    for name, beam, K, du, dv, nvw, rows, cols, _ in _paper_rows():
        K, du, dv, nvw = int(K), int(du), int(dv), int(nvw)
        dims = (K, K, 1) if beam == "fan" else (K, K, K)
        vecs = synth.circular(beam, nvw, 360.0 if name != "sec3D" else 180.0, 50.0, 50.0, du, dv, 1.0, 1.0)
        g = synth.Geometry(synth.BEAM_NAMES[beam], vecs, du, dv, dims)
        # a printed value is exact to half a unit of its last printed digit
        assert abs(g.n_rays - float(rows)) <= _half_ulp(rows)
        assert abs(g.n_vox - float(cols)) <= _half_ulp(cols)
        if name == "sec3A":
            P = Projector(g, BlockGrid(dims, (2, 1, 1)))
            A0, A1 = P.csr(range(36), 0), P.csr(range(36), 1)
            assert A0.shape[0] == 1080 and A0.shape[1] + A1.shape[1] == 256
            assert (A0.data >= 0).all() and (A1.data >= 0).all()     # non-negative


def test_adjoint_and_block_additivity():
    """<A x, y> = <x, A^T y> to 1e-12 over random blocks (FP gathers, BP scatters
    through separate code paths); sum_j A^{J_j} x_{J_j} = A x (Eq. 3)."""
    p = synth.scaled(synth.PRESETS["cfg3"], 16, n_views=8)
    g = p.geometry()
    rng = np.random.default_rng(3)
    for blocks in [(1, 1, 4), (2, 2, 2), (1, 2, 1)]:
        P = Projector(g, BlockGrid(g.dims, blocks))
        views = np.arange(8)
        for j in range(P.grid.N):
            x = rng.standard_normal(P.grid.bsize)
            y = rng.standard_normal(g.n_rays)
            ax = P.fp(views, j, x)
            aty = P.bp(views, j, y)
            lhs, rhs = float(ax @ y), float(x @ aty)
            assert abs(lhs - rhs) <= 1e-12 * max(1.0, abs(lhs)) * 100
    # block additivity vs the single-block operator
    P1 = Projector(g, BlockGrid(g.dims, (1, 1, 1)))
    P8 = Projector(g, BlockGrid(g.dims, (2, 2, 2)))
    vol = rng.standard_normal((16, 16, 16))
    full = P1.fp(np.arange(8), 0, vol.ravel())
    xb = P8.grid.to_blocks(vol)
    acc = np.zeros_like(full)
    for j in range(8):
        P8.fp(np.arange(8), j, xb[j], proj=acc, accumulate=True)
    assert np.max(np.abs(acc - full)) <= 1e-10 * np.max(np.abs(full))
    # linearity and FP(0) = 0
    x1, x2 = rng.standard_normal(P1.grid.bsize), rng.standard_normal(P1.grid.bsize)
    f = lambda x: P1.fp(np.arange(8), 0, x)
    assert np.max(np.abs(f(2 * x1 - 3 * x2) - (2 * f(x1) - 3 * f(x2)))) < 1e-9
    assert np.all(f(np.zeros_like(x1)) == 0)


def test_rects_restrict_rows():
    """FP/BP with detector rects touch exactly the rays inside the rect."""
    p = synth.scaled(synth.PRESETS["cfg3"], 16, n_views=4)
    g = p.geometry()
    P = Projector(g, BlockGrid(g.dims, (1, 1, 2)))
    x = np.ones(P.grid.bsize)
    full = P.fp(range(4), 1, x)
    rects = [(0, 16, 4, 8)] * 4
    part = P.fp(range(4), 1, x, rects=rects)
    mask = np.zeros((4, 16, 16), bool)
    mask[:, 4:8, :] = True
    mask = mask.ravel()
    assert np.array_equal(part[mask], full[mask]) and np.all(part[~mask] == 0)


def test_unequal_z_slabs():
    """Column blocks need not be equal (Eq. 3's partition J):
    z-slabs between arbitrary split planes are a partition of the volume (to/from_blocks
    round trip, zero tails), their operators sum to the single-block A (block additivity),
    the adjoint identity holds per slab, and every slab's operator equals the same box cut
    from an equal-slab grid where the boxes coincide."""
    p = synth.scaled(synth.PRESETS["cfg3"], 16, n_views=8)
    g = p.geometry()
    rng = np.random.default_rng(8)
    zs = [0, 3, 4, 9, 16]
    grid = BlockGrid(g.dims, (1, 1, 4), zs)
    assert grid.bsizes == [16 * 16 * t for t in (3, 1, 5, 7)] and grid.bsize == 16 * 16 * 7
    vol = rng.standard_normal((16, 16, 16))
    xb = grid.to_blocks(vol)
    assert np.array_equal(grid.from_blocks(xb), vol)
    assert np.all(xb[0, grid.bsizes[0]:] == 0) and grid.mask().sum() == 16 ** 3
    P = Projector(g, grid)
    views = np.arange(8)
    full = Projector(g, BlockGrid(g.dims, (1, 1, 1))).fp(views, 0, vol.ravel())
    acc = np.zeros_like(full)
    for j in range(4):
        P.fp(views, j, xb[j], proj=acc, accumulate=True)
        y = rng.standard_normal(g.n_rays)
        lhs, rhs = float(P.fp(views, j, xb[j]) @ y), float(xb[j] @ P.bp(views, j, y))
        assert abs(lhs - rhs) <= 1e-10 * max(1.0, abs(lhs))
        assert np.all(P.bp(views, j, y)[grid.bsizes[j]:] == 0)   # nothing lands in the tail
    assert np.max(np.abs(acc - full)) <= 1e-10 * np.max(np.abs(full))
    # slab [4, 8) of an equal (1,1,4) grid vs a split grid containing the same box
    Pe = Projector(g, BlockGrid(g.dims, (1, 1, 4)))
    Pu = Projector(g, BlockGrid(g.dims, (1, 1, 3), [0, 4, 8, 16]))
    xe = Pe.grid.to_blocks(vol)
    xu = Pu.grid.to_blocks(vol)
    assert np.array_equal(Pe.fp(views, 1, xe[1]), Pu.fp(views, 1, xu[1]))
    with pytest.raises(ValueError):
        BlockGrid(g.dims, (2, 1, 2), [0, 8, 16])
    with pytest.raises(ValueError):
        BlockGrid(g.dims, (1, 1, 2), [0, 9, 9])
