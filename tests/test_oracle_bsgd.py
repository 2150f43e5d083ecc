"""Pins of the oracle's BSGD layer (§IV fixed point 539-639)
against closed forms, special cases, independent re-implementations and
printed values — never against the oracle itself."""
import math
import os

import numpy as np
import pytest

import synth
from oracle import bsgd as ob
from oracle.projector import BlockGrid, Projector

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


# --------------------------------------------------------------------------- sampler
def test_splitmix64_kat():
    want = [int(l, 16) for l in open(os.path.join(GOLDEN, "splitmix64.txt")) if not l.startswith("#")]
    got = [ob.rnd(0, 0, 0, k) for k in range(4)]
    assert got == want


def test_select_properties_and_uniformity():
    n, m = 6, 2
    counts = {}
    for e in range(6000):
        s = ob.select(12345, 2, e, n, m)
        assert s == sorted(s) and len(set(s)) == m and all(0 <= v < n for v in s)
        counts[tuple(s)] = counts.get(tuple(s), 0) + 1
    assert len(counts) == math.comb(n, m)
    exp = 6000 / math.comb(n, m)
    chi2 = sum((c - exp) ** 2 / exp for c in counts.values())
    assert chi2 < 45.0                      # 14 dof, p ~ 1e-4
    assert ob.select(1, 1, 0, 5, 5) == [0, 1, 2, 3, 4]
    assert sorted(ob.permutation(7, 0, 0, 50)) == list(range(50))


def test_view_partition():
    for kind in ["random", "contiguous", "interleaved"]:
        rows = ob.view_partition(360, 5, kind, seed=3)
        flat = sorted(v for r in rows for v in r)
        assert flat == list(range(360)) and all(len(r) == 72 for r in rows)
        assert all(r == sorted(r) for r in rows)
    rows = ob.view_partition(90, 4, "random", seed=1)
    assert [len(r) for r in rows] == [23, 23, 22, 22]      # first V mod M get +1
    with pytest.raises(ValueError):
        ob.view_partition(3, 4)


def test_eq8_printed_examples():
    for line in open(os.path.join(GOLDEN, "eq8.txt")):
        if line.startswith("#") or not line.strip():
            continue
        t = line.split()
        node, M, N, alpha, gamma = int(t[0]), int(t[1]), int(t[2]), float(t[3]), float(t[4])
        aM, gN, a, g = ob.eq8_counts(node, M, N)
        assert abs(a - alpha) < 1e-12 and abs(g - gamma) < 1e-12
        assert aM == round(alpha * M) and gN == round(gamma * N)
    # NodeNum = M N -> alpha = gamma = 1
    assert ob.eq8_counts(32, 4, 8)[:2] == (4, 8)


# --------------------------------------------------------------------------- small systems
def sec3a_system(M=4, N=2, noise=True):
    """The paper's §III-A system: 2D fan, K = 16, OP = OD = 50, 30 detectors,
    10° steps -> A in R^{1080 x 256}; 17.5 dB noise."""
    vecs = synth.circular("fan", 36, 360.0, 50.0, 50.0, 30, 1, 1.0, 1.0)
    g = synth.Geometry(synth.FAN, vecs, 30, 1, (16, 16, 1))
    blocks = {1: (1, 1, 1), 2: (2, 1, 1), 4: (2, 2, 1)}[N]
    grid = BlockGrid(g.dims, blocks)
    P = Projector(g, grid)
    A = P.dense()
    x_true = synth.rasterise(synth.ellipsoids_world("shepp2d", g.dims), g.dims).ravel()
    y = A @ x_true
    if noise:
        y = synth.gaussian_noise_snr(y, 17.5, seed=5)
    return g, grid, A, x_true, y


def global_of(grid, xb):
    return grid.from_blocks(xb).ravel()


@pytest.mark.parametrize("M,N", [(4, 2), (1, 1)])
def test_alpha_gamma_one_is_gd_closed_form(M, N):
    """alpha = gamma = 1 refreshes every z and g_hat, so Algo 1 is GD
    x_{k+1} = x_k + 2 mu A^T (y - A x_k); closed form via the
    SVD of A: x_k = sum_i (1 - (1 - 2 mu s_i^2)^k)/s_i (u_i.y) v_i."""
    g, grid, A, x_true, y = sec3a_system(M, N)
    U, s, Vt = np.linalg.svd(A, full_matrices=False)
    mu = 0.5 / s[0] ** 2
    prm = ob.Params(seed=9, mu=mu, rows_per_epoch=M, cols_per_epoch=N)
    o = ob.OracleBSGD(g, grid.blocks, M, y, prm, row_kind="random")
    keep = s > 1e-10 * s[0]
    uy = U.T @ y
    f_prev = 0.5 * y @ y
    for k in range(1, 21):
        o.epoch()
        xk = (Vt[keep].T * ((1 - (1 - 2 * mu * s[keep] ** 2) ** k) / s[keep])) @ uy[keep]
        xg = global_of(grid, o.x)
        assert np.max(np.abs(xg - xk)) <= 1e-10 * np.max(np.abs(xk))
        f = 0.5 * np.sum((y - A @ xg) ** 2)
        assert f <= f_prev * (1 + 1e-12)                   # monotone (mu < 1/s_max^2)
        # the maintained r of epoch k is y - A x_{k-1} (formed before the step)
        assert abs(o.log[-1]["obj"] - f_prev) <= 1e-9 * f_prev
        f_prev = f


def test_gamma_one_is_sag():
    """gamma = 1 makes BSGD SAG ("When gamma = 1, the method becomes
    SAG"): an independent SAG over the M row blocks with stored gradients."""
    M, N = 4, 2
    g, grid, A, x_true, y = sec3a_system(M, N)
    s0 = np.linalg.norm(A, 2)
    mu = 0.3 / s0 ** 2
    prm = ob.Params(seed=4, mu=mu, rows_per_epoch=1, cols_per_epoch=N)
    o = ob.OracleBSGD(g, grid.blocks, M, y, prm)
    rows = [o.P.rows_of(r) for r in o.rows]
    # independent SAG on the dense A (global column order)
    x = np.zeros(A.shape[1])
    d = [np.zeros(A.shape[1]) for _ in range(M)]
    for k in range(60):
        (i,) = ob.select(4, 1, k, M, 1)
        Ai = A[rows[i]]
        d[i] = 2 * Ai.T @ (y[rows[i]] - Ai @ x)
        x = x + mu * sum(d)
        o.epoch()
        assert np.max(np.abs(global_of(grid, o.x) - x)) <= 1e-11 * max(1.0, np.max(np.abs(x)))


def test_fixed_point_is_least_squares():
    """§IV: the state (x_lsq, z^j = A^{J_j} x_lsq,
    g_hat^i_{J_j} = 2 (A_{I_i}^{J_j})^T (y - A x_lsq)_{I_i}) is a fixed point of
    every epoch; a perturbed x is not."""
    M, N = 4, 4
    g, grid, A, x_true, y = sec3a_system(M, N)
    x_lsq = np.linalg.lstsq(A, y, rcond=None)[0]
    s0 = np.linalg.norm(A, 2)
    prm = ob.Params(seed=2, mu=0.5 / s0 ** 2, rows_per_epoch=2, cols_per_epoch=2)

    def make(xg):
        o = ob.OracleBSGD(g, grid.blocks, M, y, prm, row_kind="interleaved")
        o.x = grid.to_blocks(xg.reshape(1, 16, 16))
        views_all = np.arange(g.n_views)
        for j in range(N):
            o.z[j] = o.P.fp(views_all, j, o.x[j])
        o.r = y - o.z.sum(0)
        for i in range(M):
            for j in range(N):
                o.ghat[i, j] = 2 * o.P.bp(o.rows[i], j, o.r)
        o.g = o.ghat.sum(0)
        return o

    o = make(x_lsq)
    x0 = o.x.copy()
    assert np.max(np.abs(o.g)) < 1e-9 * np.max(np.abs(o.ghat))      # A^T r = 0 at x_lsq
    for _ in range(30):
        o.epoch()
    assert np.max(np.abs(o.x - x0)) <= 1e-10 * np.max(np.abs(x0))
    o2 = make(x_lsq + 1e-3 * np.random.default_rng(0).standard_normal(x_lsq.shape))
    xp = o2.x.copy()
    for _ in range(30):
        o2.epoch()
    assert np.max(np.abs(o2.x - xp)) > 1e-6


def test_tiles_one_im_equals_bsgd():
    """A single sub-detector tile makes Algo 2 identical to Algo 1."""
    g, grid, A, x_true, y = sec3a_system(4, 4, noise=False)
    s0 = np.linalg.norm(A, 2)
    base = dict(seed=8, mu=0.5 / s0 ** 2, rows_per_epoch=1, cols_per_epoch=2)
    o1 = ob.OracleBSGD(g, grid.blocks, 4, y, ob.Params(**base))
    o2 = ob.OracleBSGD(g, grid.blocks, 4, y, ob.Params(im=True, **base), tiles=(1, 1))
    for _ in range(10):
        o1.epoch()
        o2.epoch()
    assert np.array_equal(o1.x, o2.x)


def test_im_table_and_containment():
    """IM weights: each row sums to 2^16 up to the floor (<= T); a block whose
    shadow lies inside one tile gets all the weight."""
    vecs = synth.circular("parallel", 8, 180.0, 0, 0, 64, 1, 1.0, 1.0)
    g = synth.Geometry(synth.PARALLEL, vecs, 64, 1, (64, 64, 1))
    P = Projector(g, BlockGrid(g.dims, (1, 2, 1)))       # halves along y
    q = ob.im_table(P, (2, 1))
    assert np.all(q.sum(axis=2) <= ob.IM_SCALE) and np.all(q.sum(axis=2) >= ob.IM_SCALE - 2)
    # view 0: rays along -x at y = iu - 31.5; detector half 0 sees exactly block 0
    assert list(q[0, 0]) == [ob.IM_SCALE, 0] and list(q[1, 0]) == [0, ob.IM_SCALE]


def test_im_area_counts_brute_force():
    """IS_AREA weights (reading A9 alternative) = number of tile rays whose chord through the
    block box exceeds 1e-6, checked against an independent vectorised slab test on the ray
    endpoints; and the containment case of test_im_table_and_containment."""
    p = synth.PRESETS["cfg2"]
    g = p.geometry()
    P = Projector(g, BlockGrid(g.dims, p.blocks))
    views = np.arange(g.n_views)
    A, B = synth.ray_endpoints(g, views)
    A = A.reshape(g.n_views, -1, 3) + np.array(g.dims) / 2.0
    B = B.reshape(g.n_views, -1, 3)
    L = np.linalg.norm(B, axis=2)
    nu = g.det_u
    T = p.tiles[0] * p.tiles[1]
    for j in range(P.grid.N):
        lo, hi = P.grid.box(j)
        t0 = np.zeros(A.shape[:2])
        t1 = np.ones(A.shape[:2])
        for c in range(2 if g.dims[2] == 1 else 3):
            with np.errstate(divide="ignore", invalid="ignore"):
                u0 = (lo[c] - A[..., c]) / B[..., c]
                u1 = (hi[c] - A[..., c]) / B[..., c]
            par = B[..., c] == 0
            inside = (A[..., c] >= lo[c]) & (A[..., c] < hi[c])
            t0 = np.where(par, np.where(inside, t0, 2.0), np.maximum(t0, np.minimum(u0, u1)))
            t1 = np.where(par, np.where(inside, t1, -1.0), np.minimum(t1, np.maximum(u0, u1)))
        chord = np.maximum(t1 - t0, 0.0) * L
        want = np.zeros((g.n_views, T))
        ch = chord.reshape(g.n_views, g.det_v, nu)
        for t, (u0_, u1_, v0_, v1_) in enumerate(ob.tile_rects(nu, g.det_v, p.tiles)):
            want[:, t] = (ch[:, v0_:v1_, u0_:u1_] > 1e-6).sum(axis=(1, 2))
        got = P.tile_mass(views, j, p.tiles, area=True)
        assert np.array_equal(got, want), j
    q = ob.im_table(P, p.tiles, area=True)
    assert np.all(q.sum(axis=2) <= ob.IM_SCALE) and np.all(q.sum(axis=2) >= ob.IM_SCALE - T)


def test_im_epoch_touches_only_tile_rows():
    g, grid, A, x_true, y = sec3a_system(4, 4, noise=False)
    prm = ob.Params(seed=3, mu=1e-4, rows_per_epoch=1, cols_per_epoch=2, im=True)
    o = ob.OracleBSGD(g, grid.blocks, 4, y, prm, tiles=(2, 1))
    o.x[:] = 1.0
    rec = o.epoch()
    rows_hit = set()
    for (j, v), t in rec["tiles"].items():
        u0, u1, _, _ = o.rects[t]
        nz = np.nonzero(o.z[j].reshape(g.n_views, 30)[v])[0]
        assert np.all((nz >= u0) & (nz < u1))
        rows_hit.add(j)
    assert rows_hit == set(rec["cols"])


# --------------------------------------------------------------------------- TV
def test_tv_grad_adjoint():
    rng = np.random.default_rng(1)
    for shape in [(1, 7, 9), (4, 5, 6)]:
        u = rng.standard_normal(shape)
        p = rng.standard_normal((3,) + shape)
        assert abs(np.sum(ob.tv_grad(u) * p) - np.sum(u * ob.tv_grad_T(p))) < 1e-10


def test_tv_prox_closed_forms():
    """w = 0 -> identity; constant image unchanged; image constant along y with a
    step between x-runs of lengths L1, L2 -> exact 1D ROF: levels move by w/L1 and
    w/L2 toward each other until they meet (TV of Eq. 6 with a zero boundary
    difference)."""
    rng = np.random.default_rng(0)
    b = rng.standard_normal((1, 8, 8))
    assert np.array_equal(ob.tv_prox(b, 0.0), b)
    c = np.full((1, 8, 8), 3.25)
    assert np.max(np.abs(ob.tv_prox(c, 0.7) - c)) < 1e-12
    step = np.zeros((1, 8, 8))
    step[..., 4:] = 1.0
    for w, lo, hi in [(0.5, 0.125, 0.875), (3.0, 0.5, 0.5)]:
        t = ob.tv_prox(step, w, iters=20000)
        assert np.max(np.abs(t[..., :4] - lo)) < 1e-9 and np.max(np.abs(t[..., 4:] - hi)) < 1e-9
    # unequal runs L1 = 2, L2 = 6 (3D volume, step along x, constant in y and z)
    s3 = np.zeros((3, 4, 8))
    s3[..., 2:] = 1.0
    t = ob.tv_prox(s3, 0.2, iters=20000)
    assert np.max(np.abs(t[..., :2] - 0.1)) < 1e-8 and np.max(np.abs(t[..., 2:] - (1 - 0.2 / 6))) < 1e-8


def test_tv_prox_20_iterations_improves_objective():
    rng = np.random.default_rng(2)
    img = synth.rasterise(synth.ellipsoids_world("shepp2d", (32, 32, 1)), (32, 32, 1))
    b = img + 0.1 * rng.standard_normal(img.shape)
    w = 0.05
    obj = lambda t: 0.5 * np.sum((t - b) ** 2) + w * ob.tv_value(t)
    t = ob.tv_prox(b, w, 20)
    assert obj(t) < obj(b)
    # non-expansive (prox of a convex function)
    b2 = b + 0.05 * rng.standard_normal(b.shape)
    t_many = ob.tv_prox(b, w, 3000)
    t2_many = ob.tv_prox(b2, w, 3000)
    assert np.linalg.norm(t_many - t2_many) <= np.linalg.norm(b - b2) * (1 + 1e-6)


# --------------------------------------------------------------------------- Algo 3
def test_auto_mu_decisions():
    """Algo 3 lines 5-12 on scripted |r| and theta."""
    kw = dict(eps=0.05, delta=0.4, t1=0.5, t2=0.0)
    # |r| decreasing twice -> increase
    assert ob.auto_mu_decision(1.0, 1.0, 2.0, 3.0, 0.9, 0.9, **kw) == pytest.approx(1.05)
    # |r| increasing twice and theta < t2 -> decrease
    assert ob.auto_mu_decision(1.0, 3.0, 2.0, 1.0, -0.1, 0.9, **kw) == pytest.approx(0.6)
    # increasing twice and |theta - theta_prev| > t1 -> decrease
    assert ob.auto_mu_decision(1.0, 3.0, 2.0, 1.0, 0.2, 0.9, **kw) == pytest.approx(0.6)
    # increasing twice but theta stable and positive -> unchanged (criterion 2 fails)
    assert ob.auto_mu_decision(1.0, 3.0, 2.0, 1.0, 0.8, 0.9, **kw) == 1.0
    # mixed -> unchanged; equalities are not strict monotonicity
    assert ob.auto_mu_decision(1.0, 2.0, 3.0, 2.5, -1.0, 0.9, **kw) == 1.0
    assert ob.auto_mu_decision(1.0, 2.0, 2.0, 2.0, -1.0, 0.9, **kw) == 1.0
    # undefined theta: only theta < t2 could fire, and it is undefined -> unchanged
    assert ob.auto_mu_decision(1.0, 3.0, 2.0, 1.0, None, None, **kw) == 1.0
    assert ob.auto_mu_decision(1.0, 3.0, 2.0, 1.0, -0.5, None, **kw) == pytest.approx(0.6)


def test_auto_mu_recovers_from_large_step():
    """Survey-time behaviour: from mu0 = 4/s_max^2 fixed-step BSGD
    diverges while auto-mu brings the objective down."""
    g, grid, A, x_true, y = sec3a_system(4, 2, noise=False)
    s0 = np.linalg.norm(A, 2)
    base = dict(seed=1, mu=4.0 / s0 ** 2, rows_per_epoch=1, cols_per_epoch=1)
    fixed = ob.OracleBSGD(g, grid.blocks, 4, y, ob.Params(**base))
    auto = ob.OracleBSGD(g, grid.blocks, 4, y, ob.Params(auto_mu=True, **base))
    for _ in range(300):
        fixed.epoch()
        auto.epoch()
    f0 = 0.5 * y @ y
    assert fixed.log[-1]["obj"] > f0
    assert auto.log[-1]["obj"] < 0.05 * f0
    assert auto.log[-1]["mu"] < base["mu"]


def test_select_stratified():
    """Stratified column selection (reading A31): one stratum is the plain
    m-of-n draw on stream 2; every stratum gets m/S distinct blocks of its own range; the
    draw inside a stratum is uniform and independent of the other strata."""
    for e in range(50):
        assert ob.select_stratified(9, e, 8, 2, 1) == ob.select(9, 2, e, 8, 2)
    n, m, S = 8, 4, 2
    counts = {}
    for e in range(6000):
        s = ob.select_stratified(4242, e, n, m, S)
        assert s == sorted(s) and len(set(s)) == m
        assert sum(v < 4 for v in s) == 2 and sum(v >= 4 for v in s) == 2
        counts[tuple(s)] = counts.get(tuple(s), 0) + 1
    assert len(counts) == math.comb(4, 2) ** 2          # every (pair, pair) combination occurs
    exp = 6000 / len(counts)
    chi2 = sum((c - exp) ** 2 / exp for c in counts.values())
    assert chi2 < 75.0                                   # 35 dof, p ~ 1e-4
    assert ob.select_stratified(1, 0, 8, 8, 8) == list(range(8))   # gamma N = N: every block
    with pytest.raises(ValueError):
        ob.select_stratified(1, 0, 8, 3, 2)


def test_tv_prox_chambolle_closed_forms():
    """The Chambolle-2004 flag converges to the same prox: the exact 1D-ROF step solutions
    (levels w/L1, w/L2 toward each other) and the FGP result at many iterations; identity
    for w = 0; a constant image is a fixed point."""
    step = np.zeros((1, 8, 8))
    step[..., 4:] = 1.0
    for w, lo, hi in [(0.5, 0.125, 0.875), (3.0, 0.5, 0.5)]:
        t = ob.tv_prox(step, w, iters=40000, method="chambolle")
        assert np.max(np.abs(t[..., :4] - lo)) < 1e-6 and np.max(np.abs(t[..., 4:] - hi)) < 1e-6
    s3 = np.zeros((3, 4, 8))
    s3[..., 2:] = 1.0
    t = ob.tv_prox(s3, 0.2, iters=40000, method="chambolle")
    assert np.max(np.abs(t[..., :2] - 0.1)) < 1e-6 and np.max(np.abs(t[..., 2:] - (1 - 0.2 / 6))) < 1e-6
    c = np.full((2, 5, 6), -1.5)
    assert np.max(np.abs(ob.tv_prox(c, 0.7, 50, method="chambolle") - c)) < 1e-12
    rng = np.random.default_rng(5)
    b = rng.standard_normal((3, 6, 7))
    assert np.array_equal(ob.tv_prox(b, 0.0, method="chambolle"), b)
    assert np.max(np.abs(ob.tv_prox(b, 0.3, 30000, method="chambolle") - ob.tv_prox(b, 0.3, 5000))) < 1e-5


# --------------------------------------------------------------------------- pins added in r02
def test_im_draw_interval_kat_and_zero_tiles():
    """Algo 2 line 5: the tile is drawn with probability q_t / sum q.  The
    draw x = bounded(rnd(seed, 3, epoch, k), sum q) (the pinned sampler) selects the tile
    whose half-open interval [c_{t-1}, c_t) of the cumulative weights contains x.  Checked
    by hand-written interval tables (not a cumulative-sum loop): zero-weight tiles are never
    drawn, and a draw on an interval's upper end belongs to the NEXT tile (an off-by-one in
    the comparison, x <= c, fails here)."""
    cases = [
        # q, [(lo, hi, tile)] with x in [lo, hi) -> tile
        ([1, 0, 1], [(0, 1, 0), (1, 2, 2)]),
        ([0, 5, 0, 3], [(0, 5, 1), (5, 8, 3)]),
        ([2, 3, 0, 0, 1], [(0, 2, 0), (2, 5, 1), (5, 6, 4)]),
        ([0, 0, 7], [(0, 7, 2)]),
    ]
    for q, table in cases:
        S = sum(q)
        seen = set()
        for k in range(400):
            x = ob.bounded(ob.rnd(99, 3, 5, k), S)
            want = [t for lo, hi, t in table if lo <= x < hi]
            assert len(want) == 1
            got = ob.im_draw(99, 5, k, np.array(q, np.uint32), False)
            assert got == want[0], (q, x, got, want)
            seen.add(got)
        assert seen == {t for _, _, t in table}          # every non-zero tile occurs
    # uniform (RAN) and zero-total weights: bounded(rnd, T)
    for k in range(50):
        u = ob.rnd(7, 3, 1, k)
        assert ob.im_draw(7, 1, k, np.array([5, 0, 0, 0], np.uint32), True) == ob.bounded(u, 4)
        assert ob.im_draw(7, 1, k, np.zeros(3, np.uint32), False) == ob.bounded(u, 3)


def test_im_draw_frequencies_match_weights():
    """The draw frequencies of Algo 2's tiles match q / sum q (chi-square, 20000 draws,
    4 tiles of weights 1:2:3:10 plus a zero tile that must never occur)."""
    q = np.array([1, 2, 0, 3, 10], np.uint32) * 4096
    n = 20000
    cnt = np.zeros(len(q))
    for k in range(n):
        cnt[ob.im_draw(2024, 7, k, q, False)] += 1
    assert cnt[2] == 0
    p = q / q.sum()
    nz = p > 0
    chi2 = float(np.sum((cnt[nz] - n * p[nz]) ** 2 / (n * p[nz])))
    assert chi2 < 21.1                          # 3 dof, p ~ 1e-4


def test_power_iteration_is_spectral_norm():
    """sigma_max(A)^2 from the oracle's power iteration (it sets every mu = omega/sigma_max^2
    of the parity suite) equals the squared spectral norm of the explicitly assembled A
    (LAPACK SVD), on the paper's §III-A system and on a small cone-beam system."""
    g, grid, A, x_true, y = sec3a_system(4, 4, noise=False)
    P = Projector(g, grid)
    ref = np.linalg.norm(A, 2) ** 2
    got = ob.power_iteration(P, 300, seed=1)
    assert abs(got - ref) <= 1e-8 * ref, (got, ref)
    p = synth.scaled(synth.PRESETS["cfg3"], 12, n_views=10)
    gc = p.geometry()
    Pc = Projector(gc, BlockGrid(gc.dims, (1, 1, 2)))
    Ac = Pc.dense()
    refc = np.linalg.norm(Ac, 2) ** 2
    gotc = ob.power_iteration(Pc, 400, seed=2)
    assert abs(gotc - refc) <= 1e-6 * refc, (gotc, refc)


def test_is_off_last_switches_to_algo1_in_the_final_global_epochs():
    """"the last few iterations without importance sampling" (reading A11):
    with is_off_last = L and total_epochs = K, epochs k > K - L (1-based, global) are plain
    Algo 1 epochs.  An IM run of K epochs equals an IM run of K - L epochs continued by L
    epochs of Algo 1 from the same state, and the IM epochs before differ from Algo 1."""
    g, grid, A, x_true, y = sec3a_system(4, 4, noise=False)
    s0 = np.linalg.norm(A, 2)
    base = dict(seed=21, mu=0.5 / s0 ** 2, rows_per_epoch=1, cols_per_epoch=2)
    K, L = 9, 3
    o = ob.OracleBSGD(g, grid.blocks, 4, y, ob.Params(im=True, is_off_last=L, total_epochs=K, **base),
                      tiles=(2, 1))
    for _ in range(K):
        o.epoch()
    assert all("tiles" in r for r in o.log[:K - L]) and all("tiles" not in r for r in o.log[K - L:])
    ref = ob.OracleBSGD(g, grid.blocks, 4, y, ob.Params(im=True, **base), tiles=(2, 1))
    for _ in range(K - L):
        ref.epoch()
    ref.p = ob.Params(im=False, **base)                 # the same state, Algo 1 from here
    for _ in range(L):
        ref.epoch()
    assert np.array_equal(ref.x, o.x)
    plain = ob.OracleBSGD(g, grid.blocks, 4, y, ob.Params(**base))
    for _ in range(K):
        plain.epoch()
    assert not np.allclose(plain.x, o.x)


# --------------------------------------------------------------------------- lean Algo 1
def test_lean_algo1_gd_closed_form_and_sag():
    """OracleBSGDLean (the touched-pairs-only storage used for the 1024^3 fixture) pinned
    like the dense oracle: alpha = gamma = 1 is GD (SVD closed form) and
    gamma = 1 is SAG (independent dense SAG)."""
    M, N = 4, 2
    g, grid, A, x_true, y = sec3a_system(M, N)
    U, s, Vt = np.linalg.svd(A, full_matrices=False)
    mu = 0.5 / s[0] ** 2
    o = ob.OracleBSGDLean(g, grid.blocks, M, y.astype(np.float32),
                          ob.Params(seed=9, mu=mu, rows_per_epoch=M, cols_per_epoch=N))
    y32 = y.astype(np.float32).astype(np.float64)
    keep = s > 1e-10 * s[0]
    uy = U.T @ y32
    for k in range(1, 21):
        rec = o.epoch()
        xk = (Vt[keep].T * ((1 - (1 - 2 * mu * s[keep] ** 2) ** k) / s[keep])) @ uy[keep]
        xg = global_of(grid, o.x)
        assert np.max(np.abs(xg - xk)) <= 1e-10 * np.max(np.abs(xk))
        xprev = (Vt[keep].T * ((1 - (1 - 2 * mu * s[keep] ** 2) ** (k - 1)) / s[keep])) @ uy[keep]
        f = 0.5 * np.sum((y32 - A @ xprev) ** 2)          # r of epoch k = y - A x_{k-1}
        assert abs(rec["obj"] - f) <= 1e-9 * f
    # gamma = 1: SAG over the M row blocks
    mu = 0.3 / s[0] ** 2
    o = ob.OracleBSGDLean(g, grid.blocks, M, y.astype(np.float32),
                          ob.Params(seed=4, mu=mu, rows_per_epoch=1, cols_per_epoch=N))
    rows = [o.P.rows_of(r) for r in o.rows]
    x = np.zeros(A.shape[1])
    d = [np.zeros(A.shape[1]) for _ in range(M)]
    for k in range(40):
        (i,) = ob.select(4, 1, k, M, 1)
        Ai = A[rows[i]]
        d[i] = 2 * Ai.T @ (y32[rows[i]] - Ai @ x)
        x = x + mu * sum(d)
        o.epoch()
        assert np.max(np.abs(global_of(grid, o.x) - x)) <= 1e-11 * max(1.0, np.max(np.abs(x)))


@pytest.mark.parametrize("aM,gN", [(1, 1), (2, 3)])
def test_lean_algo1_equals_dense_state(tmp_path, aM, gN):
    """Stochastic schedules (stale z and g-hat in lines 7 and 11): the lean storage gives
    the dense oracle's trajectory (selections identical; x, objective, RMSE to fp64
    rounding of the reordered norms), with g-hat file-backed as for the 1024^3 run."""
    p = synth.scaled(synth.PRESETS["cfg3"], K=24, n_views=30)
    g = p.geometry()
    vol = synth.rasterise(synth.ellipsoids_world("shepp3d", g.dims), g.dims).astype(np.float32)
    grid = BlockGrid(g.dims, p.blocks)
    P = Projector(g, grid)
    y = np.zeros(g.n_rays)
    xb = grid.to_blocks(vol.astype(np.float64))
    for j in range(grid.N):
        P.fp(np.arange(g.n_views), j, xb[j], proj=y, accumulate=True)
    y32 = y.astype(np.float32)
    prm = ob.Params(seed=6, mu=0.3 / 2.2e4, rows_per_epoch=aM, cols_per_epoch=gN)
    d = ob.OracleBSGD(g, p.blocks, p.M, y32.astype(np.float64), prm, row_seed=3, x_true=xb)
    lean = ob.OracleBSGDLean(g, p.blocks, p.M, y32, prm, row_seed=3, x_true32=grid.to_blocks(vol),
                             ghat_dir=str(tmp_path))
    for _ in range(25):
        a, b = d.epoch(), lean.epoch()
        assert (a["rows"], a["cols"]) == (b["rows"], b["cols"])
        assert abs(a["obj"] - b["obj"]) <= 1e-12 * a["obj"]
        assert abs(a["rmse"] - b["rmse"]) <= 1e-12 * a["rmse"]
    assert np.max(np.abs(d.x - lean.x)) <= 1e-13 * np.max(np.abs(d.x))


def test_unequal_slabs_gd_closed_form():
    """alpha = gamma = 1 BSGD over unequal z-slabs is still GD (the partition does not
    change the full-gradient step): SVD closed form to 1e-10; the RMSE is
    over the volume's voxels."""
    p = synth.scaled(synth.PRESETS["cfg3"], 8, n_views=12)
    g = p.geometry()
    zs = [0, 1, 4, 5, 8]
    grid = BlockGrid(g.dims, (1, 1, 4), zs)
    P = Projector(g, grid)
    A = P.dense()
    x_true = synth.rasterise(synth.ellipsoids_world("shepp3d", g.dims), g.dims)
    y = A @ x_true.ravel()
    U, s, Vt = np.linalg.svd(A, full_matrices=False)
    mu = 0.5 / s[0] ** 2
    o = ob.OracleBSGD(g, (1, 1, 4), 3, y, ob.Params(seed=2, mu=mu, rows_per_epoch=3, cols_per_epoch=4),
                      x_true=grid.to_blocks(x_true), z_splits=zs)
    keep = s > 1e-10 * s[0]
    uy = U.T @ y
    for k in range(1, 11):
        rec = o.epoch()
        xk = (Vt[keep].T * ((1 - (1 - 2 * mu * s[keep] ** 2) ** k) / s[keep])) @ uy[keep]
        xg = grid.from_blocks(o.x).ravel()
        assert np.max(np.abs(xg - xk)) <= 1e-10 * np.max(np.abs(xk))
        assert abs(rec["rmse"] - np.sqrt(np.mean((xg - x_true.ravel()) ** 2))) <= 1e-12
