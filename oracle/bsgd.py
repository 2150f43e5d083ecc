"""ORACLE — test infrastructure.  BSGD and its variants, step by step in the
paper's order and notation, in fp64.  Never imported by the product path.

Every function cites the passage it follows (PAPER.md line numbers, section,
algorithm / equation).  Readings of silent or ambiguous passages are the
SURVEY §8c A-numbers, listed again in DESIGN.md §"Readings".

Parity pins: see tests/test_oracle_*.py and DESIGN.md §"Oracle pins".
"""
from __future__ import annotations

import math
import os
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from .projector import BlockGrid, Projector

MASK64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15


# ----------------------------------------------------------------------------
# Random selection (Algo 1 line 3 "randomly select alpha M row
# blocks ... and gamma N column blocks"; reading A3: uniform without
# replacement, fresh each epoch; the generator is the counter-based SplitMix64
# of SURVEY §8c "RNG and sampling spec", implemented here independently).
# ----------------------------------------------------------------------------
def mix64(z: int) -> int:
    """SplitMix64 output finaliser (Steele, Lea, Flood 2014)."""
    z &= MASK64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    return z ^ (z >> 31)


def rnd(seed: int, stream: int, epoch: int, k: int) -> int:
    """rnd = mix64(seed + (ctr + 1) * golden), ctr = stream<<48 | epoch<<24 | k."""
    ctr = (stream << 48) | (epoch << 24) | k
    return mix64((seed + (ctr + 1) * GOLDEN) & MASK64)


def bounded(u: int, n: int) -> int:
    """Multiply-shift map of a 64-bit draw to [0, n): ((u >> 32) * n) >> 32."""
    return ((u >> 32) * n) >> 32


def select(seed: int, stream: int, epoch: int, n: int, m: int) -> list[int]:
    """m of n without replacement: partial Fisher-Yates on the identity, sorted."""
    a = list(range(n))
    for i in range(m):
        j = i + bounded(rnd(seed, stream, epoch, i), n - i)
        a[i], a[j] = a[j], a[i]
    return sorted(a[:m])


def select_stratified(seed: int, epoch: int, n: int, m: int, strata: int) -> list[int]:
    """Column blocks drawn per owner stratum (reading A31): blocks
    [s n/S, (s+1) n/S) form stratum s; m/S of them are drawn by partial Fisher-Yates
    with draws rnd(seed, 2, epoch, s n/S + i); strata concatenated in order (sorted)."""
    if strata < 1 or n % strata or m % strata:
        raise ValueError("strata must divide n and m")
    ns, ms = n // strata, m // strata
    out = []
    for s in range(strata):
        a = list(range(ns))
        for i in range(ms):
            j = i + bounded(rnd(seed, 2, epoch, s * ns + i), ns - i)
            a[i], a[j] = a[j], a[i]
        out += [s * ns + v for v in sorted(a[:ms])]
    return out


def permutation(seed: int, stream: int, epoch: int, n: int) -> list[int]:
    """Full Fisher-Yates permutation (unsorted) with the same draws as select()."""
    a = list(range(n))
    for i in range(n):
        j = i + bounded(rnd(seed, stream, epoch, i), n - i)
        a[i], a[j] = a[j], a[i]
    return a


# ----------------------------------------------------------------------------
# Partitions
# ----------------------------------------------------------------------------
def view_partition(n_views: int, M: int, kind: str = "random", seed: int = 0) -> list[list[int]]:
    """Row blocks I_i as sets of whole views ("randomly partitioned
    the 360 projections into 5 groups"; reading A5: seeded permutation (stream
    0) cut into M chunks, the first V mod M one longer; each list sorted)."""
    if not (1 <= M <= n_views):
        raise ValueError("M must be in [1, n_views]")
    if kind == "random":
        order = permutation(seed, 0, 0, n_views)
    elif kind in ("contiguous", "interleaved"):
        order = list(range(n_views))
    else:
        raise ValueError(kind)
    if kind == "interleaved":
        return [sorted(range(i, n_views, M)) for i in range(M)]
    base, extra = divmod(n_views, M)
    out, s = [], 0
    for i in range(M):
        c = base + (1 if i < extra else 0)
        out.append(sorted(order[s:s + c]))
        s += c
    return out


def eq8_counts(node_num: int, M: int, N: int) -> tuple[int, int, float, float]:
    """Eq. 8: gamma = min{1, NodeNum/N}, alpha = NodeNum/(M N gamma);
    block counts alpha*M, gamma*N rounded half up, at least 1 (reading A4)."""
    gamma = min(1.0, node_num / N)
    alpha = node_num / (M * N * gamma)
    aM = max(1, int(math.floor(alpha * M + 0.5)))
    gN = max(1, int(math.floor(gamma * N + 0.5)))
    return min(aM, M), min(gN, N), alpha, gamma


def tile_rects(nu: int, nv: int, tiles: tuple) -> list[tuple[int, int, int, int]]:
    """Sub-detector tiles (Fig. 2 `Impor`): a tiles_u x tiles_v
    grid; tile t = tv*tiles_u + tu covers [tu nu/Tu, (tu+1) nu/Tu) x [...]."""
    tu_n, tv_n = tiles
    out = []
    for t in range(tu_n * tv_n):
        tu, tv = t % tu_n, t // tu_n
        out.append((tu * nu // tu_n, (tu + 1) * nu // tu_n, tv * nv // tv_n, (tv + 1) * nv // tv_n))
    return out


IM_SCALE = 1 << 16


def im_table(proj: Projector, tiles: tuple, area: bool = False) -> np.ndarray:
    """Integer importance table q[j][view][t] ("the denser a
    sub-matrix is, the higher the probability ... computes the fraction of a
    volume block's projection area on each sub-detector"; reading A9: weight =
    L1 mass of A_{tile}^{J} = ones-pass chord sums; area=True: the number of tile
    rays crossing the block, chord > 1e-6 — the "projection area" reading, IS_AREA).
    q = floor(2^16 w/sum w)."""
    N, V = proj.grid.N, proj.g.n_views
    T = tiles[0] * tiles[1]
    q = np.zeros((N, V, T), dtype=np.uint32)
    views = np.arange(V)
    for j in range(N):
        w = proj.tile_mass(views, j, tiles, area)
        s = w.sum(axis=1, keepdims=True)
        with np.errstate(invalid="ignore", divide="ignore"):
            f = np.where(s > 0, np.floor(IM_SCALE * w / np.where(s > 0, s, 1.0)), 0.0)
        q[j] = f.astype(np.uint32)
    return q


def im_draw(seed: int, epoch: int, k: int, q_row: np.ndarray, uniform: bool) -> int:
    """One tile per (selected block, view) (Algo 2 line 5): by
    weight (IM) or uniformly (RAN).  Zero total weight -> uniform."""
    u = rnd(seed, 3, epoch, k)
    T = len(q_row)
    S = int(np.sum(q_row, dtype=np.int64))
    if uniform or S == 0:
        return bounded(u, T)
    x = bounded(u, S)
    c = 0
    for t in range(T):
        c += int(q_row[t])
        if x < c:
            return t
    raise AssertionError("unreachable")


# ----------------------------------------------------------------------------
# TV (Eq. 5-6) and its proximal step (Algo 4 line 16).
# ----------------------------------------------------------------------------
def tv_grad(u: np.ndarray) -> np.ndarray:
    """Backward differences per axis with a zero difference at index 0 (Eq. 6,
    PAPER.md:224-227; 3D adds the third difference).  u: (nz, ny, nx) ->
    (3, nz, ny, nx) with components (x, y, z)."""
    out = np.zeros((3,) + u.shape)
    for comp, ax in ((0, 2), (1, 1), (2, 0)):
        sl_hi = [slice(None)] * 3
        sl_lo = [slice(None)] * 3
        sl_hi[ax] = slice(1, None)
        sl_lo[ax] = slice(None, -1)
        out[comp][tuple(sl_hi)] = u[tuple(sl_hi)] - u[tuple(sl_lo)]
    return out


def tv_grad_T(p: np.ndarray) -> np.ndarray:
    """Adjoint of tv_grad: (grad^T p)_i = sum_a p_a,i [i_a >= 1] - p_a,i+e_a [i_a + 1 <= n_a - 1]."""
    out = np.zeros(p.shape[1:])
    for comp, ax in ((0, 2), (1, 1), (2, 0)):
        sl_hi = [slice(None)] * 3
        sl_lo = [slice(None)] * 3
        sl_hi[ax] = slice(1, None)
        sl_lo[ax] = slice(None, -1)
        out[tuple(sl_hi)] += p[comp][tuple(sl_hi)]
        out[tuple(sl_lo)] -= p[comp][tuple(sl_hi)]
    return out


def tv_value(u: np.ndarray) -> float:
    """TV(u) = sum_i |(grad u)_i|_2 (isotropic, Eq. 6)."""
    g = tv_grad(u)
    return float(np.sum(np.sqrt(np.sum(g * g, axis=0))))


def tv_prox(b: np.ndarray, w: float, iters: int = 20, method: str = "fgp") -> np.ndarray:
    """argmin_t 1/2|t - b|^2 + w TV(t)  (Algo 4 line 16 with w = mu*lambda:
    argmin |t-x|^2 + 2 mu lambda TV(t)), by FGP (Beck & Teboulle
    2009) on the dual: p in unit balls, t = b - w grad^T p; cold start p = q = 0,
    s_1 = 1; L = 4 * (number of axes with extent > 1); reading A16."""
    b = np.asarray(b, dtype=np.float64)
    if w == 0.0:
        return b.copy()
    L = 4.0 * sum(1 for n in b.shape if n > 1)
    if method == "chambolle":
        return _tv_prox_chambolle(b, w, iters, L)
    p = np.zeros((3,) + b.shape)
    q = np.zeros_like(p)
    s = 1.0
    for _ in range(iters):
        u = b - w * tv_grad_T(q)
        pn = q + tv_grad(u) / (L * w)
        nrm = np.sqrt(np.sum(pn * pn, axis=0))
        pn /= np.maximum(1.0, nrm)
        s_new = (1.0 + math.sqrt(1.0 + 4.0 * s * s)) / 2.0
        q = pn + ((s - 1.0) / s_new) * (pn - p)
        p = pn
        s = s_new
    return b - w * tv_grad_T(p)


def _tv_prox_chambolle(b, w, iters, L):
    """Chambolle (2004) semi-implicit dual iteration, the flag of SURVEY §8c step 7: with
    tau = 1/L (1/8 in 2D, 1/12 in 3D) and p_0 = 0,
        u = b - w grad^T p;   p <- (p + tau grad(u) / w) / (1 + tau |grad(u)| / w)
    (Chambolle's p with the sign of div = -grad^T folded in); result b - w grad^T p."""
    tau = 1.0 / L
    p = np.zeros((3,) + b.shape)
    for _ in range(iters):
        gu = tv_grad(b - w * tv_grad_T(p)) * (tau / w)
        p = (p + gu) / (1.0 + np.sqrt(np.sum(gu * gu, axis=0)))
    return b - w * tv_grad_T(p)


# ----------------------------------------------------------------------------
# Algo 3 decision (PAPER.md:189-211 `cre1`), as a pure function.
# ----------------------------------------------------------------------------
def auto_mu_decision(mu: float, r_k: float, r_kM: float, r_k2M: float,
                     theta: Optional[float], theta_prev: Optional[float],
                     eps: float, delta: float, t1: float, t2: float) -> float:
    """Lines 5-12 of Algo 3.  Strict inequalities as printed; criterion 2 terms
    with an undefined theta are false (reading A14)."""
    if r_k < r_kM < r_k2M:                      # line 5
        mu = (1.0 + eps) * mu                   # line 6
    if r_k > r_kM > r_k2M:                      # line 8 (criterion 1)
        c2 = False                              # line 9 (criterion 2)
        if theta is not None:
            if theta_prev is not None and abs(theta - theta_prev) > t1:
                c2 = True
            if theta < t2:
                c2 = True
        if c2:
            mu = (1.0 - delta) * mu             # line 10
    return mu


# ----------------------------------------------------------------------------
# The solver state and one epoch.
# ----------------------------------------------------------------------------
@dataclass
class Params:
    seed: int = 1
    mu: float = 1e-4
    rows_per_epoch: int = 1          # alpha M
    cols_per_epoch: int = 1          # gamma N
    im: bool = False                 # BSGD-IM (Algo 2)
    im_uniform: bool = False         # BSGD-RAN
    im_area: bool = False            # IS_AREA weights (reading A9 alternative)
    is_off_last: int = 0             # epochs at the end run without IS
    total_epochs: int = 0            # needed for is_off_last
    auto_mu: bool = False            # Algo 3
    eps: float = 0.05
    delta: float = 0.4
    t1: float = 0.5
    t2: float = 0.0
    tv: bool = False                 # Algo 4
    lam: float = 0.1
    tv_iters: int = 20
    tv_period: int = 0               # 0 = round(1/(alpha gamma))
    tv_method: str = "fgp"           # "chambolle": the Chambolle-2004 flag
    sgd: bool = False                # Eq. 4 mini-batch SGD baseline
    strata: int = 0                  # > 0: stratified column selection


class OracleBSGD:
    """State of Algo 1: x_est, {z^j}, {g_hat^i}, g, r.

    Initial state (Algo 1 line 1): g = 0, g_hat^i = 0, z^j = 0, r = y, x_est = 0
    (or the given x0)."""

    def __init__(self, geom, blocks, M, y, params: Params, row_kind="random",
                 row_seed=None, tiles=(1, 1), x0=None, x_true=None, z_splits=None):
        self.geom = geom
        self.grid = BlockGrid(geom.dims, blocks, z_splits)
        self.P = Projector(geom, self.grid)
        self.M, self.N = M, self.grid.N
        self.p = params
        rs = params.seed if row_seed is None else row_seed
        self.rows = view_partition(geom.n_views, M, row_kind, rs)
        self.tiles = tuple(tiles)
        self.rects = tile_rects(geom.det_u, geom.det_v, self.tiles)
        self.q = im_table(self.P, self.tiles, params.im_area) if params.im and not params.im_uniform else None
        self.y = np.asarray(y, dtype=np.float64).ravel()
        nb = self.grid.bsize
        self.x = np.zeros((self.N, nb)) if x0 is None else np.array(x0, dtype=np.float64).reshape(self.N, nb)
        self.x_true = None if x_true is None else np.asarray(x_true, dtype=np.float64).reshape(self.N, nb)
        self.z = np.zeros((self.N, geom.n_rays))
        self.ghat = np.zeros((M, self.N, nb))
        self.g = np.zeros((self.N, nb))
        self.r = self.y.copy()
        self.mu = float(params.mu)
        self.k = 0
        # Algo 3 state
        self.eud_cur = np.zeros((self.N, nb))
        self.eud_prev = None
        self.theta_prev = None
        self.rnorm_hist = {0: float(np.linalg.norm(self.y))}
        self.log = []

    # -- helpers --------------------------------------------------------------
    def tv_period(self):
        if self.p.tv_period:
            return self.p.tv_period
        alpha = self.p.rows_per_epoch / self.M
        gamma = self.p.cols_per_epoch / self.N
        return max(1, int(math.floor(1.0 / (alpha * gamma) + 0.5)))      # reading A17

    def selection(self, e):
        p = self.p
        rows = select(p.seed, 1, e, self.M, p.rows_per_epoch)
        if p.sgd:
            cols = list(range(self.N))
        elif p.strata > 0:
            cols = select_stratified(p.seed, e, self.N, p.cols_per_epoch, p.strata)
        else:
            cols = select(p.seed, 2, e, self.N, p.cols_per_epoch)
        return rows, cols

    def tiles_for(self, e, rows, cols, use_im):
        """tile[j][view] for Algo 2 line 5; None when IS is off this epoch."""
        if not use_im:
            return None
        vsel = [v for i in rows for v in self.rows[i]]
        out = {}
        for cs, j in enumerate(cols):
            for vs, v in enumerate(vsel):
                qrow = None if self.q is None else self.q[j, v]
                T = len(self.rects)
                if self.p.im_uniform or qrow is None:
                    t = im_draw(self.p.seed, e, cs * len(vsel) + vs, np.ones(T, np.uint32), True)
                else:
                    t = im_draw(self.p.seed, e, cs * len(vsel) + vs, qrow, False)
                out[(j, v)] = t
        return out

    # -- one epoch ------------------------------------------------------------
    def epoch(self, rows=None, cols=None, tiles=None):
        p = self.p
        self.k += 1
        k, e = self.k, self.k - 1
        if rows is None:
            rows, cols = self.selection(e)
            use_im = p.im and not (p.is_off_last and k > p.total_epochs - p.is_off_last)
            tiles = self.tiles_for(e, rows, cols, use_im)
        # Algo 1 lines 4-6 / Algo 2 lines 4-7:  z^j_{I_i} = A_{I_i}^{J_j} x_{J_j}
        for i in rows:
            for j in cols:
                if tiles is None:
                    self.P.fp(self.rows[i], j, self.x[j], proj=self.z[j])
                else:
                    rects = [self.rects[tiles[(j, v)]] for v in self.rows[i]]
                    self.P.fp(self.rows[i], j, self.x[j], proj=self.z[j], rects=rects)
        # line 7:  r = y - sum_{j=1}^{N} z^j
        acc = np.zeros_like(self.y)
        for j in range(self.N):
            acc += self.z[j]
        self.r = self.y - acc
        # lines 8-10:  g_hat^i_{J_j} = 2 (A_{I_i}^{J_j})^T r_{I_i}   (IM: tile rows)
        if p.sgd:
            gsgd = np.zeros_like(self.g)
        for i in rows:
            for j in cols:
                if tiles is None:
                    bp = self.P.bp(self.rows[i], j, self.r)
                else:
                    rects = [self.rects[tiles[(j, v)]] for v in self.rows[i]]
                    bp = self.P.bp(self.rows[i], j, self.r, rects=rects)
                if p.sgd:
                    gsgd[j] += 2.0 * bp          # Eq. 4: g = 2 A_I^T r_I (no memory)
                else:
                    self.ghat[i, j] = 2.0 * bp
        # line 11:  g = sum_{i=1}^{M} g_hat^i
        if p.sgd:
            self.g = gsgd
        else:
            self.g = np.zeros_like(self.g)
            for i in range(self.M):
                self.g += self.ghat[i]
        # lines 12-14:  x_{J_j} += mu g_{J_j}  for the selected J_j
        for j in cols:
            self.x[j] += self.mu * self.g[j]
        mu_used = self.mu
        # Algo 4 lines 15-17: TV prox every 1/(alpha gamma) epochs
        if p.tv and k % self.tv_period() == 0:
            vol = self.grid.from_blocks(self.x)
            vol = tv_prox(vol, self.mu * p.lam, p.tv_iters, p.tv_method)
            self.x = self.grid.to_blocks(vol)
        # Algo 3 (after the epoch): EUD, theta, criteria
        if p.auto_mu:
            self._auto_mu(k)
        rec = dict(k=k, rows=list(rows), cols=list(cols), mu=mu_used,
                   obj=0.5 * float(self.r @ self.r))
        if tiles is not None:
            rec["tiles"] = dict(tiles)
        if self.x_true is not None:   # over the volume's voxels (block tails are zero in both)
            rec["rmse"] = float(np.sqrt(np.sum((self.x - self.x_true) ** 2) / self.grid.n_vox))
        self.log.append(rec)
        return rec

    def _auto_mu(self, k):
        p = self.p
        self.eud_cur += self.g                      # Algo 3 line 2: sum of g over M epochs
        if k % self.M != 0:
            return
        theta = None
        if self.eud_prev is not None:               # line 3
            na = float(np.linalg.norm(self.eud_cur))
            nb = float(np.linalg.norm(self.eud_prev))
            if na > 0 and nb > 0:
                theta = float(np.sum(self.eud_cur * self.eud_prev)) / (na * nb)
        self.rnorm_hist[k] = float(np.linalg.norm(self.r))   # reading A13: maintained r
        if k > self.M:                              # line 4
            self.mu = auto_mu_decision(self.mu, self.rnorm_hist[k], self.rnorm_hist[k - self.M],
                                       self.rnorm_hist[k - 2 * self.M], theta, self.theta_prev,
                                       p.eps, p.delta, p.t1, p.t2)
        self.theta_prev = theta
        self.eud_prev = self.eud_cur
        self.eud_cur = np.zeros_like(self.eud_cur)

    # -- metrics --------------------------------------------------------------
    def true_objective(self):
        """1/2 |y - A x|^2 (Eq. 2) with a fresh full FP."""
        ax = np.zeros_like(self.y)
        views = np.arange(self.geom.n_views)
        for j in range(self.N):
            self.P.fp(views, j, self.x[j], proj=ax, accumulate=True)
        d = self.y - ax
        return 0.5 * float(d @ d)


def snr_db(x_true, x_rec):
    """SNR of x = 20 log10(|x_true| / |x_rec - x_true|) (§III-D)."""
    return 20.0 * math.log10(np.linalg.norm(x_true) / np.linalg.norm(x_rec - x_true))


def power_iteration(P: Projector, iters: int = 50, seed: int = 0) -> float:
    """sigma_max(A)^2 by power iteration on A^T A (for mu = omega / sigma_max^2;
    with the factor-2 gradient, GD is stable iff mu < 1/sigma_max^2, reading A1)."""
    rng = np.random.default_rng(seed)
    N = P.grid.N
    v = rng.standard_normal((N, P.grid.bsize)) * P.grid.mask()
    v /= np.linalg.norm(v)
    views = np.arange(P.g.n_views)
    lam = 0.0
    for _ in range(iters):
        ax = np.zeros(P.g.n_rays)
        for j in range(N):
            P.fp(views, j, v[j], proj=ax, accumulate=True)
        w = np.zeros_like(v)
        for j in range(N):
            w[j] = P.bp(views, j, ax)
        lam = float(np.linalg.norm(w))
        v = w / lam
    return lam


class OracleBSGDLean:
    """Algo 1 exactly as OracleBSGD runs it, with storage restricted
    to what the epochs touch, for the 1024^3 configuration (where the dense state, N
    full-length z^j and M x N g-hat blocks, would need ~130 GB in fp64):

    * z^j_{I_i} is kept per touched (i, j) pair over the rays of I_i only (z^j is zero
      elsewhere: line 5 writes only rows of selected row blocks, from z = 0, line 1);
    * g-hat^i_{J_j} per touched pair (zero otherwise, line 1), optionally file-backed;
    * line 7's r = y - sum_j z^j is evaluated on the selected row blocks, the only rows
      where it changes; 1/2 |r|^2 is kept per row block (initially |y_{I_i}|^2, r = y);
    * line 11's g = sum_i g-hat^i is formed for the selected J_j, the only blocks line 13
      reads it for.
    The sums run in the dense oracle's order (j ascending, i ascending, absent terms = the
    +0.0 the dense oracle adds), so the state equals OracleBSGD's (pinned against it in
    tests/test_oracle_bsgd.py).  Plain Algo 1 only (no IM / TV / auto-mu / SGD)."""

    def __init__(self, geom, blocks, M, y32, params: Params, row_kind="random", row_seed=None,
                 x_true32=None, ghat_dir=None):
        p = params
        if p.im or p.tv or p.auto_mu or p.sgd or p.strata:
            raise ValueError("OracleBSGDLean runs plain Algo 1 only")
        self.geom = geom
        self.grid = BlockGrid(geom.dims, blocks)
        self.P = Projector(geom, self.grid)
        self.M, self.N, self.p = M, self.grid.N, p
        rs = p.seed if row_seed is None else row_seed
        self.rows = view_partition(geom.n_views, M, row_kind, rs)
        self.y = y32                                  # fp32 data, converted per row block
        self.x_true = x_true32                        # block-major fp32 (N, bsize) or None
        self.x = np.zeros((self.N, self.grid.bsize))
        self.z, self.ghat = {}, {}
        self.ghat_dir = ghat_dir
        self.scratch = np.zeros(geom.n_rays)          # full-length ray buffer for the C calls
        self.rn2 = [float(np.sum(self._y(i) ** 2)) for i in range(M)]
        self.mu = float(p.mu)
        self.k = 0
        self.log = []

    def _y(self, i):
        return np.asarray(self.y[self.P.rows_of(self.rows[i])], dtype=np.float64)

    def _new_ghat(self, key):
        if self.ghat_dir is None:
            return np.zeros(self.grid.bsize)
        fn = os.path.join(self.ghat_dir, f"ghat_{key[0]}_{key[1]}.f64")
        return np.memmap(fn, dtype=np.float64, mode="w+", shape=(self.grid.bsize,))

    def selection(self, e):
        return (select(self.p.seed, 1, e, self.M, self.p.rows_per_epoch),
                select(self.p.seed, 2, e, self.N, self.p.cols_per_epoch))

    def epoch(self):
        self.k += 1
        e = self.k - 1
        rows, cols = self.selection(e)
        # lines 4-6: z^j_{I_i} = A_{I_i}^{J_j} x_{J_j}
        for i in rows:
            ids = self.P.rows_of(self.rows[i])
            for j in cols:
                self.P.fp(self.rows[i], j, self.x[j], proj=self.scratch)
                self.z[(i, j)] = self.scratch[ids].copy()
        # line 7 on the selected row blocks: r_{I_i} = y_{I_i} - sum_{j=1}^{N} z^j_{I_i}
        r = {}
        for i in rows:
            acc = np.zeros(len(self.rows[i]) * self.geom.det_u * self.geom.det_v)
            for j in range(self.N):
                if (i, j) in self.z:
                    acc += self.z[(i, j)]
            r[i] = self._y(i) - acc
            self.rn2[i] = float(r[i] @ r[i])
        # lines 8-10: g-hat^i_{J_j} = 2 (A_{I_i}^{J_j})^T r_{I_i}
        for i in rows:
            ids = self.P.rows_of(self.rows[i])
            self.scratch[ids] = r[i]
            for j in cols:
                bp = self.P.bp(self.rows[i], j, self.scratch)
                if (i, j) not in self.ghat:
                    self.ghat[(i, j)] = self._new_ghat((i, j))
                self.ghat[(i, j)][:] = 2.0 * bp
        # lines 11-14: g_{J_j} = sum_{i=1}^{M} g-hat^i_{J_j}; x_{J_j} += mu g_{J_j}
        for j in cols:
            g = np.zeros(self.grid.bsize)
            for i in range(self.M):
                if (i, j) in self.ghat:
                    g += self.ghat[(i, j)]
            self.x[j] += self.mu * g
        rec = dict(k=self.k, rows=list(rows), cols=list(cols), mu=self.mu, obj=0.5 * float(np.sum(self.rn2)))
        if self.x_true is not None:
            s = 0.0
            for j in range(self.N):
                d = self.x[j] - self.x_true[j]
                s += float(d @ d)
            rec["rmse"] = math.sqrt(s / self.grid.n_vox)
        self.log.append(rec)
        return rec
