"""ORACLE — test infrastructure.  The comparison solvers of the paper's §III
(GD, GD-BB, ISTA, FISTA, SVRG), written
as the textbook algorithms the paper cites, in fp64, over a generic operator.
Never imported by the product path.

The paper gives no listing for these methods, only their citations, so each
function follows the cited algorithm in the notation of this project (reading A1:
the objective is F(x) = ||y - A x||^2 in the update rules, with the negative
gradient g(x) = 2 A^T (y - A x), exactly the BP of Algo 1 line 9; the logs report
1/2 ||y - A x||^2 like the BSGD logs):

* GD (Fig. 12, 506 Fig. 18):          x+ = x + mu g(x)
* GD-BB, Barzilai & Borwein 1988:    mu_k = <s,s>/<s,w>,
      s = x_k - x_{k-1}, w = g(x_{k-1}) - g(x_k)  (the "BB1" long step); mu_0 given,
      and mu_k = mu_{k-1} whenever <s,w> <= 0
* ISTA, Combettes & Wajs 2005:       x+ = prox_{mu lam TV}(x + mu g(x))
* FISTA, Beck & Teboulle 2009:       z+ = prox_{mu lam TV}(v + mu g(v)),
      t+ = (1 + sqrt(1 + 4 t^2)) / 2,  v+ = z+ + ((t - 1)/t+)(z+ - z),  t_0 = 1, v_0 = x_0
* SVRG, Johnson & Zhang 2013, over the M row blocks
  F = sum_i F_i, F_i = ||y_I - A_I x||^2: each outer iteration takes the snapshot
  x~ = x and G~ = g(x~); each of its m inner steps draws one row block i uniformly and
  moves x <- x - mu (M (grad F_i(x) - grad F_i(x~)) + grad F(x~))
          = x - mu M h + mu G~,   h = 2 A_I^T A_I (x - x~).

The prox is the FGP TV prox of Algo 4 (`bsgd.tv_prox`, reading A16) with weight
mu * lam on the image as a volume; lam = 0 makes it the identity.  The row-block
draws of SVRG use the project's counter RNG (`bsgd.select`, stream 1 = rows, the
counter being the global inner-step index), as the GPU engine does.
"""
from __future__ import annotations

import math

import numpy as np

from . import bsgd as ob
from .projector import BlockGrid, Projector


class DenseOperator:
    """A dense matrix with a row partition (for the closed-form pins)."""

    def __init__(self, A: np.ndarray, row_sets, vol_shape=None):
        self.A = np.asarray(A, dtype=np.float64)
        self.row_sets = [np.asarray(r, dtype=np.int64) for r in row_sets]
        self.M = len(self.row_sets)
        self.vol_shape = vol_shape if vol_shape is not None else (1, 1, self.A.shape[1])

    def fp(self, x, rows=None):
        if rows is None:
            return self.A @ x
        out = np.zeros(self.A.shape[0])
        for i in rows:
            out[self.row_sets[i]] = self.A[self.row_sets[i]] @ x
        return out

    def bp(self, r, rows=None):
        if rows is None:
            return self.A.T @ r
        out = np.zeros(self.A.shape[1])
        for i in rows:
            out += self.A[self.row_sets[i]].T @ r[self.row_sets[i]]
        return out

    def to_volume(self, x):
        return x.reshape(self.vol_shape)

    def from_volume(self, v):
        return v.ravel()


class ProjectorOperator:
    """The CT operator: Siddon blocks (oracle/projector.py) with the view partition of
    the engine (bsgd.view_partition, reading A5).  Images are block-major vectors."""

    def __init__(self, geom, blocks, M, row_kind="random", row_seed=1):
        self.grid = BlockGrid(geom.dims, blocks)
        self.P = Projector(geom, self.grid)
        self.geom = geom
        self.rows = ob.view_partition(geom.n_views, M, row_kind, row_seed)
        self.M = M

    def _views(self, rows):
        if rows is None:
            return np.arange(self.geom.n_views)
        return np.array(sorted(v for i in rows for v in self.rows[i]), dtype=np.int64)

    def fp(self, x, rows=None):
        views = self._views(rows)
        xb = np.asarray(x, dtype=np.float64).reshape(self.grid.N, -1)
        out = np.zeros(self.geom.n_rays)
        for j in range(self.grid.N):
            self.P.fp(views, j, xb[j], proj=out, accumulate=True)
        return out

    def bp(self, r, rows=None):
        views = self._views(rows)
        mask = np.zeros(self.geom.n_rays)
        mask[self.P.rows_of(views)] = 1.0
        rr = np.asarray(r, dtype=np.float64) * mask
        return np.concatenate([self.P.bp(views, j, rr) for j in range(self.grid.N)])

    def to_volume(self, x):
        return self.grid.from_blocks(np.asarray(x).reshape(self.grid.N, -1))

    def from_volume(self, v):
        return self.grid.to_blocks(v).ravel()


def _neg_grad(op, y, x):
    """g(x) = 2 A^T (y - A x) and 1/2 ||y - A x||^2 (reading A1)."""
    r = y - op.fp(x)
    return 2.0 * op.bp(r), 0.5 * float(r @ r)


def _prox(op, x, w, tv_iters):
    if w == 0.0:
        return x.copy()
    return op.from_volume(ob.tv_prox(op.to_volume(x), w, tv_iters))


def gd(op, y, x0, mu, iters):
    x = np.array(x0, dtype=np.float64)
    log = []
    for _ in range(iters):
        g, f = _neg_grad(op, y, x)
        log.append({"obj": f, "mu": mu})
        x = x + mu * g
    return x, log


def gd_bb(op, y, x0, mu0, iters):
    x = np.array(x0, dtype=np.float64)
    mu = float(mu0)
    x_prev = g_prev = None
    log = []
    for _ in range(iters):
        g, f = _neg_grad(op, y, x)
        if x_prev is not None:
            s = x - x_prev
            w = g_prev - g
            sw = float(s @ w)
            if sw > 0.0:
                mu = float(s @ s) / sw
        log.append({"obj": f, "mu": mu})
        x_prev, g_prev = x, g
        x = x + mu * g
    return x, log


def ista(op, y, x0, mu, lam, iters, tv_iters=20):
    x = np.array(x0, dtype=np.float64)
    log = []
    for _ in range(iters):
        g, f = _neg_grad(op, y, x)
        log.append({"obj": f, "mu": mu})
        x = _prox(op, x + mu * g, mu * lam, tv_iters)
    return x, log


def fista(op, y, x0, mu, lam, iters, tv_iters=20):
    z = np.array(x0, dtype=np.float64)
    v = z.copy()
    t = 1.0
    log = []
    for _ in range(iters):
        g, f = _neg_grad(op, y, v)
        log.append({"obj": f, "mu": mu})
        z_new = _prox(op, v + mu * g, mu * lam, tv_iters)
        t_new = (1.0 + math.sqrt(1.0 + 4.0 * t * t)) / 2.0
        v = z_new + ((t - 1.0) / t_new) * (z_new - z)
        z, t = z_new, t_new
    return z, log


def svrg(op, y, x0, mu, outer, m, seed=1):
    x = np.array(x0, dtype=np.float64)
    M = op.M
    log = []
    step = 0
    for _ in range(outer):
        xs = x.copy()
        G, f = _neg_grad(op, y, xs)
        log.append({"obj": f, "mu": mu})
        for _ in range(m):
            i = ob.select(seed, 1, step, M, 1)[0]
            d = x - xs
            h = 2.0 * op.bp(op.fp(d, [i]), [i])
            x = x - mu * M * h + mu * G
            step += 1
    return x, log
