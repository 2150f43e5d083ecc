"""Pins of the comparison solvers (oracle/solvers.py) against closed
forms, special cases and theorems — never against a re-typing of their own update
rules.  CPU only."""
import math

import numpy as np
import pytest

from oracle import solvers as so
from oracle import bsgd as ob


def _problem(seed=0, m=30, n=12, cond=20.0):
    rng = np.random.default_rng(seed)
    U, _ = np.linalg.qr(rng.standard_normal((m, n)))
    V, _ = np.linalg.qr(rng.standard_normal((n, n)))
    sig = np.geomspace(1.0, 1.0 / cond, n)
    A = U @ np.diag(sig) @ V.T
    y = rng.standard_normal(m)
    return A, y, U, sig, V


def _gd_closed_form(U, sig, V, y, mu, k):
    """x_k = sum_i [(1 - (1 - 2 mu s_i^2)^k) / s_i] (u_i^T y) v_i  (x_0 = 0)."""
    c = (1.0 - (1.0 - 2.0 * mu * sig ** 2) ** k) / sig * (U.T @ y)
    return V @ c


def test_gd_matches_svd_closed_form():
    A, y, U, sig, V = _problem()
    op = so.DenseOperator(A, [np.arange(30)])
    mu = 0.4 / sig[0] ** 2
    x, log = so.gd(op, y, np.zeros(12), mu, 25)
    assert np.allclose(x, _gd_closed_form(U, sig, V, y, mu, 25), atol=1e-12)
    assert all(a["obj"] >= b["obj"] for a, b in zip(log, log[1:]))   # monotone (mu < 1/s_max^2)


def test_gd_bb_exact_on_scaled_orthogonal_system():
    """A^T A = c I: the BB step of iteration 1 is 1/(2c) (Newton), so x_2 = A^T y / c
    = the least-squares solution, whatever mu_0 (Barzilai & Borwein 1988)."""
    rng = np.random.default_rng(3)
    Q, _ = np.linalg.qr(rng.standard_normal((20, 7)))
    c = 3.7
    A = math.sqrt(c) * Q
    y = rng.standard_normal(20)
    op = so.DenseOperator(A, [np.arange(20)])
    x, log = so.gd_bb(op, y, np.zeros(7), 0.013, 2)
    assert np.allclose(x, A.T @ y / c, atol=1e-12)
    assert abs(log[1]["mu"] - 1.0 / (2.0 * c)) < 1e-12


def test_gd_bb_converges_to_least_squares():
    A, y, U, sig, V = _problem(seed=5, cond=10.0)
    op = so.DenseOperator(A, [np.arange(30)])
    x, _ = so.gd_bb(op, y, np.zeros(12), 0.1 / sig[0] ** 2, 200)
    x_ls = np.linalg.lstsq(A, y, rcond=None)[0]
    assert np.linalg.norm(x - x_ls) <= 1e-8 * np.linalg.norm(x_ls)


def test_ista_without_tv_is_gd():
    A, y, U, sig, V = _problem(seed=1)
    op = so.DenseOperator(A, [np.arange(30)])
    mu = 0.3 / sig[0] ** 2
    x, _ = so.ista(op, y, np.zeros(12), mu, 0.0, 15)
    assert np.allclose(x, _gd_closed_form(U, sig, V, y, mu, 15), atol=1e-12)


def test_ista_identity_operator_one_step_is_rof():
    """A = I, mu = 1/2: x_1 = prox_{lam/2 TV}(y) and x_2 = x_1 (fixed point).  On the
    8x8 step image with weight 1/2 the exact 1D-ROF levels are 1/8 and 7/8."""
    step = np.zeros((1, 8, 8))
    step[..., 4:] = 1.0
    op = so.DenseOperator(np.eye(64), [np.arange(64)], vol_shape=(1, 8, 8))
    x1, _ = so.ista(op, step.ravel(), np.zeros(64), 0.5, 1.0, 1, tv_iters=20000)
    v = x1.reshape(8, 8)
    assert np.allclose(v[:, :4], 0.125, atol=1e-9) and np.allclose(v[:, 4:], 0.875, atol=1e-9)
    x2, _ = so.ista(op, step.ravel(), x1, 0.5, 1.0, 1, tv_iters=20000)
    assert np.allclose(x2, x1, atol=1e-9)


def test_fista_rate_bound():
    """Beck & Teboulle 2009, Thm 4.4 (lam = 0, step 1/L, L = Lipschitz constant of grad F
    = 2 s_max^2):  F(z_k) - F* <= 2 L |x_0 - x*|^2 / (k + 1)^2, with F = |y - A x|^2."""
    A, y, U, sig, V = _problem(seed=2, cond=200.0)
    op = so.DenseOperator(A, [np.arange(30)])
    L = 2.0 * sig[0] ** 2
    x_ls = np.linalg.lstsq(A, y, rcond=None)[0]
    F = lambda x: float(np.sum((y - A @ x) ** 2))
    Fs = F(x_ls)
    for k in (1, 2, 5, 10, 40, 100):
        z, _ = so.fista(op, y, np.zeros(12), 1.0 / L, 0.0, k)
        assert F(z) - Fs <= 2.0 * L * float(x_ls @ x_ls) / (k + 1) ** 2 + 1e-12
    # and it is faster than GD with the same step on this ill-conditioned problem
    zg, _ = so.gd(op, y, np.zeros(12), 1.0 / L, 100)
    zf, _ = so.fista(op, y, np.zeros(12), 1.0 / L, 0.0, 100)
    assert F(zf) - Fs < F(zg) - Fs


def test_fista_first_step_is_gd_step():
    A, y, U, sig, V = _problem(seed=4)
    op = so.DenseOperator(A, [np.arange(30)])
    mu = 0.2 / sig[0] ** 2
    z, _ = so.fista(op, y, np.zeros(12), mu, 0.0, 1)
    assert np.allclose(z, _gd_closed_form(U, sig, V, y, mu, 1), atol=1e-13)


@pytest.mark.parametrize("m", [1, 3, 7])
def test_svrg_single_row_block_is_gd(m):
    """M = 1: h = 2 A^T A (x - x~) and x <- x - mu h + mu G~ = x + mu g(x): every inner
    step is a GD step, so `outer` outer iterations = outer * m GD steps."""
    A, y, U, sig, V = _problem(seed=6)
    op = so.DenseOperator(A, [np.arange(30)])
    mu = 0.3 / sig[0] ** 2
    x, _ = so.svrg(op, y, np.zeros(12), mu, 4, m)
    assert np.allclose(x, _gd_closed_form(U, sig, V, y, mu, 4 * m), atol=1e-11)


def test_svrg_converges_linearly_to_least_squares():
    """Consistent system, M = 5 row blocks: SVRG's iterates converge to x_LS (the
    variance of its gradient estimate vanishes there) with a constant step."""
    rng = np.random.default_rng(8)
    A = rng.standard_normal((40, 10))
    x_true = rng.standard_normal(10)
    y = A @ x_true
    rows = np.array_split(np.arange(40), 5)
    op = so.DenseOperator(A, rows)
    smax2 = np.linalg.norm(A, 2) ** 2
    x, log = so.svrg(op, y, np.zeros(10), 0.1 / smax2, 60, 10, seed=3)
    assert np.linalg.norm(x - x_true) <= 1e-6 * np.linalg.norm(x_true)
    objs = [r["obj"] for r in log]
    assert objs[-1] < 1e-10 * objs[0]


def test_svrg_row_draws_follow_the_sampler():
    """The inner draws are the project's counter RNG (stream 1, counter = step)."""
    draws = [ob.select(11, 1, k, 6, 1)[0] for k in range(50)]
    assert set(draws) <= set(range(6)) and len(set(draws)) == 6
