"""Sharded TV on non-slab block grids (the paper's "8 cubic blocks",
PAPER.md:449): with G virtual ranks on one GPU (bsgd_vgroup), every rank owning whole
z-layers of a bx x by x bz grid, BSGD-TV (Algo 4) + Algo 3 against the oracle, the TV prox
(Algo 4 line 16) and TV(x) (Eq. 6) per voxel, and the E_PARTITION contract for grids whose
ranks would own partial layers."""
import threading

import numpy as np
import pytest

from oracle import bsgd as ob
from oracle.projector import BlockGrid, Projector

from _problems import problem

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def bs():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1903_11874_b200 as m
    return m


def _ranks(bs, G, fn):
    """Run fn(r, stream) on G threads (one per virtual rank); re-raise the first error."""
    out, errs = [None] * G, []

    def main(r):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                out[r] = fn(r, s)
                s.synchronize()
        except Exception as e:          # noqa: BLE001 -- surfaced below
            errs.append(e)

    th = [threading.Thread(target=main, args=(r,)) for r in range(G)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    assert not errs, errs
    return out


@pytest.mark.parametrize("blocks,G", [((2, 2, 2), 2), ((2, 2, 4), 4), ((2, 1, 4), 2)])
def test_virtual_ranks_block_grid_tv_trajectory(bs, blocks, G):
    p, g, vol32, y = problem("cfg3", K=48, n_views=40)
    P = Projector(g, BlockGrid(g.dims, blocks))
    mu = float(np.float32(2.0 / ob.power_iteration(P, 30, seed=1)))
    E, M, N = 24, p.M, P.grid.N
    xtb = P.grid.to_blocks(vol32)
    prm = ob.Params(seed=3, mu=mu, rows_per_epoch=1, cols_per_epoch=N // 2, total_epochs=E, tv=True,
                    auto_mu=True, lam=0.1, tv_period=3)
    o = ob.OracleBSGD(g, blocks, M, y.astype(np.float64), prm, row_kind="random", row_seed=11,
                      x_true=xtb.astype(np.float64))
    for _ in range(E):
        o.epoch()
    group = bs.VirtualGroup(G)
    ctxs = [bs.Context.from_geometry(g, blocks, M, kind="random", row_seed=11, rank=r, world=G, vgroup=group)
            for r in range(G)]
    nb = N // G

    def run(r, s):
        yd = torch.from_numpy(y).cuda()
        xd = torch.zeros(nb * P.grid.bsize, device="cuda")
        xt = torch.from_numpy(xtb[r * nb:(r + 1) * nb].ravel().copy()).cuda()
        res = ctxs[r].run(yd, xd, epochs=E, mu0=mu, seed=3, x_true=xt, rows_per_epoch=1, cols_per_epoch=N // 2,
                          flags=bs.TV | bs.AUTO_MU, lam=0.1, tv_iters=20, tv_period=3, stream=s)
        s.synchronize()
        return res, xd.cpu().numpy().astype(np.float64)

    out = _ranks(bs, G, run)
    for c in ctxs:
        c.close()
    group.close()
    res0 = out[0][0]
    for r in range(1, G):
        assert np.array_equal(out[r][0].obj, res0.obj)
        assert np.array_equal(out[r][0].mu, res0.mu)
    assert [r_["rows"] for r_ in o.log] == res0.sel_rows.tolist()
    assert [r_["cols"] for r_ in o.log] == res0.sel_cols.tolist()
    obj = np.array([r_["obj"] for r_ in o.log])
    rmse = np.array([r_["rmse"] for r_ in o.log])
    assert np.allclose(res0.mu, [r_["mu"] for r_ in o.log], rtol=1e-12)
    x = np.concatenate([out[r][1] for r in range(G)])
    e_obj = float(np.max(np.abs(res0.obj - obj) / obj))
    e_rmse = float(np.max(np.abs(res0.rmse - rmse) / rmse))
    e_x = float(np.max(np.abs(x - o.x.ravel())) / np.max(np.abs(o.x)))
    print(f"blocks {blocks} G={G}: obj {e_obj:.3g} rmse {e_rmse:.3g} x {e_x:.3g}")
    assert e_obj < 1e-3 and e_rmse < 1e-3 and e_x < 1e-2, (e_obj, e_rmse, e_x)


@pytest.mark.parametrize("blocks,G", [((2, 2, 2), 2), ((3, 2, 4), 4)])
def test_virtual_ranks_block_grid_tv_prox_and_value(bs, blocks, G):
    """bsgd_tv_prox / bsgd_tv_value with the halo planes gathered from the bx*by blocks of a
    layer: per voxel against the oracle's whole-volume FGP prox and TV(x)."""
    dims = (36, 28, 24)
    rng = np.random.default_rng(5)
    vol = rng.random((dims[2], dims[1], dims[0])).astype(np.float32)
    import synth
    vecs = synth.circular("cone", 8, 360.0, 100.0, 60.0, 40, 30, 1.4, 1.3)
    g = synth.Geometry(synth.CONE, vecs, 40, 30, dims)
    grid = BlockGrid(dims, blocks)
    xb = grid.to_blocks(vol)
    N = grid.N
    nb = N // G
    w = 0.07
    ref = ob.tv_prox(vol.astype(np.float64), w, 20)
    tv_ref = ob.tv_value(vol.astype(np.float64))
    group = bs.VirtualGroup(G)
    ctxs = [bs.Context.from_geometry(g, blocks, 2, rank=r, world=G, vgroup=group) for r in range(G)]

    def run(r, s):
        xd = torch.from_numpy(xb[r * nb:(r + 1) * nb].ravel().copy()).cuda()
        tv = ctxs[r].tv_value(xd, stream=s)
        ctxs[r].tv_prox(xd, w, 20, stream=s)
        s.synchronize()
        return tv, xd.cpu().numpy().astype(np.float64)

    out = _ranks(bs, G, run)
    for c in ctxs:
        c.close()
    group.close()
    got = grid.from_blocks(np.concatenate([o[1] for o in out]).reshape(N, -1))
    err = float(np.max(np.abs(got - ref)))
    print(f"blocks {blocks} G={G}: prox max |d| {err:.3g}, TV rel {abs(out[0][0] - tv_ref) / tv_ref:.3g}")
    assert err < 1e-5 * max(1.0, float(np.max(np.abs(ref))))
    for r in range(G):
        assert abs(out[r][0] - tv_ref) <= 1e-9 * tv_ref


def test_partial_layer_ownership_is_rejected(bs):
    """(2,2,2) over 4 ranks: each rank would own half a z-layer (cross-rank x / y neighbours):
    the TV calls fail with E_PARTITION before any device work; plain BSGD still runs."""
    import synth
    dims = (16, 16, 16)
    vecs = synth.circular("cone", 6, 360.0, 60.0, 40.0, 24, 20, 1.3, 1.3)
    g = synth.Geometry(synth.CONE, vecs, 24, 20, dims)
    G = 4
    group = bs.VirtualGroup(G)
    ctxs = [bs.Context.from_geometry(g, (2, 2, 2), 2, rank=r, world=G, vgroup=group) for r in range(G)]
    codes = []
    for c in ctxs:
        x = torch.ones(c.owned_count * c.block_voxels, device="cuda")
        with pytest.raises(bs.BsgdError) as e:
            c.tv_prox(x, 0.1, 5)
        codes.append(e.value.code)
        assert torch.all(x == 1.0)
    assert codes == [2] * G                      # BSGD_E_PARTITION
    for c in ctxs:
        c.close()
    group.close()


@pytest.mark.parametrize("G", [2, 4, 8])
def test_band_exchange_matches_oracle_and_full_allreduce(bs, G, monkeypatch):
    """N2: the residual formed from the peers' partial sums on overlapping
    detector bands only (default for world > 1) reproduces the oracle's Algo 1 + Algo 3
    trajectory, and the full-allreduce mode (BSGD_EXCHANGE=full), on G virtual ranks of a
    scaled cfg5-shaped cone problem (8 z-slabs); it sends >= 4x fewer bytes.  LSA mode
    (BSGD_EXCHANGE=lsa): the residual kernel reads the same overlap rows straight from the
    peers' partial-sum buffers (here the other virtual ranks' buffers on the same device)."""
    p, g, vol32, y = problem("cfg5", K=64, n_views=36)
    P = Projector(g, BlockGrid(g.dims, p.blocks))
    mu = float(np.float32(1.5 / ob.power_iteration(P, 20, seed=1)))
    E = 20
    xtb = P.grid.to_blocks(vol32)
    prm = ob.Params(seed=3, mu=mu, rows_per_epoch=1, cols_per_epoch=8, total_epochs=E, auto_mu=True)
    o = ob.OracleBSGD(g, p.blocks, p.M, y.astype(np.float64), prm, row_kind="random", row_seed=11,
                      x_true=xtb.astype(np.float64))
    for _ in range(E):
        o.epoch()
    nb = p.N // G
    runs = {}
    for mode in ("band", "full", "lsa"):
        monkeypatch.setenv("BSGD_EXCHANGE", mode)
        group = bs.VirtualGroup(G)
        ctxs = [bs.Context.from_geometry(g, p.blocks, p.M, kind="random", row_seed=11, rank=r, world=G,
                                         vgroup=group) for r in range(G)]

        def run(r, s):
            yd = torch.from_numpy(y).cuda()
            xd = torch.zeros(nb * P.grid.bsize, device="cuda")
            xt = torch.from_numpy(xtb[r * nb:(r + 1) * nb].ravel().copy()).cuda()
            res = ctxs[r].run(yd, xd, epochs=E, mu0=mu, seed=3, x_true=xt, rows_per_epoch=1, cols_per_epoch=8,
                              flags=bs.AUTO_MU, stream=s)
            s.synchronize()
            return res, xd.cpu().numpy().astype(np.float64), ctxs[r].comm_stats()

        out = _ranks(bs, G, run)
        # the host plan (bsgd_exchange_plan) predicts the bytes the ranks sent
        plan = 0
        for e in range(E):
            views = [v for i in out[0][0].sel_rows[e] for v in ctxs[0].row_block_views(int(i))]
            pl = ctxs[0].exchange_plan(G, views)
            plan += pl["full_bytes"] if mode == "full" else pl["band_bytes"]   # lsa reads what band sends
        for c in ctxs:
            c.close()
        group.close()
        assert all(o_[2]["mode"] == mode for o_ in out)
        assert abs(sum(o_[2]["bytes_sent"] for o_ in out) - plan) <= 8 * G * E, (mode, plan)
        for r in range(1, G):
            assert np.array_equal(out[r][0].obj, out[0][0].obj)
            assert np.array_equal(out[r][0].mu, out[0][0].mu)
        runs[mode] = out
    for mode, out in runs.items():
        res0 = out[0][0]
        x = np.concatenate([o_[1] for o_ in out])
        obj = np.array([r_["obj"] for r_ in o.log])
        rmse = np.array([r_["rmse"] for r_ in o.log])
        assert [r_["cols"] for r_ in o.log] == res0.sel_cols.tolist()
        assert np.allclose(res0.mu, [r_["mu"] for r_ in o.log], rtol=1e-12)
        e_obj = float(np.max(np.abs(res0.obj - obj) / obj))
        e_rmse = float(np.max(np.abs(res0.rmse - rmse) / rmse))
        e_x = float(np.max(np.abs(x - o.x.ravel())) / np.max(np.abs(o.x)))
        sent = sum(o_[2]["bytes_sent"] for o_ in out)
        print(f"G={G} {mode}: obj {e_obj:.3g} rmse {e_rmse:.3g} x {e_x:.3g}; sent {sent / 1e6:.2f} MB")
        assert e_obj < 1e-3 and e_rmse < 1e-3 and e_x < 1e-2, (mode, e_obj, e_rmse, e_x)
    band = sum(o_[2]["bytes_sent"] for o_ in runs["band"])
    full = sum(o_[2]["bytes_sent"] for o_ in runs["full"])
    assert 0 < band and 4 * band <= full, (band, full)
    assert sum(o_[2]["bytes_sent"] for o_ in runs["lsa"]) == band      # the same overlap rows, read in place


# ----------------------------------------------------------------- unequal z-slabs (N3)
def _zs_problem(K=48, n_views=40):
    return problem("cfg4", K=K, n_views=n_views)


def test_unequal_slabs_operator_parity(bs):
    """FP per ray / BP per voxel on unequal z-slabs (bsgd_create_ex z_splits) against the
    oracle's operators on the same slabs (thin, thick and one-plane slabs)."""
    p, g, vol32, y = _zs_problem()
    zs = [0, 5, 6, 20, 33, 48]
    grid = BlockGrid(g.dims, (1, 1, 5), zs)
    P = Projector(g, grid)
    ctx = bs.Context.from_geometry(g, (1, 1, 5), 2, z_splits=zs)
    assert [ctx.block_box(j) for j in range(5)] == [((0, 0, zs[j]), (48, 48, zs[j + 1])) for j in range(5)]
    assert ctx.block_voxels == grid.bsize
    rng = np.random.default_rng(4)
    views = np.arange(0, 40, 3)
    rows = P.rows_of(views)
    for j in range(5):
        x = (rng.random(grid.bsize) * grid.mask()[j]).astype(np.float32)
        proj = torch.zeros(g.n_rays, device="cuda")
        ctx.forward(views, j, torch.from_numpy(x).cuda(), proj)
        got = proj.cpu().numpy().astype(np.float64)[rows]
        ref = P.fp(views, j, x.astype(np.float64))[rows]
        assert np.all(np.abs(got - ref) <= 1e-5 * ref + 1e-7 * float(x.max())), j
        r = np.zeros(g.n_rays, dtype=np.float32)
        r[rows] = rng.standard_normal(len(rows)).astype(np.float32)
        gb = torch.zeros(grid.bsize, device="cuda")
        ctx.back(views, j, torch.from_numpy(r).cuda(), gb, scale=1.0)
        gg = gb.cpu().numpy().astype(np.float64)
        gref = P.bp(views, j, r.astype(np.float64))
        gabs = P.bp(views, j, np.abs(r).astype(np.float64))
        assert np.all(np.abs(gg - gref) <= 1e-5 * gabs + 1e-7 * float(np.abs(r).max())), j
        assert np.all(gg[grid.bsizes[j]:] == 0.0)                  # nothing in the row's tail
    ctx.close()


@pytest.mark.parametrize("G", [1, 2])
def test_unequal_slabs_trajectory(bs, G):
    """BSGD-TV (Algo 4) + Algo 3 + IM (Algo 2) on unequal z-slabs vs the oracle on the same
    partition, on one rank and on 2 virtual ranks (band exchange, TV halos of the packed
    owned planes)."""
    p, g, vol32, y = _zs_problem()
    zs = [0, 7, 15, 22, 26, 31, 36, 41, 48]
    grid = BlockGrid(g.dims, (1, 1, 8), zs)
    P = Projector(g, grid)
    mu = float(np.float32(2.0 / ob.power_iteration(P, 30, seed=1)))
    E = 24
    xtb = grid.to_blocks(vol32)
    prm = ob.Params(seed=3, mu=mu, rows_per_epoch=1, cols_per_epoch=3, total_epochs=E, tv=True, auto_mu=True,
                    lam=0.1, tv_period=3, im=True)
    o = ob.OracleBSGD(g, (1, 1, 8), p.M, y.astype(np.float64), prm, row_kind="random", row_seed=11,
                      tiles=p.tiles, x_true=xtb.astype(np.float64), z_splits=zs)
    for _ in range(E):
        o.epoch()
    group = bs.VirtualGroup(G) if G > 1 else None
    ctxs = [bs.Context.from_geometry(g, (1, 1, 8), p.M, kind="random", row_seed=11, tiles=p.tiles, rank=r, world=G,
                                     vgroup=group, z_splits=zs) for r in range(G)]
    nb = 8 // G

    def run(r, s):
        yd = torch.from_numpy(y).cuda()
        xd = torch.zeros(nb * grid.bsize, device="cuda")
        xt = torch.from_numpy(xtb[r * nb:(r + 1) * nb].ravel().copy()).cuda()
        res = ctxs[r].run(yd, xd, epochs=E, mu0=mu, seed=3, x_true=xt, rows_per_epoch=1, cols_per_epoch=3,
                          flags=bs.TV | bs.AUTO_MU | bs.IS, lam=0.1, tv_iters=20, tv_period=3, stream=s)
        s.synchronize()
        return res, xd.cpu().numpy().astype(np.float64)

    out = _ranks(bs, G, run)
    for c in ctxs:
        c.close()
    if group:
        group.close()
    res0 = out[0][0]
    assert [r_["cols"] for r_ in o.log] == res0.sel_cols.tolist()
    obj = np.array([r_["obj"] for r_ in o.log])
    rmse = np.array([r_["rmse"] for r_ in o.log])
    assert np.allclose(res0.mu, [r_["mu"] for r_ in o.log], rtol=1e-12)
    x = np.concatenate([o_[1] for o_ in out]).reshape(8, -1)
    assert np.all(x * (1 - grid.mask()) == 0)                      # tails untouched
    e_obj = float(np.max(np.abs(res0.obj - obj) / obj))
    e_rmse = float(np.max(np.abs(res0.rmse - rmse) / rmse))
    e_x = float(np.max(np.abs(x - o.x)) / np.max(np.abs(o.x)))
    print(f"unequal slabs G={G}: obj {e_obj:.3g} rmse {e_rmse:.3g} x {e_x:.3g}")
    assert e_obj < 1e-3 and e_rmse < 1e-3 and e_x < 1e-2, (e_obj, e_rmse, e_x)


def test_balanced_z_splits(bs):
    """bsgd_balanced_z_splits: from a one-plane-slab context's exact visit table, 8 slabs
    whose visit counts (measured again by the COUNT traversal of the balanced context) are
    equal up to the split granularity (each boundary within half a plane's visits of its
    target: spread <= two planes' share), and closer than equal-thickness slabs.  (At cfg5's
    full size, 4-plane candidates, the bench's `balance` object measures 1.7 %.)"""
    p, g, vol32, y = problem("cfg5", K=64, n_views=36)
    fine = bs.Context.from_geometry(g, (1, 1, 64), 1)
    zs = fine.balanced_z_splits(8)
    vt = fine.visit_table().sum(axis=(1, 2)).astype(np.float64)     # visits per plane
    fine.close()
    assert zs[0] == 0 and zs[-1] == 64 and all(b > a for a, b in zip(zs, zs[1:]))

    def spread(splits):
        ctx = bs.Context.from_geometry(g, (1, 1, 8), 1, z_splits=splits)
        v = ctx.visit_table().sum(axis=(1, 2)).astype(np.float64)
        ctx.close()
        return (v.max() - v.min()) / v.mean(), v

    s_bal, v_bal = spread(zs)
    s_eq, _ = spread(list(range(0, 65, 8)))
    gran = vt.max() / (vt.sum() / 8)                                  # one plane, relative to a slab
    print(f"balanced splits {zs}: visit spread {s_bal:.4f} (equal slabs {s_eq:.4f}; one-plane granularity {gran:.4f})")
    assert s_bal <= 2 * gran + 1e-12 and s_bal < s_eq
    # the balanced context's visits are the same planes' visits regrouped (the exact COUNT
    # traversal is additive over slabs up to boundary slivers)
    for k in range(8):
        assert abs(v_bal[k] - vt[zs[k]:zs[k + 1]].sum()) <= 2e-4 * v_bal[k]


@pytest.mark.parametrize("mode", ["im", "sgd", "stratified"])
def test_band_exchange_schedules(bs, mode):
    """The band exchange under the other epoch shapes: BSGD-IM (tile rows only; Algo 2),
    Eq. 4 SGD (every block's FP fresh) and owner-stratified columns, G = 4 virtual ranks,
    against the oracle."""
    p, g, vol32, y = problem("cfg3", K=32, n_views=30)
    P = Projector(g, BlockGrid(g.dims, p.blocks))
    mu = float(np.float32(0.5 / ob.power_iteration(P, 20, seed=1)))
    E, G = 12, 4
    xtb = P.grid.to_blocks(vol32)
    kw = {"im": dict(im=True), "sgd": dict(sgd=True), "stratified": dict(strata=G)}[mode]
    flags = {"im": bs.IS, "sgd": bs.SGD, "stratified": bs.STRATIFIED}[mode]
    gN = 4 if mode != "sgd" else 8
    prm = ob.Params(seed=3, mu=mu, rows_per_epoch=1, cols_per_epoch=gN, total_epochs=E, **kw)
    o = ob.OracleBSGD(g, p.blocks, p.M, y.astype(np.float64), prm, row_kind="random", row_seed=11,
                      tiles=p.tiles, x_true=xtb.astype(np.float64))
    for _ in range(E):
        o.epoch()
    group = bs.VirtualGroup(G)
    ctxs = [bs.Context.from_geometry(g, p.blocks, p.M, kind="random", row_seed=11, tiles=p.tiles, rank=r, world=G,
                                     vgroup=group) for r in range(G)]
    nb = p.N // G

    def run(r, s):
        yd = torch.from_numpy(y).cuda()
        xd = torch.zeros(nb * P.grid.bsize, device="cuda")
        xt = torch.from_numpy(xtb[r * nb:(r + 1) * nb].ravel().copy()).cuda()
        res = ctxs[r].run(yd, xd, epochs=E, mu0=mu, seed=3, x_true=xt, rows_per_epoch=1, cols_per_epoch=gN,
                          flags=flags, strata=G if mode == "stratified" else 0, stream=s)
        s.synchronize()
        return res, xd.cpu().numpy().astype(np.float64), ctxs[r].comm_stats()

    out = _ranks(bs, G, run)
    for c in ctxs:
        c.close()
    group.close()
    assert all(o_[2]["mode"] == "band" for o_ in out)
    res0 = out[0][0]
    obj = np.array([r_["obj"] for r_ in o.log])
    rmse = np.array([r_["rmse"] for r_ in o.log])
    x = np.concatenate([o_[1] for o_ in out])
    e_obj = float(np.max(np.abs(res0.obj - obj) / obj))
    e_rmse = float(np.max(np.abs(res0.rmse - rmse) / rmse))
    e_x = float(np.max(np.abs(x - o.x.ravel())) / np.max(np.abs(o.x)))
    print(f"band exchange {mode}: obj {e_obj:.3g} rmse {e_rmse:.3g} x {e_x:.3g}")
    assert e_obj < 1e-3 and e_rmse < 1e-3 and e_x < 1e-2, (e_obj, e_rmse, e_x)


def test_unequal_slabs_other_paths(bs):
    """Unequal z-slabs through the remaining entry points: a host-buffer run equals the device
    run (per-block uploads / downloads of the thinner slabs' rows); deterministic BP runs are
    bit-identical; LOG_TRUE_OBJ's fresh A x and the seen-voxel RMSE match the oracle; and a
    full-gradient solver (FISTA-TV) gives the same iterates as on equal slabs (the partition
    does not change a full-gradient method)."""
    p, g, vol32, y = _zs_problem(K=32, n_views=30)
    zs = [0, 3, 7, 12, 16, 19, 24, 27, 32]
    grid = BlockGrid(g.dims, (1, 1, 8), zs)
    P = Projector(g, grid)
    mu = float(np.float32(1.0 / ob.power_iteration(P, 20, seed=1)))
    xtb = grid.to_blocks(vol32)
    # host buffers vs device buffers
    outs = []
    for host in (False, True):
        ctx = bs.Context.from_geometry(g, (1, 1, 8), p.M, kind="random", row_seed=2, z_splits=zs)
        if host:
            yh, xh = torch.from_numpy(y.copy()).pin_memory(), torch.zeros(8 * grid.bsize).pin_memory()
            res = ctx.run(yh, xh, epochs=10, mu0=mu, seed=4, rows_per_epoch=1, cols_per_epoch=3, flags=bs.AUTO_MU)
            xr = xh.numpy().copy()
        else:
            yd, xd = torch.from_numpy(y).cuda(), torch.zeros(8 * grid.bsize, device="cuda")
            res = ctx.run(yd, xd, epochs=10, mu0=mu, seed=4, rows_per_epoch=1, cols_per_epoch=3, flags=bs.AUTO_MU)
            xr = xd.cpu().numpy()
        outs.append((res.obj.copy(), res.mu.copy(), xr))
        ctx.close()
    assert np.array_equal(outs[0][1], outs[1][1]) and np.allclose(outs[0][0], outs[1][0], rtol=1e-5)
    assert np.max(np.abs(outs[0][2] - outs[1][2])) <= 1e-4 * np.max(np.abs(outs[0][2]))
    assert np.all(outs[1][2].reshape(8, -1) * (1 - grid.mask()) == 0)
    # deterministic BP: two runs bit-identical
    xs = []
    for _ in range(2):
        ctx = bs.Context.from_geometry(g, (1, 1, 8), p.M, kind="random", row_seed=2, z_splits=zs)
        xd = torch.zeros(8 * grid.bsize, device="cuda")
        ctx.run(torch.from_numpy(y).cuda(), xd, epochs=6, mu0=mu, seed=4, rows_per_epoch=1, cols_per_epoch=3,
                flags=bs.DETERMINISTIC)
        xs.append(xd.cpu().numpy())
        ctx.close()
    assert np.array_equal(xs[0], xs[1])
    # LOG_TRUE_OBJ: 1/2 |y - A x_k|^2 after each epoch vs the oracle
    prm = ob.Params(seed=4, mu=mu, rows_per_epoch=1, cols_per_epoch=3)
    o = ob.OracleBSGD(g, (1, 1, 8), p.M, y.astype(np.float64), prm, row_kind="random", row_seed=2, z_splits=zs)
    want = []
    for _ in range(4):
        o.epoch()
        want.append(o.true_objective())
    ctx = bs.Context.from_geometry(g, (1, 1, 8), p.M, kind="random", row_seed=2, z_splits=zs)
    xd = torch.zeros(8 * grid.bsize, device="cuda")
    res = ctx.run(torch.from_numpy(y).cuda(), xd, epochs=4, mu0=mu, seed=4, rows_per_epoch=1, cols_per_epoch=3,
                  flags=bs.LOG_TRUE_OBJ, x_true=torch.from_numpy(xtb.ravel().copy()).cuda())
    ctx.close()
    assert np.max(np.abs(res.obj_true - want) / np.array(want)) < 1e-5, (res.obj_true, want)
    # FISTA-TV: the same iterates over unequal slabs as over equal ones
    xs = []
    for split in (zs, None):
        ctx = bs.Context.from_geometry(g, (1, 1, 8), p.M, z_splits=split)
        gb = BlockGrid(g.dims, (1, 1, 8), split)
        xd = torch.zeros(8 * gb.bsize, device="cuda")
        obj, _ = ctx.solve("fista", torch.from_numpy(y).cuda(), xd, 8, mu, lam=0.05, tv_iters=10)
        xs.append((obj, gb.from_blocks(xd.cpu().numpy().reshape(8, -1))))
        ctx.close()
    assert np.allclose(xs[0][0], xs[1][0], rtol=1e-5)
    assert np.max(np.abs(xs[0][1] - xs[1][1])) <= 1e-4 * np.max(np.abs(xs[1][1]))
