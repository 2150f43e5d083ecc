"""C-ABI contract on the GPU (include/bsgd.h; SURVEY §8b Conventions): invalid arguments are
rejected with the documented status BEFORE any device work (state unchanged), degenerate
calls are no-ops, and the context keeps working after a rejected call."""
import numpy as np
import pytest

import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

E_GEOMETRY, E_PARTITION, E_DIMENSION, E_CONTRACT = 1, 2, 3, 4


@pytest.fixture(scope="module")
def bs():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1903_11874_b200 as m
    return m


def _geom(dims=(32, 32, 32), views=8, det=(24, 24)):
    vecs = synth.circular("cone", views, 360.0, 6.0 * dims[0], 4.0 * dims[0], det[0], det[1], 2.0, 2.0)
    return synth.Geometry(synth.CONE, vecs, det[0], det[1], dims)


def test_create_rejects_bad_arguments(bs):
    g = _geom()
    cases = [(dict(blocks=(1, 1, 5), M=2), E_PARTITION),          # 32 not divisible by 5
             (dict(blocks=(1, 1, 4), M=9), E_PARTITION),          # M > n_views
             (dict(blocks=(1, 1, 4), M=2, tiles=(25, 1)), E_PARTITION)]   # more tiles than columns
    for kw, code in cases:
        blocks, M = kw.pop("blocks"), kw.pop("M")
        with pytest.raises(bs.BsgdError) as e:
            bs.Context.from_geometry(g, blocks, M, **kw)
        assert e.value.code == code, (blocks, M, kw)
    bad = synth.Geometry(synth.CONE, np.full_like(g.vecs, np.nan), 24, 24, g.dims)
    with pytest.raises(bs.BsgdError) as e:
        bs.Context.from_geometry(bad, (1, 1, 4), 2)
    assert e.value.code == E_GEOMETRY


def test_run_and_operators_reject_bad_arguments_state_unchanged(bs):
    g = _geom()
    ctx = bs.Context.from_geometry(g, (1, 1, 4), 2, kind="random", row_seed=1)
    y = torch.rand(g.n_rays, device="cuda")
    x = torch.rand(ctx.owned_count * ctx.block_voxels, device="cuda")
    x0 = x.clone()
    res0 = ctx.run(y, x, epochs=2, mu0=1e-4, seed=1, rows_per_epoch=1, cols_per_epoch=2)
    x1 = x.clone()
    r1 = ctx.get_state(3)
    bad_runs = [dict(rows_per_epoch=3, cols_per_epoch=1),                 # alpha M > M
                dict(rows_per_epoch=1, cols_per_epoch=5),                 # gamma N > N
                dict(rows_per_epoch=1, cols_per_epoch=1, flags=1 << 20),  # unknown flag
                dict(rows_per_epoch=1, cols_per_epoch=3, flags=bs.STRATIFIED, strata=2)]
    for kw in bad_runs:
        with pytest.raises(bs.BsgdError) as e:
            ctx.run(y, x, epochs=2, mu0=1e-4, seed=1, **kw)
        assert e.value.code == E_CONTRACT, kw
    with pytest.raises(bs.BsgdError) as e:
        ctx.run(y, x, epochs=1, mu0=float("nan"), seed=1, rows_per_epoch=1, cols_per_epoch=1)
    assert e.value.code == E_CONTRACT
    torch.cuda.synchronize()
    assert torch.equal(x, x1) and np.array_equal(ctx.get_state(3), r1)   # nothing ran
    # operators: view out of range, block not owned
    proj = torch.zeros(g.n_rays, device="cuda")
    with pytest.raises(bs.BsgdError) as e:
        ctx.forward([0, 99], 0, x[:ctx.block_voxels], proj)
    assert e.value.code == E_DIMENSION
    with pytest.raises(bs.BsgdError) as e:
        ctx.forward([0], 7, x[:ctx.block_voxels], proj)
    assert e.value.code == E_DIMENSION
    with pytest.raises(bs.BsgdError) as e:
        ctx.tv_prox(x, -1.0, 5)
    assert e.value.code == E_CONTRACT
    with pytest.raises(bs.BsgdError):
        ctx.set_state(3, 0, np.zeros(5, np.float32))                   # wrong byte count
    # degenerate calls are no-ops; the context still works after the rejections
    res = ctx.run(y, x, epochs=0, mu0=1e-4, seed=1, rows_per_epoch=1, cols_per_epoch=1, flags=bs.RESUME)
    assert len(res.obj) == 0 and torch.equal(x, x1)
    x.copy_(x0)
    res2 = ctx.run(y, x, epochs=2, mu0=1e-4, seed=1, rows_per_epoch=1, cols_per_epoch=2)
    assert np.allclose(res2.obj, res0.obj, rtol=1e-6) and torch.allclose(x, x1, rtol=1e-5, atol=1e-7)
    ctx.close()


def test_every_block_every_view_degenerate_schedules(bs):
    """gamma N = N and alpha M = M (full GD step per epoch), M = n_views (one view per row
    block), one block: all run and decrease the objective on consistent data."""
    g = _geom(dims=(16, 16, 16), views=6, det=(16, 16))
    for blocks, M, aM, gN in [((1, 1, 2), 6, 6, 2), ((1, 1, 1), 6, 1, 1), ((2, 2, 2), 3, 3, 8)]:
        ctx = bs.Context.from_geometry(g, blocks, M, kind="contiguous")
        xt = torch.rand(ctx.owned_count * ctx.block_voxels, device="cuda")
        y = torch.zeros(g.n_rays, device="cuda")
        for j in range(ctx.owned_count):   # y = A x_true through the library's own FP
            ctx.forward(list(range(g.n_views)), j, xt[j * ctx.block_voxels:(j + 1) * ctx.block_voxels], y,
                        accumulate=True)
        x = torch.zeros_like(xt)
        sig = ctx.power_iteration(30)
        res = ctx.run(y, x, epochs=6, mu0=0.5 / sig, seed=2, rows_per_epoch=aM, cols_per_epoch=gN)
        assert res.obj[-1] < res.obj[0], (blocks, M, res.obj)
        ctx.close()
