"""Small end-to-end workload for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck): every kernel family of the library on a scaled cone problem -- the FP / BP
traversals (v3 + steep v2 companions, COUNT, deterministic BP), the residual, the block
update, Algo 3's reductions, the IM weights, the fused FGP TV prox (two-iteration passes,
float4 and scalar layouts), the generic TV path of non-slab grids, TV(x), the solvers, and the virtual-rank
collectives (band exchange, halos).

    compute-sanitizer --tool racecheck python tools/sanitize.py
"""
import os
import sys
import threading

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synth  # noqa: E402
import paper_1903_11874_b200 as bs  # noqa: E402


def main():
    torch.cuda.set_device(0)
    p = synth.scaled(synth.PRESETS["cfg4"], K=32, n_views=24)
    g = p.geometry()
    ells = synth.ellipsoids_world("shepp3d", g.dims)
    y = torch.from_numpy(synth.analytic_projection(g, ells).ravel().astype(np.float32)).cuda()
    for blocks in [(1, 1, 8), (2, 2, 2)]:
        ctx = bs.Context.from_geometry(g, blocks, p.M, kind="random", row_seed=1, tiles=p.tiles)
        x = torch.zeros(ctx.owned_count * ctx.block_voxels, device="cuda")
        ctx.run(y, x, epochs=4, mu0=1e-5, seed=1, rows_per_epoch=1, cols_per_epoch=4,
                flags=bs.TV | bs.AUTO_MU | bs.IS, lam=0.1, tv_iters=3, tv_period=2)
        ctx.run(y, x, epochs=2, mu0=1e-5, seed=2, rows_per_epoch=2, cols_per_epoch=8,
                flags=bs.DETERMINISTIC | bs.RESUME)
        ctx.run(y, x, epochs=2, mu0=1e-5, seed=3, flags=bs.SGD | bs.TV_CHAMBOLLE | bs.TV, lam=0.1, tv_iters=2)
        ctx.tv_value(x)
        ctx.visit_table()
        ctx.solve("fista", y, x, 2, 1e-5, lam=0.1, tv_iters=2)
        ctx.close()
    # unequal z-slabs (forward / back single operators share a padded scratch)
    zs = [0, 3, 9, 20, 32]
    ctx = bs.Context.from_geometry(g, (1, 1, 4), p.M, kind="random", row_seed=1, z_splits=zs)
    x = torch.zeros(ctx.owned_count * ctx.block_voxels, device="cuda")
    ctx.run(y, x, epochs=3, mu0=1e-5, seed=1, rows_per_epoch=1, cols_per_epoch=2, flags=bs.TV | bs.AUTO_MU,
            lam=0.1, tv_iters=2, tv_period=2)
    proj = torch.zeros(g.n_rays, device="cuda")
    for j in range(4):
        ctx.forward([0, 5], j, x[j * ctx.block_voxels:(j + 1) * ctx.block_voxels], proj)
    ctx.close()
    torch.cuda.synchronize()
    # two-iteration TV passes (k_tv_fgp_z2) over several 60 x 12 tiles and z-chunks, odd count
    gt = synth.Geometry(2, synth.circular("cone", 4, 360.0, 800.0, 500.0, 8, 8, 1.0, 1.0), 8, 8, (136, 30, 40))
    ctx = bs.Context.from_geometry(gt, (1, 1, 2), 1)
    xt = torch.rand(136 * 30 * 40, device="cuda")
    ctx.tv_prox(xt, 0.2, 5)
    ctx.close()
    torch.cuda.synchronize()
    # virtual ranks: band exchange + TV halos
    G = 2
    group = bs.VirtualGroup(G)
    ctxs = [bs.Context.from_geometry(g, p.blocks, p.M, kind="random", row_seed=1, rank=r, world=G, vgroup=group)
            for r in range(G)]

    def rank_main(r):
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            xr = torch.zeros(ctxs[r].owned_count * ctxs[r].block_voxels, device="cuda")
            ctxs[r].run(y, xr, epochs=3, mu0=1e-5, seed=1, rows_per_epoch=1, cols_per_epoch=4,
                        flags=bs.TV | bs.AUTO_MU, lam=0.1, tv_iters=2, tv_period=2, stream=s)
            s.synchronize()

    th = [threading.Thread(target=rank_main, args=(r,)) for r in range(G)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for c in ctxs:
        c.close()
    group.close()
    torch.cuda.synchronize()
    print("sanitize workload done")


if __name__ == "__main__":
    main()
