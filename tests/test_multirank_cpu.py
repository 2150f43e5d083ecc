"""Multi-rank host logic on CPU (gloo, world size 2): the pieces of the sharded
path that are not kernels.  Each rank uses the C-ABI host functions for its
selection and ownership, the oracle for its partial projections (stand-in for
the owned-block FP kernels), and gloo for the exchanges the engine does with
NCCL: the residual allreduce of partial sums ("ALLREDUCE") and the
z-slab halo schedule of the sharded FGP TV prox."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import synth
        import paper_1903_11874_b200 as bs
        from oracle import bsgd as ob
        from oracle.projector import BlockGrid, Projector
        out = {}
        # ---- NCCL id bootstrap through the process group (as bench.py does)
        r, w, nid = bs.dist_from_process_group()
        ids = [None] * world
        dist.all_gather_object(ids, nid)
        out["id_same"] = ids[0] == ids[1] and len(ids[0]) == 128
        # ---- ownership + selection identical on every rank
        p = synth.scaled(synth.PRESETS["cfg3"], 16, n_views=20)
        g = p.geometry()
        N, M = 4, 5
        first, cnt = bs.owned_blocks(N, world, rank)
        owned = list(range(first, first + cnt))
        sels = [(bs.sample(9, 1, e, M, 1), bs.sample(9, 2, e, N, 2)) for e in range(6)]
        allsel = [None] * world
        dist.all_gather_object(allsel, sels)
        out["sel_same"] = allsel[0] == allsel[1]
        allown = [None] * world
        dist.all_gather_object(allown, owned)
        out["partition_ok"] = sorted(sum(allown, [])) == list(range(N))
        # ---- distributed residual: r_I = y_I - allreduce(sum_{owned j} z^j_I)
        P = Projector(g, BlockGrid(g.dims, (1, 1, N)))
        rng = np.random.default_rng(0)
        xb = rng.random((N, P.grid.bsize))
        y = rng.random(g.n_rays)
        rows = ob.view_partition(g.n_views, M, "random", 9)
        views = rows[sels[0][0][0]]
        part = np.zeros(g.n_rays)
        for j in owned:
            P.fp(views, j, xb[j], proj=part, accumulate=True)
        rid = P.rows_of(views)
        t = torch.from_numpy(part[rid].copy())
        dist.all_reduce(t)
        r_dist = y[rid] - t.numpy()
        full = np.zeros(g.n_rays)
        for j in range(N):
            P.fp(views, j, xb[j], proj=full, accumulate=True)
        out["residual_err"] = float(np.max(np.abs(r_dist - (y[rid] - full[rid]))))
        # ---- sharded FGP TV prox with the engine's halo schedule
        vol = rng.random((8, 6, 5))
        z0, z1 = rank * 4, rank * 4 + 4
        out["tv_err"] = float(np.max(np.abs(_tv_sharded(vol[z0:z1], 0.3, 20, rank, world, vol.shape)
                                            - ob.tv_prox(vol, 0.3, 20)[z0:z1])))
        out["tv_fused_err"] = float(np.max(np.abs(_tv_sharded_fused(vol[z0:z1], 0.3, 20, rank, world, vol.shape)
                                                  - ob.tv_prox(vol, 0.3, 20)[z0:z1])))
        # ---- stratified selection (strata = world): each rank owns gamma N / G of the draw
        st = [bs.sample_stratified(9, e, N, 2, world) for e in range(20)]
        out["strat_own"] = all(sum(1 for j in c if j in owned) == 2 // world for c in st)
        allst = [None] * world
        dist.all_gather_object(allst, st)
        out["strat_same"] = allst[0] == allst[1]
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def _tv_sharded(b, w, iters, rank, world, gshape):
    """FGP on a z-slab with halos: q_z of plane z1 from rank+1 before the u pass,
    u of plane z0-1 from rank-1 before the p/q pass (the engine's tv_prox order)."""
    import math
    nzl = b.shape[0]
    z0 = rank * nzl
    L = 4.0 * sum(1 for n in gshape if n > 1)
    p = np.zeros((3,) + b.shape)
    q = np.zeros_like(p)
    s = 1.0

    def halo(plane_send, down):
        recv = torch.zeros(plane_send.shape, dtype=torch.float64)
        send = torch.from_numpy(np.ascontiguousarray(plane_send))
        reqs = []
        if down:
            if rank > 0:
                reqs.append(dist.isend(send, rank - 1))
            if rank < world - 1:
                reqs.append(dist.irecv(recv, rank + 1))
        else:
            if rank < world - 1:
                reqs.append(dist.isend(send, rank + 1))
            if rank > 0:
                reqs.append(dist.irecv(recv, rank - 1))
        for r in reqs:
            r.wait()
        return recv.numpy()

    def gradT(f, hq):
        out = np.zeros(b.shape)
        for comp, ax in ((0, 2), (1, 1)):
            sh = [slice(None)] * 3; sl = [slice(None)] * 3
            sh[ax] = slice(1, None); sl[ax] = slice(None, -1)
            out[tuple(sh)] += f[comp][tuple(sh)]
            out[tuple(sl)] -= f[comp][tuple(sh)]
        fz = f[2].copy()
        for k in range(nzl):
            gz = z0 + k
            if gz >= 1:
                out[k] += fz[k]
            if gz + 1 <= gshape[0] - 1:
                out[k] -= fz[k + 1] if k + 1 < nzl else hq
        return out

    def grad(u, hu):
        g = np.zeros((3,) + b.shape)
        for comp, ax in ((0, 2), (1, 1)):
            sh = [slice(None)] * 3; sl = [slice(None)] * 3
            sh[ax] = slice(1, None); sl[ax] = slice(None, -1)
            g[comp][tuple(sh)] = u[tuple(sh)] - u[tuple(sl)]
        for k in range(nzl):
            if z0 + k >= 1:
                g[2][k] = u[k] - (u[k - 1] if k >= 1 else hu)
        return g

    for _ in range(iters):
        hq = halo(q[2][0], True)
        u = b - w * gradT(q, hq)
        hu = halo(u[-1], False)
        pn = q + grad(u, hu) / (L * w)
        pn /= np.maximum(1.0, np.sqrt(np.sum(pn * pn, axis=0)))
        s1 = (1 + math.sqrt(1 + 4 * s * s)) / 2
        q = pn + ((s - 1) / s1) * (pn - p)
        p = pn
        s = s1
    hq = halo(p[2][0], True)
    return b - w * gradT(p, hq)


def _tv_sharded_fused(b, w, iters, rank, world, gshape):
    """FGP on a z-slab with the fused kernel's halo schedule (engine tv_prox, z-slab path):
    b of plane z0-1 once; per iteration q (3 components) of plane z0-1 from rank-1 and q_z
    of plane z1 from rank+1; u is evaluated on planes z0-1 .. z1-1 locally (never exchanged)."""
    import math
    nzl, ny, nx = b.shape
    z0 = rank * nzl
    L = 4.0 * sum(1 for n in gshape if n > 1)
    p = np.zeros((3,) + b.shape)
    q = np.zeros_like(p)
    s = 1.0

    def xchg(plane, down):
        recv = torch.zeros(plane.shape, dtype=torch.float64)
        send = torch.from_numpy(np.ascontiguousarray(plane))
        src, dst = (rank + 1, rank - 1) if down else (rank - 1, rank + 1)
        reqs = []
        if 0 <= dst < world:
            reqs.append(dist.isend(send, dst))
        if 0 <= src < world:
            reqs.append(dist.irecv(recv, src))
        for r in reqs:
            r.wait()
        return recv.numpy()

    def u_planes(f, bb, zs, fz_next):
        """b - w grad^T f on planes zs .. zs+len-1 (f: (3, n, ny, nx)); fz_next = f_z of the
        plane after the last one."""
        n = f.shape[1]
        out = np.zeros((n, ny, nx))
        for comp, ax in ((0, 2), (1, 1)):
            sh = [slice(None)] * 3; sl = [slice(None)] * 3
            sh[ax] = slice(1, None); sl[ax] = slice(None, -1)
            out[tuple(sh)] += f[comp][tuple(sh)]
            out[tuple(sl)] -= f[comp][tuple(sh)]
        for k in range(n):
            gz = zs + k
            if gz >= 1:
                out[k] += f[2][k]
            if gz + 1 <= gshape[0] - 1:
                out[k] -= f[2][k + 1] if k + 1 < n else fz_next
        return bb - w * out

    hb = xchg(b[-1], False)                       # b of plane z0 - 1
    for _ in range(iters):
        hq = np.stack([xchg(q[c][-1], False) for c in range(3)])   # q of plane z0 - 1
        hz = xchg(q[2][0], True)                  # q_z of plane z1
        fe = np.concatenate([hq[:, None], q], axis=1)
        ue = u_planes(fe, np.concatenate([hb[None], b]), z0 - 1, hz)
        u, um = ue[1:], ue[:-1]                   # u on own planes; u one plane below
        gr = np.zeros((3,) + b.shape)
        gr[0][:, :, 1:] = u[:, :, 1:] - u[:, :, :-1]
        gr[1][:, 1:, :] = u[:, 1:, :] - u[:, :-1, :]
        for k in range(nzl):
            if z0 + k >= 1:
                gr[2][k] = u[k] - um[k]
        pn = q + gr / (L * w)
        pn /= np.maximum(1.0, np.sqrt(np.sum(pn * pn, axis=0)))
        s1 = (1 + math.sqrt(1 + 4 * s * s)) / 2
        q = pn + ((s - 1) / s1) * (pn - p)
        p = pn
        s = s1
    hz = xchg(p[2][0], True)
    return u_planes(p, b, z0, hz)


def test_two_ranks_gloo():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for pr in procs:
        pr.join(timeout=60)
    for r in range(world):
        o = res[r]
        assert o["id_same"] and o["sel_same"] and o["partition_ok"]
        assert o["residual_err"] < 1e-12
        assert o["tv_err"] < 1e-12
        assert o["tv_fused_err"] < 1e-12
        assert o["strat_own"] and o["strat_same"]


def _band_worker(rank, world, port, q):
    """The band exchange of the residual on CPU: each rank's band from the
    library's pure-host bsgd_rank_bands_host, its partial projection by the oracle (the FP
    kernels' stand-in), the overlap rows exchanged with gloo send/recv, r formed on the band."""
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import synth
        import paper_1903_11874_b200 as bs
        from oracle.projector import BlockGrid, Projector
        out = {}
        p = synth.scaled(synth.PRESETS["cfg5"], 32, n_views=12)
        g = p.geometry()
        N = 8
        s = N // world
        owned = range(rank * s, (rank + 1) * s)
        band = bs.rank_bands(g, (1, 1, N), world, rank)
        allb = [None] * world
        dist.all_gather_object(allb, band.tolist())
        bands = np.array(allb)                                   # [world][view][2]
        P = Projector(g, BlockGrid(g.dims, (1, 1, N)))
        rng = np.random.default_rng(1)
        xb = rng.random((N, P.grid.bsize))
        y = rng.random(g.n_rays)
        views = np.arange(g.n_views)
        nu, nv = g.det_u, g.det_v
        part = np.zeros(g.n_rays)
        for j in owned:
            P.fp(views, j, xb[j], proj=part, accumulate=True)
        part = part.reshape(g.n_views, nv, nu)
        # (1) the partial projection vanishes outside the band (what the exchange relies on)
        outside = 0.0
        for v in views:
            lo, hi = band[v]
            outside = max(outside, float(np.abs(part[v, :lo]).max(initial=0.0)),
                          float(np.abs(part[v, hi:]).max(initial=0.0)))
        out["outside"] = outside
        # (2) send my partial sums on the overlap rows to the peer, receive the peer's
        peer = 1 - rank
        recv = {}
        for v in views:
            lo, hi = max(band[v][0], bands[peer][v][0]), min(band[v][1], bands[peer][v][1])
            if lo >= hi:
                continue
            snd = torch.from_numpy(np.ascontiguousarray(part[v, lo:hi]))
            rcv = torch.zeros_like(snd)
            reqs = [dist.isend(snd, peer), dist.irecv(rcv, peer)] if rank == 0 else \
                [dist.irecv(rcv, peer), dist.isend(snd, peer)]
            for r_ in reqs:
                r_.wait()
            recv[v] = (lo, rcv.numpy())
        # (3) r on my band = y - (sum over ranks, ascending) vs the full residual
        full = np.zeros(g.n_rays)
        for j in range(N):
            P.fp(views, j, xb[j], proj=full, accumulate=True)
        r_full = (y - full).reshape(g.n_views, nv, nu)
        err, overlap_rows = 0.0, 0
        yv = y.reshape(g.n_views, nv, nu)
        for v in views:
            lo, hi = band[v]
            acc = np.zeros((hi - lo, nu))
            contrib = {rank: part[v, lo:hi]}
            if v in recv:
                olo, data = recv[v]
                pc = np.zeros((hi - lo, nu))
                pc[olo - lo:olo - lo + data.shape[0]] = data
                contrib[peer] = pc
                overlap_rows += data.shape[0]
            for h in sorted(contrib):
                acc = acc + contrib[h]
            err = max(err, float(np.abs((yv[v, lo:hi] - acc) - r_full[v, lo:hi]).max(initial=0.0)))
        out["band_err"] = err
        out["overlap_rows"] = overlap_rows
        out["band_rows"] = int(sum(hi - lo for lo, hi in band))
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def test_two_ranks_band_exchange_gloo():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_band_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for pr in procs:
        pr.join(timeout=60)
    for r in range(world):
        o = res[r]
        assert o["outside"] == 0.0                         # p_g is zero outside band_g
        assert o["band_err"] < 1e-12                       # r on the band = the full residual
        assert 0 < o["overlap_rows"] < o["band_rows"]      # something, but far less than all, is sent
    assert res[0]["overlap_rows"] == res[1]["overlap_rows"]   # the overlap is symmetric
