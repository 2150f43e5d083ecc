"""Debug tool (not the oracle, not the product): a numpy emulation of the v3 projector's
fixed-point slice stepping (csrc/project.cu k_project3), used to localise parity failures
on the CPU.  Emits per-ray segment lists (voxel offset within the block, length)."""
from __future__ import annotations

import sys

import numpy as np

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import synth  # noqa: E402


def rays(g, view):
    vec = g.vecs[view]
    nu, nv = g.det_u, g.det_v
    iu, iv = np.meshgrid(np.arange(nu), np.arange(nv))
    ou = iu.ravel() - (nu - 1) / 2.0
    ov = iv.ravel() - (nv - 1) / 2.0
    d = vec[3:6][None, :] + ou[:, None] * vec[6:9][None, :] + ov[:, None] * vec[9:12][None, :]
    a = np.broadcast_to(vec[0:3], d.shape).copy()
    b = d - a
    a = a + np.array(g.dims) / 2.0
    return a, b


def v3_segments(g, view, lo, hi, emulate=True):
    vec = g.vecs[view]
    mainX = abs(vec[3] - vec[0]) > abs(vec[4] - vec[1])
    a, b = rays(g, view)
    lo = np.array(lo, float)
    hi = np.array(hi, float)
    perm = [1, 0, 2] if mainX else [0, 1, 2]
    a = a[:, perm]
    b = b[:, perm]
    lo = lo[perm]
    hi = hi[perm]
    n = len(a)
    with np.errstate(divide="ignore", invalid="ignore"):
        inv = np.where(b != 0, 1.0 / b, 0.0)
        amin = np.zeros(n)
        amax = np.ones(n)
        ok = np.ones(n, bool)
        for c in range(3):
            z = b[:, c] == 0
            ok &= ~z | ((a[:, c] >= lo[c]) & (a[:, c] < hi[c]))
            t0 = (lo[c] - a[:, c]) * inv[:, c]
            t1 = (hi[c] - a[:, c]) * inv[:, c]
            amin = np.where(z, amin, np.maximum(amin, np.minimum(t0, t1)))
            amax = np.where(z, amax, np.minimum(amax, np.maximum(t0, t1)))
    hit = ok & (amin < amax)
    lim = np.abs(b[:, 1]) * (1 - 1 / 1073741824.0)
    steep = (b[:, 1] == 0) | ~(np.abs(b[:, 0]) < lim) | ~(np.abs(b[:, 2]) < lim)
    out = {}
    bdx, bdy = int(hi[0] - lo[0]), int(hi[1] - lo[1])
    plane = bdx * bdy
    for r in np.nonzero(hit & ~steep)[0]:
        out[r] = one_ray(a[r], b[r], inv[r], amin[r], amax[r], lo, hi, bdx, plane)
    return out, mainX, hit, steep


def cell_enter(c, d, lo, hi):
    f = np.floor(c)
    i = int(f)
    if d < 0 and f == c:
        i -= 1
    return min(max(i, int(lo)), int(hi) - 1)


def cell_exit(c, d, lo, hi):
    i = int(np.ceil(c)) - 1 if d > 0 else int(np.floor(c))
    return min(max(i, int(lo)), int(hi) - 1)


def one_ray(a, b, inv, amin, amax, lo, hi, bdx, plane):
    f32 = np.float32
    sy = 1 if b[1] > 0 else -1
    ainv1 = abs(inv[1])
    j0 = cell_enter(a[1] + amin * b[1], sy, lo[1], hi[1])
    j1 = cell_exit(a[1] + amax * b[1], sy, lo[1], hi[1])
    if sy * (j1 - j0) < 0:
        j1 = j0
    yin0 = j0 if sy > 0 else j0 + 1
    yin1 = j1 if sy > 0 else j1 + 1
    ap = (yin0 - a[1]) * inv[1]
    kx, kz = b[0] * ainv1, b[2] * ainv1
    mx, mz = kx < 0, kz < 0
    xr = a[0] + ap * b[0] - lo[0]
    zr = a[2] + ap * b[2] - lo[2]
    xm = -xr if mx else xr
    zm = -zr if mz else zr
    T = 2.0 ** 64
    KX = int(round(abs(kx) * T))
    KZ = int(round(abs(kz) * T))

    def plane_dist(c, K):
        f = np.floor(c)
        cell = int(f)
        rem = 1.0 - (c - f)
        if rem >= 1.0:
            return 0, cell - (1 if K else 0)
        return int(round(rem * T)), cell

    DX, cxm = plane_dist(xm, KX)
    DZ, czm = plane_dist(zm, KZ)
    ix = -cxm - 1 if mx else cxm
    iz = -czm - 1 if mz else czm
    ikx = f32(1.0 / float(KX)) if KX else f32(0)
    ikz = f32(1.0 / float(KZ)) if KZ else f32(0)
    sxo = -1 if mx else 1
    pstep = -plane if mz else plane
    o = iz * plane + (j0 - int(lo[1])) * bdx + ix
    slo = f32(min(max((amin - ap) * abs(b[1]), 0.0), 1.0))
    aq = (yin1 - a[1]) * inv[1]
    shil = f32(min(max((amax - aq) * abs(b[1]), 0.0), 1.0))
    if j1 == j0:
        shil = max(shil, slo)
    Ls = f32(np.sqrt(b @ b) * ainv1)
    nk = sy * (j1 - j0)
    segs = []
    if True:
        for k in range(nk + 1):
            shi = shil if k == nk else f32(1)
            cx, cz = DX < KX, DZ < KZ
            ux = f32(f32(DX) * ikx)
            uz = f32(f32(DZ) * ikz)
            ex = ux if cx else f32(2)
            ez = uz if cz else f32(2)
            xfirst = ex <= ez
            m1, m2 = min(ex, ez), max(ex, ez)
            c1 = min(max(m1, slo), shi)
            c2 = min(max(m2, slo), shi)
            l0, l1, l2 = f32(c1 - slo), f32(c2 - c1), f32(shi - c2)
            dox = sxo if cx else 0
            doz = pstep if cz else 0
            o1 = o + (dox if xfirst else doz)
            o2 = o + dox + doz
            segs.append((o, l0 * Ls))
            if cx or cz:
                segs.append((o1, l1 * Ls))
            if cx and cz:
                segs.append((o2, l2 * Ls))
            o = o2 + sy * bdx
            DX = (DX - KX) % (1 << 64)
            DZ = (DZ - KZ) % (1 << 64)
            slo = f32(0)
    return segs
