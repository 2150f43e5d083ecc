"""Host model of a brick-major projector at cfg5 ("Shared-memory staging"):
for a brick of the slab staged in shared memory and one view, every ray whose line meets
the brick walks only the brick's slices (main in-plane axis, as k_project3), so each ray
segment needs its own set-up and a warp of 32 adjacent detector columns walks the union of
its lanes' slice ranges.  Reports, per brick shape and view angle, the mean slices per
segment (what the per-segment set-up is amortised over) and the lane efficiency
(useful lane-slices / lanes x walked slices) that the current whole-slab walk does not pay.

    python tools/brick_model.py
"""
import math
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402


def brick_stats(p, view_deg, lo, hi):
    """Slices per segment and warp lane efficiency for the rays of one view through the
    box [lo, hi) (voxel units, volume corner at 0)."""
    n = p.dims[0]
    c, s = math.cos(math.radians(view_deg)), math.sin(math.radians(view_deg))
    src = np.array([p.OP * c, p.OP * s, 0.0]) + n / 2.0
    det_c = np.array([-p.OD * c, -p.OD * s, 0.0]) + n / 2.0
    u = p.pitch[0] * np.array([-s, c, 0.0])
    v = p.pitch[1] * np.array([0.0, 0.0, 1.0])
    nu, nv = p.det
    # detector rows / columns that can see the box (corner projection bounding rectangle)
    iu = np.arange(nu)
    iv = np.arange(nv)
    corners = np.array([[x, y, z] for x in (lo[0], hi[0]) for y in (lo[1], hi[1]) for z in (lo[2], hi[2])], float)
    # ray through pixel (a, b): d = det_c + (a - (nu-1)/2) u + (b - (nv-1)/2) v - src
    normal = det_c - src
    t = (normal @ normal) / ((corners - src) @ normal)
    hit = src + (corners - src) * t[:, None] - det_c
    ua = hit @ u / (u @ u) + (nu - 1) / 2.0
    vb = hit @ v / (v @ v) + (nv - 1) / 2.0
    iu = iu[(iu >= math.floor(ua.min()) - 1) & (iu <= math.ceil(ua.max()) + 1)]
    iv = iv[(iv >= math.floor(vb.min()) - 1) & (iv <= math.ceil(vb.max()) + 1)]
    A, B = np.meshgrid(iu - (nu - 1) / 2.0, iv - (nv - 1) / 2.0)
    d = det_c[None, None, :] + A[..., None] * u + B[..., None] * v - src
    main = 0 if abs(c) > abs(s) else 1            # walk axis: the larger direction component (k_project3)
    with np.errstate(divide="ignore", invalid="ignore"):
        t0 = (np.asarray(lo, float) - src) / d
        t1 = (np.asarray(hi, float) - src) / d
    tmin = np.nanmax(np.minimum(t0, t1), axis=-1)
    tmax = np.nanmin(np.maximum(t0, t1), axis=-1)
    ok = tmax > tmin
    pa = src[main] + tmin * d[..., main]
    pb = src[main] + tmax * d[..., main]
    k0 = np.floor(np.minimum(pa, pb))
    k1 = np.ceil(np.maximum(pa, pb)) - 1
    slices = np.where(ok, k1 - k0 + 1, 0)
    nseg = int(ok.sum())
    if nseg == 0:
        return None
    useful, walked = 0.0, 0.0
    for r in range(slices.shape[0]):
        for w0 in range(0, slices.shape[1], 32):
            m = ok[r, w0:w0 + 32]
            if not m.any():
                continue
            a, b = k0[r, w0:w0 + 32][m], k1[r, w0:w0 + 32][m]
            useful += float((b - a + 1).sum())
            walked += 32.0 * float(b.max() - a.min() + 1)
    return {"segments": nseg, "slices_per_segment": float(slices[ok].mean()), "lane_eff": useful / walked}


def main():
    p = synth.PRESETS["cfg5"]
    n = p.dims[0]
    shapes = {"32x32x32": (32, 32, 32), "64x64x8": (64, 64, 8), "whole slab (k_project3)": (n, n, 128)}
    print(f"cfg5: OP {p.OP}, OD {p.OD}, pitch {p.pitch}, det {p.det}")
    for name, (bx, by, bz) in shapes.items():
        rows = []
        for view in (0.0, 22.5, 45.0):
            # a brick near the slab centre of the slab above the mid-plane (z 512..640)
            lo = (n / 2 - bx / 2 + 100 if bx < n else 0, n / 2 - by / 2 + 60 if by < n else 0, 512 + (128 - bz) // 2)
            hi = (lo[0] + bx, lo[1] + by, lo[2] + bz)
            st = brick_stats(p, view, lo, hi)
            rows.append((view, st))
        for view, st in rows:
            print(f"{name:>24s} view {view:5.1f} deg: {st['segments']:8d} segments, "
                  f"{st['slices_per_segment']:7.1f} slices / segment, lane efficiency {st['lane_eff']:.3f}")


if __name__ == "__main__":
    main()
