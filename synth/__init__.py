"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NONE of the method's arithmetic (no Siddon tracing, no BSGD
step, no sampler, no TV prox).  It only produces the *inputs* of a run:

* per-view geometry vectors (the scan geometry),
* phantoms rasterised at voxel centres (modified Shepp-Logan 2D/3D, seeded
  random ellipsoids),
* analytic line integrals of those phantoms (closed form, independent of both
  projectors; used as data y for the 3D configs),
* noise (Gaussian at an exact SNR, P:272/P:392/P:506; Poisson transmission
  noise),
* the five workload presets of BASELINE.json ``configs``.

Geometry convention (voxel units, voxel edge 1, volume centred at the
rotation centre O, Fig. 3 "O is the centre of the object and the
rotation centre"): voxel (ix, iy, iz) covers world
[ix - nx/2, ix + 1 - nx/2) x [...] x [...].  A view vector is 12 doubles:
``src`` (fan/cone) or unit ray direction (parallel), detector centre, detector
u step, detector v step.  Ray (view, iv, iu) goes through the detector pixel
centre ``det + (iu - (nu-1)/2) u + (iv - (nv-1)/2) v``.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field, replace
from typing import Optional

import numpy as np

PARALLEL, FAN, CONE = 0, 1, 2
BEAM_NAMES = {"parallel": PARALLEL, "fan": FAN, "cone": CONE}


# ----------------------------------------------------------------------------
# geometry
# ----------------------------------------------------------------------------
def cos_sin_deg(theta_deg: float) -> tuple[float, float]:
    """cos/sin of an angle in degrees with exact values at multiples of 90°.

    The angle is reduced to [0, 360), split into a quadrant k and a remainder
    r in [0, 90); r == 0 gives exactly (1, 0); the result is rotated by k
    quarter turns exactly.  (rays lying on voxel planes at
    0°/90° must be exact so that the half-open tie rule decides them.)
    """
    t = math.fmod(theta_deg, 360.0)
    if t < 0.0:
        t += 360.0
    k = math.floor(t / 90.0)
    r = t - 90.0 * k
    if r < 0.0:
        k -= 1
        r = t - 90.0 * k
    if r >= 90.0:
        k += 1
        r = t - 90.0 * k
    if r == 0.0:
        c, s = 1.0, 0.0
    else:
        rad = r * (math.pi / 180.0)
        c, s = math.cos(rad), math.sin(rad)
    for _ in range(k):
        c, s = -s, c
    return c, s


def circular(beam: str | int, n_views: int, arc_deg: float, OP: float, OD: float,
             det_u: int, det_v: int, pitch_u: float, pitch_v: float) -> np.ndarray:
    """Circular-orbit per-view vectors, shape (n_views, 12), float64.

    theta_v = v * arc / n_views (counter-clockwise from +x).  Fan/cone: source
    OP*(cos, sin, 0), detector centre -OD*(cos, sin, 0) (Fig. 3, P:425:
    source and detector centre on the middle slice).  Parallel: direction
    -(cos, sin, 0), detector centre at O.  u = pitch_u*(-sin, cos, 0),
    v = pitch_v*(0, 0, 1).
    """
    b = BEAM_NAMES[beam] if isinstance(beam, str) else int(beam)
    out = np.zeros((n_views, 12), dtype=np.float64)
    for vi in range(n_views):
        th = vi * arc_deg / n_views
        c, s = cos_sin_deg(th)
        if b == PARALLEL:
            out[vi, 0:3] = (-c, -s, 0.0)
            out[vi, 3:6] = (0.0, 0.0, 0.0)
        else:
            out[vi, 0:3] = (OP * c, OP * s, 0.0)
            out[vi, 3:6] = (-OD * c, -OD * s, 0.0)
        out[vi, 6:9] = (pitch_u * -s, pitch_u * c, 0.0)
        out[vi, 9:12] = (0.0, 0.0, pitch_v)
    return out


def laminography(n_views: int, tilt_deg: float, OP: float, OD: float, det_u: int, det_v: int,
                 pitch_u: float, pitch_v: float) -> np.ndarray:
    """Cone-beam laminography vectors (PAPER.md:75 motivates arbitrary
    trajectories): the rotation axis is z, the beam is inclined by `tilt_deg` out of the
    xy-plane.  Source OP*(cos a cos t, cos a sin t, sin a), detector centre opposite at
    -OD*(same), u = pitch_u*(-sin t, cos t, 0), v = pitch_v*(-sin a cos t, -sin a sin t,
    cos a) (orthogonal to u and to the central ray).  Shape (n_views, 12), float64."""
    ca, sa = cos_sin_deg(tilt_deg)
    out = np.zeros((n_views, 12), dtype=np.float64)
    for vi in range(n_views):
        c, s = cos_sin_deg(vi * 360.0 / n_views)
        d = np.array([ca * c, ca * s, sa])
        out[vi, 0:3] = OP * d
        out[vi, 3:6] = -OD * d
        out[vi, 6:9] = (pitch_u * -s, pitch_u * c, 0.0)
        out[vi, 9:12] = (pitch_v * -sa * c, pitch_v * -sa * s, pitch_v * ca)
    return out


@dataclass(frozen=True)
class Geometry:
    beam: int
    vecs: np.ndarray          # (n_views, 12) float64
    det_u: int
    det_v: int
    dims: tuple               # (nx, ny, nz)

    @property
    def n_views(self) -> int:
        return int(self.vecs.shape[0])

    @property
    def n_rays(self) -> int:
        return self.n_views * self.det_u * self.det_v

    @property
    def n_vox(self) -> int:
        nx, ny, nz = self.dims
        return nx * ny * nz


# ----------------------------------------------------------------------------
# phantoms (intensity, semi-axes a b c, centre x0 y0 z0, rotation about z in
# degrees) in normalised [-1, 1] coordinates.
# ----------------------------------------------------------------------------
# Modified Shepp-Logan (Toft 1996), 2D: (A, a, b, x0, y0, phi)
SHEPP_LOGAN_2D = [
    (1.0, 0.69, 0.92, 0.0, 0.0, 0.0),
    (-0.8, 0.6624, 0.8740, 0.0, -0.0184, 0.0),
    (-0.2, 0.1100, 0.3100, 0.22, 0.0, -18.0),
    (-0.2, 0.1600, 0.4100, -0.22, 0.0, 18.0),
    (0.1, 0.2100, 0.2500, 0.0, 0.35, 0.0),
    (0.1, 0.0460, 0.0460, 0.0, 0.1, 0.0),
    (0.1, 0.0460, 0.0460, 0.0, -0.1, 0.0),
    (0.1, 0.0460, 0.0230, -0.08, -0.605, 0.0),
    (0.1, 0.0230, 0.0230, 0.0, -0.606, 0.0),
    (0.1, 0.0230, 0.0460, 0.06, -0.605, 0.0),
]
# 3D modified Shepp-Logan (rotation about z only): (A, a, b, c, x0, y0, z0, phi)
SHEPP_LOGAN_3D = [
    (1.0, 0.6900, 0.920, 0.810, 0.0, 0.0, 0.0, 0.0),
    (-0.8, 0.6624, 0.874, 0.780, 0.0, -0.0184, 0.0, 0.0),
    (-0.2, 0.1100, 0.310, 0.220, 0.22, 0.0, 0.0, -18.0),
    (-0.2, 0.1600, 0.410, 0.280, -0.22, 0.0, 0.0, 18.0),
    (0.1, 0.2100, 0.250, 0.410, 0.0, 0.35, -0.15, 0.0),
    (0.1, 0.0460, 0.046, 0.050, 0.0, 0.1, 0.25, 0.0),
    (0.1, 0.0460, 0.046, 0.050, 0.0, -0.1, 0.25, 0.0),
    (0.1, 0.0460, 0.023, 0.050, -0.08, -0.605, 0.0, 0.0),
    (0.1, 0.0230, 0.023, 0.020, 0.0, -0.606, 0.0, 0.0),
    (0.1, 0.0230, 0.046, 0.020, 0.06, -0.605, 0.0, 0.0),
]


def ellipsoids_world(kind: str, dims, seed: int = 20190327, count: int = 32) -> np.ndarray:
    """Ellipsoid table in world (voxel) units: rows (rho, a, b, c, x0, y0, z0, phi_deg)."""
    nx, ny, nz = dims
    hx, hy, hz = nx / 2.0, ny / 2.0, max(nz / 2.0, 0.5)
    rows = []
    if kind == "shepp2d":
        for A, a, b, x0, y0, phi in SHEPP_LOGAN_2D:
            rows.append((A, a * hx, b * hy, 1.0, x0 * hx, y0 * hy, 0.0, phi))
    elif kind == "shepp3d":
        for A, a, b, c, x0, y0, z0, phi in SHEPP_LOGAN_3D:
            rows.append((A, a * hx, b * hy, c * hz, x0 * hx, y0 * hy, z0 * hz, phi))
    elif kind == "random":
        rng = np.random.default_rng(seed)
        K = min(nx, ny)
        for _ in range(count):
            rho = rng.uniform(0.1, 1.0)
            a, b = rng.uniform(0.05, 0.3, size=2) * K
            c = rng.uniform(0.05, 0.3) * (nz if nz > 1 else K)
            if nz == 1:
                c = 1.0
            x0, y0 = rng.uniform(-0.45, 0.45, size=2) * K
            z0 = rng.uniform(-0.45, 0.45) * nz if nz > 1 else 0.0
            phi = rng.uniform(0.0, 180.0)
            rows.append((rho, a, b, c, x0, y0, z0, phi))
    else:
        raise ValueError(kind)
    return np.asarray(rows, dtype=np.float64)


def rasterise(ells: np.ndarray, dims) -> np.ndarray:
    """Point-sample the (additive) ellipsoid phantom at voxel centres.

    Returns float64 array of shape (nz, ny, nx) (x fastest)."""
    nx, ny, nz = dims
    xs = np.arange(nx) + 0.5 - nx / 2.0
    ys = np.arange(ny) + 0.5 - ny / 2.0
    zs = np.arange(nz) + 0.5 - nz / 2.0 if nz > 1 else np.zeros(1)
    img = np.zeros((len(zs), ny, nx), dtype=np.float64)
    # z-chunked (the 1024^3 grid would need ~80 GB of temporaries at once); every voxel gets
    # exactly the same element-wise arithmetic as an unchunked evaluation
    step = max(1, (1 << 24) // max(1, nx * ny))
    for z_lo in range(0, len(zs), step):
        z_hi = min(len(zs), z_lo + step)
        Z, Y, X = np.meshgrid(zs[z_lo:z_hi], ys, xs, indexing="ij")
        sub = img[z_lo:z_hi]
        for rho, a, b, c, x0, y0, z0, phi in ells:
            cp, sp = math.cos(math.radians(phi)), math.sin(math.radians(phi))
            dx, dy, dz = X - x0, Y - y0, Z - z0
            xr = cp * dx + sp * dy
            yr = -sp * dx + cp * dy
            inside = (xr / a) ** 2 + (yr / b) ** 2 + (dz / c) ** 2 <= 1.0
            sub[inside] += rho
    return img


def rasterise_torch(ells: np.ndarray, dims, device: str = "cuda"):
    """rasterise() evaluated with torch on `device`: the same fp64 element-wise operations in
    the same order (each torch op is one correctly rounded IEEE operation, as in numpy), so
    the voxel values are identical; returns a float32 torch tensor (nz, ny, nx) on `device`.
    (The 1024^3 phantom takes ~40 min single-threaded in numpy.)"""
    import torch
    nx, ny, nz = dims
    f64 = dict(dtype=torch.float64, device=device)
    xs = torch.arange(nx, **f64) + 0.5 - nx / 2.0
    ys = torch.arange(ny, **f64) + 0.5 - ny / 2.0
    zs = torch.arange(nz, **f64) + 0.5 - nz / 2.0 if nz > 1 else torch.zeros(1, **f64)
    out = torch.empty((len(zs), ny, nx), dtype=torch.float32, device=device)
    step = max(1, (1 << 24) // max(1, nx * ny))
    for z_lo in range(0, len(zs), step):
        z_hi = min(len(zs), z_lo + step)
        Z, Y, X = torch.meshgrid(zs[z_lo:z_hi], ys, xs, indexing="ij")
        sub = torch.zeros(Z.shape, **f64)
        for rho, a, b, c, x0, y0, z0, phi in ells:
            cp, sp = math.cos(math.radians(phi)), math.sin(math.radians(phi))
            dx, dy, dz = X - float(x0), Y - float(y0), Z - float(z0)
            xr = cp * dx + sp * dy
            yr = -sp * dx + cp * dy
            inside = (xr / float(a)) * (xr / float(a)) + (yr / float(b)) * (yr / float(b)) \
                + (dz / float(c)) * (dz / float(c)) <= 1.0
            sub[inside] += float(rho)
        out[z_lo:z_hi] = sub.to(torch.float32)
    return out


def ray_endpoints(geom: Geometry, views: np.ndarray):
    """World-coordinate ray parametrisation p(alpha) = A + alpha*B, alpha in [0,1].

    Fan/cone: A = source, B = pixel - source.  Parallel: A = pixel - R*dir,
    B = 2R*dir with R = |volume diagonal|/2 + 1.
    Returns (A, B) each of shape (len(views), det_v, det_u, 3)."""
    v = geom.vecs[np.asarray(views)]
    nu, nv = geom.det_u, geom.det_v
    ou = np.arange(nu) - (nu - 1) / 2.0
    ov = np.arange(nv) - (nv - 1) / 2.0
    pix = (v[:, None, None, 3:6]
           + ou[None, None, :, None] * v[:, None, None, 6:9]
           + ov[None, :, None, None] * v[:, None, None, 9:12])
    if geom.beam == PARALLEL:
        nx, ny, nz = geom.dims
        R = 0.5 * math.sqrt(nx * nx + ny * ny + nz * nz) + 1.0
        d = np.broadcast_to(v[:, None, None, 0:3], pix.shape)
        return pix - R * d, 2.0 * R * d
    src = np.broadcast_to(v[:, None, None, 0:3], pix.shape)
    return src, pix - src


def analytic_projection(geom: Geometry, ells: np.ndarray, views=None, device: str = "cpu",
                        chunk_rays: int = 1 << 22, out_torch=None):
    """Closed-form line integrals of the additive ellipsoid phantom.

    For each ellipsoid (rho, semi-axes D, centre c, rotation R about z) the
    ray maps to unit-sphere coordinates p' = D^-1 R^T (A - c), d' = D^-1 R^T B;
    |p' + t d'|^2 = 1 gives t1 < t2, clipped to [0, 1]; the contribution is
    rho (t2 - t1) |B|.  Returns float64 numpy array (len(views), det_v, det_u).
    Uses torch (fp64) so the 1024^3 preset can run on a GPU.  If ``out_torch``
    (a float32 torch tensor of n_views*det_v*det_u elements) is given, the
    result is written there (indexed by view) instead of a numpy array."""
    import torch
    if views is None:
        views = np.arange(geom.n_views)
    views = np.asarray(views)
    out = None if out_torch is not None else np.zeros((len(views), geom.det_v, geom.det_u), dtype=np.float64)
    per_view = geom.det_u * geom.det_v
    vchunk = max(1, chunk_rays // per_view)
    E = torch.as_tensor(ells, dtype=torch.float64, device=device)
    vecs = torch.as_tensor(geom.vecs, dtype=torch.float64, device=device)
    ou = torch.arange(geom.det_u, dtype=torch.float64, device=device) - (geom.det_u - 1) / 2.0
    ov = torch.arange(geom.det_v, dtype=torch.float64, device=device) - (geom.det_v - 1) / 2.0
    for s in range(0, len(views), vchunk):
        vs = views[s:s + vchunk]
        v = vecs[torch.as_tensor(vs, device=device)]
        pix = (v[:, None, None, 3:6] + ou[None, None, :, None] * v[:, None, None, 6:9]
               + ov[None, :, None, None] * v[:, None, None, 9:12])
        if geom.beam == PARALLEL:
            nx, ny, nz = geom.dims
            R = 0.5 * math.sqrt(nx * nx + ny * ny + nz * nz) + 1.0
            d = v[:, None, None, 0:3].expand_as(pix)
            A, B = pix - R * d, 2.0 * R * d
        else:
            src = v[:, None, None, 0:3].expand_as(pix)
            A, B = src, pix - src
        A = A.reshape(-1, 3)
        B = B.reshape(-1, 3)
        blen = torch.linalg.norm(B, dim=1)
        acc = torch.zeros(A.shape[0], dtype=torch.float64, device=device)
        for e in range(E.shape[0]):
            rho, a, b, c, x0, y0, z0, phi = [E[e, k] for k in range(8)]
            cp, sp = torch.cos(torch.deg2rad(phi)), torch.sin(torch.deg2rad(phi))
            px, py, pz = A[:, 0] - x0, A[:, 1] - y0, A[:, 2] - z0
            qx = (cp * px + sp * py) / a
            qy = (-sp * px + cp * py) / b
            qz = pz / c
            dx = (cp * B[:, 0] + sp * B[:, 1]) / a
            dy = (-sp * B[:, 0] + cp * B[:, 1]) / b
            dz = B[:, 2] / c
            aa = dx * dx + dy * dy + dz * dz
            bb = 2.0 * (qx * dx + qy * dy + qz * dz)
            cc = qx * qx + qy * qy + qz * qz - 1.0
            disc = bb * bb - 4.0 * aa * cc
            ok = disc > 0
            sq = torch.sqrt(torch.clamp(disc, min=0.0))
            t1 = ((-bb - sq) / (2.0 * aa)).clamp(0.0, 1.0)
            t2 = ((-bb + sq) / (2.0 * aa)).clamp(0.0, 1.0)
            acc += torch.where(ok, rho * (t2 - t1) * blen, torch.zeros_like(acc))
        if out_torch is not None:
            ot = out_torch.view(geom.n_views, per_view)
            ot[torch.as_tensor(vs, device=ot.device)] = acc.reshape(len(vs), per_view).to(ot.device, torch.float32)
        else:
            out[s:s + len(vs)] = acc.reshape(len(vs), geom.det_v, geom.det_u).cpu().numpy()
    return out if out_torch is None else out_torch


# ----------------------------------------------------------------------------
# noise
# ----------------------------------------------------------------------------
def gaussian_noise_snr(y: np.ndarray, snr_db: float, seed: int) -> np.ndarray:
    """y + e with e Gaussian scaled so 20 log10(|y| / |e|) = snr_db exactly."""
    rng = np.random.default_rng(seed)
    e = rng.standard_normal(y.shape)
    e *= np.linalg.norm(y) / (np.linalg.norm(e) * 10.0 ** (snr_db / 20.0))
    return y + e


def poisson_noise(y: np.ndarray, I0: float, seed: int, max_integral: float = 3.0) -> np.ndarray:
    """Transmission Poisson noise: scale = max_integral / max(y),
    N ~ Poisson(I0 exp(-scale y)), y' = -ln(max(N, 1) / I0) / scale."""
    rng = np.random.default_rng(seed)
    scale = max_integral / max(float(np.max(y)), 1e-30)
    counts = rng.poisson(I0 * np.exp(-scale * y))
    return -np.log(np.maximum(counts, 1) / I0) / scale


# ----------------------------------------------------------------------------
# workload presets (BASELINE.json configs)
# ----------------------------------------------------------------------------
@dataclass(frozen=True)
class Preset:
    name: str
    beam: str
    dims: tuple
    n_views: int
    arc_deg: float
    det: tuple             # (det_u, det_v)
    pitch: tuple           # (pitch_u, pitch_v)
    OP: float
    OD: float
    blocks: tuple          # (bx, by, bz)
    M: int
    tiles: tuple           # (tiles_u, tiles_v) for importance sampling
    rows_per_epoch: int    # alpha*M
    cols_per_epoch: int    # gamma*N
    phantom: str
    noise: Optional[tuple] = None   # ("gauss", snr_db, seed) | ("poisson", I0, seed)
    data: str = "consistent"         # "consistent" (y = A x_true by the oracle) | "analytic"
    epochs: int = 20

    def geometry(self) -> Geometry:
        vecs = circular(self.beam, self.n_views, self.arc_deg, self.OP, self.OD,
                        self.det[0], self.det[1], self.pitch[0], self.pitch[1])
        return Geometry(BEAM_NAMES[self.beam], vecs, self.det[0], self.det[1], tuple(self.dims))

    @property
    def N(self) -> int:
        return self.blocks[0] * self.blocks[1] * self.blocks[2]


PRESETS = {
    # cfg1: 2D parallel 64x64 Shepp-Logan, 90 angles x 95 detectors, 2x2 blocks, 4 row blocks
    "cfg1": Preset("cfg1", "parallel", (64, 64, 1), 90, 180.0, (95, 1), (1.0, 1.0), 0.0, 0.0,
                   (2, 2, 1), 4, (2, 1), 1, 1, "shepp2d"),
    # cfg2: 2D fan 256x256, 360 angles x 367 detectors, 4x4 blocks, IS vs uniform, Poisson
    "cfg2": Preset("cfg2", "fan", (256, 256, 1), 360, 360.0, (367, 1), (2.0, 1.0), 400.0, 400.0,
                   (4, 4, 1), 4, (2, 1), 1, 2, "shepp2d", ("poisson", 2e3, 7)),
    # cfg3: 3D cone 256^3, 360 x 256^2, 8 z-slabs, BSGD vs SGD
    "cfg3": Preset("cfg3", "cone", (256, 256, 256), 360, 360.0, (256, 256), (1.5625, 1.5625),
                   1536.0, 1000.0, (1, 1, 8), 5, (1, 4), 1, 2, "shepp3d"),
    # cfg4: 3D cone 512^3, 720 x 512^2, TV + auto-mu
    "cfg4": Preset("cfg4", "cone", (512, 512, 512), 720, 360.0, (512, 512), (1.5625, 1.5625),
                   3072.0, 2000.0, (1, 1, 8), 10, (1, 4), 1, 2, "shepp3d",
                   ("gauss", 28.1, 11), "analytic"),
    # cfg5: 3D cone 1024^3, 720 x 1024^2, image sharded over 1/2/4/8 GPUs
    "cfg5": Preset("cfg5", "cone", (1024, 1024, 1024), 720, 360.0, (1024, 1024), (1.5625, 1.5625),
                   6144.0, 4000.0, (1, 1, 8), 10, (1, 4), 1, 8, "random", None, "analytic"),
}


def scaled(p: Preset, K: int, det: Optional[int] = None, n_views: Optional[int] = None) -> Preset:
    """A smaller copy of a 3D cone preset with the same §III-E proportions
    (OP = 6K, OD = 1000K/256, pitch 400/256 * K/n_det)."""
    det = det or K
    nv = n_views or p.n_views
    pitch = (400.0 / 256.0) * K / det
    return replace(p, name=f"{p.name}@{K}", dims=(K, K, K), det=(det, det), pitch=(pitch, pitch),
                   OP=6.0 * K, OD=1000.0 * K / 256.0, n_views=nv)
