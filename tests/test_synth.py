"""The seeded input generators (synth/: inputs only, shared by the oracle and the CUDA
path): the torch phantom rasteriser used for the 1024^3 fixtures gives the numpy one's
values exactly, and the z-chunked numpy rasteriser equals an unchunked evaluation."""
import math

import numpy as np

import synth


def test_rasterise_torch_equals_numpy():
    for dims, kind in [((48, 40, 36), "random"), ((1100, 1100, 16), "shepp3d"), ((64, 64, 1), "shepp2d")]:
        e = synth.ellipsoids_world(kind, dims)
        a = synth.rasterise(e, dims).astype(np.float32)
        b = synth.rasterise_torch(e, dims, device="cpu").numpy()
        assert np.array_equal(a, b), dims


def test_rasterise_chunking_is_exact():
    dims = (1100, 1100, 16)          # 13 planes per chunk -> 2 chunks
    e = synth.ellipsoids_world("shepp3d", dims)
    nx, ny, nz = dims
    xs = np.arange(nx) + 0.5 - nx / 2
    ys = np.arange(ny) + 0.5 - ny / 2
    zs = np.arange(nz) + 0.5 - nz / 2
    Z, Y, X = np.meshgrid(zs, ys, xs, indexing="ij")
    img = np.zeros((nz, ny, nx))
    for rho, a, b, c, x0, y0, z0, phi in e:
        cp, sp = math.cos(math.radians(phi)), math.sin(math.radians(phi))
        dx, dy, dz = X - x0, Y - y0, Z - z0
        xr, yr = cp * dx + sp * dy, -sp * dx + cp * dy
        img[(xr / a) ** 2 + (yr / b) ** 2 + (dz / c) ** 2 <= 1.0] += rho
    assert np.array_equal(synth.rasterise(e, dims), img)
