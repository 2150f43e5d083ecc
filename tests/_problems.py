"""Seeded problem builders for the parity tests (inputs only: geometry,
phantom, data).  y is produced by the ORACLE (consistent data)
or by synth's analytic projections — never by the CUDA path."""
from __future__ import annotations

import numpy as np

import synth
from oracle.projector import BlockGrid, Projector


def phantom(preset, geom):
    kind = preset.phantom
    return synth.rasterise(synth.ellipsoids_world(kind, geom.dims), geom.dims)


def consistent_data(geom, blocks, vol32, views=None):
    """y = A x_true by the oracle (fp64), from the fp32-rounded phantom."""
    P = Projector(geom, BlockGrid(geom.dims, blocks))
    xb = P.grid.to_blocks(vol32.astype(np.float64))
    views = np.arange(geom.n_views) if views is None else views
    y = np.zeros(geom.n_rays)
    for j in range(P.grid.N):
        P.fp(views, j, xb[j], proj=y, accumulate=True)
    return y


def problem(name, **scaled_kw):
    p = synth.PRESETS[name]
    if scaled_kw:
        p = synth.scaled(p, **scaled_kw)
    g = p.geometry()
    vol32 = phantom(p, g).astype(np.float32)
    if p.data == "consistent":
        y = consistent_data(g, p.blocks, vol32)
    else:
        ells = synth.ellipsoids_world(p.phantom, g.dims)
        y = synth.analytic_projection(g, ells).ravel()
    if p.noise is not None:
        kind, a, seed = p.noise
        if kind == "gauss":
            y = synth.gaussian_noise_snr(y, a, seed)
        else:
            y = synth.poisson_noise(y, a, seed)
    return p, g, vol32, y.astype(np.float32)
