"""ORACLE — test infrastructure.  ctypes wrapper of oracle/siddon.c.

The block operators of the paper's partition (§II Eq. 3):
``A_I^J x_J`` (FP) and ``(A_I^J)^T r_I`` (BP) computed on the fly by
merged-alpha Siddon in fp64.  Column blocks J_j are equal
axis-aligned boxes of a bx x by x bz grid, stored block-major (block j, then
[z][y][x] inside); row blocks are sets of whole views.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import build

_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        P = C.POINTER
        d, i, i64 = C.c_double, C.c_int, C.c_int64
        _lib.oracle_ray.argtypes = [i, P(d), i, i, i, i, P(i), P(d), P(d)]
        _lib.oracle_trace.argtypes = [P(d), P(d), P(i), P(i), P(i64), P(d), i]
        _lib.oracle_trace.restype = i
        common = [i, P(d), i, i, P(i), P(i), P(i)]
        _lib.oracle_fp.argtypes = common + [P(i), i, P(i), P(d), P(d), i]
        _lib.oracle_bp.argtypes = common + [P(i), i, P(i), P(d), P(d)]
        _lib.oracle_tile_mass.argtypes = common + [P(i), i, i, i, i, P(d)]
        _lib.oracle_csr_count.argtypes = common + [P(i), i, P(i64)]
        _lib.oracle_csr_fill.argtypes = common + [P(i), i, P(i64), P(i64), P(d)]
        _lib.oracle_count.argtypes = common + [P(i), i, P(i)]
        _lib.oracle_count.restype = i64
    return _lib


def _p(a, ct):
    return a.ctypes.data_as(C.POINTER(ct))


class BlockGrid:
    """Boxes of a bx x by x bz block grid over the (nx, ny, nz) volume: equal boxes, or, for
    z-slab grids (1, 1, N), slabs between the given z_splits (0 = s_0 < ... < s_N = nz; the
    column partition J of Eq. 3, need not be uniform).
    Block-major arrays are (N, bsize) with bsize the LARGEST block's voxel count: block j's
    [z][y][x] values fill the first bsizes[j] entries of its row, the rest are zero."""

    def __init__(self, dims, blocks, z_splits=None):
        self.dims = tuple(int(v) for v in dims)
        self.blocks = tuple(int(v) for v in blocks)
        self.N = self.blocks[0] * self.blocks[1] * self.blocks[2]
        if z_splits is None:
            for n, b in zip(self.dims, self.blocks):
                if b < 1 or n % b:
                    raise ValueError("volume dims must be divisible by the block grid")
            self.z_splits = None
            self.bdims = tuple(n // b for n, b in zip(self.dims, self.blocks))
        else:
            zs = [int(v) for v in z_splits]
            if self.blocks[:2] != (1, 1) or len(zs) != self.blocks[2] + 1 or zs[0] != 0 or zs[-1] != self.dims[2] \
                    or any(b <= a for a, b in zip(zs, zs[1:])):
                raise ValueError("z_splits: a z-slab grid and 0 = s_0 < ... < s_N = nz")
            self.z_splits = zs
            self.bdims = (self.dims[0], self.dims[1], max(b - a for a, b in zip(zs, zs[1:])))
        self.bsize = self.bdims[0] * self.bdims[1] * self.bdims[2]
        self.bsizes = [int(np.prod(self.box(j)[1] - self.box(j)[0])) for j in range(self.N)]
        self.n_vox = self.dims[0] * self.dims[1] * self.dims[2]

    def box(self, j):
        if self.z_splits is not None:
            lo = np.array([0, 0, self.z_splits[j]], dtype=np.int32)
            return lo, np.array([self.dims[0], self.dims[1], self.z_splits[j + 1]], dtype=np.int32)
        bx, by, _ = self.blocks
        jx, jy, jz = j % bx, (j // bx) % by, j // (bx * by)
        lo = np.array([jx * self.bdims[0], jy * self.bdims[1], jz * self.bdims[2]], dtype=np.int32)
        return lo, lo + np.array(self.bdims, dtype=np.int32)

    def to_blocks(self, vol):
        """(nz, ny, nx) volume -> (N, bsize) block-major (zero tail for smaller blocks)."""
        vol = np.asarray(vol).reshape(self.dims[2], self.dims[1], self.dims[0])
        out = np.zeros((self.N, self.bsize), dtype=vol.dtype)
        for j in range(self.N):
            lo, hi = self.box(j)
            out[j, :self.bsizes[j]] = vol[lo[2]:hi[2], lo[1]:hi[1], lo[0]:hi[0]].ravel()
        return out

    def from_blocks(self, blk):
        blk = np.asarray(blk).reshape(self.N, self.bsize)
        vol = np.empty((self.dims[2], self.dims[1], self.dims[0]), dtype=blk.dtype)
        for j in range(self.N):
            lo, hi = self.box(j)
            vol[lo[2]:hi[2], lo[1]:hi[1], lo[0]:hi[0]] = blk[j, :self.bsizes[j]].reshape(
                hi[2] - lo[2], hi[1] - lo[1], hi[0] - lo[0])
        return vol

    def mask(self):
        """(N, bsize) 1.0 on block voxels, 0.0 on the tails of smaller blocks."""
        m = np.zeros((self.N, self.bsize))
        for j in range(self.N):
            m[j, :self.bsizes[j]] = 1.0
        return m


class Projector:
    """A_I^J / (A_I^J)^T for a geometry (synth.Geometry) and a BlockGrid."""

    def __init__(self, geom, grid: BlockGrid):
        self.g = geom
        self.grid = grid
        self.vecs = np.ascontiguousarray(geom.vecs, dtype=np.float64)
        self.dims = np.array(geom.dims, dtype=np.int32)
        self.nu, self.nv = geom.det_u, geom.det_v
        lib()

    def _common(self, j):
        lo, hi = self.grid.box(j)
        return (self.g.beam, _p(self.vecs, C.c_double), self.nu, self.nv,
                _p(self.dims, C.c_int), _p(lo, C.c_int), _p(hi, C.c_int)), (lo, hi)

    @staticmethod
    def _rects(rects, n):
        if rects is None:
            return None, None
        r = np.ascontiguousarray(np.asarray(rects, dtype=np.int32).reshape(n, 4))
        return r, _p(r, C.c_int)

    def ray(self, view, iu, iv):
        a = np.zeros(3)
        b = np.zeros(3)
        lib().oracle_ray(self.g.beam, _p(np.ascontiguousarray(self.vecs[view]), C.c_double),
                         self.nu, self.nv, iu, iv, _p(self.dims, C.c_int),
                         _p(a, C.c_double), _p(b, C.c_double))
        return a, b

    def fp(self, views, j, xblk, proj=None, rects=None, accumulate=False):
        """proj[rays of views] (=|+=) A_{views}^{J_j} x_J; proj is full length (fp64)."""
        views = np.ascontiguousarray(np.asarray(views, dtype=np.int32))
        if proj is None:
            proj = np.zeros(self.g.n_rays, dtype=np.float64)
        xblk = np.ascontiguousarray(xblk, dtype=np.float64)
        (common, boxes) = self._common(j)
        r, rp = self._rects(rects, len(views))
        lib().oracle_fp(*common, _p(views, C.c_int), len(views), rp, _p(xblk, C.c_double),
                        _p(proj, C.c_double), int(accumulate))
        return proj

    def bp(self, views, j, proj, gblk=None, rects=None):
        """gblk += (A_{views}^{J_j})^T proj[rays of views] (no factor 2)."""
        views = np.ascontiguousarray(np.asarray(views, dtype=np.int32))
        if gblk is None:
            gblk = np.zeros(self.grid.bsize, dtype=np.float64)
        proj = np.ascontiguousarray(proj, dtype=np.float64)
        common, _ = self._common(j)
        r, rp = self._rects(rects, len(views))
        lib().oracle_bp(*common, _p(views, C.c_int), len(views), rp, _p(proj, C.c_double),
                        _p(gblk, C.c_double))
        return gblk

    def tile_mass(self, views, j, tiles, area=False):
        views = np.ascontiguousarray(np.asarray(views, dtype=np.int32))
        T = tiles[0] * tiles[1]
        w = np.zeros(len(views) * T, dtype=np.float64)
        common, _ = self._common(j)
        lib().oracle_tile_mass(*common, _p(views, C.c_int), len(views), tiles[0], tiles[1], int(area),
                               _p(w, C.c_double))
        return w.reshape(len(views), T)

    def count(self, views, j, rects=None):
        views = np.ascontiguousarray(np.asarray(views, dtype=np.int32))
        common, _ = self._common(j)
        r, rp = self._rects(rects, len(views))
        return int(lib().oracle_count(*common, _p(views, C.c_int), len(views), rp))

    def csr(self, views, j):
        """Explicit A_{views}^{J_j} as scipy.sparse.csr_matrix (rows: views x det, row-major)."""
        import scipy.sparse as sp
        views = np.ascontiguousarray(np.asarray(views, dtype=np.int32))
        nrows = len(views) * self.nu * self.nv
        cnt = np.zeros(nrows, dtype=np.int64)
        common, _ = self._common(j)
        lib().oracle_csr_count(*common, _p(views, C.c_int), len(views), _p(cnt, C.c_int64))
        indptr = np.zeros(nrows + 1, dtype=np.int64)
        np.cumsum(cnt, out=indptr[1:])
        indices = np.zeros(int(indptr[-1]), dtype=np.int64)
        data = np.zeros(int(indptr[-1]), dtype=np.float64)
        lib().oracle_csr_fill(*common, _p(views, C.c_int), len(views), _p(indptr, C.c_int64),
                              _p(indices, C.c_int64), _p(data, C.c_double))
        return sp.csr_matrix((data, indices, indptr), shape=(nrows, self.grid.bsize))

    def rows_of(self, views):
        """Global ray ids of the listed views (view order, then iv, iu)."""
        per = self.nu * self.nv
        views = np.asarray(views, dtype=np.int64)
        return (views[:, None] * per + np.arange(per)[None, :]).ravel()

    def dense(self, views=None):
        """Dense fp64 A restricted to the listed views, columns in GLOBAL
        [z][y][x] order (small systems only)."""
        if views is None:
            views = np.arange(self.g.n_views)
        nrows = len(views) * self.nu * self.nv
        A = np.zeros((nrows, self.g.n_vox))
        # global [z][y][x] index of every block voxel
        gidx = self.grid.to_blocks(np.arange(self.g.n_vox).reshape(self.g.dims[::-1]))
        for j in range(self.grid.N):
            Aj = self.csr(views, j).toarray()
            nb = self.grid.bsizes[j]
            A[:, gidx[j, :nb]] += Aj[:, :nb]
        return A
