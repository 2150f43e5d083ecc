"""B200-native BSGD hot path (Gao, Biguri, Blumensath, arXiv 1903.11874).

Thin ctypes binding over ``libbsgd.so`` (the C ABI declared in
``include/bsgd.h``).  Argument marshalling only: every step of the path runs in
the library's CUDA kernels.  PyTorch supplies device memory (the library's
state is allocated through the torch caching allocator), streams and the
process group used to broadcast the NCCL id.

There is deliberately no CPU fallback: importing this package without the
built library raises.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libbsgd.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                      "(nvcc, sm_100a). There is no CPU fallback.")

_lib = C.CDLL(LIB_PATH)

PARALLEL, FAN, CONE = 0, 1, 2
IS, IS_UNIFORM, TV, AUTO_MU, SGD, RESUME, TIMING, STRATIFIED, IS_AREA, TV_CHAMBOLLE, DETERMINISTIC = \
    1, 2, 4, 8, 16, 32, 64, 128, 256, 512, 1024
LOG_TRUE_OBJ = 2048
STATUS = {0: "OK", 1: "E_GEOMETRY", 2: "E_PARTITION", 3: "E_DIMENSION", 4: "E_CONTRACT", 5: "E_CUDA",
          6: "E_NCCL", 7: "E_OOM", 8: "E_POISONED"}


class BsgdError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"bsgd {STATUS.get(code, code)}: {msg}")
        self.code = code


# ---------------------------------------------------------------- C structs
class Geometry(C.Structure):
    _fields_ = [("beam", C.c_int32), ("n_views", C.c_int32), ("det_u", C.c_int32), ("det_v", C.c_int32),
                ("vecs", C.POINTER(C.c_double))]


class Dims(C.Structure):
    _fields_ = [("nx", C.c_int32), ("ny", C.c_int32), ("nz", C.c_int32)]


class BlockGrid(C.Structure):
    _fields_ = [("bx", C.c_int32), ("by", C.c_int32), ("bz", C.c_int32)]


class RowGrid(C.Structure):
    _fields_ = [("M", C.c_int32), ("kind", C.c_int32), ("seed", C.c_uint64), ("tiles_u", C.c_int32),
                ("tiles_v", C.c_int32)]


class CreateOpts(C.Structure):
    _fields_ = [("z_splits", C.POINTER(C.c_int32))]


class Dist(C.Structure):
    _fields_ = [("rank", C.c_int32), ("world", C.c_int32), ("nccl_id", C.POINTER(C.c_uint8)),
                ("vgroup", C.c_void_p)]


ALLOC_FN = C.CFUNCTYPE(C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p)
FREE_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p)


class Alloc(C.Structure):
    _fields_ = [("alloc", ALLOC_FN), ("free", FREE_FN), ("user", C.c_void_p)]


class Info(C.Structure):
    _fields_ = [("N", C.c_int32), ("M", C.c_int32), ("n_views", C.c_int32), ("det_u", C.c_int32),
                ("det_v", C.c_int32), ("owned_first", C.c_int32), ("owned_count", C.c_int32),
                ("tiles", C.c_int32), ("block_voxels", C.c_int64), ("n_rays", C.c_int64),
                ("owned_voxels", C.c_int64), ("block_dims", C.c_int32 * 3), ("device_bytes", C.c_uint64)]


class Selection(C.Structure):
    _fields_ = [("n_rows", C.c_int32), ("rows", C.POINTER(C.c_int32)), ("n_cols", C.c_int32),
                ("cols", C.POINTER(C.c_int32)), ("im_tiles", C.POINTER(C.c_int32))]


class RunParams(C.Structure):
    _fields_ = [("seed", C.c_uint64), ("epochs", C.c_int32), ("rows_per_epoch", C.c_int32),
                ("cols_per_epoch", C.c_int32), ("mu0", C.c_double), ("flags", C.c_uint32),
                ("lambda_", C.c_double), ("tv_iters", C.c_int32), ("tv_period", C.c_int32),
                ("eps", C.c_double), ("delta", C.c_double), ("t1", C.c_double), ("t2", C.c_double),
                ("is_off_last_epochs", C.c_int32), ("strata", C.c_int32), ("total_epochs", C.c_int32)]


class RunLog(C.Structure):
    _fields_ = [("obj", C.POINTER(C.c_double)), ("rmse", C.POINTER(C.c_double)), ("mu", C.POINTER(C.c_double)),
                ("sel_rows", C.POINTER(C.c_int32)), ("sel_cols", C.POINTER(C.c_int32)),
                ("visits", C.POINTER(C.c_uint64)), ("t_ms", C.POINTER(C.c_double)),
                ("obj_true", C.POINTER(C.c_double)), ("tv", C.POINTER(C.c_double)),
                ("rmse_seen", C.POINTER(C.c_double))]


class SolveParams(C.Structure):
    _fields_ = [("solver", C.c_int32), ("iters", C.c_int32), ("mu0", C.c_double), ("lambda_", C.c_double),
                ("tv_iters", C.c_int32), ("svrg_m", C.c_int32), ("seed", C.c_uint64)]


SOLVERS = {"gd": 0, "gd_bb": 1, "ista": 2, "fista": 3, "svrg": 4}

P = C.POINTER
_ctx = C.c_void_p
SIGS = {
    "bsgd_abi_version": ([], C.c_int32),
    "bsgd_kernel_launches": ([], C.c_uint64),
    "bsgd_last_error": ([_ctx], C.c_char_p),
    "bsgd_geometry_circular": ([C.c_int32, C.c_int32, C.c_double, C.c_double, C.c_double, C.c_int32, C.c_int32,
                                C.c_double, C.c_double, P(C.c_double)], C.c_int),
    "bsgd_sample": ([C.c_uint64, C.c_int32, C.c_int32, C.c_int32, C.c_int32, P(C.c_int32)], C.c_int),
    "bsgd_sample_stratified": ([C.c_uint64, C.c_int32, C.c_int32, C.c_int32, C.c_int32, P(C.c_int32)], C.c_int),
    "bsgd_view_partition": ([C.c_int32, C.c_int32, C.c_int32, C.c_uint64, P(C.c_int32), P(C.c_int32)], C.c_int),
    "bsgd_eq8": ([C.c_int32, C.c_int32, C.c_int32, P(C.c_int32), P(C.c_int32)], C.c_int),
    "bsgd_owned_blocks": ([C.c_int32, C.c_int32, C.c_int32, P(C.c_int32), P(C.c_int32)], C.c_int),
    "bsgd_nccl_unique_id": ([P(C.c_uint8)], C.c_int),
    "bsgd_create": ([P(Geometry), Dims, BlockGrid, RowGrid, P(Dist), P(Alloc), P(_ctx)], C.c_int),
    "bsgd_create_ex": ([P(Geometry), Dims, BlockGrid, RowGrid, P(Dist), P(Alloc), P(CreateOpts), P(_ctx)], C.c_int),
    "bsgd_block_box": ([_ctx, C.c_int32, P(C.c_int32), P(C.c_int32)], C.c_int),
    "bsgd_rank_bands_host": ([P(Geometry), Dims, BlockGrid, C.c_int32, C.c_int32, P(C.c_int32)], C.c_int),
    "bsgd_balanced_z_splits": ([_ctx, C.c_int32, P(C.c_int32), C.c_void_p], C.c_int),
    "bsgd_destroy": ([_ctx], None),
    "bsgd_vgroup_create": ([C.c_int32, P(C.c_void_p)], C.c_int),
    "bsgd_vgroup_destroy": ([C.c_void_p], None),
    "bsgd_get_info": ([_ctx, P(Info)], C.c_int),
    "bsgd_row_block_views": ([_ctx, C.c_int32, P(C.c_int32), P(C.c_int32)], C.c_int),
    "bsgd_forward": ([_ctx, C.c_int32, P(C.c_int32), P(C.c_int32), C.c_int32, C.c_void_p, C.c_void_p, C.c_int32,
                      C.c_void_p], C.c_int),
    "bsgd_back": ([_ctx, C.c_int32, P(C.c_int32), P(C.c_int32), C.c_int32, C.c_void_p, C.c_void_p, C.c_float,
                   C.c_int32, C.c_void_p], C.c_int),
    "bsgd_im_weights": ([_ctx, P(C.c_double), P(C.c_uint32)], C.c_int),
    "bsgd_im_table": ([_ctx, C.c_int32, P(C.c_double), P(C.c_uint32)], C.c_int),
    "bsgd_visit_table": ([_ctx, P(C.c_uint64)], C.c_int),
    "bsgd_reset": ([_ctx, C.c_void_p, C.c_void_p], C.c_int),
    "bsgd_step": ([_ctx, C.c_void_p, C.c_void_p, P(Selection), C.c_float, C.c_uint32, C.c_void_p], C.c_int),
    "bsgd_run": ([_ctx, C.c_void_p, C.c_void_p, C.c_void_p, P(RunParams), P(RunLog), C.c_void_p], C.c_int),
    "bsgd_get_state": ([_ctx, C.c_int32, C.c_int32, C.c_void_p, C.c_size_t], C.c_int),
    "bsgd_set_state": ([_ctx, C.c_int32, C.c_int32, C.c_void_p, C.c_size_t], C.c_int),
    "bsgd_power_iteration": ([_ctx, C.c_int32, C.c_uint64, P(C.c_double), C.c_void_p], C.c_int),
    "bsgd_allreduce_time": ([_ctx, C.c_int64, C.c_int32, C.c_void_p, P(C.c_double)], C.c_int),
    "bsgd_comm_stats": ([_ctx, P(C.c_uint64), P(C.c_uint64), P(C.c_int32)], C.c_int),
    "bsgd_exchange_plan": ([_ctx, C.c_int32, C.c_int32, P(C.c_int32), P(C.c_uint64), P(C.c_uint64)], C.c_int),
    "bsgd_tv_prox": ([_ctx, C.c_void_p, C.c_double, C.c_int32, C.c_int32, C.c_void_p], C.c_int),
    "bsgd_tv_value": ([_ctx, C.c_void_p, P(C.c_double), C.c_void_p], C.c_int),
    "bsgd_solve": ([_ctx, C.c_void_p, C.c_void_p, P(SolveParams), P(C.c_double), P(C.c_double), C.c_void_p],
                   C.c_int),
}
for _name, (_args, _res) in SIGS.items():
    _f = getattr(_lib, _name)
    _f.argtypes = _args
    _f.restype = _res


def _check(code, ctx=None):
    if code != 0:
        msg = _lib.bsgd_last_error(ctx)
        raise BsgdError(code, msg.decode() if msg else "")


def _i32(a):
    a = np.ascontiguousarray(np.asarray(a, dtype=np.int32))
    return a, a.ctypes.data_as(P(C.c_int32))


def _ptr(t):
    """Device or host address of a torch tensor / numpy array / int."""
    if t is None:
        return None
    if isinstance(t, int):
        return t
    if isinstance(t, np.ndarray):
        return t.ctypes.data
    return t.data_ptr()


def _stream(stream):
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


# ---------------------------------------------------------------- pure host functions
def abi_version() -> int:
    return _lib.bsgd_abi_version()


def kernel_launches() -> int:
    """Kernels this library launched so far in this process."""
    return int(_lib.bsgd_kernel_launches())


def geometry_circular(beam, n_views, arc_deg, OP, OD, det_u, det_v, pitch_u, pitch_v) -> np.ndarray:
    out = np.zeros((n_views, 12), dtype=np.float64)
    b = {"parallel": PARALLEL, "fan": FAN, "cone": CONE}.get(beam, beam)
    _check(_lib.bsgd_geometry_circular(int(b), n_views, arc_deg, OP, OD, det_u, det_v, pitch_u, pitch_v,
                                       out.ctypes.data_as(P(C.c_double))))
    return out


def rank_bands(geom, blocks, world, rank) -> np.ndarray:
    """[n_views][2] detector row band of rank `rank` (bsgd_rank_bands_host; pure host)."""
    vecs = np.ascontiguousarray(geom.vecs, dtype=np.float64)
    g = Geometry(int(geom.beam), vecs.shape[0], int(geom.det_u), int(geom.det_v), vecs.ctypes.data_as(P(C.c_double)))
    out = np.zeros((vecs.shape[0], 2), dtype=np.int32)
    _check(_lib.bsgd_rank_bands_host(C.byref(g), Dims(*geom.dims), BlockGrid(*blocks), int(world), int(rank),
                                     out.ctypes.data_as(P(C.c_int32))))
    return out


def sample(seed, stream, epoch, n, m) -> list[int]:
    out = np.zeros(max(m, 1), dtype=np.int32)
    _check(_lib.bsgd_sample(seed, stream, epoch, n, m, out.ctypes.data_as(P(C.c_int32))))
    return out[:m].tolist()


def sample_stratified(seed, epoch, n, m, strata) -> list[int]:
    out = np.zeros(max(m, 1), dtype=np.int32)
    _check(_lib.bsgd_sample_stratified(seed, epoch, n, m, strata, out.ctypes.data_as(P(C.c_int32))))
    return out[:m].tolist()


def view_partition(n_views, M, kind=0, seed=0) -> list[list[int]]:
    v = np.zeros(n_views, dtype=np.int32)
    o = np.zeros(M + 1, dtype=np.int32)
    kind = {"random": 0, "contiguous": 1, "interleaved": 2}.get(kind, kind)
    _check(_lib.bsgd_view_partition(n_views, M, int(kind), seed, v.ctypes.data_as(P(C.c_int32)),
                                    o.ctypes.data_as(P(C.c_int32))))
    return [v[o[i]:o[i + 1]].tolist() for i in range(M)]


def eq8(nodes, M, N) -> tuple[int, int]:
    a, g = C.c_int32(), C.c_int32()
    _check(_lib.bsgd_eq8(nodes, M, N, C.byref(a), C.byref(g)))
    return a.value, g.value


def owned_blocks(N, world, rank) -> tuple[int, int]:
    f, c = C.c_int32(), C.c_int32()
    _check(_lib.bsgd_owned_blocks(N, world, rank, C.byref(f), C.byref(c)))
    return f.value, c.value


def nccl_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    _check(_lib.bsgd_nccl_unique_id(buf))
    return bytes(buf)


def dist_from_process_group():
    """(rank, world, nccl_id) with the id made on rank 0 and broadcast through
    the current torch.distributed process group."""
    import torch
    import torch.distributed as dist
    rank, world = dist.get_rank(), dist.get_world_size()
    if world == 1:
        return 0, 1, None
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.zeros(128, dtype=torch.uint8, device=dev)
    if rank == 0:
        t.copy_(torch.frombuffer(bytearray(nccl_unique_id()), dtype=torch.uint8))
    dist.broadcast(t, 0)
    return rank, world, bytes(t.cpu().numpy().tobytes())


# ---------------------------------------------------------------- torch allocator bridge
class _TorchAllocator:
    def __init__(self, device):
        import torch
        self.device = device
        self.torch = torch

        def _alloc(nbytes, stream, user):
            try:
                return self.torch.cuda.caching_allocator_alloc(int(nbytes), self.device)
            except Exception:
                return None

        def _free(ptr, nbytes, stream, user):
            try:
                self.torch.cuda.caching_allocator_delete(int(ptr))
            except Exception:
                pass

        self._a = ALLOC_FN(_alloc)
        self._f = FREE_FN(_free)
        self.struct = Alloc(self._a, self._f, None)


# ---------------------------------------------------------------- context
@dataclass
class RunResult:
    obj: np.ndarray
    rmse: np.ndarray
    mu: np.ndarray
    sel_rows: np.ndarray
    sel_cols: np.ndarray
    visits: np.ndarray
    t_ms: Optional[np.ndarray]
    obj_true: Optional[np.ndarray] = None   # 1/2 |y - A x_k|^2 (LOG_TRUE_OBJ)
    tv: Optional[np.ndarray] = None         # TV(x_k) (LOG_TRUE_OBJ)
    rmse_seen: Optional[np.ndarray] = None  # RMSE over the voxels rays cross (LOG_TRUE_OBJ + x_true)


class VirtualGroup:
    """`world` logical ranks in this process on one GPU (bsgd_vgroup_create): create one
    Context(..., rank=r, world=world, vgroup=group) per rank and drive each from its own
    thread and CUDA stream; their collectives meet inside the library."""

    def __init__(self, world):
        h = C.c_void_p()
        _check(_lib.bsgd_vgroup_create(int(world), C.byref(h)))
        self.h, self.world = h.value, int(world)

    def close(self):
        if getattr(self, "h", None):
            _lib.bsgd_vgroup_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Context:
    """One BSGD problem on this process's GPU (bsgd_create ... bsgd_destroy)."""

    def __init__(self, beam, vecs, det, dims, blocks, M, kind=0, row_seed=0, tiles=(1, 1),
                 rank=0, world=1, nccl_id=None, torch_alloc=True, device=None, vgroup=None, z_splits=None):
        import torch
        self.device = torch.cuda.current_device() if device is None else device
        self.vecs = np.ascontiguousarray(vecs, dtype=np.float64)
        b = {"parallel": PARALLEL, "fan": FAN, "cone": CONE}.get(beam, beam)
        kind = {"random": 0, "contiguous": 1, "interleaved": 2}.get(kind, kind)
        g = Geometry(int(b), self.vecs.shape[0], int(det[0]), int(det[1]), self.vecs.ctypes.data_as(P(C.c_double)))
        self._idbuf = None
        dist = None
        if world > 1 and vgroup is not None:      # virtual rank (VirtualGroup)
            dist = Dist(rank, world, None, vgroup.h)
            self._vgroup = vgroup                  # keep the group alive while this ctx lives
        elif world > 1:
            self._idbuf = (C.c_uint8 * 128).from_buffer_copy(nccl_id)
            dist = Dist(rank, world, C.cast(self._idbuf, P(C.c_uint8)), None)
        self._alloc = _TorchAllocator(self.device) if torch_alloc else None
        h = _ctx()
        with torch.cuda.device(self.device):
            opts = None
            if z_splits is not None:   # unequal z-slabs (bsgd_create_opts.z_splits)
                self._zsp, zp = _i32(z_splits)
                opts = CreateOpts(zp)
            _check(_lib.bsgd_create_ex(C.byref(g), Dims(*dims), BlockGrid(*blocks),
                                       RowGrid(M, int(kind), row_seed, int(tiles[0]), int(tiles[1])),
                                       C.byref(dist) if dist else None,
                                       C.byref(self._alloc.struct) if self._alloc else None,
                                       C.byref(opts) if opts else None, C.byref(h)))
        self.h = h
        inf = Info()
        _check(_lib.bsgd_get_info(self.h, C.byref(inf)), self.h)
        self.info = inf
        self.N, self.M = inf.N, inf.M
        self.block_voxels = inf.block_voxels
        self.n_rays = inf.n_rays
        self.owned_first, self.owned_count = inf.owned_first, inf.owned_count
        self.block_dims = tuple(inf.block_dims)
        self.det = (int(det[0]), int(det[1]))

    @classmethod
    def from_geometry(cls, geom, blocks, M, **kw):
        """geom: synth.Geometry-like (beam, vecs, det_u, det_v, dims)."""
        return cls(geom.beam, geom.vecs, (geom.det_u, geom.det_v), geom.dims, blocks, M, **kw)

    def close(self):
        if getattr(self, "h", None):
            _lib.bsgd_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _c(self, code):
        _check(code, self.h)

    def block_box(self, j):
        """(lo, hi) of column block j in grid coordinates (bsgd_block_box)."""
        lo, hi = (C.c_int32 * 3)(), (C.c_int32 * 3)()
        self._c(_lib.bsgd_block_box(self.h, int(j), lo, hi))
        return tuple(lo), tuple(hi)

    def balanced_z_splits(self, n_slabs, stream=None):
        """Work-balanced z-splits for n_slabs slabs from this (one-rank, z-slab) context's
        exact visit table (bsgd_balanced_z_splits)."""
        out = (C.c_int32 * (int(n_slabs) + 1))()
        self._c(_lib.bsgd_balanced_z_splits(self.h, int(n_slabs), out, _stream(stream)))
        return list(out)

    def row_block_views(self, i) -> list[int]:
        n = C.c_int32()
        self._c(_lib.bsgd_row_block_views(self.h, i, None, C.byref(n)))
        out = np.zeros(n.value, dtype=np.int32)
        self._c(_lib.bsgd_row_block_views(self.h, i, out.ctypes.data_as(P(C.c_int32)), C.byref(n)))
        return out.tolist()

    def forward(self, views, col_block, x_block, proj, rects=None, accumulate=False, stream=None):
        v, vp = _i32(views)
        r, rp = _i32(rects) if rects is not None else (None, None)
        self._c(_lib.bsgd_forward(self.h, len(v), vp, rp, col_block, _ptr(x_block), _ptr(proj), int(accumulate),
                                  _stream(stream)))

    def back(self, views, col_block, proj, g_block, rects=None, scale=1.0, accumulate=False, stream=None):
        v, vp = _i32(views)
        r, rp = _i32(rects) if rects is not None else (None, None)
        self._c(_lib.bsgd_back(self.h, len(v), vp, rp, col_block, _ptr(proj), _ptr(g_block), float(scale),
                               int(accumulate), _stream(stream)))

    def visit_table(self):
        """uint64 [owned block][view][tile] ray-voxel intersection counts (bsgd_visit_table)."""
        T = self.info.tiles
        out = np.zeros((self.owned_count, self.info.n_views, T), dtype=np.uint64)
        self._c(_lib.bsgd_visit_table(self.h, out.ctypes.data_as(P(C.c_uint64))))
        return out

    def im_weights(self, area=False):
        """(w, q) of the IM table: L1 mass (default) or, area=True, the BSGD_IS_AREA counts."""
        T = self.info.tiles
        n = self.owned_count * self.info.n_views * T
        w = np.zeros(n, dtype=np.float64)
        q = np.zeros(n, dtype=np.uint32)
        self._c(_lib.bsgd_im_table(self.h, int(bool(area)), w.ctypes.data_as(P(C.c_double)),
                                   q.ctypes.data_as(P(C.c_uint32))))
        shape = (self.owned_count, self.info.n_views, T)
        return w.reshape(shape), q.reshape(shape)

    def reset(self, y, stream=None):
        self._c(_lib.bsgd_reset(self.h, _ptr(y), _stream(stream)))

    def step(self, y, x, rows, cols, mu, tiles=None, sgd=False, stream=None):
        r, rp = _i32(rows)
        c, cp = _i32(cols if cols is not None else [])
        t, tp = _i32(tiles) if tiles is not None else (None, None)
        sel = Selection(len(r), rp, len(c), cp, tp)
        self._c(_lib.bsgd_step(self.h, _ptr(y), _ptr(x), C.byref(sel), float(mu), SGD if sgd else 0,
                               _stream(stream)))

    def run(self, y, x, epochs, mu0, seed=1, x_true=None, rows_per_epoch=0, cols_per_epoch=0, flags=0,
            lam=0.1, tv_iters=20, tv_period=0, eps=0.05, delta=0.4, t1=0.5, t2=0.0, is_off_last=0,
            strata=0, total_epochs=0, stream=None) -> RunResult:
        prm = RunParams(seed, epochs, rows_per_epoch, cols_per_epoch, mu0, flags, lam, tv_iters, tv_period,
                        eps, delta, t1, t2, is_off_last, strata, total_epochs)
        aM = rows_per_epoch or eq8(self.info.N // self.owned_count, self.M, self.N)[0]
        gN = cols_per_epoch or eq8(self.info.N // self.owned_count, self.M, self.N)[1]
        E = max(epochs, 1)
        obj, rmse, mu = np.zeros(E), np.zeros(E), np.zeros(E)
        sr = np.zeros(E * aM, dtype=np.int32)
        sc = np.zeros(E * gN, dtype=np.int32)
        vis = np.zeros(E, dtype=np.uint64)
        tms = np.zeros(E * 6) if flags & TIMING else None
        otrue = np.zeros(E) if flags & LOG_TRUE_OBJ else None
        otv = np.zeros(E) if flags & LOG_TRUE_OBJ else None
        oseen = np.zeros(E) if flags & LOG_TRUE_OBJ else None
        log = RunLog(obj.ctypes.data_as(P(C.c_double)), rmse.ctypes.data_as(P(C.c_double)),
                     mu.ctypes.data_as(P(C.c_double)), sr.ctypes.data_as(P(C.c_int32)),
                     sc.ctypes.data_as(P(C.c_int32)), vis.ctypes.data_as(P(C.c_uint64)),
                     tms.ctypes.data_as(P(C.c_double)) if tms is not None else None,
                     otrue.ctypes.data_as(P(C.c_double)) if otrue is not None else None,
                     otv.ctypes.data_as(P(C.c_double)) if otv is not None else None,
                     oseen.ctypes.data_as(P(C.c_double)) if oseen is not None else None)
        self._c(_lib.bsgd_run(self.h, _ptr(y), _ptr(x), _ptr(x_true), C.byref(prm), C.byref(log), _stream(stream)))
        return RunResult(obj[:epochs], rmse[:epochs], mu[:epochs], sr.reshape(E, aM)[:epochs],
                         sc.reshape(E, gN)[:epochs], vis[:epochs],
                         tms.reshape(E, 6)[:epochs] if tms is not None else None,
                         otrue[:epochs] if otrue is not None else None,
                         otv[:epochs] if otv is not None else None,
                         oseen[:epochs] if (oseen is not None and x_true is not None) else None)

    def solve(self, solver, y, x, iters, mu0, lam=0.0, tv_iters=20, svrg_m=0, seed=1, stream=None):
        """Comparison solver `solver` in {"gd", "gd_bb", "ista", "fista", "svrg"} (bsgd_solve;
        SURVEY §8f N1).  y, x: device tensors; x holds x_0 and receives the result.
        Returns (obj, mu) per iteration."""
        prm = SolveParams(SOLVERS[solver], iters, mu0, lam, tv_iters, svrg_m, seed)
        obj, mu = np.zeros(max(iters, 1)), np.zeros(max(iters, 1))
        self._c(_lib.bsgd_solve(self.h, _ptr(y), _ptr(x), C.byref(prm), obj.ctypes.data_as(P(C.c_double)),
                                mu.ctypes.data_as(P(C.c_double)), _stream(stream)))
        return obj[:iters], mu[:iters]

    def get_state(self, what, index=0):
        sizes = {0: (self.n_rays, np.float32), 1: (self.block_voxels, np.float32), 2: (self.block_voxels, np.float32),
                 3: (self.n_rays, np.float32), 4: (self.M, np.float64), 5: (1, np.float64)}
        n, dt = sizes[what]
        out = np.zeros(n, dtype=dt)
        self._c(_lib.bsgd_get_state(self.h, what, index, out.ctypes.data, out.nbytes))
        return out

    def set_state(self, what, index, arr):
        dt = np.float64 if what in (4, 5) else np.float32
        a = np.ascontiguousarray(arr, dtype=dt)
        self._c(_lib.bsgd_set_state(self.h, what, index, a.ctypes.data, a.nbytes))

    def tv_prox(self, x, w, iters=20, method="fgp", stream=None):
        """x (CUDA float32, the owned blocks block-major) <- prox_{w TV}(x) in place by
        `iters` FGP (or Chambolle-2004) iterations (bsgd_tv_prox; Algo 4 line 16)."""
        m = {"fgp": 0, "chambolle": 1}[method]
        self._c(_lib.bsgd_tv_prox(self.h, _ptr(x), float(w), int(iters), m, _stream(stream)))
        return x

    def tv_value(self, x, stream=None) -> float:
        """TV(x) of the whole volume (bsgd_tv_value; Eq. 6)."""
        out = C.c_double()
        self._c(_lib.bsgd_tv_value(self.h, _ptr(x), C.byref(out), _stream(stream)))
        return out.value

    def allreduce_time(self, count, iters=5, stream=None) -> float:
        """Mean ms of one sum-allreduce of `count` floats of the residual's partial-sum
        buffer (bsgd_allreduce_time; the ALLREDUCE of PAPER.md:99 on its own)."""
        out = C.c_double()
        self._c(_lib.bsgd_allreduce_time(self.h, int(count), int(iters), _stream(stream), C.byref(out)))
        return out.value

    def comm_stats(self) -> dict:
        """Residual-exchange bytes / messages this rank sent so far and the mode
        (bsgd_comm_stats)."""
        b, m, band = C.c_uint64(), C.c_uint64(), C.c_int32()
        self._c(_lib.bsgd_comm_stats(self.h, C.byref(b), C.byref(m), C.byref(band)))
        return {"bytes_sent": int(b.value), "messages": int(m.value),
                "mode": {0: "full", 1: "band", 2: "lsa"}[int(band.value)]}

    def exchange_plan(self, world, views) -> dict:
        """Bytes one epoch's residual exchange would send over `world` ranks for the given
        selected views: band mode vs the full ring allreduce (bsgd_exchange_plan)."""
        v, vp = _i32(views)
        b, f = C.c_uint64(), C.c_uint64()
        self._c(_lib.bsgd_exchange_plan(self.h, int(world), len(v), vp, C.byref(b), C.byref(f)))
        return {"band_bytes": int(b.value), "full_bytes": int(f.value)}

    def power_iteration(self, iters=30, seed=0, stream=None) -> float:
        out = C.c_double()
        self._c(_lib.bsgd_power_iteration(self.h, iters, seed, C.byref(out), _stream(stream)))
        return out.value
