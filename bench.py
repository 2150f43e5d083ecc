#!/usr/bin/env python
"""BSGD hot-path benchmark (BASELINE.json metric: "BSGD epochs/s and ray-voxel
intersections/s (FP+BP) at 1/2/4/8 B200").

A step = one BSGD epoch (Algo 1) over the cfg5 workload
(3D cone 1024^3, 720 views x 1024^2, M = 10 row blocks of 72 views, N = 8
z-slabs, alpha M = 1, gamma N = 8): selection -> FP of the 8 slabs over the 72
views -> residual (+ NCCL allreduce when N > 1) -> matched BP -> g / x update.
All of it runs in libbsgd.so; Python only marshals arguments.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...   (one process per GPU)

Prints ONE JSON line on rank 0.  --impl reference times the fp64 CPU oracle
(oracle/) on the host cores on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "BSGD epochs/s and ray-voxel intersections/s (FP+BP) at 1/2/4/8 B200"
WORKLOAD = ("cfg5: 3D cone-beam 1024^3 volume, 720 projections of 1024x1024, M=10 row blocks "
            "(72 views), N=8 z-slab blocks, alpha*M=1, gamma*N=8 per epoch")


def workload(p) -> str:
    """The `config.workload` string of a preset (cfg5 is the headline workload)."""
    if p.name == "cfg5":
        return WORKLOAD
    d = "x".join(str(v) for v in p.dims if v > 1)
    return (f"{p.name}: {p.beam} {d} volume, {p.n_views} projections of {p.det[0]}x{p.det[1]}, M={p.M} row "
            f"blocks, N={p.N} blocks {p.blocks}, alpha*M={p.rows_per_epoch}, gamma*N={p.cols_per_epoch} per epoch")


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback (B200_PROFILING.md)"


def load_traffic():
    """DRAM bytes per visit of the FP / BP launches from the newest committed ncu
    capture (profiles/traffic_<tag>.json, written by tools/traffic_from_ncu.py)."""
    d = os.path.join(ROOT, "profiles")
    names = sorted(n for n in os.listdir(d) if n.startswith("traffic_") and n.endswith(".json")) \
        if os.path.isdir(d) else []
    for name in reversed(names):
        try:
            return json.load(open(os.path.join(d, name)))
        except Exception:
            pass
    return {}


class ClockSampler:
    """SM clocks and clock-event (throttle) reasons sampled during the timed region: NVML
    every 20 ms (pynvml, from nvidia_ml_py), else nvidia-smi every 0.2 s."""

    REASONS = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"),
               ("hw_power_brake_slowdown", "nvmlClocksEventReasonHwPowerBrakeSlowdown"))
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap,utilization.gpu")

    def __init__(self, index):
        self.index = index
        self.rows = []            # (sm_mhz, max_mhz, reasons set, util %)
        self._stop = threading.Event()
        self._ready = threading.Event()   # set once the sampler runs (short timed regions)
        self._t = None
        self.source = "none"

    def _run_nvml(self, nv):
        h = nv.nvmlDeviceGetHandleByIndex(self.index)
        mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        bits = [(name, getattr(nv, attr)) for name, attr in self.REASONS if hasattr(nv, attr)]
        while not self._stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                ev = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                util = nv.nvmlDeviceGetUtilizationRates(h).gpu
                self.rows.append((float(sm), float(mx), {n for n, b in bits if ev & b}, util))
            except Exception:
                pass
            self._ready.set()
            self._stop.wait(0.02)

    def _run_smi(self):
        names = [n for n, _ in self.REASONS[:4]]
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.FIELDS,
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                r = [c.strip() for c in out.split(",")] if out else []
                if len(r) >= 7 and r[0].replace(".", "").isdigit():
                    act = {names[k] for k in range(4) if "Active" in r[2 + k] and "Not" not in r[2 + k]}
                    self.rows.append((float(r[0]), float(r[1]), act, int(r[6]) if r[6].isdigit() else 100))
            except Exception:
                pass
            self._ready.set()
            self._stop.wait(0.2)

    def _run(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            self.source = "nvml"
            self._run_nvml(nv)
        except Exception:
            self.source = "nvidia-smi"
            self._run_smi()

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        self._ready.wait(timeout=5.0)
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no clock samples"]}
        sm = [r[0] for r in self.rows]
        busy = [r[0] for r in self.rows if r[3] > 50]
        reasons = sorted(set().union(*(r[2] for r in self.rows)))
        frac = {n: round(sum(1 for r in self.rows if n in r[2]) / len(self.rows), 3) for n in reasons}
        return {"sm_mhz": float(np.median(busy or sm)), "sm_max_mhz": self.rows[0][1], "reasons": reasons,
                "reason_sample_fraction": frac, "sm_mhz_min": float(min(sm)), "samples": len(self.rows),
                "source": self.source}


# --------------------------------------------------------------------------- oracle (CPU) timing
_ORACLE_CACHE = None
# cfg5 views sampled for the CPU timing, spread over a quarter orbit (the cube's 4-fold
# symmetry: a view's visit count depends on its angle mod 90 deg, e.g. +27 % at 45 deg vs
# 0 deg), in bit-reversed order so that every prefix of the list spans the quarter
SAMPLE_VIEWS = (0, 90, 45, 135, 23, 113, 68, 158)


def _cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def _oracle_setup():
    """Per sampled view: a one-view geometry (same rays as in the full geometry; keeps the
    projection buffer at one view), its projector, and its exact FP visit count through
    the 8 slabs (the oracle's own count, computed once, outside every timed region)."""
    global _ORACLE_CACHE
    if _ORACLE_CACHE is None:
        import synth
        from oracle.projector import BlockGrid, Projector
        p = synth.PRESETS["cfg5"]
        g = p.geometry()
        projs, counts = [], []
        for v in SAMPLE_VIEWS:
            gv = synth.Geometry(g.beam, g.vecs[v:v + 1].copy(), g.det_u, g.det_v, g.dims)
            P = Projector(gv, BlockGrid(g.dims, p.blocks))
            projs.append(P)
            counts.append(sum(P.count([0], j) for j in range(p.N)))
        # visits of one epoch (FP; BP visits are the same segments) = 72 views x the mean
        # visits per view over the sampled quarter orbit
        epoch_fp = (g.n_views // p.M) * float(np.mean(counts))
        _ORACLE_CACHE = (p, g, projs, counts, epoch_fp, np.full(projs[0].grid.bsize, 0.5))
    return _ORACLE_CACHE


def oracle_sample(target_s=12.0, max_views=len(SAMPLE_VIEWS), first=0):
    """fp64 CPU oracle: FP + BP of whole sampled cfg5 views through all 8 z-slabs (the same
    per-view work as the GPU epoch) on all host cores, until `target_s` has elapsed.
    Visits are the oracle's own per-view counts.  Returns a dict."""
    p, g, projs, counts, epoch_fp, x = _oracle_setup()
    proj = np.zeros(g.det_u * g.det_v)
    visits, done, t0 = 0, [], time.perf_counter()
    while len(done) < max_views:
        k = (first + len(done)) % len(projs)
        P = projs[k]
        proj[:] = 0.0
        for j in range(p.N):
            P.fp([0], j, x, proj=proj, accumulate=True)
        for j in range(p.N):
            P.bp([0], j, proj)
        visits += 2 * counts[k]
        done.append(SAMPLE_VIEWS[k])
        if time.perf_counter() - t0 > target_s:
            break
    dt = time.perf_counter() - t0
    threads = int(os.environ.get("OMP_NUM_THREADS", "0")) or (os.cpu_count() or 1)
    return {"vps": visits / dt, "visits": visits, "seconds": dt, "views": done, "threads": threads,
            "epochs_per_s": visits / dt / (2.0 * epoch_fp), "epoch_fp_visits": epoch_fp}


def oracle_one_thread(seconds=3.0):
    """The same oracle on ONE host thread (a subprocess with OMP_NUM_THREADS=1): FP + BP of
    detector-row bands of sampled views; visits/s per core."""
    env = dict(os.environ, OMP_NUM_THREADS="1")
    code = ("import json,sys; sys.path.insert(0, %r); import bench; "
            "print(json.dumps(bench._band_sample(%r)))" % (ROOT, seconds))
    try:
        out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300)
        return json.loads(out.stdout.strip().splitlines()[-1])
    except Exception as exc:   # noqa: BLE001  (auxiliary figure)
        return {"error": f"{type(exc).__name__}: {exc}"[:200]}


def _band_sample(seconds):
    """FP + BP of 8-row detector bands of the sampled views (the counts outside the timing)."""
    import synth
    from oracle.projector import BlockGrid, Projector
    p = synth.PRESETS["cfg5"]
    g = p.geometry()
    x = None
    visits, timed, n = 0, 0.0, 0
    while timed < seconds:
        v = SAMPLE_VIEWS[n % len(SAMPLE_VIEWS)]
        gv = synth.Geometry(g.beam, g.vecs[v:v + 1].copy(), g.det_u, g.det_v, g.dims)
        P = Projector(gv, BlockGrid(g.dims, p.blocks))
        if x is None:
            x = np.full(P.grid.bsize, 0.5)
        rect = [(0, g.det_u, 480 + 8 * (n % 8), 488 + 8 * (n % 8))]
        cnt = sum(P.count([0], j, rects=rect) for j in range(p.N))
        t1 = time.perf_counter()
        proj = np.zeros(g.det_u * g.det_v)
        for j in range(p.N):
            P.fp([0], j, x, proj=proj, rects=rect, accumulate=True)
        for j in range(p.N):
            P.bp([0], j, proj, rects=rect)
        timed += time.perf_counter() - t1
        visits += 2 * cnt
        n += 1
    return {"vps_per_core": visits / timed, "bands": n, "threads": 1}


def oracle_env():
    """Both CPU legs run the oracle on all host cores with OMP_PROC_BIND=close (set before
    liboracle.so, and so its OpenMP runtime, is first loaded; torch.distributed.run exports
    OMP_NUM_THREADS=1 to every rank; BENCH_OMP_THREADS overrides)."""
    os.environ["OMP_NUM_THREADS"] = os.environ.get("BENCH_OMP_THREADS", str(os.cpu_count() or 1))
    os.environ["OMP_PROC_BIND"] = os.environ.get("BENCH_OMP_PROC_BIND", "close")


def measure_oracle(steps, warmup):
    """The one CPU measurement both legs report (the --impl reference arm and our line's
    cpu_baseline): each step = FP + BP of one whole sampled cfg5 view through the 8 slabs
    (views taken in SAMPLE_VIEWS order after the warm-up ones); value = median visits/s over
    the steps / (FP + BP visits of one epoch, from the oracle's own per-view counts)."""
    oracle_env()
    _oracle_setup()
    per_step, vps_all, views = [], [], []
    for it in range(warmup + steps):
        r = oracle_sample(target_s=4.0, max_views=1, first=it)
        if it >= warmup:
            per_step.append(r["seconds"])
            vps_all.append(r["vps"])
            views += r["views"]
    p, g, projs, counts, epoch_fp, _ = _oracle_setup()
    vps = float(np.median(vps_all))
    cores = int(os.environ.get("OMP_NUM_THREADS", "0")) or (os.cpu_count() or 1)
    sample = (f"each step = one whole cfg5 view (1024x1024 rays) FP+BP through all 8 z-slabs, fp64 merged-alpha "
              f"Siddon, OpenMP on {cores} host threads ({_cpu_model()}, OMP_PROC_BIND="
              f"{os.environ['OMP_PROC_BIND']}); views {views}; visits from the oracle's own per-view count; "
              f"epoch = {g.n_views // p.M} views x the mean visits per view of the quarter-orbit sample "
              f"{list(SAMPLE_VIEWS)} = {epoch_fp:.4g} FP visits; value = median over the steps")
    return {"value": vps / (2.0 * epoch_fp), "vps": vps, "cores": cores, "sample": sample,
            "ms_per_step": 1e3 * float(np.mean(per_step)), "epoch_fp_visits": epoch_fp}


def run_reference(args, rank, world):
    if rank != 0:
        return 0
    m = measure_oracle(args.steps, args.warmup)
    value, vps, cores, sample = m["value"], m["vps"], m["cores"], m["sample"]
    per_step = [m["ms_per_step"] / 1e3]
    line = {"metric": METRIC, "impl": "reference", "value": value, "unit": "epochs/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * float(np.mean(per_step)),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "intersections_per_s": vps,
            "config": {"workload": WORKLOAD, "sample": sample},
            "cpu_baseline": {"value": value, "unit": "epochs/s", "cores": cores, "kind": "oracle",
                             "sample": sample, "cpu_model": _cpu_model()},
            "e2e": {"value": value, "unit": "epochs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------------------- our arm
def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist
    import synth
    import paper_1903_11874_b200 as bs

    torch.cuda.set_device(local_rank)
    p = synth.PRESETS[args.config]
    g = p.geometry()
    if world > 1:
        r, w, nid = bs.dist_from_process_group()
    else:
        r, w, nid = 0, 1, None
    z_splits = None
    if args.balanced:   # slab thicknesses with equal ray-voxel intersections
        fine_n = max(p.N, p.dims[2] // 4)
        fine = bs.Context.from_geometry(g, (1, 1, fine_n), 1)   # 4-plane candidate slabs, exact visits
        z_splits = fine.balanced_z_splits(p.N)
        fine.close()
        del fine
        torch.cuda.empty_cache()
    ctx = bs.Context.from_geometry(g, p.blocks, p.M, kind="random", row_seed=1, tiles=p.tiles,
                                   rank=r, world=w, nccl_id=nid, z_splits=z_splits)
    n_owned = ctx.owned_count * ctx.block_voxels
    # synthetic data shaped like the paper's workload: analytic projections of 32
    # seeded random ellipsoids (replicated y), x0 = 0 (Algo 1 line 1)
    y = torch.empty(g.n_rays, dtype=torch.float32, device="cuda")
    if args.cheap_data:   # profiling runs: seeded uniform data (Siddon work does not depend on values)
        y.uniform_(0.0, 100.0, generator=torch.Generator(device="cuda").manual_seed(7))
    else:
        ells = synth.ellipsoids_world("random" if p.dims[2] > 1 else "shepp2d", g.dims)
        synth.analytic_projection(g, ells, device="cuda", out_torch=y, chunk_rays=1 << 23)
    x = torch.zeros(n_owned, dtype=torch.float32, device="cuda")
    # below 1/sigma_max^2 (Rayleigh lower bounds of sigma_max^2)
    mu0 = 0.25 / {"cfg1": 5451.0, "cfg2": 9.09e4, "cfg3": 8.93e4, "cfg4": 3.59e5}.get(args.config, 7.35e5)
    aM, gN = p.rows_per_epoch, p.cols_per_epoch
    # cfg4's schedule: BSGD-TV (Algo 4, lambda = 0.1; period
    # round(1/(alpha gamma)) = 40 epochs) + automatic mu (Algo 3)
    sched = (bs.TV | bs.AUTO_MU) if args.config == "cfg4" else 0
    if args.det:   # order-independent 64-bit fixed-point BP reductions (bit-reproducible runs)
        sched |= bs.DETERMINISTIC
    if args.eq8:   # Eq. 8 with NodeNum = G, columns stratified by owner (N3)
        aM, gN = 0, 0
        sched |= bs.STRATIFIED
    lam = 0.1
    stream = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # warm-up epochs (untimed; also builds/initialises everything)
    ctx.run(y, x, epochs=args.warmup, mu0=mu0, seed=7, rows_per_epoch=aM, cols_per_epoch=gN, flags=sched, lam=lam)
    launches0 = bs.kernel_launches()
    comm0 = ctx.comm_stats()
    barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clk:
        barrier()
        ev0.record(stream)
        res = ctx.run(y, x, epochs=args.steps, mu0=mu0, seed=7, rows_per_epoch=aM, cols_per_epoch=gN,
                      flags=sched | bs.RESUME, lam=lam)
        ev1.record(stream)
        barrier()
    launches = bs.kernel_launches() - launches0
    # the per-phase CUDA events (BSGD_TIMING) come from a separate run of the same epochs: the
    # timed run above is the library's own path (small problems run as one CUDA graph)
    res_t = ctx.run(y, x, epochs=args.steps, mu0=mu0, seed=7, rows_per_epoch=aM, cols_per_epoch=gN,
                    flags=sched | bs.RESUME | bs.TIMING, lam=lam)
    barrier()
    t_ms = ev0.elapsed_time(ev1)
    t = torch.tensor([t_ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    t_ms = float(t.item())
    visits_fp = float(res.visits.sum())       # this rank's FP visits (BP visits are equal)
    vt = torch.tensor([visits_fp], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(vt)
    visits_all = 2.0 * float(vt.item())       # FP + BP, all ranks
    epochs_per_s = args.steps / (t_ms / 1e3)
    # per-kernel roofline for the dominant kernel (live CUDA events on the launch stream)
    ph = res_t.t_ms                            # [steps][fp, residual, bp, step, tv/eud, total]
    fp_ms, res_ms, bp_ms, st_ms = (float(np.mean(ph[:, k])) for k in range(4))
    vis_ep = float(np.mean(res.visits))
    peak, peak_src = load_peaks()
    prof = load_traffic()
    # The dominant kernel is the projector pair: the FP and the BP launches are one and the
    # same Siddon traversal (each ~48 % of the step) and SURVEY §8d's unit of work is the
    # FP+BP visit pair (4 B gathered + 8 B reduced = 12 B).  Reporting the pair keeps the
    # line stable when the two are within noise of each other; fp_frac / bp_frac below.
    dms = fp_ms + bp_ms
    dbytes = 12.0 * vis_ep
    achieved = dbytes / (dms / 1e3) / 1e9
    traffic = None
    if all(prof.get(k, {}).get("dram_bytes_per_visit") is not None for k in ("fp", "bp")):
        traffic = (prof["fp"]["dram_bytes_per_visit"] + prof["bp"]["dram_bytes_per_visit"]) * vis_ep
    # e2e: the same metric through the C ABI with HOST buffers (pinned), copies inside
    e2e = None
    if not args.no_e2e:
        yh = y.cpu().pin_memory()
        xh = torch.zeros(n_owned, dtype=torch.float32).pin_memory()
        # untimed warm-up of the host-buffer path (one-time staging allocations, copy stream)
        ctx.run(yh, xh, epochs=1, mu0=mu0, seed=7, rows_per_epoch=aM, cols_per_epoch=gN, flags=sched, lam=lam)
        xh.zero_()
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        ctx.run(yh, xh, epochs=args.steps, mu0=mu0, seed=7, rows_per_epoch=aM, cols_per_epoch=gN, flags=sched,
                lam=lam)
        e1.record(stream)
        barrier()
        te = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e = {"value": args.steps / (float(te.item()) / 1e3), "unit": "epochs/s",
               "h2d_bytes_per_step": int(4 * g.n_rays / args.steps) + int(4 * n_owned / args.steps),
               "d2h_bytes_per_step": int(4 * n_owned / args.steps),
               "what": ("bsgd_run(y, x on pinned host memory): y and x uploaded (on a copy stream, "
                        "overlapped with the first epoch), K epochs, x copied back")}
        del yh, xh
    allreduce = None
    if world > 1:   # the epoch's exchange on its own: the partial sums of one row block
        count = (g.n_views // p.M) * g.det_u * g.det_v
        ms = ctx.allreduce_time(count, iters=5, stream=stream)
        tt = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
        nbytes = 4.0 * count
        allreduce = {"bytes": nbytes, "ms": ms, "algbw_gbs": nbytes / (ms / 1e3) / 1e9,
                     "bus_gbs": nbytes / (ms / 1e3) * 2 * (world - 1) / world / 1e9,
                     "vs_gbs": 900.0, "measured_ref_gbs": 725.0,
                     "what": "bsgd_allreduce_time: ncclAllReduce (sum, fp32) of the residual's partial-sum buffer "
                             "(72 views x 1024^2 rays), 5 back-to-back calls timed with CUDA events on the launch "
                             "stream, max over ranks; busbw = S/t x 2(G-1)/G",
                     "residual_phase_ms": res_ms}
    # N2: the residual exchange.  world > 1: the bytes all ranks sent in the timed
    # epochs (bsgd_comm_stats, band mode by default); always: the library's host plan of one
    # epoch's exchange at G = 2, 4, 8 for this config (band overlap rows vs the ring allreduce),
    # averaged over the M row blocks
    # per-slab ray-voxel intersections over all views (the exact COUNT traversal): the load
    # balance of a G-rank z-slab sharding (N3); balanced slabs with --balanced
    balance = None
    try:
        if world == 1 and p.blocks[:2] == (1, 1):
            v = ctx.visit_table().sum(axis=(1, 2)).astype(np.float64)
            shares = v / v.sum()
            balance = {"z_splits": [int(ctx.block_box(j)[0][2]) for j in range(p.N)] + [int(p.dims[2])],
                       "slab_visit_shares": [round(float(x), 5) for x in shares],
                       "visit_spread": float((v.max() - v.min()) / v.mean()),
                       "ideal_speedup": {str(G): float(1.0 / max(shares.reshape(G, -1).sum(axis=1)))
                                         for G in (2, 4, 8) if p.N % G == 0}}
    except Exception as exc:   # noqa: BLE001 -- auxiliary
        balance = {"error": f"{type(exc).__name__}: {exc}"[:300]}
    exchange = {"plan_per_epoch": {}}
    try:
        for G in (2, 4, 8):
            if p.N % G:
                continue
            bb = fb = 0
            for i in range(p.M):
                pl = ctx.exchange_plan(G, ctx.row_block_views(i))
                bb += pl["band_bytes"]
                fb += pl["full_bytes"]
            exchange["plan_per_epoch"][str(G)] = {"band_bytes": bb / p.M, "full_allreduce_bytes": fb / p.M,
                                                   "reduction": (fb / bb) if bb else None}
        if world > 1:
            cs = ctx.comm_stats()
            sent = torch.tensor([float(cs["bytes_sent"] - comm0["bytes_sent"])], dtype=torch.float64, device="cuda")
            dist.all_reduce(sent)
            exchange.update({"mode": cs["mode"], "timed_bytes_per_epoch_all_ranks": float(sent.item()) / args.steps})
    except Exception as exc:   # noqa: BLE001 -- auxiliary
        exchange["error"] = f"{type(exc).__name__}: {exc}"[:300]
    tv = None
    if not args.no_tv:   # an auxiliary measurement: never lose the main line over it
        try:
            tv = time_tv(bs, ctx, x, mu0 * lam, p, aM, gN, world, stream, t_ms / args.steps, peak)
        except Exception as exc:   # noqa: BLE001
            tv = {"error": f"{type(exc).__name__}: {exc}"[:300]}
    ctx.close()
    if rank != 0:
        return 0
    cpu = None
    if world == 1 and not args.no_cpu and args.config == "cfg5":
        # the same measurement as the --impl reference arm (measure_oracle), fewer steps
        r = measure_oracle(steps=3, warmup=1)
        one = oracle_one_thread()
        cpu = {"value": r["value"], "unit": "epochs/s", "cores": r["cores"], "kind": "oracle",
               "sample": r["sample"] + f" (this run's GPU epochs: {vis_ep:.4g} FP visits)",
               "intersections_per_s": r["vps"], "cpu_model": _cpu_model(), "one_thread": one}
    line = {
        "metric": METRIC, "value": epochs_per_s, "unit": "epochs/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t_ms / args.steps, "higher_is_better": True,
        "scaling": "weak" if args.eq8 else "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "intersections_per_s": visits_all / (t_ms / 1e3),
        "config": {"workload": workload(p) + (f" [Eq. 8 schedule at NodeNum = {world}: alpha*M = "
                                              f"{res.sel_rows.shape[1]}, gamma*N = {res.sel_cols.shape[1]}, "
                                              "columns stratified by owner]" if args.eq8 else "")
                   + (" [BSGD_DETERMINISTIC: fixed-point BP]" if args.det else "")
                   + (" [work-balanced slab thicknesses]" if args.balanced else ""),
                   "global_batch": int(res.sel_rows.shape[1]) * (g.n_views // p.M),
                   "parallelism": f"z-slab{world}" if p.blocks[:2] == (1, 1) else f"blocks{world}",
                   "l2": ("inputs larger than L2 (537 MB slabs, 3.0 GB y); no flush needed" if p.name == "cfg5"
                          else "auxiliary workload: inputs may be L2-resident, no flush (not the headline)"),
                   "visits_per_epoch_fp": visits_all / 2.0 / args.steps,   # all ranks
                   "fp64": "ray parameters fp64, values fp32"},
        "phase_ms": {"fp": fp_ms, "residual_allreduce": res_ms, "bp": bp_ms, "step": st_ms},
        "allreduce": allreduce,
        "exchange": exchange,
        "balance": balance,
        "roofline": {"bound": "hbm",
                     "kernel": "projector pair k_project3<FP> + k_project3<BP> (+ k_project2 steep-only companions)",
                     "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "peak_source": peak_src,
                     "algorithmic_bytes": f"12 B x {vis_ep:.4g} visit pairs per FP+BP launch pair",
                     "time_ms": dms,
                     "fp_frac": (4.0 * vis_ep / (fp_ms / 1e3) / 1e9) / peak,
                     "bp_frac": (8.0 * vis_ep / (bp_ms / 1e3) / 1e9) / peak,
                     "fp_plus_bp_frac": (12.0 * vis_ep / ((fp_ms + bp_ms) / 1e3) / 1e9) / peak},
        "tv_prox": tv,
        "clocks": clk.summary(),
        "gpu_launches": int(launches),
        "e2e": e2e,
        "cpu_baseline": cpu,
    }
    print(json.dumps(line), flush=True)
    return 0


def time_tv(bs, ctx, x, w, p, aM, gN, world, stream, epoch_ms, peak, iters=20, calls=3):
    """The TV proximal call of Algo 4 line 16 on this rank's owned volume,
    timed on its own (CUDA events on the launch stream, max over ranks): 20 FGP iterations.
    Algorithmic HBM bytes per call of the path that runs (TV):
      one rank (k_tv_fgp_z2, two iterations per pass): read p_{k-1}, p_{k-2} (24 B) + b (4 B),
        write p_k, p_{k+1} (24 B) = 52 B per voxel per pair; the first pair reads only b (28 B);
      several ranks (k_tv_fgp_z, one iteration per launch): read p_{k-1}, p_{k-2}, b, write p_k
        = 40 B per voxel; k = 1 reads only b (16 B), k = 2 reads p_1 and b (28 B);
    plus the final x = b - w grad^T p in place (read b, 3 p, write x: 20 B)."""
    import torch
    import torch.distributed as dist
    xt = x.clone()
    ctx.tv_prox(xt, w, iters)                  # untimed: allocates the dual fields
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l0 = bs.kernel_launches()
    e0.record(stream)
    for _ in range(calls):
        ctx.tv_prox(xt, w, iters)
    e1.record(stream)
    torch.cuda.synchronize()
    launches = (bs.kernel_launches() - l0) // calls
    t = torch.tensor([e0.elapsed_time(e1) / calls], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    n = x.numel()
    pairs = world == 1 and p.blocks[:2] == (1, 1) and p.dims[0] % 4 == 0 and os.environ.get("BSGD_TV_Z2", "1") != "0"
    if pairs:
        per_voxel = 28.0 + 52.0 * (iters // 2 - 1) + (40.0 if iters % 2 else 0.0) + 20.0
        kernel = "k_tv_fgp_z2 (two FGP iterations per pass) x iters/2 + k_tv_out"
        what = "52 B per voxel per two FGP iterations (28 B in the first pair) + 20 B final"
    else:
        per_voxel = 16.0 + 28.0 + 40.0 * (iters - 2) + 20.0
        kernel = ("k_tv_fgp_z (one FGP iteration per launch) x iters + k_tv_out" if p.blocks[:2] == (1, 1)
                  else "k_tv_u + k_tv_pq per iteration + k_tv_u")
        what = "40 B per voxel per FGP iteration (16 B at k = 1, 28 B at k = 2) + 20 B final"
    nbytes = n * per_voxel
    period = max(1, round(p.M * p.N / (aM * gN)))
    del xt
    return {"ms_per_call": ms, "iters": iters, "w": w, "voxels_per_rank": n, "launches_per_call": int(launches),
            "kernel": kernel, "algorithmic_bytes": f"{nbytes:.4g} B per call ({what})",
            "achieved_gbs": nbytes / (ms / 1e3) / 1e9, "frac": nbytes / (ms / 1e3) / 1e9 / peak,
            "period_epochs": period,
            "epochs_per_s_tv_amortised": 1e3 / (epoch_ms + ms / period)}


def self_launch(args) -> int:
    """`bench.py --gpus N` outside torchrun: launch N ranks of this same command line with
    torch.distributed.run (one process per GPU, rendezvous on 127.0.0.1), rank 0 prints."""
    import socket
    if not args.dry_run:
        import torch
        have = torch.cuda.device_count()
        if have < args.gpus:
            sys.stderr.write(f"bench.py: --gpus {args.gpus} requested but only {have} CUDA device(s) are "
                             f"visible; refusing to time fewer GPUs than requested\n")
            return 1
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def dry_run(args, rank, world) -> int:
    """--dry-run: the multi-rank plumbing only (gloo on CPU): every rank contributes 1 to an
    all-reduce; rank 0 prints what would be timed."""
    import torch
    import torch.distributed as dist
    t = torch.ones(1)
    if world > 1:
        dist.all_reduce(t)
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": world, "ranks_seen": int(t.item()),
                          "steps": args.steps, "warmup": args.warmup}), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-tv", action="store_true", help="skip the separate TV-prox timing")
    ap.add_argument("--det", action="store_true", help="BSGD_DETERMINISTIC (fixed-point BP reductions)")
    ap.add_argument("--eq8", action="store_true",
                    help="Eq. 8 schedule (gamma N = G, alpha M from Eq. 8), stratified by owner: weak scaling")
    ap.add_argument("--cheap-data", action="store_true", help="uniform random y instead of analytic projections")
    ap.add_argument("--balanced", action="store_true",
                    help="work-balanced z-slab thicknesses (bsgd_balanced_z_splits; SURVEY §8f N3)")
    ap.add_argument("--dry-run", action="store_true", help="multi-rank launch check on CPU (gloo), no GPU work")
    ap.add_argument("--config", default="cfg5", choices=["cfg1", "cfg2", "cfg3", "cfg4", "cfg5"],
                    help="workload (cfg5 = the BASELINE.json headline; the others for DESIGN tables)")
    args = ap.parse_args()
    if args.gpus < 1:
        ap.error("--gpus must be >= 1")
    env_world = os.environ.get("WORLD_SIZE")
    if env_world is None and args.gpus > 1 and args.impl == "ours":
        return self_launch(args)
    rank = int(os.environ.get("RANK", "0"))
    world = int(env_world) if env_world is not None else 1
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank, world if env_world is not None else args.gpus)
    if world != args.gpus:
        sys.stderr.write(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}; refusing to mislabel the run\n")
        return 1
    if args.dry_run:
        if world > 1:
            import torch.distributed as dist
            dist.init_process_group("gloo")
        try:
            return dry_run(args, rank, world)
        finally:
            if world > 1:
                import torch.distributed as dist
                dist.destroy_process_group()
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        return run_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    sys.exit(main())
