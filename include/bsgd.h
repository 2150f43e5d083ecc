/*
 * bsgd.h — C ABI of the B200-native BSGD hot path (Gao, Biguri, Blumensath,
 * arXiv 1903.11874, "Block stochastic gradient descent for large-scale
 * tomographic reconstruction in a parallel network").
 *
 * Problem (§I, Eq. 1-2):  min_x 1/2 ||y - A x||^2, where A is the
 * non-negative Siddon system matrix, never stored: A x (forward projection, FP)
 * and A^T r (back projection, BP) are computed on the fly by CUDA kernels.
 * Partition (§II, Eq. 3): M row blocks I_i (sets of whole views,
 * PAPER.md:449) x N column blocks J_j (equal boxes of a bx x by x bz grid).
 *
 * Conventions shared by every call
 *  - Units: voxel edge = 1; volume centred at the rotation centre; voxel
 *    (ix,iy,iz) covers [ix - nx/2, ix+1 - nx/2) x ... (half-open).
 *  - Projections: float32, layout [view][v][u] (u fastest), ray id
 *    (view*det_v + iv)*det_u + iu, full length n_views*det_v*det_u.
 *  - Images: float32, BLOCK-MAJOR: block j = (jz*by + jy)*bx + jx, then
 *    [z][y][x] inside the block.  For z-slab grids (1,1,N) this is the plain
 *    [z][y][x] volume.  A rank owns the contiguous blocks
 *    [rank*N/world, (rank+1)*N/world); "x_owned" is those blocks back to back.
 *  - Pointers: "device" = CUDA device memory of the ctx's device; "host" = CPU
 *    memory.  bsgd_run accepts y / x_owned / x_true in either (detected with
 *    cudaPointerGetAttributes; host buffers are copied in and x copied back).
 *  - Streams: every enqueueing call takes a cudaStream_t as void* (NULL = the
 *    legacy default stream).  Calls are asynchronous unless stated otherwise.
 *    Consecutive calls on one ctx may use different streams: each call's stream
 *    first waits for the work the previous call enqueued (the calls share the
 *    ctx's launch tables and scratch buffers), so a ctx's calls execute in
 *    call order whatever streams they name.
 *  - Ownership: the caller owns every buffer it passes; the ctx owns its
 *    internal state (z^j, g_hat^i, g, r, transposed image copy, scratch),
 *    allocated at create through `bsgd_alloc` (NULL = cudaMalloc).
 *  - Errors: every call returns bsgd_status; nothing throws across the ABI.
 *    Invalid arguments are rejected before any device work (state unchanged).
 *    A CUDA or NCCL failure poisons the ctx (BSGD_E_POISONED afterwards).
 *    bsgd_last_error() gives a message.
 *  - Concurrency: one ctx per process per GPU; not thread-safe.  Collective
 *    calls (bsgd_create with world > 1, bsgd_step, bsgd_run) must be issued in
 *    the same order on every rank.
 */
#ifndef BSGD_H
#define BSGD_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BSGD_ABI_VERSION 4   /* 4: bsgd_create_ex (unequal z-slabs), band exchange queries */

typedef struct bsgd_ctx_s* bsgd_ctx;

typedef enum {
    BSGD_OK = 0,
    BSGD_E_GEOMETRY = 1,   /* n_views < 1, zero detector elements, non-finite vectors, zero ray direction */
    BSGD_E_PARTITION = 2,  /* M < 1 or M > n_views, dims not divisible by the block grid, N % world != 0   */
    BSGD_E_DIMENSION = 3,  /* block / row block / view id out of range, rect outside the detector          */
    BSGD_E_CONTRACT = 4,   /* invalid selection (duplicate / unsorted), mu not finite, bad flags            */
    BSGD_E_CUDA = 5,
    BSGD_E_NCCL = 6,
    BSGD_E_OOM = 7,
    BSGD_E_POISONED = 8
} bsgd_status;

typedef enum { BSGD_PARALLEL = 0, BSGD_FAN = 1, BSGD_CONE = 2 } bsgd_beam;

/* Scan geometry (Fig. 3; §III-E).  vecs: host
 * fp64 [n_views][12] = {src (fan/cone) or unit ray direction (parallel),
 * detector centre, detector u step, detector v step}, copied at create.
 * Ray (view, iv, iu) passes through det + (iu-(nu-1)/2) u + (iv-(nv-1)/2) v;
 * fan/cone rays start at src; 2D = det_v 1 and nz 1.                          */
typedef struct { int32_t beam, n_views, det_u, det_v; const double* vecs; } bsgd_geometry;
typedef struct { int32_t nx, ny, nz; } bsgd_dims;
typedef struct { int32_t bx, by, bz; } bsgd_block_grid;
/* Row blocks ("randomly partitioned the 360 projections into 5
 * groups"): kind 0 = seeded random partition, 1 = contiguous, 2 = interleaved.
 * tiles_u x tiles_v = sub-detector tiles of BSGD-IM (Fig. 2). */
typedef struct { int32_t M, kind; uint64_t seed; int32_t tiles_u, tiles_v; } bsgd_row_grid;
/* Virtual ranks: `world` logical ranks in ONE process on one GPU,
 * each a bsgd_ctx driven by its own host thread and CUDA stream.  The collectives of the
 * NCCL path become device copies between the ranks' buffers, ordered by events and host
 * barriers: the allreduce is a fixed-order (rank-ascending) device sum, the halo
 * send/recv a peer copy.  Exercises ownership, partial sums, allreduces and TV halos
 * exactly as G GPUs would, on one GPU.  A rank that never reaches a collective makes the
 * others fail with BSGD_E_NCCL after 120 s.                                              */
typedef struct bsgd_vgroup_s* bsgd_vgroup;
bsgd_status bsgd_vgroup_create(int32_t world, bsgd_vgroup* out);
void bsgd_vgroup_destroy(bsgd_vgroup group);   /* after every member ctx is destroyed   */

/* Multi-GPU: one process per GPU; nccl_id = 128 bytes from bsgd_nccl_unique_id
 * on rank 0, broadcast by the caller (NULL when world == 1).  vgroup: non-NULL for a
 * virtual rank (bsgd_vgroup_create; nccl_id is then ignored).                   */
typedef struct { int32_t rank, world; const uint8_t* nccl_id; bsgd_vgroup vgroup; } bsgd_dist;
/* Device allocator used for ALL ctx state (Python points it at the torch
 * caching allocator).  NULL = cudaMalloc/cudaFree.                           */
typedef struct {
    void* (*alloc)(size_t bytes, void* stream, void* user);
    void (*free)(void* ptr, size_t bytes, void* stream, void* user);
    void* user;
} bsgd_alloc;

/* ---- pure host functions (no ctx, no device) ---------------------------- */
int32_t bsgd_abi_version(void);
/* Number of CUDA kernels this library has launched in this process (all
 * contexts); the bench reports the count inside its timed region.           */
uint64_t bsgd_kernel_launches(void);
const char* bsgd_last_error(bsgd_ctx ctx /* NULL = thread-local last error */);
/* Circular orbit per-view vectors: theta_v = v*arc/n_views
 * degrees with exact-quadrant trig; src = OP(cos,sin,0), det = -OD(cos,sin,0),
 * u = pitch_u(-sin,cos,0), v = pitch_v(0,0,1); parallel: dir = -(cos,sin,0),
 * det = 0.  vecs_out: host [n_views][12].                                     */
bsgd_status bsgd_geometry_circular(int32_t beam, int32_t n_views, double arc_deg, double OP, double OD,
                                   int32_t det_u, int32_t det_v, double pitch_u, double pitch_v,
                                   double* vecs_out);
/* SplitMix64 counter RNG (reading A3): m of n without replacement, sorted.
 * stream 0 = view partition, 1 = row blocks, 2 = column blocks, 3 = IM tiles. */
bsgd_status bsgd_sample(uint64_t seed, int32_t stream, int32_t epoch, int32_t n, int32_t m, int32_t* out);
/* Stratified column-block selection (BSGD_STRATIFIED, reading A31): the n
 * blocks are cut into `strata` equal consecutive strata (the owners' block ranges) and
 * m / strata blocks are drawn in each, by the partial Fisher-Yates of bsgd_sample over the
 * stratum with draw counters k = s * (n / strata) + i on stream 2; out sorted.  strata = 1
 * equals bsgd_sample(seed, 2, epoch, n, m).  Errors: strata must divide n and m.          */
bsgd_status bsgd_sample_stratified(uint64_t seed, int32_t epoch, int32_t n, int32_t m, int32_t strata,
                                   int32_t* out);
/* Row-block partition: views_out [n_views] (blocks back to back, each sorted),
 * offsets_out [M+1].                                                          */
bsgd_status bsgd_view_partition(int32_t n_views, int32_t M, int32_t kind, uint64_t seed,
                                int32_t* views_out, int32_t* offsets_out);
/* Eq. 8: gamma = min{1, nodes/N}, alpha = nodes/(M N gamma);
 * counts alpha*M and gamma*N rounded half up, at least 1 (reading A4).        */
bsgd_status bsgd_eq8(int32_t nodes, int32_t M, int32_t N, int32_t* rows_per_epoch, int32_t* cols_per_epoch);
/* Blocks owned by a rank: [*first, *first + *count).                          */
bsgd_status bsgd_owned_blocks(int32_t N, int32_t world, int32_t rank, int32_t* first, int32_t* count);
/* 128-byte NCCL unique id (call on rank 0 only, then broadcast).             */
bsgd_status bsgd_nccl_unique_id(uint8_t* out128);

/* ---- context ------------------------------------------------------------- */
bsgd_status bsgd_create(const bsgd_geometry* geom, bsgd_dims dims, bsgd_block_grid blocks,
                        bsgd_row_grid rows, const bsgd_dist* dist /* NULL = single GPU */,
                        const bsgd_alloc* alloc /* NULL = cudaMalloc */, bsgd_ctx* out);
/* Options of bsgd_create_ex.
 * z_splits: host [bz + 1] plane indices 0 = s_0 < s_1 < ... < s_bz = nz, or NULL.  Column
 *   blocks J_j of Eq. 3 need not be equal: with a z-slab grid (1, 1, bz),
 *   block j is the slab of planes [s_j, s_{j+1}) (slab thicknesses chosen so
 *   every rank traverses the same number of ray-voxel intersections, bsgd_balanced_z_splits).
 *   Block-major buffers (x_owned, x_true, g-hat / g of bsgd_get_state) then keep the stride of
 *   the THICKEST slab (bsgd_info.block_voxels): block j's [z][y][x] values, then zeros to the
 *   end of its row (inputs must carry zero tails; outputs keep them).                      */
typedef struct {
    const int32_t* z_splits;
} bsgd_create_opts;
/* bsgd_create with options (NULL opts = bsgd_create).  Errors as bsgd_create, plus
 * BSGD_E_PARTITION for z_splits on a non-slab grid, not running 0..nz or not increasing.   */
bsgd_status bsgd_create_ex(const bsgd_geometry* geom, bsgd_dims dims, bsgd_block_grid blocks,
                           bsgd_row_grid rows, const bsgd_dist* dist, const bsgd_alloc* alloc,
                           const bsgd_create_opts* opts, bsgd_ctx* out);
/* Box of column block j in grid coordinates: lo [3], hi [3] (half-open).                  */
bsgd_status bsgd_block_box(bsgd_ctx ctx, int32_t j, int32_t* lo, int32_t* hi);
/* Work-balanced z-splits: ctx must be a one-rank z-slab context whose slabs
 * are the candidate boundaries (e.g. nz/8 slabs of 8 planes); from its exact visit table (the
 * COUNT traversal of every view, bsgd_visit_table) it picks splits [n_slabs + 1] so that the
 * cumulative ray-voxel intersections of slab k end nearest to (k+1)/n_slabs of the total.
 * Synchronises the stream.  Errors: BSGD_E_PARTITION (non-slab grid, world > 1, n_slabs > N),
 * BSGD_E_CONTRACT (NULL, n_slabs < 1).                                                    */
bsgd_status bsgd_balanced_z_splits(bsgd_ctx ctx, int32_t n_slabs, int32_t* splits, void* stream);
void bsgd_destroy(bsgd_ctx ctx);

typedef struct {
    int32_t N, M, n_views, det_u, det_v, owned_first, owned_count, tiles;
    int64_t block_voxels, n_rays, owned_voxels;
    int32_t block_dims[3];
    uint64_t device_bytes;   /* bytes of ctx-owned device state */
} bsgd_info;
bsgd_status bsgd_get_info(bsgd_ctx ctx, bsgd_info* out);
/* Views of row block i: out [n] (n = size of I_i, sorted); *n returns the size. */
bsgd_status bsgd_row_block_views(bsgd_ctx ctx, int32_t i, int32_t* out, int32_t* n);

/* ---- single operators (no collective; device pointers; caller's stream) ---
 * views: host [n_views] view ids; rects: host [n_views][4] detector rect
 * (u0,u1,v0,v1) half-open per view, or NULL = whole detector.
 * bsgd_forward: proj[rays] (=|+=) A_{views,rects}^{J_j} x_block      (Algo 1 l.5)
 *   x_block: device block j (block layout); proj: device, full length; rays
 *   outside the views/rects are not touched.
 * bsgd_back:    g_block (=|+=) scale * (A_{views,rects}^{J_j})^T proj (Algo 1 l.9, PAPER.md:143;
 *   the algorithm uses scale = 2).                                            */
bsgd_status bsgd_forward(bsgd_ctx ctx, int32_t n_views, const int32_t* views, const int32_t* rects,
                         int32_t col_block, const float* x_block, float* proj, int32_t accumulate,
                         void* stream);
bsgd_status bsgd_back(bsgd_ctx ctx, int32_t n_views, const int32_t* views, const int32_t* rects,
                      int32_t col_block, const float* proj, float* g_block, float scale,
                      int32_t accumulate, void* stream);
/* Exact per-(owned block, view, tile) ones-pass masses w = sum over the tile's
 * rays of the chord through the block box (the L1 norm of A_tile^J; reading A9),
 * and the integer importance table q = floor(2^16 w / sum_t w) used by the
 * sampler.  host out: [owned_count][n_views][tiles].                        */
bsgd_status bsgd_im_weights(bsgd_ctx ctx, double* w_out, uint32_t* q_out);
/* As bsgd_im_weights for a chosen weight kind: 0 = L1 mass (chord sums, the default of
 * BSGD_IS), 1 = projection area (count of tile rays with chord > 1e-6, BSGD_IS_AREA).     */
bsgd_status bsgd_im_table(bsgd_ctx ctx, int32_t kind, double* w_out, uint32_t* q_out);
/* The visit table behind the intersections/s metric (SURVEY §8b, §8d "exact visit counts"):
 * nnz_out[b][view][tile] (host, owned blocks x n_views x tiles) = number of ray-voxel
 * intersections of block first+b, view `view`, detector tile `tile` -- Siddon segments longer
 * than 1e-6 of a main-axis slice, from one COUNT traversal at the first call (cached).  */
bsgd_status bsgd_visit_table(bsgd_ctx ctx, uint64_t* nnz_out);

/* ---- algorithm state ------------------------------------------------------ */
/* Algo 1 line 1: z^j = 0, g_hat^i = 0, g = 0, r = y, epoch = 0.
 * y: device, full length, replicated on every rank.                          */
bsgd_status bsgd_reset(bsgd_ctx ctx, const float* y, void* stream);

enum {
    BSGD_IS = 1,            /* BSGD-IM, Algo 2                     */
    BSGD_IS_UNIFORM = 2,    /* BSGD-RAN: uniform tile draws            */
    BSGD_TV = 4,            /* BSGD-TV, Algo 4                     */
    BSGD_AUTO_MU = 8,       /* Algo 3                             */
    BSGD_SGD = 16,          /* Eq. 4 mini-batch SGD baseline       */
    BSGD_RESUME = 32,       /* bsgd_run: continue from the current state (no reset)   */
    BSGD_TIMING = 64,       /* bsgd_run: per-phase CUDA-event times into the log      */
    BSGD_STRATIFIED = 128,  /* column blocks drawn per owner stratum (bsgd_sample_stratified,
                               run_params.strata): under Eq. 8 with gamma N = G
                               every rank gets gamma N / G blocks, none idles (reading A31) */
    BSGD_IS_AREA = 256,     /* with BSGD_IS: weights = number of tile rays that cross the block
                               (chord > 1e-6), the "projection area" reading of PAPER.md:162,
                               instead of the default L1 mass (reading A9)                  */
    BSGD_TV_CHAMBOLLE = 512, /* with BSGD_TV: Chambolle-2004 dual iteration instead of FGP  */
    BSGD_LOG_TRUE_OBJ = 2048, /* bsgd_run: log obj_true[k] = 1/2 ||y - A x_k||^2 (GAP^2 / 2,
                               PAPER.md:508) from a fresh FP of every view and block after
                               every epoch (validation only: ~M x an epoch's FP)           */
    BSGD_DETERMINISTIC = 1024 /* bsgd_run / bsgd_step: BP by 64-bit fixed-point reductions
                               (scale 2^e from max|r|, resolution ~1e-15 max|r|): g_hat, g and
                               x do not depend on the order of the BP threads; bit-identical
                               runs (SURVEY §8b Determinism).  64-bit REDs double the BP's L2
                               reduction traffic: cfg5 BP 105 -> 197 ms, 4.6 -> 3.2 epochs/s */
};

/* One epoch of Algo 1 / Algo 2 with an explicit selection (identical on all
 * ranks).  rows: sorted row-block ids; cols: sorted column-block ids;
 * im_tiles: NULL (Algo 1) or host [n_cols][V_sel] tile ids, V_sel = number of
 * views of the selected row blocks in ascending row-block order (Algo 2 l.5).
 * flags: BSGD_SGD, BSGD_DETERMINISTIC.  Contains the residual allreduce when world > 1. */
typedef struct {
    int32_t n_rows; const int32_t* rows;
    int32_t n_cols; const int32_t* cols;
    const int32_t* im_tiles;
} bsgd_selection;
bsgd_status bsgd_step(bsgd_ctx ctx, const float* y, float* x_owned, const bsgd_selection* sel,
                      float mu, uint32_t flags, void* stream);

typedef struct {
    uint64_t seed;
    int32_t epochs;
    int32_t rows_per_epoch, cols_per_epoch;   /* alpha*M, gamma*N; 0 = Eq. 8 with NodeNum = world */
    double mu0;
    uint32_t flags;
    double lambda;                            /* TV weight lambda of Eq. 5          */
    int32_t tv_iters, tv_period;              /* FGP iterations (20); period 0 = round(1/(alpha gamma)) */
    double eps, delta, t1, t2;                /* Algo 3 constants (reading A12: .05, .4, .5, 0)   */
    int32_t is_off_last_epochs;               /* final epochs without IS           */
    int32_t strata;                           /* BSGD_STRATIFIED: number of strata (0 = world)   */
    int32_t total_epochs;                     /* planned run length in GLOBAL epochs, for
                                                 is_off_last_epochs: IS is off in the epochs
                                                 k > total_epochs - is_off_last_epochs (k the
                                                 1-based global epoch, counting across RESUME
                                                 calls).  0 = this call ends the run (total =
                                                 global epoch at entry + epochs)               */
} bsgd_run_params;

/* Per-epoch log; every pointer is host memory and nullable.                  */
typedef struct {
    double* obj;        /* [epochs] 1/2 ||r||^2 of the maintained r (reading A30)       */
    double* rmse;       /* [epochs] RMSE(x, x_true) over all voxels (needs x_true)       */
    double* mu;         /* [epochs] step used in the epoch                              */
    int32_t* sel_rows;  /* [epochs][rows_per_epoch]                                     */
    int32_t* sel_cols;  /* [epochs][cols_per_epoch]                                     */
    uint64_t* visits;   /* [epochs] FP ray-voxel intersections (BP visits are equal)     */
    double* t_ms;       /* [epochs][6] fp, residual(+allreduce), bp, step, tv, total     */
    double* obj_true;   /* [epochs] 1/2 ||y - A x||^2 after the epoch (BSGD_LOG_TRUE_OBJ)   */
    double* tv;         /* [epochs] TV(x) after the epoch (Eq. 6; with BSGD_LOG_TRUE_OBJ)     */
    double* rmse_seen;  /* [epochs] RMSE(x, x_true) over the voxels some ray crosses (A^T 1 > 0;
                           reading A32), with BSGD_LOG_TRUE_OBJ and x_true                   */
} bsgd_run_log;

/* Run params->epochs epochs of BSGD (Algo 1) or its variants selected by
 * flags, sampling with the counter RNG from params->seed.  y, x_owned, x_true
 * may be host or device pointers (host: copied in / x copied back).
 * Synchronises `stream` before returning (the log is host memory).
 * Errors: BSGD_E_CONTRACT for bad parameters (unknown flags, mu0 <= 0, negative lambda or
 * tv_iters with BSGD_TV, bad strata); BSGD_E_PARTITION for BSGD_TV when world > 1 and a
 * rank would own part of a z-layer of the block grid (see bsgd_tv_prox).              */
bsgd_status bsgd_run(bsgd_ctx ctx, const float* y, float* x_owned, const float* x_true,
                     const bsgd_run_params* params, bsgd_run_log* log, void* stream);

/* Inspection (tests): copy internal state to / from host memory.
 * what: 0 = z^j of owned block slot `index` (n_rays floats, full length; the library stores
 *           only each view's detector footprint of the block, zero elsewhere, so set_state
 *           keeps just the footprint part of the given vector);
 *       1 = g_hat^i of (i = index / owned_count, owned slot = index % owned_count);
 *       2 = g of owned slot `index`;  3 = r (n_rays floats);
 *       4 = per-row-block ||r_I||^2 (M doubles);  5 = current mu (1 double).
 * bytes must match the item's size exactly.  Synchronous.                    */
bsgd_status bsgd_get_state(bsgd_ctx ctx, int32_t what, int32_t index, void* host_dst, size_t bytes);
bsgd_status bsgd_set_state(bsgd_ctx ctx, int32_t what, int32_t index, const void* host_src, size_t bytes);

/* sigma_max(A)^2 by `iters` power iterations on A^T A (all views, all blocks;
 * collective when world > 1).  Synchronous.                                   */
bsgd_status bsgd_power_iteration(bsgd_ctx ctx, int32_t iters, uint64_t seed, double* sigma_max_sq,
                                 void* stream);

/* The residual exchange of Algo 1 line 7 on its own (the ALLREDUCE of the partial
 * projections): `iters` sum-allreduces of the first `count` floats of the
 * ctx's partial-sum buffer over the ctx's communicator (NCCL, or the virtual-rank group),
 * enqueued on `stream` and timed there with CUDA events; *ms_out = mean milliseconds per
 * allreduce.  For the bench's bus-bandwidth figure; clobbers only that scratch buffer.
 * Collective: every rank calls it with the same count / iters.  Synchronous.
 * Errors: BSGD_E_CONTRACT if the ctx has no collective path (world == 1 without
 * BSGD_FORCE_NCCL), count < 1 or count > n_rays, iters < 1.                      */
bsgd_status bsgd_allreduce_time(bsgd_ctx ctx, int64_t count, int32_t iters, void* stream, double* ms_out);

/* Residual exchange accounting (the ALLREDUCE of PAPER.md:99), cumulative since
 * bsgd_create, host-side counters of what this rank SENT for line 7 of the epochs it ran:
 * band mode (world > 1, default): the partial projection sums on the detector rows where this
 * rank's band (the rows its blocks project into) overlaps a peer's, one message per (peer,
 * view); LSA mode (environment BSGD_EXCHANGE=lsa): the same overlap rows, read by this rank's
 * residual kernel directly from each peer's partial-sum buffer (an NCCL symmetric window;
 * counted as the bytes this rank READ, one "message" per peer); full mode (BSGD_EXCHANGE=full):
 * the ring allreduce's 2 (G-1)/G of the selected rows' buffer per epoch.  *band_mode
 * (nullable) = 1 in band mode, 2 in LSA mode, 0 in full mode.  In band and LSA mode the
 * residual r is formed on this rank's band rows only (bsgd_get_state's r is valid there;
 * rows no band covers keep r = y).  Errors: BSGD_E_CONTRACT for NULL outputs.            */
bsgd_status bsgd_comm_stats(bsgd_ctx ctx, uint64_t* bytes_sent, uint64_t* messages, int32_t* band_mode);

/* Pure host function (no GPU): the detector band of rank `rank` of `world` -- per view v the
 * rows [bands_out[2v], bands_out[2v+1]) that its owned blocks [rank N/world, (rank+1) N/world)
 * project into (the union of the blocks' footprint rows, the same fp64 computation the band
 * exchange uses; [0, 0) when no row does).  bands_out: host [n_views][2].  Errors:
 * BSGD_E_CONTRACT, BSGD_E_GEOMETRY, BSGD_E_PARTITION as bsgd_create.                       */
bsgd_status bsgd_rank_bands_host(const bsgd_geometry* geom, bsgd_dims dims, bsgd_block_grid blocks, int32_t world,
                                 int32_t rank, int32_t* bands_out);

/* Host-only plan of the residual exchange for a hypothetical ownership of this ctx's block
 * grid by `world` ranks (rank g owns blocks [g N/world, (g+1) N/world)), for one epoch whose
 * selected row blocks hold the n_sel views `views` (host int32): *band_bytes = bytes all
 * ranks together send in band mode (the same band / overlap computation the band exchange
 * uses), *full_bytes = the ring allreduce's world x 2 (world-1)/world x n_sel x rays-per-view
 * x 4 B.  Pure host work; no collective.  Errors: BSGD_E_CONTRACT (NULL outputs, views out of
 * range), BSGD_E_PARTITION (N % world != 0).                                             */
bsgd_status bsgd_exchange_plan(bsgd_ctx ctx, int32_t world, int32_t n_sel, const int32_t* views,
                               uint64_t* band_bytes, uint64_t* full_bytes);

/* TV proximal step (Algo 4 line 16; TV of Eq. 5-6):
 * x_owned <- argmin_t 1/2 ||t - x_owned||^2 + w TV(t), by `iters` cold-start FGP iterations
 * on the dual (reading A16; the same call bsgd_run makes every tv_period epochs, with
 * w = mu lambda).  TV is the isotropic backward-difference TV of Eq. 6 over the WHOLE volume
 * (zero difference at index 0).  x_owned: device, this rank's owned blocks, block-major (the
 * layout of bsgd_run's x_owned), modified in place; enqueued on `stream`.  Collective when
 * world > 1 (z-plane halos by ncclSend/Recv; every rank calls it).  w = 0 or iters = 0
 * leaves x unchanged.  method: 0 = FGP (default of bsgd_run), 1 = Chambolle 2004 (tau = 1/8
 * in 2D, 1/12 in 3D; SURVEY §8c step 7's flag; bsgd_run with BSGD_TV_CHAMBOLLE).
 * Errors: BSGD_E_CONTRACT for NULL x, w < 0 or not finite, iters < 0 or an unknown method;
 * BSGD_E_PARTITION when world > 1 and a rank would own part of a z-layer of the block grid
 * (N / world not a multiple of bx * by): the stencil's only cross-rank neighbours must lie
 * in z.  z-slabs (1, 1, N) always qualify; so do the paper's 2x2x2 cubes at world = 2.    */
bsgd_status bsgd_tv_prox(bsgd_ctx ctx, float* x_owned, double w, int32_t iters, int32_t method,
                         void* stream);
/* TV(x) = sum over voxels of |grad x|_2 (isotropic backward differences, zero at index 0;
 * Eq. 6) of the whole volume: x_owned device (owned blocks, block-major),
 * *out host.  Collective when world > 1 (one halo plane + a 1-double allreduce).  Synchronous.
 * Errors: as bsgd_tv_prox (BSGD_E_PARTITION for partial z-layers per rank).               */
bsgd_status bsgd_tv_value(bsgd_ctx ctx, const float* x_owned, double* out, void* stream);

/* Comparison solvers on the same operators (the methods the paper
 * compares against in Figs. 12 and 18, cited but not listed
 * there; the textbook forms are in oracle/solvers.py).  With g(x) = 2 A^T (y - A x)
 * (reading A1) and the full operator A (all M row blocks, all N column blocks):
 *   GD     x+ = x + mu g(x)
 *   GD_BB  GD with the Barzilai-Borwein step mu_k = <s,s>/<s,w>, s = x_k - x_{k-1},
 *          w = g(x_{k-1}) - g(x_k); mu_0 = mu0; mu kept when <s,w> <= 0
 *   ISTA   x+ = prox_{mu lambda TV}(x + mu g(x))
 *   FISTA  z+ = prox_{mu lambda TV}(v + mu g(v)), t+ = (1 + sqrt(1 + 4t^2))/2,
 *          v+ = z+ + ((t - 1)/t+)(z+ - z), v_0 = x_0, t_0 = 1
 *   SVRG   per outer iteration x~ = x, G~ = g(x~); then svrg_m (0 = M) inner steps
 *          drawing one row block i (sampler stream 1, counter = global inner step):
 *          x <- x - mu M 2 A_I^T A_I (x - x~) + mu G~
 * The prox is Algo 4's FGP prox (tv_iters iterations; lambda = 0: none).
 * y (replicated, full length) and x_owned (owned blocks, block-major) are DEVICE
 * buffers; x_owned holds x_0 on entry and the result on return.  obj[k] (host,
 * nullable) = 1/2 ||y - A p_k||^2 at the point p_k whose full gradient iteration k
 * evaluates (x_k; v_k for FISTA; x~ for SVRG outer iteration k); mu[k] the step.
 * The BSGD state of the ctx is reset afterwards (as after bsgd_run without
 * BSGD_RESUME).  Synchronises the stream.  Collective (world > 1).            */
typedef enum {
    BSGD_SOLVER_GD = 0, BSGD_SOLVER_GD_BB = 1, BSGD_SOLVER_ISTA = 2, BSGD_SOLVER_FISTA = 3, BSGD_SOLVER_SVRG = 4
} bsgd_solver;
typedef struct {
    int32_t solver;
    int32_t iters;          /* outer iterations (SVRG) / iterations                      */
    double mu0;             /* step (GD_BB: initial step)                                 */
    double lambda;          /* TV weight of ISTA / FISTA (0 = plain)                      */
    int32_t tv_iters;       /* FGP iterations of the prox (20)                            */
    int32_t svrg_m;         /* SVRG inner steps per outer iteration (0 = M)               */
    uint64_t seed;          /* SVRG row-block draws                                       */
} bsgd_solve_params;
bsgd_status bsgd_solve(bsgd_ctx ctx, const float* y, float* x_owned, const bsgd_solve_params* params,
                       double* obj, double* mu, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* BSGD_H */
