// Internal declarations of the BSGD B200 library (not part of the ABI).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "bsgd.h"

namespace bsgd {

struct Error {
    bsgd_status code;
    std::string msg;
};

[[noreturn]] void fail(bsgd_status code, const std::string& msg);
void cuda_check(cudaError_t e, const char* what, const char* file, int line);
#define BSGD_CUDA(x) ::bsgd::cuda_check((x), #x, __FILE__, __LINE__)
void note_launch();   // counts this library's kernel launches (bsgd_kernel_launches)

// ---------------------------------------------------------------- host helpers
namespace host {
void cos_sin_deg(double theta, double* c, double* s);
void circular(int beam, int n_views, double arc, double OP, double OD, int nu, int nv, double pu,
              double pv, double* out);
uint64_t mix64(uint64_t z);
uint64_t rnd(uint64_t seed, uint32_t stream, uint32_t epoch, uint32_t k);
uint32_t bounded(uint64_t u, uint32_t n);
void select(uint64_t seed, int stream, int epoch, int n, int m, int32_t* out);
void select_stratified(uint64_t seed, int epoch, int n, int m, int strata, int32_t* out);
void view_partition(int n_views, int M, int kind, uint64_t seed, int32_t* views, int32_t* offsets);
void eq8(int nodes, int M, int N, int* aM, int* gN);
int im_draw(uint64_t seed, int epoch, uint32_t k, const uint32_t* q, int T, bool uniform);
}  // namespace host

// ---------------------------------------------------------------- kernels
struct KGeom {
    const double* vecs;  // device [n_views][12]
    int beam, nu, nv, n_views;
    int dims[3];
    double R;            // parallel-beam half length (|diag|/2 + 1)
};

// Footprint-restricted storage of z^j: per (owned block, view) the detector
// rectangle [u0,u1) x [v0,v1) the block's box projects into (the launch-culling footprint,
// u0/u1 multiples of 32 or nu) and the offset of its (u0, v0) element in the packed buffer;
// rays outside it have z^j = 0 and are not stored.
struct ZRect {
    int u0, u1, v0, v1;
    long long base;
    long long pad_;
};

// One column block as seen by a projection launch.
struct BlockDesc {
    const float* xN;     // FP source, block layout [z][y][x]
    const float* xT;     // FP source, transposed layout [z][x][y]
    float* outN;         // BP target (normal layout)
    float* outT;         // BP target (transposed layout)
    float* z;            // FP target: full-length projection vector (zr == NULL) or the packed
                         // footprint storage of the block's z (zr = its [n_views] ZRect table)
    const ZRect* zr;
    int lo[3], hi[3];    // box in grid coordinates
    int band_lo;         // first detector-row band with work for this block
    // Strides of the library's PADDED image copies (xN/xT, outN/outT point at voxel (0,0,0)
    // of the block interior): every row carries PAD_X zero floats on each side and every
    // block PAD_Z zero planes below and above, so a traversal step up to one cell outside
    // the block in the row or plane direction reads 0 (FP) / lands in the ignored border
    // (BP).  Normal layout [z][y][x]: row = bx + 2 PAD_X, plane = row * by; transposed
    // [z][x][y]: row = by + 2 PAD_X, plane = row * bx.
    int rowN, planeN, rowT, planeT;
};
constexpr int PAD_X = 32;  // keeps padded rows and their interiors 128-byte aligned (bx % 32 == 0)
constexpr int PAD_Z = 1;

struct ProjLaunch {
    KGeom g;
    int n_slots;               // views in this launch (grid.y)
    const int* views;          // device [n_slots]
    const int4* rects;         // device [n_blocks][n_slots] (u0,u1,v0,v1)
    int n_blocks;              // grid.z
    const BlockDesc* blocks;   // device [n_blocks]
    int max_rect_rays;
    int rows_per_band;         // R: detector rows per band (band-major CTA order)
    int n_chunks;              // CTAs per (band, slot)
    int n_bands;               // max bands per block (grid.x = n_bands * n_slots * n_chunks)
    const float* rproj;        // BP input (full length)
    float scale;               // BP scale (2 in Algo 1)
    int accumulate;            // FP: add into z instead of overwriting
    unsigned long long* visits;  // nullable counter
    const float* det_scale;    // PROJ_BPD: device scalar S (a power of two); the BP targets
                               // are then int64 fixed-point accumulators (value * S)
    uint2* v2_list;            // the warps k_project3 leaves to the v2 companion: (blockIdx.x,
    unsigned* v2_count;        //   blockIdx.z << 3 | warp), appended by k_project3; capacity =
                               //   the launch's warps (grid.x grid.z 8); nullptr: grid companion
};

// PROJ_BPD: the BP with order-independent (deterministic) 64-bit fixed-point reductions
enum { PROJ_FP = 0, PROJ_BP = 1, PROJ_COUNT = 2, PROJ_BPD = 3 };
#ifdef __CUDACC__
__host__ __device__
#endif
constexpr bool is_bp(int mode) { return mode == PROJ_BP || mode == PROJ_BPD; }
void launch_project(int mode, const ProjLaunch& L, cudaStream_t st);

// Block update / transpose modes of k_block_update.
enum { UPD_BSGD = 0, UPD_SGD = 1, UPD_OUT = 2, UPD_XT = 3, UPD_SGD_ACC = 4 };
struct UpdLaunch {
    int bd[3];            // block dims (x, y, z)
    int rowN, planeN, rowT, planeT;   // padded strides of accN / xN and accT / xT (see BlockDesc)
    float* accN;          // normal-layout BP accumulator, padded (interior zeroed after reading)
    float* accT;          // transposed-layout BP accumulator, padded (interior zeroed after reading)
    float* ghat;          // g_hat^i_J (UPD_BSGD)
    float* g;             // g_J
    float* x;             // x_J (normal layout)
    float* xT;            // x_J transposed, padded (written when x changes / UPD_XT)
    float* xN;            // x_J copy, padded (FP source)
    float* out;           // UPD_OUT target
    float mu;
    int final_;           // apply x += mu g and refresh xT
    int accumulate;       // UPD_OUT: add into out
};
void launch_block_update(int mode, const UpdLaunch& U, cudaStream_t st);

struct ResLaunch {
    int n_slots;
    const int* views;       // device [n_slots]
    const int* slot_row;    // device [n_slots] row-block id of the slot
    int per;                // rays per view
    const float* z;         // owned z vectors: packed footprint storage (ZRect table zr)
    const ZRect* zr;        // [s][n_views]
    int n_views;
    int nu;                 // detector columns (rays per view = per = nu * nv)
    long long n_rays;
    int s;                  // owned blocks
    const float* y;
    float* r;
    float* pc;              // compact partial sums [n_slots*per] (world > 1)
    double* normsq;         // [M]
    double* part;           // [n_slots][RES_GX] per-CTA partial ||r||^2 (fixed-order final sum)
    int M;                  // row blocks (normsq entries)
    int mode;               // 0 = fused r = y - sum z (world 1); 1 = pc = sum z; 2 = r = y - pc
};
constexpr int RES_GX = 64;   // max CTAs per view slot of k_residual
void launch_residual(const ResLaunch& R, cudaStream_t st);
// N2 band exchange (world > 1): the residual on the detector rows this rank's
// blocks project into.  Row v of slot k: covered_by = {h : bands[k][h] contains v}; if this
// rank is in it, r = y - sum_{h in covered_by, ascending} data[h][k][v][.] (the same sum, in
// the same order, on every rank sharing the row) and ||r||^2 counts it iff this rank is the
// lowest h; rows no band covers keep r = y and rank 0 counts them.
struct BandLaunch {
    int n_slots, per, nu, G, me;
    const int* views;           // [n_slots]
    const int2* bands;          // [n_slots][G] (lo, hi) detector rows of every rank's band
    const int2* range;          // [n_slots] rows this rank visits
    const float* const* data;   // [G] partial sums: own pc (compact [n_slots * per]) / the
                                // packed received chunks
    const long long* adj;       // [n_slots][G] element offset of peer h's chunk of slot k
                                // (element (k, v, u) at data[h][k per + v nu + u + adj])
    const float* y;
    float* r;
    double* part;               // [n_slots][RES_GX] per-CTA partial ||r||^2
};
void launch_residual_band(const BandLaunch& B, cudaStream_t st);
void launch_copy_rows(double* dst, const double* src, const int* rows, int n, cudaStream_t st);
// dst[t[3c+1] + i] = src[t[3c] + i], i < t[3c+2], for the n chunks c of the device table t
void launch_copy_chunks(const float* src, float* dst, const long long* t, int n, cudaStream_t st);
// R.normsq[i] = fixed-order sum of R.part over the slots of row block i (gx CTAs per slot)
void launch_normsq_final(const ResLaunch& R, int gx, cudaStream_t st);
// deterministic BP: S (power of two) from max|r| over n rays, V views and rpc (an upper bound on
// the rays of one view crossing one cell); out += a / S
void launch_det_scale(const float* r, long long n, int V, double rpc, float scale, unsigned* mx, float* S,
                      cudaStream_t st);
void launch_acc64_to_f32(const long long* a, float* out, long long n, const float* S, cudaStream_t st);

void launch_zero_rows(double* normsq, const int* rows, int n, cudaStream_t st);
void launch_zero_rects(float* proj, const int* views, const int4* rects, int n, int nu, int nv, cudaStream_t st);
void launch_obj(const double* normsq, int M, double* out, cudaStream_t st);
void launch_axpy_eud(float* eud, const float* g, long long n, cudaStream_t st);
void launch_dot3(const float* a, const float* b, long long n, double* out3, cudaStream_t st);
void launch_sqdiff(const float* a, const float* b, long long n, double* out, cudaStream_t st);
void launch_fill_random(float* v, long long n, uint64_t seed, cudaStream_t st);
void launch_fill(float* v, long long n, float val, cudaStream_t st);
void launch_sqdiff_masked(const float* a, const float* b, const float* mask, long long n, double* out,
                          cudaStream_t st);
void launch_lincomb(float* out, float a, const float* x, float b, const float* y, float c, const float* z,
                    long long n, cudaStream_t st);
void launch_bb_dots(const float* x, const float* xp, const float* gp, const float* g, long long n, double* out2,
                    cudaStream_t st);
void launch_scale(float* v, long long n, const double* inv_norm_src, cudaStream_t st);

struct ImLaunch {
    KGeom g;
    int n_blocks;
    const BlockDesc* blocks;   // boxes only
    int tiles_u, tiles_v;
    double* w;
    int area;                  // 1: count rays with chord > 1e-6 (IS_AREA) instead of chord sums                 // [n_blocks][n_views][T]
};
void launch_im_weights(const ImLaunch& I, cudaStream_t st);

// TV prox on the owned volume (block-major layout, global block grid).
struct TvLaunch {
    int dims[3];        // global volume dims
    int bdims[3];       // block dims
    int bgrid[3];       // block grid
    int z0, z1;         // owned global z range (z-slab sharding) or [0, nz)
    long long block0;   // first owned block id
    const float* b;     // input image (owned, block-major)
    float* u;           // scratch (owned)
    float* p;           // 3 * owned
    float* q;           // 3 * owned
    float* out;         // output image
    const float* halo_q_next;  // q plane z1 (3 comps) or NULL
    const float* halo_u_prev;  // u plane z0-1 or NULL
    float* q_out;              // fused FGP: the next q (3 * owned; q is read-only then)
    const float* halo_prev;    // fused FGP: qx, qy, qz, b of plane z0-1 (4 planes) or NULL
    float wf, sf, betaf;       // fused FGP in fp32: w, 1/(L w), beta
    int chambolle;             // 1: Chambolle-2004 step p <- (p + s g)/(1 + s|g|) on q (p unused)
    int first;                 // fused path, first iteration: q = p = 0 (not read; no memsets)
    double w;           // weight mu*lambda
    double L;           // Lipschitz bound 4*(#axes > 1)
    double beta;        // FISTA momentum (s_k - 1)/s_{k+1}
    long long n;        // owned voxels
};
void launch_tv_u(const TvLaunch& T, const float* src_q, float* dst, cudaStream_t st);
void launch_tv_pq(const TvLaunch& T, cudaStream_t st);
// out[y * nx + x] = owned[(x, y, z)] for global plane z inside the owned range (block-major
// owned field; T: dims, bdims, bgrid, block0, n) -- a z-plane halo of a non-slab block grid
void launch_pack_plane(const TvLaunch& T, const float* owned, int z, float* out, cudaStream_t st);
// *out += TV(x) over the owned voxels (T: dims, bdims, bgrid, block0, n, halo_u_prev = x of plane z0-1)
void launch_tv_value(const TvLaunch& T, const float* x, double* out, cudaStream_t st);
// out[i] = sum_{g = 0..G-1} ptrs[g][i] in ascending g (virtual-rank allreduce), G <= 8
void launch_sum_ptrs(void* out, const void* const* ptrs, int G, long long n, bool dbl, cudaStream_t st);
// One fused FGP iteration (u, projection, momentum) for z-slab layouts (bgrid = 1 x 1 x N):
// reads q, p, b (+ halos), writes q_out, p.
void launch_tv_fgp(const TvLaunch& T, cudaStream_t st);
// x = b - w grad^T q (T.q = the final p) for z-slab layouts
void launch_tv_out(const TvLaunch& T, float* out, cudaStream_t st);
// z-marching FGP iteration (z-slab layouts, nx % 4 == 0; the default FGP path): the dual
// state is (p_{k-1}, p_{k-2}) in three rotating buffers -- q_k = p_{k-1} + beta (p_{k-1} -
// p_{k-2}) is formed where it is read, p_k is written to the third buffer -- and each CTA
// walks a column of ZC planes of one x-y tile, carrying u(z-1) in registers.
struct TvzLaunch {
    int nx, ny, nz;            // global volume dims
    int z0, z1;                // owned planes
    long long n;               // owned voxels (component stride of the P buffers)
    const float* b;            // owned b = x (prox input), [z][y][x] from plane z0
    const float* P1;           // p_{k-1} (3 components)
    const float* P2;           // p_{k-2}
    float* Pn;                 // p_k (output)
    const float* halo_prev;    // plane z0-1: P1x, P1y, P1z, P2x, P2y, P2z, b (7 planes) or NULL
    const float* halo_next;    // plane z1: P1z, P2z (2 planes) or NULL
    float w, s, beta;          // w = mu lambda, s = 1/(L w), beta = beta_{k-1}
    int stage;                 // 1: k = 1 (q = 0); 2: k = 2 (q = p_1, p_0 = 0 not read); 0: k >= 3
    int zc;                    // planes per CTA
    int pf;                    // L2 prefetch distance in planes (0 = none)
};
void launch_tv_fgp_z(const TvzLaunch& T, cudaStream_t st);
// Two FGP iterations k, k+1 per pass (temporal blocking; one rank owning the whole volume as
// one [z][y][x] array): reads p_{k-1}, p_{k-2}, b, writes p_k and p_{k+1} -- 52 B per voxel
// per two iterations instead of 2 x 40.  Each CTA marches up a column of zc planes of a
// 56 x 12 x-y tile (nx % 4 == 0); the loaded region carries a 2-voxel halo (the two stencils' reach),
// iteration k runs one plane ahead of iteration k+1; q_k, u_k, q_{k+1}, u_{k+1} live in
// shared-memory rings, p_{k-1} and b (read only at the loading thread's own voxels) in registers.
struct Tvz2Launch {
    int nx, ny, nz;
    long long n;               // voxels (component stride of the P buffers)
    const float* b;            // prox input
    const float* P1;           // p_{k-1}
    const float* P2;           // p_{k-2}
    float* Pa;                 // p_k (output)
    float* Pb;                 // p_{k+1} (output)
    float w, s;                // w = mu lambda, s = 1/(L w)
    float beta0, beta1;        // beta_{k-1} (q_k) and beta_k (q_{k+1})
    int stage;                 // of iteration k: 1 (q_k = 0, p_{k-1} = 0), 2 (q_k = p_{k-1}), 0
    int zc;                    // planes per CTA
    int pf;                    // L2 prefetch distance in planes (0 = none)
};
void launch_tv_fgp_z2(const Tvz2Launch& T, cudaStream_t st);
// out[h] = this device's address of rank h's copy of an NCCL symmetric window (LSA exchange;
// w: the ncclWindow_t, n: world size)
void launch_lsa_ptrs(void* w, int n, void** out, cudaStream_t st);

}  // namespace bsgd
