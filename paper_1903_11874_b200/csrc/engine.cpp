// BSGD epoch engine and the extern "C" boundary (include/bsgd.h).
//
// One process per GPU.  A rank owns the contiguous column blocks
// [rank*N/G, (rank+1)*N/G) ("each parallel node calculates a
// forward projection A_I^{J_j} x_{J_j}.  The summation over j is then
// calculated ... using an ALLREDUCE procedure").  Every epoch: host selection
// (Algo 1 line 3) -> FP of the owned selected blocks (line 5) -> partial sum of
// the owned z^j over the selected rows -> ncclAllReduce (the only per-epoch
// exchange) -> r_I = y_I - sum_j z^j_I (line 7) -> BP (line 9) -> g / x update
// (lines 11-14).  Algo 3 (auto mu) and Algo 4 (TV prox) hook in after the step.
#include <math.h>
#include <nccl.h>
#include <string.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <mutex>
#include <cstdio>
#include <memory>
#include <new>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "internal.h"

namespace bsgd {

static thread_local std::string g_last_error;
static std::atomic<unsigned long long> g_launches{0};

void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

void fail(bsgd_status code, const std::string& msg) { throw Error{code, msg}; }

void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
    if (e != cudaSuccess) {
        char buf[512];
        snprintf(buf, sizeof buf, "%s failed: %s (%s:%d)", what, cudaGetErrorString(e), file, line);
        fail(e == cudaErrorMemoryAllocation ? BSGD_E_OOM : BSGD_E_CUDA, buf);
    }
}

#define BSGD_NCCL(x)                                                                          \
    do {                                                                                      \
        ncclResult_t r_ = (x);                                                                \
        if (r_ != ncclSuccess) ::bsgd::fail(BSGD_E_NCCL, std::string(#x " failed: ") +        \
                                                         ncclGetErrorString(r_));             \
    } while (0)

}  // namespace bsgd

using namespace bsgd;

// Virtual-rank group (bsgd_vgroup_create): `world` contexts of one process share it.
// NVTX range per phase of an epoch (host-side markers for nsys / ncu --nvtx; header-only
// NVTX 3, a no-op unless a tool is attached)
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};

struct bsgd_vgroup_s {
    int world = 1;
    std::mutex m;
    std::condition_variable cv;
    int arrived = 0;
    unsigned long long gen = 0;
    std::vector<const void*> src;          // per rank: the buffer it offers in the current collective
    std::vector<cudaEvent_t> ev1, ev2;     // per rank: "offered buffer ready", "my reads are done"
    void barrier() {
        std::unique_lock<std::mutex> lk(m);
        const unsigned long long g = gen;
        if (++arrived == world) {
            arrived = 0;
            ++gen;
            cv.notify_all();
            return;
        }
        if (!cv.wait_for(lk, std::chrono::seconds(120), [&] { return gen != g; }))
            fail(BSGD_E_NCCL, "virtual group: barrier timeout (a rank did not reach the collective)");
    }
};

struct bsgd_ctx_s {
    // ---- configuration
    int beam = 0, n_views = 0, nu = 0, nv = 0;
    std::vector<double> vecs;
    int dims[3] = {0, 0, 0}, bgrid[3] = {1, 1, 1}, bd[3] = {0, 0, 0};
    // Unequal z-slabs (work-balanced slabs): block j spans planes
    // [zsp[j], zsp[j+1]); bd[2] is then the thickest slab and every block-major buffer keeps
    // the stride bsize of that slab (a thinner slab's row ends in zeros nobody reads).
    bool zsplit = false;
    std::vector<int> zsp;
    int N = 1, M = 1, kind = 0, tiles_u = 1, tiles_v = 1, T = 1;
    uint64_t row_seed = 0;
    int rank = 0, world = 1, first = 0, s = 1;
    bool coll = false;     // collective code path (world > 1, or BSGD_FORCE_NCCL=1 with one rank)
    bsgd_vgroup vg = nullptr;   // virtual rank: collectives through the in-process group
    void* vg_tmp = nullptr;
    double* d_rpart = nullptr;   // k_residual per-CTA partials of ||r||^2
    // N2 band exchange (world > 1).  Rank h's partial sum p_h = sum of its owned
    // z^j is zero outside the detector rows its blocks project into (band_h(view): the union
    // of the footprint rows of its blocks), and its BP reads r only there.  So instead of an
    // allreduce of the whole detector, each rank receives the peers' p on the rows where their
    // bands overlap its own and forms r on its band rows only (r is then valid on the band;
    // rows no band covers stay r = y).  ||r_I||^2: each row counted by the lowest rank whose
    // band covers it, one M-double allreduce.  BSGD_EXCHANGE=full keeps the full allreduce.
    bool band = false;
    // LSA mode (BSGD_EXCHANGE=lsa, band mode over NCCL): the band residual kernel reads the
    // peers' partial sums straight from their memory over NVLink -- pc is an NCCL symmetric
    // window (ncclMemAlloc + ncclCommWindowRegister), each peer's copy addressed through
    // ncclGetPeerPointer -- so there is no pack kernel, no send / receive buffers and no
    // ncclSend / ncclRecv; a one-float allreduce orders "every rank wrote pc" before the reads,
    // the ||r_I||^2 allreduce that follows orders the reads before the next epoch's writes.
    // Virtual ranks emulate it with each other's pc pointers (same device).
    bool lsa = false;
    void* pc_win = nullptr;                // ncclWindow_t of pc (NCCL ranks)
    bool pc_ncclmem = false;               // pc from ncclMemAlloc
    std::vector<const float*> lsa_pc;      // per rank: its pc as this device addresses it
    float* d_bar = nullptr;                // the one-float "partials written" allreduce
    std::vector<int2> bands;         // [world][n_views] (lo, hi)
    float *ex_send = nullptr, *ex_recv = nullptr;   // packed overlap chunks (sent / received)
    long long ex_cap = 0;
    double* d_npart = nullptr;       // [M] this rank's partial ||r_I||^2
    unsigned long long comm_bytes = 0, comm_msgs = 0;   // residual exchange, sent by this rank
    float* gap_proj = nullptr;   // BSGD_LOG_TRUE_OBJ: A x (full length)
    float* tvv_halo = nullptr;   // tv_value: x plane z0-1 from the previous rank
    double* d_tvv = nullptr;     // per-epoch TV(x) (BSGD_LOG_TRUE_OBJ with log->tv)
    double* d_tvv1 = nullptr;    // bsgd_tv_value
    float* seen = nullptr;       // A^T 1 over all views (owned voxels): > 0 where a ray passes
    double* d_seenlog = nullptr; // per-epoch [sum (x - x_true)^2, count] over the seen voxels
    double* d_gap = nullptr;     // ... and 1/2-less |y - A x|^2 per epoch
    int d_gap_n = 0;
    // deterministic BP (BSGD_DETERMINISTIC): int64 fixed-point twins of accN / accT
    bool det = false;
    long long* acc64N = nullptr;
    long long* acc64T = nullptr;
    float* d_det_scale = nullptr;
    unsigned* d_det_max = nullptr;
    double rays_per_cell = 0.0;   // upper bound on the rays of one view crossing one cell (set at create)
    size_t vg_tmp_bytes = 0;
    long long bsize = 0, n_rays = 0, per = 0;
    double R = 0.0;
    std::vector<std::vector<int>> rows;   // views of each row block (sorted)
    std::vector<int> view_row;             // row block of each view
    // ---- memory
    bsgd_alloc alloc{nullptr, nullptr, nullptr};
    struct Buf { void* p; size_t bytes; };
    std::vector<Buf> bufs;
    uint64_t bytes = 0;
    // ---- device state
    double* d_vecs = nullptr;
    float *xT = nullptr, *g = nullptr, *ghat = nullptr, *z = nullptr, *r = nullptr;
    float *accN = nullptr, *accT = nullptr, *pc = nullptr;
    float *eud_cur = nullptr, *eud_prev = nullptr;
    float *tv_u = nullptr, *tv_p = nullptr, *tv_q = nullptr, *tv_hq = nullptr, *tv_hu = nullptr,
          *tv_q2 = nullptr, *tv_hp = nullptr, *tv_pk = nullptr, *tvz_hp = nullptr, *tvz_hn = nullptr,
          *tv_xc = nullptr, *tv_q3 = nullptr;
    float *fp_scratchT = nullptr, *fp_scratchN = nullptr, *pw_v = nullptr, *pw_proj = nullptr, *pw_vT = nullptr,
          *pw_vN = nullptr;
    float* xN = nullptr;   // slack-padded copy of x_owned (FP source for main-Y views)
    float *y_dev = nullptr, *x_dev = nullptr, *xt_dev = nullptr;
    float *sv_a = nullptr, *sv_b = nullptr, *sv_c = nullptr, *sv_d = nullptr, *y_zero = nullptr;   // solvers
    double* d_normsq = nullptr;
    // footprint-restricted z^j storage: ZRect per (owned block, view)
    std::vector<ZRect> h_zr;
    ZRect* d_zr = nullptr;
    long long z_size = 0;
    double* d_normsq0 = nullptr;         // ||y_I||^2 of a deferred reset (host-buffer runs)
    cudaStream_t copy_st = nullptr;      // H2D uploads of host-buffer runs
    std::vector<cudaEvent_t> x_events;
    std::vector<cudaEvent_t> up_ev;      // [s] x blocks, [s] y, [s + 1] start
    void ensure_copy_stream() {
        if (copy_st) return;
        BSGD_CUDA(cudaStreamCreateWithFlags(&copy_st, cudaStreamNonBlocking));
        up_ev.resize(s + 3);   // x blocks, y of the first epoch's rows, misc, the rest of y
        for (auto& e : up_ev) BSGD_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        d_normsq0 = dnew<double>(M);
    }
    int* d_rows_tmp = nullptr;         // M ints: a row-block list for one launch
    uint2* v2_list = nullptr;          // ProjLaunch::v2_list (the v2 companion's warps)
    unsigned* v2_count = nullptr;
    long long v2_cap = 0;
    double* d_red = nullptr;           // 8 doubles scratch
    double* d_log = nullptr;           // per-epoch [obj, rmse] scratch
    long long d_log_cap = 0;
    unsigned long long* d_visits = nullptr;
    unsigned long long* count_target = nullptr;   // per (block, slot) counters of a COUNT launch
    std::vector<unsigned long long> vtab;          // visits [owned block][view][tile]
    bool vtab_ready = false;
    // launch tables
    char* d_tab = nullptr;
    size_t tab_bytes = 0;
    // ---- host state
    std::vector<double> h_normsq;
    double mu = 0.0;
    int epoch = 0;
    std::vector<uint32_t> q;            // IM table [s][n_views][T]
    std::vector<double> w;
    bool q_ready = false;
    int q_kind = 0;
    // Algo 3 state
    bool have_prev_eud = false, have_theta_prev = false;
    double theta_prev = 0.0;
    std::vector<double> rnorm_hist;     // ||r||^{k} at k = 0, M, 2M, ...
    ncclComm_t comm = nullptr;
    // Calls may come on different streams, but they share the launch-table arena (d_tab), the
    // BP accumulators and the FP scratch copies: every call first waits for the work the
    // previous call enqueued (an event recorded on its stream), so a table or accumulator is
    // never rewritten while a kernel of an earlier call on another stream still reads it.
    cudaEvent_t order_ev = nullptr;
    cudaStream_t order_st = nullptr;
    bool order_valid = false;
    void stream_enter(cudaStream_t st) {
        if (order_valid && order_st != st) BSGD_CUDA(cudaStreamWaitEvent(st, order_ev, 0));
    }
    void stream_leave(cudaStream_t st) {
        if (!order_ev && cudaEventCreateWithFlags(&order_ev, cudaEventDisableTiming) != cudaSuccess) {
            cudaGetLastError();
            order_ev = nullptr;
            return;
        }
        if (cudaEventRecord(order_ev, st) != cudaSuccess) {
            cudaGetLastError();
            order_valid = false;
            return;
        }
        order_st = st;
        order_valid = true;
    }
    bool poisoned = false;
    std::string err;

    // ------------------------------------------------------------ memory
    void* dalloc(size_t n) {
        if (n == 0) n = 16;
        n = (n + 255) & ~(size_t)255;
        void* p = nullptr;
        if (alloc.alloc) {
            p = alloc.alloc(n, nullptr, alloc.user);
            if (!p) fail(BSGD_E_OOM, "allocator callback returned NULL");
        } else {
            cudaError_t e = cudaMalloc(&p, n);
            if (e != cudaSuccess) {
                cudaGetLastError();
                fail(BSGD_E_OOM, "cudaMalloc of " + std::to_string(n) + " bytes failed");
            }
        }
        bufs.push_back({p, n});
        bytes += n;
        return p;
    }
    template <class T> T* dnew(long long count, bool zero = true) {
        T* p = (T*)dalloc(sizeof(T) * (size_t)count);
        if (zero) BSGD_CUDA(cudaMemset(p, 0, sizeof(T) * (size_t)count));
        return p;
    }
    // Image buffers the projector reads or scatters into are PADDED copies (BlockDesc):
    // per block, rows carry PAD_X zero floats on each side and PAD_Z zero planes bound the
    // block, so a traversal step up to one cell past a row / plane face reads 0 (FP) or lands
    // in the ignored border (BP).  That lets the FP/BP slice loop skip entry/exit clamping.
    // Each whole buffer also carries `slack` zeroed floats on both sides (a safety margin
    // of one padded plane).  pN / pT give the interior origin of owned block b.
    int rowN = 0, planeN = 0, rowT = 0, planeT = 0;
    long long padN = 0, padT = 0, orgN = 0, orgT = 0, slack = 0;
    float* dnew_pad(int nblocks, bool transposed) {
        float* p = dnew<float>((long long)nblocks * (transposed ? padT : padN) + 2 * slack);
        return p + slack;
    }
    float* pN(float* base, long long b) const { return base + b * padN + orgN; }
    float* pT(float* base, long long b) const { return base + b * padT + orgT; }
    // the LSA window and its memory go before the communicator
    void release_comm() {
        if (pc_win && comm) ncclCommWindowDeregister(comm, (ncclWindow_t)pc_win);
        pc_win = nullptr;
        if (pc_ncclmem) ncclMemFree(pc);
        pc_ncclmem = false;
        if (comm) ncclCommDestroy(comm);
        comm = nullptr;
    }
    void release() {
        if (order_ev) cudaEventDestroy(order_ev);
        order_ev = nullptr;
        for (auto& e : up_ev) cudaEventDestroy(e);
        up_ev.clear();
        if (copy_st) cudaStreamDestroy(copy_st);
        copy_st = nullptr;
        for (auto& b : bufs) {
            if (alloc.free) alloc.free(b.p, b.bytes, nullptr, alloc.user);
            else cudaFree(b.p);
        }
        bufs.clear();
    }

    KGeom kgeom() const {
        KGeom k;
        k.vecs = d_vecs;
        k.beam = beam;
        k.nu = nu;
        k.nv = nv;
        k.n_views = n_views;
        for (int c = 0; c < 3; ++c) k.dims[c] = dims[c];
        k.R = R;
        return k;
    }
    int nz_of(int j) const { return zsplit ? zsp[j + 1] - zsp[j] : bd[2]; }
    long long vox_of(int j) const { return (long long)bd[0] * bd[1] * nz_of(j); }
    void box(int j, int lo[3], int hi[3]) const {
        if (zsplit) {
            lo[0] = lo[1] = 0;
            lo[2] = zsp[j];
            hi[0] = dims[0];
            hi[1] = dims[1];
            hi[2] = zsp[j + 1];
            return;
        }
        int jx = j % bgrid[0], jy = (j / bgrid[0]) % bgrid[1], jz = j / (bgrid[0] * bgrid[1]);
        lo[0] = jx * bd[0]; lo[1] = jy * bd[1]; lo[2] = jz * bd[2];
        for (int c = 0; c < 3; ++c) hi[c] = lo[c] + bd[c];
    }
    bool owned(int j) const { return j >= first && j < first + s; }

    // Detector pixels (u0,u1,v0,v1) whose rays can meet the box [lo,hi) (grid coords):
    // bounding box of the projected corners + 1 pixel margin, u aligned to warps.
    // Falls back to the whole detector when a corner is not in front of the source.
    int band_rows = 8;   // BSGD_BAND_ROWS (measured: 1: 3.31, 2: 3.46, 4: 3.54, 8: 3.56, 16: 3.54 epochs/s)
    int4 footprint(const int lo[3], const int hi[3], int view) const {
        const int4 full = make_int4(0, nu, 0, nv);
        const double* q = &vecs[12 * (size_t)view];
        const double *d = q + 3, *u = q + 6, *v = q + 9;
        auto dot = [](const double* a, const double* b) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]; };
        double n[3] = {u[1] * v[2] - u[2] * v[1], u[2] * v[0] - u[0] * v[2], u[0] * v[1] - u[1] * v[0]};
        const double uu = dot(u, u), vv = dot(v, v), uv = dot(u, v), det = uu * vv - uv * uv;
        if (!(det > 0)) return full;
        double amn = 1e300, amx = -1e300, bmn = 1e300, bmx = -1e300;
        for (int c = 0; c < 8; ++c) {
            double P[3] = {(c & 1 ? hi[0] : lo[0]) - dims[0] / 2.0, (c & 2 ? hi[1] : lo[1]) - dims[1] / 2.0,
                           (c & 4 ? hi[2] : lo[2]) - dims[2] / 2.0};
            double Q[3];
            if (beam == BSGD_PARALLEL) {
                const double dn = dot(q, n);
                if (fabs(dn) < 1e-12) return full;
                double dp[3] = {d[0] - P[0], d[1] - P[1], d[2] - P[2]};
                const double mu_ = dot(dp, n) / dn;
                for (int k = 0; k < 3; ++k) Q[k] = P[k] + mu_ * q[k];
            } else {
                double ps[3] = {P[0] - q[0], P[1] - q[1], P[2] - q[2]}, ds[3] = {d[0] - q[0], d[1] - q[1], d[2] - q[2]};
                const double den = dot(ps, n), num = dot(ds, n);
                if (!(den * num > 0)) return full;
                const double lam = num / den;
                for (int k = 0; k < 3; ++k) Q[k] = q[k] + lam * ps[k];
            }
            double r[3] = {Q[0] - d[0], Q[1] - d[1], Q[2] - d[2]};
            const double ru = dot(r, u), rv = dot(r, v);
            const double al = (ru * vv - rv * uv) / det, be = (rv * uu - ru * uv) / det;
            amn = std::min(amn, al); amx = std::max(amx, al);
            bmn = std::min(bmn, be); bmx = std::max(bmx, be);
        }
        const double cu = (nu - 1) / 2.0, cv = (nv - 1) / 2.0;
        auto clampi = [](double x, int lo_, int hi_) { return (int)std::min<double>(std::max<double>(x, lo_), hi_); };
        int u0 = clampi(floor(amn + cu) - 1, 0, nu), u1 = clampi(ceil(amx + cu) + 2, 0, nu);
        int v0 = clampi(floor(bmn + cv) - 1, 0, nv), v1 = clampi(ceil(bmx + cv) + 2, 0, nv);
        u0 = (u0 / 32) * 32;
        u1 = std::min(nu, ((u1 + 31) / 32) * 32);
        return make_int4(u0, u1, v0, v1);
    }

    // Upper bound on the number of rays of one view that cross one cell (the deterministic BP's
    // fixed-point range, k_det_scale).  A cell's projection spans at most sqrt(3) * magnification
    // voxel units along each detector axis, i.e. ceil(sqrt(3) m / |u|) + 1 pixel columns and as
    // many rows (+1 for a partial pixel); m = 1 for parallel beams and |s - d_c| / (distance of
    // the source from the volume's bounding sphere) for fan / cone.  A source inside that sphere
    // has no bound: every ray of the view is counted.
    double compute_rays_per_cell() const {
        const double Rv = 0.5 * sqrt((double)dims[0] * dims[0] + (double)dims[1] * dims[1] + (double)dims[2] * dims[2]);
        double worst = 1.0;
        for (int v = 0; v < n_views; ++v) {
            const double* q = &vecs[12 * (size_t)v];
            const double pu = sqrt(q[6] * q[6] + q[7] * q[7] + q[8] * q[8]);
            const double pv = sqrt(q[9] * q[9] + q[10] * q[10] + q[11] * q[11]);
            double m = 1.0;
            if (beam != BSGD_PARALLEL) {
                const double ds = sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2]) - Rv;
                const double sd = sqrt((q[3] - q[0]) * (q[3] - q[0]) + (q[4] - q[1]) * (q[4] - q[1]) +
                                       (q[5] - q[2]) * (q[5] - q[2]));
                if (!(ds > 0.0)) return (double)nu * nv;
                m = sd / ds;
            }
            const double cu = nu > 1 && pu > 0 ? std::min<double>(nu, ceil(1.7320508075688772 * m / pu) + 2.0) : 1.0;
            const double cv = nv > 1 && pv > 0 ? std::min<double>(nv, ceil(1.7320508075688772 * m / pv) + 2.0) : 1.0;
            worst = std::max(worst, cu * cv);
        }
        return worst;
    }

    // pack host tables into the device arena; returns device pointers
    template <class T> T* tab_put(size_t& off, const std::vector<T>& v, std::vector<char>& staging) {
        off = (off + 15) & ~(size_t)15;
        size_t nb = sizeof(T) * v.size();
        if (off + nb > staging.size()) staging.resize(off + nb);
        if (nb) memcpy(staging.data() + off, v.data(), nb);
        T* dp = (T*)(d_tab + off);
        off += nb;
        return dp;
    }
    void tab_upload(const std::vector<char>& staging, size_t used, cudaStream_t st) {
        if (used > tab_bytes) fail(BSGD_E_CONTRACT, "launch table overflow");
        BSGD_CUDA(cudaMemcpyAsync(d_tab, staging.data(), used, cudaMemcpyHostToDevice, st));
    }

    // ------------------------------------------------------------ operators
    // FP for `blocks` (owned slots) over `views`; rects[b][slot] (empty = full detector).
    void fp(const std::vector<int>& views, const std::vector<int>& slots, const std::vector<int4>& rects,
            std::vector<const float*> xN, std::vector<const float*> xTs, std::vector<float*> zout,
            int accumulate, cudaStream_t st, size_t tab_off = 0) {
        project(PROJ_FP, views, slots, rects, xN, xTs, {}, {}, zout, nullptr, 0.f, accumulate, st, tab_off);
    }

    void project(int mode, const std::vector<int>& views, const std::vector<int>& slots,
                 const std::vector<int4>& rects, const std::vector<const float*>& xN,
                 const std::vector<const float*>& xTs, const std::vector<float*>& oN,
                 const std::vector<float*>& oT, const std::vector<float*>& zout, const float* rproj,
                 float scale, int accumulate, cudaStream_t st, size_t tab_off = 0) {
        const int nb = (int)slots.size(), ns = (int)views.size();
        if (nb == 0 || ns == 0) return;
        std::vector<BlockDesc> bl(nb);
        for (int b = 0; b < nb; ++b) {
            BlockDesc& d = bl[b];
            box(first + slots[b], d.lo, d.hi);
            d.xN = xN.empty() ? nullptr : xN[b];
            d.xT = xTs.empty() ? nullptr : xTs[b];
            d.outN = oN.empty() ? nullptr : oN[b];
            d.outT = oT.empty() ? nullptr : oT[b];
            d.z = zout.empty() ? nullptr : zout[b];
            d.zr = (!zout.empty() && zout[b] == z) ? d_zr + (size_t)slots[b] * n_views : nullptr;
            d.rowN = rowN; d.planeN = planeN; d.rowT = rowT; d.planeT = planeT;
        }
        std::vector<int4> rc = rects;
        int maxr = 0;
        if (rc.empty()) rc.assign((size_t)nb * ns, make_int4(0, nu, 0, nv));
        // footprint culling: only detector pixels whose rays can meet the block box
        const int R = band_rows;
        int maxw = 0, nbands = 0;
        for (int b = 0; b < nb; ++b) {
            int vlo = nv, vhi = 0;
            for (int k = 0; k < ns; ++k) {
                int4& q = rc[(size_t)b * ns + k];
                int4 f = footprint(bl[b].lo, bl[b].hi, views[k]);
                q.x = std::max(q.x, f.x); q.y = std::min(q.y, f.y);
                q.z = std::max(q.z, f.z); q.w = std::min(q.w, f.w);
                if (q.x >= q.y || q.z >= q.w) { q = make_int4(0, 0, 0, 0); continue; }
                maxw = std::max(maxw, q.y - q.x);
                vlo = std::min(vlo, q.z);
                vhi = std::max(vhi, q.w);
            }
            bl[b].band_lo = vlo < vhi ? vlo / R : 0;
            if (vlo < vhi) nbands = std::max(nbands, (vhi - 1) / R - vlo / R + 1);
        }
        for (auto& q : rc) maxr = std::max(maxr, (q.y - q.x) * (q.w - q.z));
        if (maxr == 0) return;
        std::vector<char> staging;
        size_t off = tab_off;
        staging.resize(off);
        ProjLaunch L;
        L.g = kgeom();
        L.n_slots = ns;
        L.views = tab_put(off, views, staging);
        L.rects = tab_put(off, rc, staging);
        L.n_blocks = nb;
        L.blocks = tab_put(off, bl, staging);
        L.max_rect_rays = maxr;
        L.rows_per_band = R;
        L.n_chunks = (R * maxw + 255) / 256;
        L.n_bands = nbands;
        L.rproj = rproj;
        L.scale = scale;
        L.accumulate = accumulate;
        L.visits = (mode == PROJ_COUNT) ? count_target : nullptr;
        L.det_scale = d_det_scale;
        // the warps k_project3 hands to the v2 companion are listed (capacity: every warp of
        // the launch); BSGD_V2_LIST=0 keeps the grid companion (A/B)
        static const bool v2l = !(getenv("BSGD_V2_LIST") && atoi(getenv("BSGD_V2_LIST")) == 0);
        L.v2_list = nullptr;
        L.v2_count = nullptr;
        if (v2l) {
            const long long warps = (long long)nbands * ns * L.n_chunks * nb * 8;
            if (warps > v2_cap) {
                v2_list = dnew<uint2>(warps, false);
                v2_cap = warps;
            }
            if (!v2_count) v2_count = dnew<unsigned>(1);
            L.v2_list = v2_list;
            L.v2_count = v2_count;
        }
        if (off > tab_bytes) fail(BSGD_E_CONTRACT, "launch table overflow");
        BSGD_CUDA(cudaMemcpyAsync(d_tab + tab_off, staging.data() + tab_off, off - tab_off,
                                  cudaMemcpyHostToDevice, st));
        launch_project(mode, L, st);
    }

    float* ghat_of(int i, int b) { return ghat + ((long long)i * s + b) * bsize; }

    void update(int mode, int b, float* x, float mu_, int final_, float* out, int accumulate,
                cudaStream_t st, float* accN_ = nullptr, float* accT_ = nullptr, float* xT_ = nullptr,
                int ghat_i = 0, float* xN_ = nullptr) {
        UpdLaunch U;
        U.bd[0] = bd[0]; U.bd[1] = bd[1]; U.bd[2] = nz_of(first + b);
        U.rowN = rowN; U.planeN = planeN; U.rowT = rowT; U.planeT = planeT;
        U.accN = accN_ ? accN_ : pN(accN, b);
        U.accT = accT_ ? accT_ : pT(accT, b);
        U.ghat = ghat ? ghat_of(ghat_i, b) : nullptr;
        U.g = g + b * bsize;
        U.x = x;
        U.xT = xT_ ? xT_ : pT(xT, b);
        U.xN = xN_ ? xN_ : (xT_ ? nullptr : pN(xN, b));
        U.out = out;
        U.mu = mu_;
        U.final_ = final_;
        U.accumulate = accumulate;
        launch_block_update(mode, U, st);
    }

    void refresh_xT(float* x_owned, const std::vector<int>& slots, cudaStream_t st) {
        for (int b : slots) update(UPD_XT, b, x_owned + b * bsize, 0.f, 1, nullptr, 0, st);
    }

    void allreduce_f(float* p, size_t n, cudaStream_t st) {
        if (vg) vg_allreduce(p, n, false, st);
        else if (coll) BSGD_NCCL(ncclAllReduce(p, p, n, ncclFloat, ncclSum, comm, st));
    }
    void allreduce_d(double* p, size_t n, cudaStream_t st) {
        if (vg) vg_allreduce(p, n, true, st);
        else if (coll) BSGD_NCCL(ncclAllReduce(p, p, n, ncclDouble, ncclSum, comm, st));
    }

    // ---- virtual ranks: the two collective shapes as events + host barriers + device work
    void vg_offer(const void* p, cudaStream_t st) {
        BSGD_CUDA(cudaEventRecord(vg->ev1[rank], st));
        vg->src[rank] = p;
        vg->barrier();
    }
    void vg_release(cudaStream_t st) {   // nobody reuses an offered buffer before all have read it
        BSGD_CUDA(cudaEventRecord(vg->ev2[rank], st));
        vg->barrier();
        for (int g = 0; g < world; ++g) BSGD_CUDA(cudaStreamWaitEvent(st, vg->ev2[g], 0));
    }
    void vg_allreduce(void* p, size_t n, bool dbl, cudaStream_t st) {
        const size_t bytes = n * (dbl ? sizeof(double) : sizeof(float));
        if (bytes > vg_tmp_bytes) {
            vg_tmp = dalloc(bytes);
            vg_tmp_bytes = bytes;
        }
        vg_offer(p, st);
        const void* srcs[8];
        for (int g = 0; g < world; ++g) {
            srcs[g] = vg->src[g];
            BSGD_CUDA(cudaStreamWaitEvent(st, vg->ev1[g], 0));
        }
        launch_sum_ptrs(vg_tmp, srcs, world, (long long)n, dbl, st);   // rank-ascending order
        vg_release(st);
        BSGD_CUDA(cudaMemcpyAsync(p, vg_tmp, bytes, cudaMemcpyDeviceToDevice, st));
    }

    // Rows [lo, hi) of the detector that the blocks [h s_, (h+1) s_) of rank h of a G_-rank
    // ownership project into, per view ([G_][n_views]).
    std::vector<int2> rank_bands(int G_, int s_) const {
        std::vector<int2> out((size_t)G_ * n_views, make_int2(0, 0));
        for (int h = 0; h < G_; ++h)
            for (int v = 0; v < n_views; ++v) {
                int lo_ = nv, hi_ = 0;
                for (int b = 0; b < s_; ++b) {
                    int lo[3], hi[3];
                    box(h * s_ + b, lo, hi);
                    const int4 f = footprint(lo, hi, v);
                    if (f.x >= f.y || f.z >= f.w) continue;
                    lo_ = std::min(lo_, f.z);
                    hi_ = std::max(hi_, f.w);
                }
                out[(size_t)h * n_views + v] = lo_ < hi_ ? make_int2(lo_, hi_) : make_int2(0, 0);
            }
        return out;
    }
    void compute_bands() { bands = rank_bands(world, s); }
    int2 band_of(int h, int v) const { return bands[(size_t)h * n_views + v]; }
    static int2 isect(int2 a, int2 b) { return make_int2(std::max(a.x, b.x), std::min(a.y, b.y)); }

    // The exchange plan of rank g for the selected views: per peer h (ascending) the chunks of
    // its compact partial sums pc on the overlap rows band_g ∩ band_h (slot order), packed back to
    // back; peer h's region starts at off[h].  Symmetric: g's chunk list for h equals h's for g.
    struct Chunk { long long src, cnt, k, lo; };
    struct ExPlan {
        std::vector<std::vector<Chunk>> ch;
        std::vector<long long> off;
        long long total = 0;
    };
    ExPlan plan_for(int g, const std::vector<int>& vsel) const {
        ExPlan P;
        P.ch.resize(world);
        P.off.assign(world + 1, 0);
        for (int h = 0; h < world; ++h) {
            P.off[h] = P.total;
            if (h == g) continue;
            for (int k = 0; k < (int)vsel.size(); ++k) {
                const int2 o = isect(band_of(g, vsel[k]), band_of(h, vsel[k]));
                if (o.x >= o.y) continue;
                P.ch[h].push_back({(long long)k * per + (long long)o.x * nu, (long long)(o.y - o.x) * nu, k, o.x});
                P.total += (long long)(o.y - o.x) * nu;
            }
        }
        P.off[world] = P.total;
        return P;
    }

    // Send this rank's pc on the overlap rows to every peer whose band overlaps and receive theirs:
    // the chunks are packed (k_copy_chunks) into one buffer, one ncclSend / ncclRecv per peer, into
    // ex_recv (peer h's chunks at off[h]); the virtual-rank group copies each peer's region from its
    // offered pack buffer.  Returns the plan (the residual kernel reads ex_recv through it).
    ExPlan band_exchange(const std::vector<int>& vsel, std::vector<char>& staging, size_t& off, cudaStream_t st) {
        ExPlan P = plan_for(rank, vsel);
        if (P.total > ex_cap) {   // sized once for the largest plan (every view selected)
            std::vector<int> all(n_views);
            for (int v = 0; v < n_views; ++v) all[v] = v;
            ex_cap = std::max(P.total, plan_for(rank, all).total);
            ex_send = dnew<float>(ex_cap, false);
            ex_recv = dnew<float>(ex_cap, false);
        }
        std::vector<long long> tab;      // (src, dst, cnt) triples
        for (int h = 0; h < world; ++h) {
            long long d = P.off[h];
            for (auto& c : P.ch[h]) {
                tab.push_back(c.src);
                tab.push_back(d);
                tab.push_back(c.cnt);
                d += c.cnt;
                comm_bytes += 4ull * (unsigned long long)c.cnt;
            }
            if (!P.ch[h].empty()) ++comm_msgs;
        }
        if (!tab.empty()) {   // the chunk table goes after this epoch's residual tables in d_tab
            const size_t start = off;
            const long long* dt = tab_put(off, tab, staging);
            if (off > tab_bytes) fail(BSGD_E_CONTRACT, "launch table overflow (exchange plan)");
            BSGD_CUDA(cudaMemcpyAsync(d_tab + start, staging.data() + start, off - start, cudaMemcpyHostToDevice, st));
            launch_copy_chunks(pc, ex_send, dt, (int)(tab.size() / 3), st);
        }
        if (vg) {
            vg_offer(ex_send, st);
            for (int h = 0; h < world; ++h) {
                const long long n = P.off[h + 1] - P.off[h];
                if (n == 0) continue;
                const ExPlan Q = plan_for(h, vsel);                 // where h packed its chunks for me
                BSGD_CUDA(cudaStreamWaitEvent(st, vg->ev1[h], 0));
                BSGD_CUDA(cudaMemcpyAsync(ex_recv + P.off[h], (const float*)vg->src[h] + Q.off[rank],
                                          sizeof(float) * n, cudaMemcpyDeviceToDevice, st));
            }
            vg_release(st);
            return P;
        }
        BSGD_NCCL(ncclGroupStart());
        for (int h = 0; h < world; ++h) {
            const long long n = P.off[h + 1] - P.off[h];
            if (n == 0) continue;
            BSGD_NCCL(ncclSend(ex_send + P.off[h], (size_t)n, ncclFloat, h, comm, st));
            BSGD_NCCL(ncclRecv(ex_recv + P.off[h], (size_t)n, ncclFloat, h, comm, st));
        }
        BSGD_NCCL(ncclGroupEnd());
        return P;
    }

    // line 7 with the band exchange (Rl: the k_residual launch of this epoch, pc filled):
    // r on this rank's band rows and ||r_I||^2 of the selected row blocks (into d_normsq)
    void band_residual(ResLaunch& Rl, const std::vector<int>& vsel, const std::vector<int>& sel_rows,
                       const int* drows, std::vector<char>& staging, size_t& off, cudaStream_t st) {
        const int V = (int)vsel.size();
        const ExPlan P = lsa ? plan_for(rank, vsel) : band_exchange(vsel, staging, off, st);
        std::vector<const float*> peer(world, nullptr);
        if (lsa) {   // every rank's pc written, then read in place from its memory
            if (vg) {
                vg_offer(pc, st);
                for (int h = 0; h < world; ++h) {
                    BSGD_CUDA(cudaStreamWaitEvent(st, vg->ev1[h], 0));
                    peer[h] = (const float*)vg->src[h];
                }
            } else {
                BSGD_NCCL(ncclAllReduce(d_bar, d_bar, 1, ncclFloat, ncclSum, comm, st));
                peer = lsa_pc;
            }
            for (int h = 0; h < world; ++h)   // bytes this rank reads from peer h's memory
                if (P.off[h + 1] > P.off[h]) {
                    comm_bytes += 4ull * (unsigned long long)(P.off[h + 1] - P.off[h]);
                    ++comm_msgs;
                }
        }
        std::vector<int2> bt((size_t)V * world), rg(V);
        for (int k = 0; k < V; ++k) {
            for (int h = 0; h < world; ++h) bt[(size_t)k * world + h] = band_of(h, vsel[k]);
            rg[k] = rank == 0 ? make_int2(0, nv) : band_of(rank, vsel[k]);
        }
        // element (slot k, row v, column u) of peer h's partial sums sits at ex_recv[k per + v nu +
        // u + adj[k][h]] (only rows of band_me ∩ band_h are read); own pc: adj = 0
        // (LSA: peer h's own pc, adj = 0)
        std::vector<long long> adj((size_t)V * world, 0);
        for (int h = 0; h < world && !lsa; ++h) {
            long long d = P.off[h];
            for (auto& c : P.ch[h]) {
                adj[(size_t)c.k * world + h] = d - c.src;
                d += c.cnt;
            }
        }
        std::vector<const float*> dp(world, nullptr);
        for (int h = 0; h < world; ++h)
            dp[h] = h == rank ? pc : (P.off[h + 1] > P.off[h] ? (lsa ? peer[h] : ex_recv) : nullptr);
        const size_t start = off;
        BandLaunch B;
        B.n_slots = V;
        B.per = (int)per;
        B.nu = nu;
        B.G = world;
        B.me = rank;
        B.views = Rl.views;
        B.bands = tab_put(off, bt, staging);
        B.range = tab_put(off, rg, staging);
        B.data = tab_put(off, dp, staging);
        B.adj = tab_put(off, adj, staging);
        if (off > tab_bytes) fail(BSGD_E_CONTRACT, "launch table overflow");
        BSGD_CUDA(cudaMemcpyAsync(d_tab + start, staging.data() + start, off - start, cudaMemcpyHostToDevice, st));
        B.y = Rl.y;
        B.r = Rl.r;
        B.part = d_rpart;
        launch_residual_band(B, st);
        if (lsa && vg) vg_release(st);
        ResLaunch Rn = Rl;
        Rn.normsq = d_npart;
        launch_zero_rows(d_npart, drows, (int)sel_rows.size(), st);
        launch_normsq_final(Rn, RES_GX, st);
        allreduce_d(d_npart, (size_t)M, st);
        launch_copy_rows(d_normsq, d_npart, drows, (int)sel_rows.size(), st);
    }

    // ------------------------------------------------------------ one epoch
    // Algo 1 / Algo 2 / Eq. 4 with an explicit selection.  tiles: [n_cols][V_sel] or empty.
    // Host-buffer runs (bsgd_run with y / x in host memory) overlap the uploads with the
    // first epoch: xev (per owned block) makes the FP wait block by block for its x
    // upload (refreshing the projector copies of every owned block), yev makes the
    // residual wait for y, and y_reset runs the deferred r = y of Algo 1 line 1 there
    // (its ||y_I||^2 are kept in d_normsq0 for Algo 3's ||r||^0).
    struct Upload {
        const std::vector<cudaEvent_t>* xev = nullptr;
        cudaEvent_t yev = nullptr;       // host y: the views of this (first) epoch's selected rows
        bool y_reset = false;
        // last epoch of a host-x run: each block's x goes to the host as soon as its final
        // update is done (the BP of the final row block then runs block by block), so the
        // download overlaps the remaining BP launches
        float* x_host_out = nullptr;
    };
    void epoch_step(const float* y, float* x_owned, const std::vector<int>& sel_rows,
                    const std::vector<int>& sel_cols, const std::vector<int>& tiles, float mu_,
                    bool sgd, cudaStream_t st, cudaEvent_t* ev, bool refresh = true,
                    const Upload* up = nullptr) {
        std::vector<int> vsel, slot_row;
        for (int i : sel_rows)
            for (int v : rows[i]) {
                vsel.push_back(v);
                slot_row.push_back(i);
            }
        const int V = (int)vsel.size();
        std::vector<int> cols = sgd ? std::vector<int>() : sel_cols;
        if (sgd) for (int j = 0; j < N; ++j) cols.push_back(j);
        // owned selected blocks and their global column slot
        std::vector<int> oslots, ocs;
        for (int cs = 0; cs < (int)cols.size(); ++cs)
            if (owned(cols[cs])) {
                oslots.push_back(cols[cs] - first);
                ocs.push_back(cs);
            }
        const int nb = (int)oslots.size();
        // x^T of the selected blocks must match x (the caller may have changed x);
        // bsgd_run keeps it in sync itself (refresh = false)
        if (refresh && !(up && up->xev)) refresh_xT(x_owned, oslots, st);
        auto rect_for = [&](int b, int vs) -> int4 {
            if (tiles.empty()) return make_int4(0, nu, 0, nv);
            int t = tiles[(size_t)ocs[b] * V + vs];
            int tu = t % tiles_u, tv = t / tiles_u;
            return make_int4((int)((long long)tu * nu / tiles_u), (int)((long long)(tu + 1) * nu / tiles_u),
                             (int)((long long)tv * nv / tiles_v), (int)((long long)(tv + 1) * nv / tiles_v));
        };
        if (ev) BSGD_CUDA(cudaEventRecord(ev[0], st));
        NvtxRange nv_epoch("bsgd epoch");
        // ---- lines 4-6: z^j_{I_i} = A_{I_i}^{J_j} x_{J_j}  (IM: tile rows only)
        std::unique_ptr<NvtxRange> nv_phase(new NvtxRange("fp (Algo 1 l.5)"));
        if (up && up->xev) {   // block by block as the x upload lands
            for (int b = 0; b < s; ++b) {
                BSGD_CUDA(cudaStreamWaitEvent(st, (*up->xev)[b], 0));
                refresh_xT(x_owned, {b}, st);
                for (int q = 0; q < nb; ++q) {
                    if (oslots[q] != b) continue;
                    std::vector<int4> rc(V);
                    for (int vs = 0; vs < V; ++vs) rc[vs] = rect_for(q, vs);
                    project(PROJ_FP, vsel, {b}, rc, {pN(xN, b)}, {pT(xT, b)}, {}, {}, {z},
                            nullptr, 0.f, 0, st, 0);
                }
            }
        } else {
            std::vector<int4> rc((size_t)nb * V);
            std::vector<const float*> xs, xts;
            std::vector<float*> zs;
            for (int b = 0; b < nb; ++b) {
                for (int vs = 0; vs < V; ++vs) rc[(size_t)b * V + vs] = rect_for(b, vs);
                xs.push_back(pN(xN, oslots[b]));
                xts.push_back(pT(xT, oslots[b]));
                zs.push_back(z);   // packed footprint storage (ZRect table of the slot)
            }
            project(PROJ_FP, vsel, oslots, rc, xs, xts, {}, {}, zs, nullptr, 0.f, 0, st, 0);
        }
        if (up && up->yev) {
            BSGD_CUDA(cudaStreamWaitEvent(st, up->yev, 0));
            if (up->y_reset) {   // the selected rows now; the others after this epoch (bsgd_run)
                reset_r(y, st, &sel_rows);
                BSGD_CUDA(cudaMemcpyAsync(d_normsq0, d_normsq, sizeof(double) * M, cudaMemcpyDeviceToDevice, st));
            }
        }
        if (ev) BSGD_CUDA(cudaEventRecord(ev[1], st));
        nv_phase.reset(new NvtxRange("residual + exchange (Algo 1 l.7)"));
        // ---- line 7: r = y - sum_j z^j on the selected rows (+ allreduce of the partials)
        {
            std::vector<char> staging(tab_bytes / 2);
            size_t off = tab_bytes / 2;
            staging.resize(off);
            ResLaunch Rl;
            Rl.n_slots = V;
            Rl.views = tab_put(off, vsel, staging);
            Rl.slot_row = tab_put(off, slot_row, staging);
            int* drows = tab_put(off, sel_rows, staging);
            BSGD_CUDA(cudaMemcpyAsync(d_tab + tab_bytes / 2, staging.data() + tab_bytes / 2,
                                      off - tab_bytes / 2, cudaMemcpyHostToDevice, st));
            Rl.per = (int)per;
            Rl.z = z;
            Rl.zr = d_zr;
            Rl.n_views = n_views;
            Rl.nu = nu;
            Rl.n_rays = n_rays;
            Rl.s = s;
            Rl.y = y;
            Rl.r = r;
            Rl.pc = pc;
            Rl.normsq = d_normsq;
            Rl.part = d_rpart;
            Rl.M = M;
            launch_zero_rows(d_normsq, drows, (int)sel_rows.size(), st);
            if (!coll) {
                Rl.mode = 0;
                launch_residual(Rl, st);
            } else if (band) {
                Rl.mode = 1;
                launch_residual(Rl, st);
                band_residual(Rl, vsel, sel_rows, drows, staging, off, st);
            } else {
                Rl.mode = 1;
                launch_residual(Rl, st);
                allreduce_f(pc, (size_t)V * per, st);
                if (world > 1) {   // ring allreduce: 2 (G-1)/G of the buffer sent per rank
                    comm_bytes += (unsigned long long)(8.0 * (double)V * per * (world - 1) / world);
                    ++comm_msgs;
                }
                Rl.mode = 2;
                launch_residual(Rl, st);
            }
        }
        if (ev) BSGD_CUDA(cudaEventRecord(ev[2], st));
        nv_phase.reset(new NvtxRange("bp + step (Algo 1 l.9-14)"));
        // ---- lines 8-10: g_hat^i_{J_j} = 2 (A_{I_i}^{J_j})^T r_{I_i}, then lines 11-14
        std::vector<float*> oN, oT;
        std::vector<const float*> none;
        for (int b = 0; b < nb; ++b) {
            oN.push_back(pN(accN, oslots[b]));
            oT.push_back(pT(accT, oslots[b]));
        }
        if (sgd) {   // Eq. 4: g = 2 A_I^T r_I over all selected rows, no memory
            std::vector<int4> rc((size_t)nb * V, make_int4(0, nu, 0, nv));
            bp(vsel, oslots, rc, oN, oT, st);
            if (ev) BSGD_CUDA(cudaEventRecord(ev[3], st));
            for (int b = 0; b < nb; ++b)
                update(UPD_SGD, oslots[b], x_owned + oslots[b] * bsize, mu_, 1, nullptr, 0, st);
        } else {
            int vs0 = 0;
            for (size_t ii = 0; ii < sel_rows.size(); ++ii) {
                const int i = sel_rows[ii];
                const int Vi = (int)rows[i].size();
                std::vector<int> vi(vsel.begin() + vs0, vsel.begin() + vs0 + Vi);
                std::vector<int4> rc((size_t)nb * Vi);
                for (int b = 0; b < nb; ++b)
                    for (int k = 0; k < Vi; ++k) rc[(size_t)b * Vi + k] = rect_for(b, vs0 + k);
                const int fin = (ii + 1 == sel_rows.size());
                if (fin && up && up->x_host_out) {
                    // blocks this epoch does not update are final already
                    BSGD_CUDA(cudaEventRecord(up_ev[s + 1], st));
                    BSGD_CUDA(cudaStreamWaitEvent(copy_st, up_ev[s + 1], 0));
                    for (int q = 0; q < s; ++q)
                        if (std::find(oslots.begin(), oslots.end(), q) == oslots.end())
                            BSGD_CUDA(cudaMemcpyAsync(up->x_host_out + (size_t)q * bsize, x_owned + (size_t)q * bsize,
                                                      sizeof(float) * bsize, cudaMemcpyDeviceToHost, copy_st));
                    for (int b = 0; b < nb; ++b) {
                        std::vector<int4> rcb(rc.begin() + (size_t)b * Vi, rc.begin() + (size_t)(b + 1) * Vi);
                        bp(vi, {oslots[b]}, rcb, {oN[b]}, {oT[b]}, st);
                        update(UPD_BSGD, oslots[b], x_owned + oslots[b] * bsize, mu_, fin, nullptr, 0, st,
                               nullptr, nullptr, nullptr, i);
                        BSGD_CUDA(cudaEventRecord(up_ev[b], st));
                        BSGD_CUDA(cudaStreamWaitEvent(copy_st, up_ev[b], 0));
                        BSGD_CUDA(cudaMemcpyAsync(up->x_host_out + (size_t)oslots[b] * bsize,
                                                  x_owned + (size_t)oslots[b] * bsize, sizeof(float) * bsize,
                                                  cudaMemcpyDeviceToHost, copy_st));
                    }
                    if (ev) BSGD_CUDA(cudaEventRecord(ev[3], st));
                } else {
                    bp(vi, oslots, rc, oN, oT, st);
                    if (ev && fin) BSGD_CUDA(cudaEventRecord(ev[3], st));
                    for (int b = 0; b < nb; ++b)
                        update(UPD_BSGD, oslots[b], x_owned + oslots[b] * bsize, mu_, fin, nullptr, 0, st,
                               nullptr, nullptr, nullptr, i);
                }
                vs0 += Vi;
            }
        }
        if (ev) BSGD_CUDA(cudaEventRecord(ev[4], st));
    }

    // BP of views `vv` into the accumulators of `slots` (oN / oT: their accN / accT interiors):
    // fp32 REDs, or with `det` 64-bit fixed-point REDs into int64 twins converted afterwards,
    // which makes g_hat independent of the order of the ray threads (SURVEY §8b Determinism)
    void bp(const std::vector<int>& vv, const std::vector<int>& slots, const std::vector<int4>& rc,
            const std::vector<float*>& oN, const std::vector<float*>& oT, cudaStream_t st) {
        if (!det) {
            project(PROJ_BP, vv, slots, rc, {}, {}, oN, oT, {}, r, 2.f, 0, st, 0);
            return;
        }
        const size_t rawN = (size_t)s * padN + 2 * slack, rawT = (size_t)s * padT + 2 * slack;
        if (!acc64N) {
            acc64N = dnew<long long>((long long)rawN) + slack;
            acc64T = dnew<long long>((long long)rawT) + slack;
            d_det_scale = dnew<float>(1);
            d_det_max = dnew<unsigned>(1);
        }
        launch_det_scale(r, n_rays, (int)vv.size(), rays_per_cell, 2.f, d_det_max, d_det_scale, st);
        std::vector<float*> dN, dT;
        for (size_t k = 0; k < slots.size(); ++k) {   // the int64 twin at the same element offsets
            dN.push_back(reinterpret_cast<float*>(acc64N + (oN[k] - accN)));
            dT.push_back(reinterpret_cast<float*>(acc64T + (oT[k] - accT)));
        }
        project(PROJ_BPD, vv, slots, rc, {}, {}, dN, dT, {}, r, 2.f, 0, st, 0);
        for (size_t k = 0; k < slots.size(); ++k) {   // whole padded block regions (borders too)
            const long long bN = (long long)slots[k] * padN, bT = (long long)slots[k] * padT;
            launch_acc64_to_f32(acc64N + bN, accN + bN, padN, d_det_scale, st);
            launch_acc64_to_f32(acc64T + bT, accT + bT, padT, d_det_scale, st);
        }
        BSGD_CUDA(cudaMemsetAsync(acc64N - slack, 0, sizeof(long long) * rawN, st));
        BSGD_CUDA(cudaMemsetAsync(acc64T - slack, 0, sizeof(long long) * rawT, st));
    }

    void reset(const float* y, cudaStream_t st) {
        reset_state(st);
        reset_r(y, st);
    }
    // Algo 1 line 1 without y: z = 0, g_hat = 0, g = 0 and the host-side schedule state
    void reset_state(cudaStream_t st) {
        BSGD_CUDA(cudaMemsetAsync(z, 0, sizeof(float) * (size_t)z_size, st));
        BSGD_CUDA(cudaMemsetAsync(ghat, 0, sizeof(float) * (size_t)M * s * bsize, st));
        BSGD_CUDA(cudaMemsetAsync(g, 0, sizeof(float) * (size_t)s * bsize, st));
        if (eud_cur) BSGD_CUDA(cudaMemsetAsync(eud_cur, 0, sizeof(float) * (size_t)s * bsize, st));
        epoch = 0;
        have_prev_eud = false;
        have_theta_prev = false;
        rnorm_hist.clear();
    }
    // ... and r = y on every row block with ||r_I||^2 (needs y on the device)
    // only: the row blocks to reset (nullptr: all; d_normsq of the others is left untouched)
    void reset_r(const float* y, cudaStream_t st, const std::vector<int>* only = nullptr) {
        if (!only) BSGD_CUDA(cudaMemsetAsync(d_normsq, 0, sizeof(double) * M, st));
        // r = y - sum z = y on every row block, with ||r_I||^2 (Algo 1 line 1)
        std::vector<int> all, srow;
        std::vector<int> blocks_;
        if (only) blocks_ = *only;
        else for (int i = 0; i < M; ++i) blocks_.push_back(i);
        for (int i : blocks_)
            for (int v : rows[i]) {
                all.push_back(v);
                srow.push_back(i);
            }
        if (all.empty()) return;
        std::vector<char> staging;
        size_t off = 0;
        ResLaunch Rl;
        Rl.n_slots = (int)all.size();
        Rl.views = tab_put(off, all, staging);
        Rl.slot_row = tab_put(off, srow, staging);
        tab_upload(staging, off, st);
        Rl.per = (int)per;
        Rl.z = z;
        Rl.zr = d_zr;
        Rl.n_views = n_views;
        Rl.nu = nu;
        Rl.n_rays = n_rays;
        Rl.s = 0;                  // no z terms: r = y exactly (Algo 1 line 1, z = 0), even when a
                                   // deferred reset runs after the first FP has filled some z
        Rl.y = y;
        Rl.r = r;
        Rl.pc = pc;
        Rl.normsq = d_normsq;
        Rl.part = d_rpart;
        Rl.M = M;
        Rl.mode = 0;
        launch_residual(Rl, st);   // no allreduce needed
    }

    // Exact ray-voxel intersection counts (positive-length Siddon segments) per
    // (owned block, view, detector tile), from one COUNT traversal of every view; the
    // FP/BP hot loops do not count.  Used for the visits/s metric.
    void ensure_visit_table(cudaStream_t st) {
        if (vtab_ready) return;
        std::vector<int> all(n_views), slots(s);
        for (int v = 0; v < n_views; ++v) all[v] = v;
        for (int b = 0; b < s; ++b) slots[b] = b;
        unsigned long long* dc = dnew<unsigned long long>((long long)s * n_views);
        vtab.assign((size_t)s * n_views * T, 0ull);
        std::vector<unsigned long long> h((size_t)s * n_views);
        for (int t = 0; t < T; ++t) {
            const int tu = t % tiles_u, tv = t / tiles_u;
            const int4 r = make_int4((int)((long long)tu * nu / tiles_u), (int)((long long)(tu + 1) * nu / tiles_u),
                                     (int)((long long)tv * nv / tiles_v), (int)((long long)(tv + 1) * nv / tiles_v));
            std::vector<int4> rc((size_t)s * n_views, r);
            BSGD_CUDA(cudaMemsetAsync(dc, 0, sizeof(unsigned long long) * s * n_views, st));
            count_target = dc;
            project(PROJ_COUNT, all, slots, rc, {}, {}, {}, {}, {}, nullptr, 0.f, 0, st, 0);
            count_target = nullptr;
            BSGD_CUDA(cudaMemcpyAsync(h.data(), dc, sizeof(unsigned long long) * h.size(), cudaMemcpyDeviceToHost, st));
            BSGD_CUDA(cudaStreamSynchronize(st));
            for (int b = 0; b < s; ++b)
                for (int v = 0; v < n_views; ++v) vtab[((size_t)b * n_views + v) * T + t] = h[(size_t)b * n_views + v];
        }
        vtab_ready = true;
    }

    // IM table of the given kind (0: L1 mass = ones-pass chord sums; 1: IS_AREA = count of
    // tile rays crossing the block), recomputed when the kind changes
    void ensure_im_table(cudaStream_t st, int kind = 0) {
        if (q_ready && q_kind == kind) return;
        double* dw = dnew<double>((long long)s * n_views * T);
        std::vector<BlockDesc> bl(s);
        for (int b = 0; b < s; ++b) box(first + b, bl[b].lo, bl[b].hi);
        std::vector<char> staging;
        size_t off = 0;
        ImLaunch I;
        I.g = kgeom();
        I.n_blocks = s;
        I.blocks = tab_put(off, bl, staging);
        I.tiles_u = tiles_u;
        I.tiles_v = tiles_v;
        I.w = dw;
        I.area = kind;
        BSGD_CUDA(cudaMemsetAsync(dw, 0, sizeof(double) * (size_t)s * n_views * T, st));
        tab_upload(staging, off, st);
        launch_im_weights(I, st);
        w.assign((size_t)s * n_views * T, 0.0);
        BSGD_CUDA(cudaMemcpyAsync(w.data(), dw, sizeof(double) * w.size(), cudaMemcpyDeviceToHost, st));
        BSGD_CUDA(cudaStreamSynchronize(st));
        q.assign(w.size(), 0u);
        for (size_t e = 0; e < w.size(); e += T) {
            double S = 0.0;
            for (int t = 0; t < T; ++t) S += w[e + t];
            for (int t = 0; t < T; ++t) q[e + t] = S > 0 ? (uint32_t)floor(65536.0 * w[e + t] / S) : 0u;
        }
        q_ready = true;
        q_kind = kind;
    }

    // FGP TV prox (Algo 4 line 16) on the owned volume: x <- argmin 1/2|t-x|^2 + w TV(t)
    // ------------------------------------------------------------ comparison solvers
    // (oracle/solvers.py).  gout = 2 A_I^T (yv - A_I p) over the views of the
    // row blocks `rsel` and all owned column blocks (+ the residual allreduce when world > 1);
    // ||yv_I - A_I p||^2 lands in d_normsq[i] for i in rsel.  Clobbers z, r and the BP
    // accumulators (the BSGD state is reset after a solve).
    void row_grad(const float* yv, float* p, float* gout, const std::vector<int>& rsel, cudaStream_t st) {
        std::vector<int> vsel, slot_row, slots(s);
        for (int i : rsel)
            for (int v : rows[i]) {
                vsel.push_back(v);
                slot_row.push_back(i);
            }
        for (int b = 0; b < s; ++b) slots[b] = b;
        const int V = (int)vsel.size();
        refresh_xT(p, slots, st);
        std::vector<int4> rc((size_t)s * V, make_int4(0, nu, 0, nv));
        {
            std::vector<const float*> xs, xts;
            std::vector<float*> zs;
            for (int b = 0; b < s; ++b) {
                xs.push_back(pN(xN, b));
                xts.push_back(pT(xT, b));
                zs.push_back(z);
            }
            project(PROJ_FP, vsel, slots, rc, xs, xts, {}, {}, zs, nullptr, 0.f, 0, st, 0);
        }
        {
            std::vector<char> staging(tab_bytes / 2);
            size_t off = tab_bytes / 2;
            staging.resize(off);
            ResLaunch Rl;
            Rl.n_slots = V;
            Rl.views = tab_put(off, vsel, staging);
            Rl.slot_row = tab_put(off, slot_row, staging);
            int* drows = tab_put(off, rsel, staging);
            if (off > tab_bytes) fail(BSGD_E_CONTRACT, "launch table overflow");
            BSGD_CUDA(cudaMemcpyAsync(d_tab + tab_bytes / 2, staging.data() + tab_bytes / 2,
                                      off - tab_bytes / 2, cudaMemcpyHostToDevice, st));
            Rl.per = (int)per;
            Rl.z = z;
            Rl.zr = d_zr;
            Rl.n_views = n_views;
            Rl.nu = nu;
            Rl.n_rays = n_rays;
            Rl.s = s;
            Rl.y = yv;
            Rl.r = r;
            Rl.pc = pc;
            Rl.normsq = d_normsq;
            Rl.part = d_rpart;
            Rl.M = M;
            launch_zero_rows(d_normsq, drows, (int)rsel.size(), st);
            Rl.mode = coll ? 1 : 0;
            launch_residual(Rl, st);
            if (coll) {
                allreduce_f(pc, (size_t)V * per, st);
                Rl.mode = 2;
                launch_residual(Rl, st);
            }
        }
        std::vector<float*> oN, oT;
        std::vector<const float*> none;
        for (int b = 0; b < s; ++b) {
            oN.push_back(pN(accN, b));
            oT.push_back(pT(accT, b));
        }
        project(PROJ_BP, vsel, slots, rc, none, none, oN, oT, {}, r, 2.f, 0, st, 0);
        for (int b = 0; b < s; ++b) update(UPD_OUT, b, p + b * bsize, 0.f, 1, gout + b * bsize, 0, st);
    }

    // host copy of 1/2 sum_i d_normsq[i] (the objective after a full row_grad)
    double half_normsq(cudaStream_t st) {
        BSGD_CUDA(cudaMemcpyAsync(h_normsq.data(), d_normsq, sizeof(double) * M, cudaMemcpyDeviceToHost, st));
        BSGD_CUDA(cudaStreamSynchronize(st));
        double s2 = 0;
        for (double v : h_normsq) s2 += v;
        return 0.5 * s2;
    }

    void solve(int solver, const float* y, float* x, int iters, double mu0, double lam, int tv_iters, int m,
               uint64_t seed, double* obj_log, double* mu_log, cudaStream_t st) {
        const long long n = (long long)s * bsize;
        auto need = [&](float*& b) { if (!b) b = dnew<float>(n, false); };
        std::vector<int> all(M);
        for (int i = 0; i < M; ++i) all[i] = i;
        double mu = mu0;
        if (solver == BSGD_SOLVER_GD || solver == BSGD_SOLVER_ISTA) {
            need(sv_a);                                       // g
            for (int k = 0; k < iters; ++k) {
                row_grad(y, x, sv_a, all, st);
                if (obj_log) obj_log[k] = half_normsq(st);
                if (mu_log) mu_log[k] = mu;
                launch_lincomb(x, 1.f, x, (float)mu, sv_a, 0.f, nullptr, n, st);   // x + mu g
                if (solver == BSGD_SOLVER_ISTA) tv_prox(x, mu * lam, tv_iters, st);
            }
        } else if (solver == BSGD_SOLVER_GD_BB) {
            need(sv_a); need(sv_b); need(sv_c);               // g, x_prev, g_prev
            for (int k = 0; k < iters; ++k) {
                row_grad(y, x, sv_a, all, st);
                if (obj_log) obj_log[k] = half_normsq(st);
                if (k > 0) {                                  // BB1: <s,s> / <s,w>
                    BSGD_CUDA(cudaMemsetAsync(d_red, 0, 2 * sizeof(double), st));
                    launch_bb_dots(x, sv_b, sv_c, sv_a, n, d_red, st);
                    allreduce_d(d_red, 2, st);
                    double h2[2];
                    BSGD_CUDA(cudaMemcpyAsync(h2, d_red, sizeof(h2), cudaMemcpyDeviceToHost, st));
                    BSGD_CUDA(cudaStreamSynchronize(st));
                    if (h2[1] > 0.0) mu = h2[0] / h2[1];
                }
                if (mu_log) mu_log[k] = mu;
                BSGD_CUDA(cudaMemcpyAsync(sv_b, x, sizeof(float) * n, cudaMemcpyDeviceToDevice, st));
                std::swap(sv_a, sv_c);                        // g_prev <- g
                launch_lincomb(x, 1.f, x, (float)mu, sv_c, 0.f, nullptr, n, st);
            }
        } else if (solver == BSGD_SOLVER_FISTA) {
            need(sv_a); need(sv_b); need(sv_c);               // g, v, z_new
            BSGD_CUDA(cudaMemcpyAsync(sv_b, x, sizeof(float) * n, cudaMemcpyDeviceToDevice, st));   // v_0 = x_0
            double t = 1.0;
            for (int k = 0; k < iters; ++k) {
                row_grad(y, sv_b, sv_a, all, st);             // g(v)
                if (obj_log) obj_log[k] = half_normsq(st);
                if (mu_log) mu_log[k] = mu;
                launch_lincomb(sv_c, 1.f, sv_b, (float)mu, sv_a, 0.f, nullptr, n, st);   // v + mu g(v)
                if (lam > 0.0) tv_prox(sv_c, mu * lam, tv_iters, st);   // z+ (lam = 0: identity)
                const double t1 = (1.0 + sqrt(1.0 + 4.0 * t * t)) / 2.0, beta = (t - 1.0) / t1;
                // v+ = z+ + beta (z+ - z)   (z = x)
                launch_lincomb(sv_b, (float)(1.0 + beta), sv_c, (float)(-beta), x, 0.f, nullptr, n, st);
                BSGD_CUDA(cudaMemcpyAsync(x, sv_c, sizeof(float) * n, cudaMemcpyDeviceToDevice, st));
                t = t1;
            }
        } else if (solver == BSGD_SOLVER_SVRG) {
            need(sv_a); need(sv_b); need(sv_c); need(sv_d);   // G~, x~, d = x - x~, g_I(d)
            if (!y_zero) y_zero = dnew<float>(n_rays, true);
            const int inner = m > 0 ? m : M;
            long long step = 0;
            for (int k = 0; k < iters; ++k) {
                BSGD_CUDA(cudaMemcpyAsync(sv_b, x, sizeof(float) * n, cudaMemcpyDeviceToDevice, st));
                row_grad(y, sv_b, sv_a, all, st);             // G~ = g(x~)
                if (obj_log) obj_log[k] = half_normsq(st);
                if (mu_log) mu_log[k] = mu;
                for (int t = 0; t < inner; ++t, ++step) {
                    int i = 0;
                    host::select(seed, 1, (int)step, M, 1, &i);
                    launch_lincomb(sv_c, 1.f, x, -1.f, sv_b, 0.f, nullptr, n, st);   // d = x - x~
                    row_grad(y_zero, sv_c, sv_d, std::vector<int>{i}, st);          // 2 A_I^T (0 - A_I d) = -h
                    // x <- x - mu M h + mu G~ = x + mu M (-h) + mu G~
                    launch_lincomb(x, 1.f, x, (float)(mu * M), sv_d, (float)mu, sv_a, n, st);
                }
            }
        } else {
            fail(BSGD_E_CONTRACT, "unknown solver");
        }
        reset(y, st);                                         // back to the initial BSGD state
        epoch = 0;
    }

    // Sharded TV (the stencil's only cross-rank neighbours are in z) needs every rank to own
    // whole z-layers of the block grid: z-slabs, or any bx x by x bz grid with N/G a multiple
    // of bx*by (e.g. the paper's 2x2x2 octants at G = 2).  The owned region is then the global
    // z-range [z0, z1) and the halos are whole z-planes.
    bool tv_shardable() const {
        return world == 1 || (bgrid[0] == 1 && bgrid[1] == 1) || s % (bgrid[0] * bgrid[1]) == 0;
    }
    int owned_z0() const { return zsplit ? zsp[first] : (first / (bgrid[0] * bgrid[1])) * bd[2]; }
    int owned_z1() const { return zsplit ? zsp[first + s] : ((first + s) / (bgrid[0] * bgrid[1])) * bd[2]; }
    // Unequal slabs: the TV stencil runs on the owned planes packed contiguously (tv_xc);
    // copy the blocks' rows in / out (their real parts; the zero tails stay as they are)
    void zsplit_pack(const float* x_owned, float* xc, bool in, cudaStream_t st) {
        long long o = 0;
        for (int b = 0; b < s; ++b) {
            const long long nb = vox_of(first + b);
            if (in) BSGD_CUDA(cudaMemcpyAsync(xc + o, x_owned + b * bsize, sizeof(float) * nb, cudaMemcpyDeviceToDevice, st));
            else BSGD_CUDA(cudaMemcpyAsync((float*)x_owned + b * bsize, xc + o, sizeof(float) * nb, cudaMemcpyDeviceToDevice, st));
            o += nb;
        }
    }
    long long owned_real() const { return (long long)dims[0] * dims[1] * (owned_z1() - owned_z0()); }
    // Global plane z (inside the owned z-range) of an owned block-major field as a contiguous
    // [y][x] plane: in place for z-slab layouts, else gathered from the bx*by blocks of its
    // layer into tv_pk (stream-ordered: the previous exchange reading tv_pk is complete).
    const float* plane_of(const float* owned, int z, cudaStream_t st) {
        const long long plane = (long long)dims[0] * dims[1];
        if (bgrid[0] == 1 && bgrid[1] == 1) return owned + (long long)(z - owned_z0()) * plane;
        if (!tv_pk) tv_pk = dnew<float>(plane, false);
        TvLaunch T{};
        for (int c = 0; c < 3; ++c) {
            T.dims[c] = dims[c];
            T.bdims[c] = bd[c];
            T.bgrid[c] = bgrid[c];
        }
        T.block0 = first;
        T.n = (long long)s * bsize;
        launch_pack_plane(T, owned, z, tv_pk, st);
        return tv_pk;
    }

    // method 0: FGP (Beck-Teboulle, reading A16); 1: Chambolle 2004 (tau = 1/L), the flag of
    // one dual field (tv_q, double-buffered on the fused path)
    void tv_prox(float* x_owned, double wgt, int iters, cudaStream_t st, int method = 0) {
        NvtxRange nv_("tv prox (Algo 4 l.16)");
        if (wgt == 0.0 || iters <= 0) return;
        if (zsplit) {
            if (!tv_xc) tv_xc = dnew<float>(owned_real(), false);
            zsplit_pack(x_owned, tv_xc, true, st);
            tv_prox_on(tv_xc, owned_real(), wgt, iters, st, method);
            zsplit_pack(x_owned, tv_xc, false, st);
            return;
        }
        tv_prox_on(x_owned, (long long)s * bsize, wgt, iters, st, method);
    }
    // the prox on an owned volume whose blocks are stored back to back (n voxels)
    void tv_prox_on(float* x_owned, long long n, double wgt, int iters, cudaStream_t st, int method) {
        // z-slab layouts (the owned volume is one [z][y][x] array) take the fused iteration
        const bool fused = bgrid[0] == 1 && bgrid[1] == 1;
        const long long plane = (long long)dims[0] * dims[1];
        if (wgt == 0.0 || iters <= 0) return;   // the identity: no dual fields needed
        if (!tv_p) {
            tv_p = dnew<float>(3 * n, false);
            tv_q = dnew<float>(3 * n, false);
            tv_hq = dnew<float>(plane);
            if (fused) {
                tv_q2 = dnew<float>(3 * n, false);
                tv_hp = dnew<float>(4 * plane);
            } else {
                tv_u = dnew<float>(n, false);
                tv_hu = dnew<float>(plane);
            }
        }
        // b = x itself: read-only during the iterations, and the final x = b - w grad^T p reads
        // b only at the voxel it writes.  The fused path's first iteration treats q = p = 0
        // without reading them, so the dual fields need no clearing there.
        if (!fused) {
            BSGD_CUDA(cudaMemsetAsync(tv_p, 0, sizeof(float) * 3 * n, st));
            BSGD_CUDA(cudaMemsetAsync(tv_q, 0, sizeof(float) * 3 * n, st));
        }
        TvLaunch Tl{};
        for (int c = 0; c < 3; ++c) {
            Tl.dims[c] = dims[c];
            Tl.bdims[c] = bd[c];
            Tl.bgrid[c] = bgrid[c];
        }
        Tl.block0 = first;
        Tl.b = x_owned;
        Tl.u = tv_u;
        Tl.p = tv_p;
        Tl.q = tv_q;
        Tl.out = x_owned;
        Tl.halo_q_next = tv_hq;
        Tl.halo_u_prev = tv_hu;
        Tl.w = wgt;
        int axes = (dims[0] > 1) + (dims[1] > 1) + (dims[2] > 1);
        Tl.L = 4.0 * axes;
        Tl.n = n;
        Tl.z0 = owned_z0();
        Tl.z1 = owned_z1();
        Tl.chambolle = method == 1;
        double sk = 1.0;
        if (fused && method == 0 && dims[0] % 4 == 0 && !getenv("BSGD_TV_PLANEWISE")) {
            // z-marching FGP (k_tv_fgp_z): p_{k-1}, p_{k-2}, p_k rotate through tv_q, tv_q2, tv_p
            if (!tvz_hp) {
                tvz_hp = dnew<float>(7 * plane);
                tvz_hn = dnew<float>(2 * plane);
            }
            float* buf[3] = {tv_q, tv_q2, tv_p};
            // one rank owning the whole volume: two iterations per pass (k_tv_fgp_z2, temporal
            // blocking), p_k in buf4[k % 4]; an odd last iteration takes k_tv_fgp_z
            const bool z2 = world == 1 && iters >= 2 && Tl.z0 == 0 && Tl.z1 == dims[2] &&
                            !(getenv("BSGD_TV_Z2") && atoi(getenv("BSGD_TV_Z2")) == 0);
            float* buf4[4] = {tv_q, tv_q2, tv_p, nullptr};
            if (z2) {
                if (!tv_q3) tv_q3 = dnew<float>(3 * n, false);
                buf4[3] = tv_q3;
            }
            auto b4 = [&](int j) { return buf4[((j % 4) + 4) % 4]; };
            std::vector<double> sk_(iters + 3, 1.0);   // s_1 = 1, s_{j+1} = (1 + sqrt(1 + 4 s_j^2)) / 2
            for (int j = 1; j + 1 < (int)sk_.size(); ++j) sk_[j + 1] = (1.0 + sqrt(1.0 + 4.0 * sk_[j] * sk_[j])) / 2.0;
            auto beta_of = [&](int j) { return j >= 1 ? (sk_[j] - 1.0) / sk_[j + 1] : 0.0; };   // beta_j
            TvzLaunch Z{};
            Z.nx = dims[0];
            Z.ny = dims[1];
            Z.nz = dims[2];
            Z.z0 = Tl.z0;
            Z.z1 = Tl.z1;
            Z.n = n;
            Z.b = x_owned;
            Z.halo_prev = tvz_hp;
            Z.halo_next = tvz_hn;
            Z.w = (float)wgt;
            Z.s = (float)(1.0 / (Tl.L * wgt));
            Z.zc = std::max(1, std::min(16, (Tl.z1 - Tl.z0) / 4));
            if (const char* e = getenv("BSGD_TV_ZC")) Z.zc = std::max(1, atoi(e));   // A/B hooks
            Z.pf = 2;
            if (const char* e = getenv("BSGD_TV_PF")) Z.pf = std::max(0, atoi(e));
            if (world > 1) halo_exchange(x_owned + n - plane, tvz_hp + 6 * plane, plane, false, st);   // b of z0-1
            if (z2) {
                Tvz2Launch Y{};
                Y.nx = dims[0];
                Y.ny = dims[1];
                Y.nz = dims[2];
                Y.n = n;
                Y.b = x_owned;
                Y.w = (float)wgt;
                Y.s = (float)(1.0 / (Tl.L * wgt));
                Y.zc = std::max(1, std::min(32, dims[2] / 8));
                if (const char* e = getenv("BSGD_TV_Z2C")) Y.zc = std::max(1, atoi(e));   // A/B hooks
                Y.pf = 1;
                if (const char* e = getenv("BSGD_TV_PF")) Y.pf = std::max(0, atoi(e));
                int k = 1;
                for (; k + 1 <= iters; k += 2) {
                    Y.P1 = b4(k - 1);
                    Y.P2 = b4(k - 2);
                    Y.Pa = b4(k);
                    Y.Pb = b4(k + 1);
                    Y.stage = k == 1 ? 1 : (k == 2 ? 2 : 0);
                    Y.beta0 = (float)beta_of(k - 1);
                    Y.beta1 = (float)beta_of(k);
                    launch_tv_fgp_z2(Y, st);
                }
                if (k == iters) {                            // odd count: the last iteration alone
                    Z.P1 = b4(k - 1);
                    Z.P2 = b4(k - 2);
                    Z.Pn = b4(k);
                    Z.stage = k == 1 ? 1 : (k == 2 ? 2 : 0);
                    Z.beta = (float)beta_of(k - 1);
                    launch_tv_fgp_z(Z, st);
                }
                float* pf = b4(iters);                       // p_K
                Tl.first = 0;
                Tl.q = pf;
                Tl.wf = (float)wgt;
                launch_tv_out(Tl, x_owned, st);
                return;
            }
            double s_prev = 1.0;                             // s_{k-1}
            for (int k = 1; k <= iters; ++k) {
                double beta = 0.0;                           // beta_{k-1} = (s_{k-1} - 1) / s_k
                if (k >= 2) {
                    const double s_k = (1.0 + sqrt(1.0 + 4.0 * s_prev * s_prev)) / 2.0;
                    beta = (s_prev - 1.0) / s_k;
                    s_prev = s_k;
                }
                Z.P1 = buf[(k + 2) % 3];                     // p_{k-1}
                Z.P2 = buf[(k + 1) % 3];                     // p_{k-2}
                Z.Pn = buf[k % 3];                           // p_k
                Z.stage = k == 1 ? 1 : (k == 2 ? 2 : 0);
                Z.beta = (float)beta;
                if (world > 1 && k >= 2) {
                    for (int c = 0; c < 3; ++c) {            // P1, P2 of plane z0-1 from the previous rank
                        halo_exchange(Z.P1 + c * n + n - plane, tvz_hp + c * plane, plane, false, st);
                        halo_exchange(Z.P2 + c * n + n - plane, tvz_hp + (3 + c) * plane, plane, false, st);
                    }
                    halo_exchange(Z.P1 + 2 * n, tvz_hn, plane, true, st);           // z components of
                    halo_exchange(Z.P2 + 2 * n, tvz_hn + plane, plane, true, st);   // plane z1
                }
                launch_tv_fgp_z(Z, st);
            }
            float* pf = buf[iters % 3];                      // p_K
            Tl.first = 0;
            if (world > 1) halo_exchange(pf + 2 * n, tv_hq, plane, true, st);
            Tl.q = pf;
            Tl.wf = (float)wgt;
            launch_tv_out(Tl, x_owned, st);
            return;
        }
        if (fused) {
            Tl.halo_prev = tv_hp;
            halo_exchange(x_owned + n - plane, tv_hp + 3 * plane, plane, false, st);   // b of plane z0-1
            float *qa = tv_q, *qb = tv_q2;
            for (int it = 0; it < iters; ++it) {
                const double sk1 = (1.0 + sqrt(1.0 + 4.0 * sk * sk)) / 2.0;
                Tl.beta = (sk - 1.0) / sk1;
                for (int c = 0; c < 3; ++c)       // q of plane z0-1 from the previous rank
                    halo_exchange(qa + c * n + n - plane, tv_hp + c * plane, plane, false, st);
                halo_exchange(qa + 2 * n, tv_hq, plane, true, st);   // q_z of plane z1 from the next
                Tl.q = qa;
                Tl.q_out = qb;
                Tl.first = it == 0;
                Tl.wf = (float)wgt;
                Tl.sf = (float)(1.0 / (Tl.L * wgt));
                Tl.betaf = (float)Tl.beta;
                launch_tv_fgp(Tl, st);
                std::swap(qa, qb);
                sk = sk1;
            }
            Tl.first = 0;
            float* pf = method == 1 ? qa : tv_p;          // the final dual field
            halo_exchange(pf + 2 * n, tv_hq, plane, true, st);
            Tl.q = pf;
            Tl.wf = (float)wgt;
            launch_tv_out(Tl, x_owned, st);
            return;
        }
        for (int it = 0; it < iters; ++it) {
            const double sk1 = (1.0 + sqrt(1.0 + 4.0 * sk * sk)) / 2.0;
            Tl.beta = (sk - 1.0) / sk1;
            // u = b - w grad^T q   (needs q_z of plane z1 from the next rank)
            if (world > 1) halo_exchange(plane_of(tv_q + 2 * n, Tl.z0, st), tv_hq, plane, /*down*/ true, st);
            launch_tv_u(Tl, tv_q, tv_u, st);
            // p, q update (needs u of plane z0-1 from the previous rank)
            if (world > 1) halo_exchange(plane_of(tv_u, Tl.z1 - 1, st), tv_hu, plane, false, st);
            launch_tv_pq(Tl, st);
            sk = sk1;
        }
        float* pf = method == 1 ? tv_q : tv_p;                // Chambolle updates q in place
        if (world > 1) halo_exchange(plane_of(pf + 2 * n, Tl.z0, st), tv_hq, plane, true, st);
        launch_tv_u(Tl, pf, x_owned, st);
    }

    // A^T 1 over every view into `seen` (once): the voxels some ray crosses (reading A32)
    void ensure_seen(cudaStream_t st) {
        if (seen) return;
        seen = dnew<float>((long long)s * bsize, false);
        float* ones = dnew<float>(n_rays, false);
        launch_fill(ones, n_rays, 1.f, st);
        std::vector<int> all(n_views);
        for (int v = 0; v < n_views; ++v) all[v] = v;
        for (int b = 0; b < s; ++b) {
            project(PROJ_BP, all, {b}, {}, {}, {}, {pN(accN, b)}, {pT(accT, b)}, {}, ones, 1.f, 0, st, 0);
            update(UPD_OUT, b, nullptr, 0.f, 0, seen + b * bsize, 0, st);
        }
    }

    // TV(x) (Eq. 6) of the whole volume into *d_out (device; summed over ranks)
    void tv_value(const float* x_owned, double* d_out, cudaStream_t st) {
        if (zsplit) {
            if (!tv_xc) tv_xc = dnew<float>(owned_real(), false);
            zsplit_pack(x_owned, tv_xc, true, st);
            x_owned = tv_xc;
        }
        const long long n = zsplit ? owned_real() : (long long)s * bsize, plane = (long long)dims[0] * dims[1];
        if (!tv_shardable())
            fail(BSGD_E_PARTITION, "sharded TV needs whole z-layers of blocks per rank (N/G divisible by bx*by)");
        if (!tvv_halo) tvv_halo = dnew<float>(plane);
        TvLaunch Tl{};
        for (int c = 0; c < 3; ++c) {
            Tl.dims[c] = dims[c];
            Tl.bdims[c] = bd[c];
            Tl.bgrid[c] = bgrid[c];
        }
        Tl.block0 = first;
        Tl.n = n;
        Tl.z0 = owned_z0();
        Tl.z1 = owned_z1();
        Tl.halo_u_prev = tvv_halo;
        if (world > 1) halo_exchange(plane_of(x_owned, Tl.z1 - 1, st), tvv_halo, plane, false, st);   // x of plane z0-1
        BSGD_CUDA(cudaMemsetAsync(d_out, 0, sizeof(double), st));
        launch_tv_value(Tl, x_owned, d_out, st);
        allreduce_d(d_out, 1, st);
    }

    // z-slab halo: `down` = send my first plane (src) to rank-1 and receive rank+1's first
    // plane into dst; otherwise send my last plane (src) to rank+1, receive from rank-1.
    void halo_exchange(const float* src, float* dst, long long plane, bool down, cudaStream_t st) {
        if (world == 1) return;
        if (vg) {
            vg_offer(src, st);
            const int from = down ? rank + 1 : rank - 1;
            if (from >= 0 && from < world) {
                BSGD_CUDA(cudaStreamWaitEvent(st, vg->ev1[from], 0));
                BSGD_CUDA(cudaMemcpyAsync(dst, vg->src[from], sizeof(float) * plane, cudaMemcpyDeviceToDevice, st));
            }
            vg_release(st);
            return;
        }
        BSGD_NCCL(ncclGroupStart());
        if (down) {
            if (rank > 0) BSGD_NCCL(ncclSend(src, plane, ncclFloat, rank - 1, comm, st));
            if (rank < world - 1) BSGD_NCCL(ncclRecv(dst, plane, ncclFloat, rank + 1, comm, st));
        } else {
            if (rank < world - 1) BSGD_NCCL(ncclSend(src, plane, ncclFloat, rank + 1, comm, st));
            if (rank > 0) BSGD_NCCL(ncclRecv(dst, plane, ncclFloat, rank - 1, comm, st));
        }
        BSGD_NCCL(ncclGroupEnd());
    }
};

// ============================================================================
// C ABI
// ============================================================================
namespace {

template <class F> bsgd_status guard(bsgd_ctx ctx, F&& f) {
    if (ctx && ctx->poisoned) {
        g_last_error = "context poisoned by an earlier CUDA/NCCL error: " + ctx->err;
        return BSGD_E_POISONED;
    }
    try {
        f();
        return BSGD_OK;
    } catch (const Error& e) {
        g_last_error = e.msg;
        if (ctx) {
            ctx->err = e.msg;
            if (e.code == BSGD_E_CUDA || e.code == BSGD_E_NCCL) ctx->poisoned = true;
        }
        return e.code;
    } catch (const std::bad_alloc&) {
        g_last_error = "host allocation failed";
        return BSGD_E_OOM;
    } catch (...) {
        g_last_error = "unknown exception";
        return BSGD_E_CUDA;
    }
}

cudaStream_t S(void* p) { return (cudaStream_t)p; }

// Orders a call's stream after the previous call's work on the same context (see
// bsgd_ctx_s::stream_enter); records this call's end on its stream when the scope closes.
struct Ordered {
    bsgd_ctx c;
    cudaStream_t st;
    Ordered(bsgd_ctx c_, cudaStream_t st_) : c(c_), st(st_) { c->stream_enter(st); }
    ~Ordered() { c->stream_leave(st); }
};

bool is_device_ptr(const void* p) {
    cudaPointerAttributes a;
    cudaError_t e = cudaPointerGetAttributes(&a, p);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

void check_views(bsgd_ctx c, int n, const int32_t* views, const int32_t* rects) {
    if (n < 0 || (n > 0 && !views)) fail(BSGD_E_CONTRACT, "views pointer is NULL");
    for (int k = 0; k < n; ++k) {
        if (views[k] < 0 || views[k] >= c->n_views) fail(BSGD_E_DIMENSION, "view id out of range");
        if (rects) {
            const int32_t* q = rects + 4 * k;
            if (q[0] < 0 || q[1] > c->nu || q[0] > q[1] || q[2] < 0 || q[3] > c->nv || q[2] > q[3])
                fail(BSGD_E_DIMENSION, "detector rect outside the detector");
        }
    }
}

void check_sorted_unique(const int32_t* v, int n, int hi, const char* what) {
    for (int k = 0; k < n; ++k) {
        if (v[k] < 0 || v[k] >= hi) fail(BSGD_E_CONTRACT, std::string(what) + " id out of range");
        if (k && v[k] <= v[k - 1]) fail(BSGD_E_CONTRACT, std::string(what) + " must be sorted and unique");
    }
}

}  // namespace

#pragma GCC visibility push(default)
extern "C" {

int32_t bsgd_abi_version(void) { return BSGD_ABI_VERSION; }

uint64_t bsgd_kernel_launches(void) { return g_launches.load(); }

const char* bsgd_last_error(bsgd_ctx ctx) {
    if (ctx && !ctx->err.empty()) return ctx->err.c_str();
    return g_last_error.c_str();
}

bsgd_status bsgd_geometry_circular(int32_t beam, int32_t n_views, double arc_deg, double OP, double OD,
                                   int32_t det_u, int32_t det_v, double pitch_u, double pitch_v,
                                   double* vecs_out) {
    return guard(nullptr, [&] {
        if (n_views < 1 || det_u < 1 || det_v < 1 || !vecs_out) fail(BSGD_E_GEOMETRY, "bad counts");
        if (beam != BSGD_PARALLEL && (!(OP > 0) || !(OD > 0)))
            fail(BSGD_E_GEOMETRY, "non-positive source/detector distance");
        if (beam < 0 || beam > 2) fail(BSGD_E_GEOMETRY, "unknown beam");
        host::circular(beam, n_views, arc_deg, OP, OD, det_u, det_v, pitch_u, pitch_v, vecs_out);
    });
}

bsgd_status bsgd_sample(uint64_t seed, int32_t stream, int32_t epoch, int32_t n, int32_t m, int32_t* out) {
    return guard(nullptr, [&] {
        if (n < 1 || m < 0 || m > n || !out || stream < 0 || epoch < 0 || epoch >= (1 << 24))
            fail(BSGD_E_CONTRACT, "bad sample arguments");
        host::select(seed, stream, epoch, n, m, out);
    });
}

bsgd_status bsgd_sample_stratified(uint64_t seed, int32_t epoch, int32_t n, int32_t m, int32_t strata,
                                   int32_t* out) {
    return guard(nullptr, [&] {
        if (n < 1 || m < 0 || m > n || !out || epoch < 0 || epoch >= (1 << 24) || strata < 1 || n % strata ||
            m % strata)
            fail(BSGD_E_CONTRACT, "bad stratified sample arguments");
        host::select_stratified(seed, epoch, n, m, strata, out);
    });
}

bsgd_status bsgd_view_partition(int32_t n_views, int32_t M, int32_t kind, uint64_t seed, int32_t* views_out,
                                int32_t* offsets_out) {
    return guard(nullptr, [&] {
        if (M < 1 || M > n_views) fail(BSGD_E_PARTITION, "M must be in [1, n_views]");
        if (kind < 0 || kind > 2) fail(BSGD_E_CONTRACT, "unknown partition kind");
        host::view_partition(n_views, M, kind, seed, views_out, offsets_out);
    });
}

bsgd_status bsgd_eq8(int32_t nodes, int32_t M, int32_t N, int32_t* aM, int32_t* gN) {
    return guard(nullptr, [&] {
        if (nodes < 1 || M < 1 || N < 1) fail(BSGD_E_CONTRACT, "counts must be >= 1");
        host::eq8(nodes, M, N, aM, gN);
    });
}

bsgd_status bsgd_owned_blocks(int32_t N, int32_t world, int32_t rank, int32_t* first, int32_t* count) {
    return guard(nullptr, [&] {
        if (world < 1 || rank < 0 || rank >= world || N < 1) fail(BSGD_E_CONTRACT, "bad rank/world");
        if (N % world) fail(BSGD_E_PARTITION, "N must be divisible by the number of ranks");
        *count = N / world;
        *first = rank * (N / world);
    });
}

bsgd_status bsgd_nccl_unique_id(uint8_t* out128) {
    return guard(nullptr, [&] {
        ncclUniqueId id;
        BSGD_NCCL(ncclGetUniqueId(&id));
        memcpy(out128, &id, sizeof id);
    });
}

bsgd_status bsgd_create(const bsgd_geometry* geom, bsgd_dims dims, bsgd_block_grid blocks, bsgd_row_grid rowg,
                        const bsgd_dist* dist, const bsgd_alloc* alloc, bsgd_ctx* out) {
    return bsgd_create_ex(geom, dims, blocks, rowg, dist, alloc, nullptr, out);
}

bsgd_status bsgd_create_ex(const bsgd_geometry* geom, bsgd_dims dims, bsgd_block_grid blocks, bsgd_row_grid rowg,
                           const bsgd_dist* dist, const bsgd_alloc* alloc, const bsgd_create_opts* opts,
                           bsgd_ctx* out) {
    std::unique_ptr<bsgd_ctx_s> c(new bsgd_ctx_s());
    bsgd_status st = guard(nullptr, [&] {
        const int32_t* zsp_in = opts ? opts->z_splits : nullptr;
        if (!geom || !out || !geom->vecs) fail(BSGD_E_GEOMETRY, "NULL geometry");
        if (geom->n_views < 1 || geom->det_u < 1 || geom->det_v < 1) fail(BSGD_E_GEOMETRY, "bad counts");
        if (geom->beam < 0 || geom->beam > 2) fail(BSGD_E_GEOMETRY, "unknown beam");
        for (long long k = 0; k < 12LL * geom->n_views; ++k)
            if (!isfinite(geom->vecs[k])) fail(BSGD_E_GEOMETRY, "non-finite geometry vector");
        if (dims.nx < 1 || dims.ny < 1 || dims.nz < 1) fail(BSGD_E_PARTITION, "bad volume dims");
        if (blocks.bx < 1 || blocks.by < 1 || blocks.bz < 1 || dims.nx % blocks.bx || dims.ny % blocks.by ||
            (!zsp_in && dims.nz % blocks.bz))
            fail(BSGD_E_PARTITION, "volume dims must be divisible by the block grid");
        if (zsp_in) {
            if (blocks.bx != 1 || blocks.by != 1) fail(BSGD_E_PARTITION, "z_splits need a z-slab grid (1, 1, N)");
            if (zsp_in[0] != 0 || zsp_in[blocks.bz] != dims.nz) fail(BSGD_E_PARTITION, "z_splits must run from 0 to nz");
            for (int k = 0; k < blocks.bz; ++k)
                if (zsp_in[k + 1] <= zsp_in[k]) fail(BSGD_E_PARTITION, "z_splits must increase strictly");
        }
        if (rowg.M < 1 || rowg.M > geom->n_views) fail(BSGD_E_PARTITION, "M must be in [1, n_views]");
        if (rowg.kind < 0 || rowg.kind > 2) fail(BSGD_E_PARTITION, "unknown row partition kind");
        if (rowg.tiles_u < 1 || rowg.tiles_v < 1 || rowg.tiles_u > geom->det_u || rowg.tiles_v > geom->det_v)
            fail(BSGD_E_PARTITION, "bad tile grid");
        c->beam = geom->beam;
        c->n_views = geom->n_views;
        c->nu = geom->det_u;
        c->nv = geom->det_v;
        c->vecs.assign(geom->vecs, geom->vecs + 12LL * geom->n_views);
        c->dims[0] = dims.nx; c->dims[1] = dims.ny; c->dims[2] = dims.nz;
        c->bgrid[0] = blocks.bx; c->bgrid[1] = blocks.by; c->bgrid[2] = blocks.bz;
        for (int k = 0; k < 3; ++k) c->bd[k] = c->dims[k] / c->bgrid[k];
        if (zsp_in) {   // unequal z-slabs: blocks keep the stride of the thickest one
            c->zsplit = true;
            c->zsp.assign(zsp_in, zsp_in + blocks.bz + 1);
            c->bd[2] = 0;
            for (int k = 0; k < blocks.bz; ++k) c->bd[2] = std::max(c->bd[2], c->zsp[k + 1] - c->zsp[k]);
        }
        c->N = blocks.bx * blocks.by * blocks.bz;
        c->M = rowg.M;
        c->kind = rowg.kind;
        c->row_seed = rowg.seed;
        c->tiles_u = rowg.tiles_u;
        c->tiles_v = rowg.tiles_v;
        c->T = rowg.tiles_u * rowg.tiles_v;
        c->bsize = (long long)c->bd[0] * c->bd[1] * c->bd[2];
        c->per = (long long)c->nu * c->nv;
        c->n_rays = c->per * c->n_views;
        c->R = 0.5 * sqrt((double)dims.nx * dims.nx + (double)dims.ny * dims.ny + (double)dims.nz * dims.nz) + 1.0;
        for (int v = 0; v < c->n_views; ++v) {     // zero-length rays are invalid geometry
            const double* q = &c->vecs[12 * v];
            if (c->beam == BSGD_PARALLEL && q[0] == 0 && q[1] == 0 && q[2] == 0)
                fail(BSGD_E_GEOMETRY, "zero parallel ray direction");
        }
        if (dist && dist->world > 1) {
            c->rank = dist->rank;
            c->world = dist->world;
            if (c->rank < 0 || c->rank >= c->world) fail(BSGD_E_CONTRACT, "bad rank");
            if (c->N % c->world) fail(BSGD_E_PARTITION, "N must be divisible by the number of ranks");
            if (dist->vgroup) {
                if (dist->vgroup->world != c->world) fail(BSGD_E_CONTRACT, "world differs from the virtual group's");
                if (c->world > 8) fail(BSGD_E_CONTRACT, "virtual groups hold at most 8 ranks");
                c->vg = dist->vgroup;
            } else if (!dist->nccl_id) {
                fail(BSGD_E_CONTRACT, "nccl_id required when world > 1");
            }
        }
        c->s = c->N / c->world;
        c->first = c->rank * c->s;
        c->rays_per_cell = c->compute_rays_per_cell();
        if (const char* e = getenv("BSGD_BAND_ROWS")) c->band_rows = std::max(1, atoi(e));
        if (c->bsize >= (1LL << 31)) fail(BSGD_E_PARTITION, "a column block must hold fewer than 2^31 voxels");
        // row blocks
        std::vector<int32_t> vv(c->n_views), off(c->M + 1);
        host::view_partition(c->n_views, c->M, c->kind, c->row_seed, vv.data(), off.data());
        c->rows.resize(c->M);
        c->view_row.resize(c->n_views);
        for (int i = 0; i < c->M; ++i)
            for (int k = off[i]; k < off[i + 1]; ++k) {
                c->rows[i].push_back(vv[k]);
                c->view_row[vv[k]] = i;
            }
        if (alloc) c->alloc = *alloc;
        // device state
        const long long sb = (long long)c->s * c->bsize;
        c->d_vecs = c->dnew<double>(12LL * c->n_views, false);
        BSGD_CUDA(cudaMemcpy(c->d_vecs, c->vecs.data(), sizeof(double) * c->vecs.size(), cudaMemcpyHostToDevice));
        c->rowN = c->bd[0] + 2 * PAD_X;
        c->planeN = c->rowN * c->bd[1];
        c->rowT = c->bd[1] + 2 * PAD_X;
        c->planeT = c->rowT * c->bd[0];
        c->padN = (long long)c->planeN * (c->bd[2] + 2 * PAD_Z);
        c->padT = (long long)c->planeT * (c->bd[2] + 2 * PAD_Z);
        c->orgN = (long long)PAD_Z * c->planeN + PAD_X;
        c->orgT = (long long)PAD_Z * c->planeT + PAD_X;
        if (c->padN >= (1LL << 31) || c->padT >= (1LL << 31))
            fail(BSGD_E_PARTITION, "a padded block must hold < 2^31 voxels (32-bit offsets)");
        c->slack = (((long long)std::max(c->planeN, c->planeT) + 64 + 63) / 64) * 64;
        c->xT = c->dnew_pad(c->s, true);
        c->xN = c->dnew_pad(c->s, false);
        c->g = c->dnew<float>(sb);
        c->ghat = c->dnew<float>((long long)c->M * sb);
        {   // z^j only inside each block's detector footprint per view (the launch-culling
            // rectangle): at cfg5 about 1.3 full-length vectors for 8 slabs instead of 8
            c->h_zr.resize((size_t)c->s * c->n_views);
            long long off = 0;
            for (int b = 0; b < c->s; ++b) {
                int lo[3], hi[3];
                c->box(c->first + b, lo, hi);
                for (int v = 0; v < c->n_views; ++v) {
                    int4 f = c->footprint(lo, hi, v);
                    if (f.x >= f.y || f.z >= f.w) f = make_int4(0, 0, 0, 0);
                    ZRect& q = c->h_zr[(size_t)b * c->n_views + v];
                    q.u0 = f.x; q.u1 = f.y; q.v0 = f.z; q.v1 = f.w;
                    q.base = off;
                    q.pad_ = 0;
                    off += (long long)(f.y - f.x) * (f.w - f.z);
                }
            }
            c->z_size = std::max(off, 1LL);
            c->z = c->dnew<float>(c->z_size);
            c->d_zr = c->dnew<ZRect>((long long)c->h_zr.size(), false);
            BSGD_CUDA(cudaMemcpy(c->d_zr, c->h_zr.data(), sizeof(ZRect) * c->h_zr.size(), cudaMemcpyHostToDevice));
        }
        c->r = c->dnew<float>(c->n_rays);
        c->accN = c->dnew_pad(c->s, false);
        c->accT = c->dnew_pad(c->s, true);
        if (const char* e = getenv("BSGD_FORCE_NCCL")) c->coll = atoi(e) != 0;   // test hook
        if (c->world > 1) c->coll = true;
        const char* exch = getenv("BSGD_EXCHANGE");
        c->lsa = c->coll && exch && std::string(exch) == "lsa";
        // LSA over NCCL: pc comes from ncclMemAlloc once the communicator exists (below)
        c->pc = c->coll && !(c->lsa && !c->vg) ? c->dnew<float>(c->n_rays) : nullptr;
        if (c->world > 1) {
            const char* e = exch;
            c->band = !(e && std::string(e) == "full");
            if (c->band) {
                c->compute_bands();
                c->d_npart = c->dnew<double>(c->M);
            }
        }
        c->d_normsq = c->dnew<double>(c->M);
        c->d_rpart = c->dnew<double>((long long)c->n_views * RES_GX);
        c->d_red = c->dnew<double>(16);
        c->d_visits = c->dnew<unsigned long long>(1);
        c->tab_bytes = 2 * (size_t)(64 + 16 * ((size_t)c->n_views * (2 + 4LL * c->s + 1 + 4LL * c->world) +
                                              64LL * c->s + c->M + c->world) + 4096);
        c->d_tab = (char*)c->dalloc(c->tab_bytes);
        c->h_normsq.assign(c->M, 0.0);
        if (c->vg) {
            std::lock_guard<std::mutex> lk(c->vg->m);
            BSGD_CUDA(cudaEventCreateWithFlags(&c->vg->ev1[c->rank], cudaEventDisableTiming));
            BSGD_CUDA(cudaEventCreateWithFlags(&c->vg->ev2[c->rank], cudaEventDisableTiming));
        } else if (c->world > 1) {
            ncclUniqueId id;
            memcpy(&id, dist->nccl_id, sizeof id);
            BSGD_NCCL(ncclCommInitRank(&c->comm, c->world, id, c->rank));
        } else if (c->coll) {   // one-rank communicator: exercises the collective path on 1 GPU
            ncclUniqueId id;
            BSGD_NCCL(ncclGetUniqueId(&id));
            BSGD_NCCL(ncclCommInitRank(&c->comm, 1, id, 0));
        }
        if (c->lsa && !c->vg) {   // pc as an NCCL symmetric window, every rank's copy addressable
            const size_t bytes = sizeof(float) * (size_t)c->n_rays;
            BSGD_NCCL(ncclMemAlloc((void**)&c->pc, bytes));
            c->pc_ncclmem = true;
            BSGD_CUDA(cudaMemset(c->pc, 0, bytes));
            ncclWindow_t w = nullptr;
            BSGD_NCCL(ncclCommWindowRegister(c->comm, c->pc, bytes, &w, NCCL_WIN_COLL_SYMMETRIC));
            c->pc_win = w;
            void** dptr = (void**)c->dalloc(sizeof(void*) * (size_t)c->world);
            launch_lsa_ptrs(w, c->world, dptr, 0);
            std::vector<void*> hp((size_t)c->world);
            BSGD_CUDA(cudaMemcpy(hp.data(), dptr, sizeof(void*) * hp.size(), cudaMemcpyDeviceToHost));
            for (void* q : hp) c->lsa_pc.push_back((const float*)q);
            // the window's own-rank address is a second mapping of pc: a value written through
            // it must read back through pc
            const float probe = 1234.5f;
            float back = 0.f;
            BSGD_CUDA(cudaMemcpy((void*)c->lsa_pc[c->rank], &probe, sizeof probe, cudaMemcpyHostToDevice));
            BSGD_CUDA(cudaMemcpy(&back, c->pc, sizeof back, cudaMemcpyDeviceToHost));
            if (back != probe) fail(BSGD_E_NCCL, "LSA exchange: the window's own-rank address does not alias pc");
            BSGD_CUDA(cudaMemset(c->pc, 0, sizeof(float)));
            c->d_bar = c->dnew<float>(1);
        }
        BSGD_CUDA(cudaDeviceSynchronize());
    });
    if (st != BSGD_OK) {
        c->release_comm();
        c->release();
        return st;
    }
    *out = c.release();
    return BSGD_OK;
}

bsgd_status bsgd_vgroup_create(int32_t world, bsgd_vgroup* out) {
    return guard(nullptr, [&] {
        if (!out || world < 1 || world > 8) fail(BSGD_E_CONTRACT, "virtual group: 1 <= world <= 8");
        auto* g = new bsgd_vgroup_s();
        g->world = world;
        g->src.assign(world, nullptr);
        g->ev1.assign(world, nullptr);
        g->ev2.assign(world, nullptr);
        *out = g;
    });
}

void bsgd_vgroup_destroy(bsgd_vgroup g) {
    if (!g) return;
    cudaDeviceSynchronize();
    for (auto e : g->ev1) if (e) cudaEventDestroy(e);
    for (auto e : g->ev2) if (e) cudaEventDestroy(e);
    delete g;
}

void bsgd_destroy(bsgd_ctx ctx) {
    if (!ctx) return;
    cudaDeviceSynchronize();
    ctx->release_comm();
    ctx->release();
    delete ctx;
}

bsgd_status bsgd_get_info(bsgd_ctx c, bsgd_info* o) {
    return guard(c, [&] {
        if (!c || !o) fail(BSGD_E_CONTRACT, "NULL");
        o->N = c->N; o->M = c->M; o->n_views = c->n_views; o->det_u = c->nu; o->det_v = c->nv;
        o->owned_first = c->first; o->owned_count = c->s; o->tiles = c->T;
        o->block_voxels = c->bsize; o->n_rays = c->n_rays; o->owned_voxels = c->bsize * c->s;
        for (int k = 0; k < 3; ++k) o->block_dims[k] = c->bd[k];
        o->device_bytes = c->bytes;
    });
}

bsgd_status bsgd_row_block_views(bsgd_ctx c, int32_t i, int32_t* out, int32_t* n) {
    return guard(c, [&] {
        if (!c || !n) fail(BSGD_E_CONTRACT, "NULL");
        if (i < 0 || i >= c->M) fail(BSGD_E_DIMENSION, "row block out of range");
        *n = (int32_t)c->rows[i].size();
        if (out) memcpy(out, c->rows[i].data(), sizeof(int32_t) * c->rows[i].size());
    });
}

bsgd_status bsgd_forward(bsgd_ctx c, int32_t n, const int32_t* views, const int32_t* rects, int32_t col_block,
                         const float* x_block, float* proj, int32_t accumulate, void* stream) {
    return guard(c, [&] {
        if (!c || !x_block || !proj) fail(BSGD_E_CONTRACT, "NULL");
        check_views(c, n, views, rects);
        if (!c->owned(col_block)) fail(BSGD_E_DIMENSION, "column block not owned by this rank");
        Ordered order_(c, S(stream));
        if (n == 0) return;
        if (!c->fp_scratchT) {
            c->fp_scratchT = c->pT(c->dnew_pad(1, true), 0);
            c->fp_scratchN = c->pN(c->dnew_pad(1, false), 0);
        }
        const int b = col_block - c->first;
        cudaStream_t st = S(stream);
        if (c->zsplit && c->nz_of(col_block) < c->bd[2]) {
            // the scratch copies are shared by all blocks: the planes past a thinner slab
            // (its zero border first) must not hold a thicker slab's values
            const int nzj = c->nz_of(col_block);
            BSGD_CUDA(cudaMemsetAsync(c->fp_scratchN - PAD_X + (long long)nzj * c->planeN, 0,
                                      sizeof(float) * (size_t)(c->bd[2] - nzj) * c->planeN, st));
            BSGD_CUDA(cudaMemsetAsync(c->fp_scratchT - PAD_X + (long long)nzj * c->planeT, 0,
                                      sizeof(float) * (size_t)(c->bd[2] - nzj) * c->planeT, st));
        }
        c->update(UPD_XT, b, const_cast<float*>(x_block), 0.f, 1, nullptr, 0, st, nullptr, nullptr,
                  c->fp_scratchT, 0, c->fp_scratchN);
        std::vector<int> vv(views, views + n);
        std::vector<int4> rc;
        if (rects)
            for (int k = 0; k < n; ++k) rc.push_back(make_int4(rects[4 * k], rects[4 * k + 1], rects[4 * k + 2], rects[4 * k + 3]));
        else
            rc.assign(n, make_int4(0, c->nu, 0, c->nv));
        if (!accumulate) {   // overwrite semantics: rays of the rects outside the footprint become 0
            std::vector<char> staging;
            size_t off = c->tab_bytes / 2;
            staging.resize(off);
            const int* dv = c->tab_put(off, vv, staging);
            const int4* dr = c->tab_put(off, rc, staging);
            BSGD_CUDA(cudaMemcpyAsync(c->d_tab + c->tab_bytes / 2, staging.data() + c->tab_bytes / 2,
                                      off - c->tab_bytes / 2, cudaMemcpyHostToDevice, st));
            launch_zero_rects(proj, dv, dr, n, c->nu, c->nv, st);
        }
        c->project(PROJ_FP, vv, {b}, rc, {c->fp_scratchN}, {c->fp_scratchT}, {}, {}, {proj}, nullptr, 0.f,
                   accumulate, st, 0);
    });
}

bsgd_status bsgd_back(bsgd_ctx c, int32_t n, const int32_t* views, const int32_t* rects, int32_t col_block,
                      const float* proj, float* g_block, float scale, int32_t accumulate, void* stream) {
    return guard(c, [&] {
        if (!c || !proj || !g_block) fail(BSGD_E_CONTRACT, "NULL");
        check_views(c, n, views, rects);
        if (!c->owned(col_block)) fail(BSGD_E_DIMENSION, "column block not owned by this rank");
        if (!isfinite(scale)) fail(BSGD_E_CONTRACT, "scale not finite");
        Ordered order_(c, S(stream));
        const int b = col_block - c->first;
        cudaStream_t st = S(stream);
        std::vector<int> vv(views, views + n);
        std::vector<int4> rc;
        if (rects)
            for (int k = 0; k < n; ++k) rc.push_back(make_int4(rects[4 * k], rects[4 * k + 1], rects[4 * k + 2], rects[4 * k + 3]));
        float* aN = c->pN(c->accN, b);
        float* aT = c->pT(c->accT, b);
        if (n > 0) c->project(PROJ_BP, vv, {b}, rc, {}, {}, {aN}, {aT}, {}, proj, scale, 0, st, 0);
        c->update(UPD_OUT, b, nullptr, 0.f, 0, g_block, accumulate, st);
    });
}

bsgd_status bsgd_im_weights(bsgd_ctx c, double* w_out, uint32_t* q_out) {
    return bsgd_im_table(c, 0, w_out, q_out);
}

bsgd_status bsgd_im_table(bsgd_ctx c, int32_t kind, double* w_out, uint32_t* q_out) {
    return guard(c, [&] {
        if (!c || kind < 0 || kind > 1) fail(BSGD_E_CONTRACT, "bad arguments");
        Ordered order_(c, nullptr);
        c->ensure_im_table(nullptr, kind);
        if (w_out) memcpy(w_out, c->w.data(), sizeof(double) * c->w.size());
        if (q_out) memcpy(q_out, c->q.data(), sizeof(uint32_t) * c->q.size());
    });
}

bsgd_status bsgd_visit_table(bsgd_ctx c, uint64_t* nnz_out) {
    return guard(c, [&] {
        if (!c || !nnz_out) fail(BSGD_E_CONTRACT, "NULL");
        Ordered order_(c, nullptr);
        c->ensure_visit_table(nullptr);
        for (size_t k = 0; k < c->vtab.size(); ++k) nnz_out[k] = c->vtab[k];
    });
}

bsgd_status bsgd_reset(bsgd_ctx c, const float* y, void* stream) {
    return guard(c, [&] {
        if (!c || !y) fail(BSGD_E_CONTRACT, "NULL");
        Ordered order_(c, S(stream));
        c->reset(y, S(stream));
    });
}

bsgd_status bsgd_step(bsgd_ctx c, const float* y, float* x_owned, const bsgd_selection* sel, float mu,
                      uint32_t flags, void* stream) {
    return guard(c, [&] {
        if (!c || !y || !x_owned || !sel) fail(BSGD_E_CONTRACT, "NULL");
        if (!isfinite(mu)) fail(BSGD_E_CONTRACT, "mu not finite");
        if (flags & ~(uint32_t)(BSGD_SGD | BSGD_DETERMINISTIC))
            fail(BSGD_E_CONTRACT, "bsgd_step accepts BSGD_SGD and BSGD_DETERMINISTIC only");
        const bool sgd = flags & BSGD_SGD;
        c->det = (flags & BSGD_DETERMINISTIC) != 0;
        if (sel->n_rows < 1 || !sel->rows) fail(BSGD_E_CONTRACT, "empty row selection");
        check_sorted_unique(sel->rows, sel->n_rows, c->M, "row block");
        if (!sgd) {
            if (sel->n_cols < 1 || !sel->cols) fail(BSGD_E_CONTRACT, "empty column selection");
            check_sorted_unique(sel->cols, sel->n_cols, c->N, "column block");
        }
        std::vector<int> rows(sel->rows, sel->rows + sel->n_rows);
        std::vector<int> cols;
        if (!sgd) cols.assign(sel->cols, sel->cols + sel->n_cols);
        std::vector<int> tiles;
        if (sel->im_tiles && !sgd) {
            int V = 0;
            for (int i : rows) V += (int)c->rows[i].size();
            tiles.assign(sel->im_tiles, sel->im_tiles + (size_t)V * cols.size());
            for (int t : tiles)
                if (t < 0 || t >= c->T) fail(BSGD_E_CONTRACT, "tile id out of range");
        }
        Ordered order_(c, S(stream));
        c->epoch_step(y, x_owned, rows, cols, tiles, mu, sgd, S(stream), nullptr);
        c->epoch += 1;
    });
}

bsgd_status bsgd_solve(bsgd_ctx c, const float* y, float* x_owned, const bsgd_solve_params* P, double* obj,
                       double* mu, void* stream) {
    return guard(c, [&] {
        if (!c || !y || !x_owned || !P) fail(BSGD_E_CONTRACT, "NULL");
        if (!is_device_ptr(y) || !is_device_ptr(x_owned)) fail(BSGD_E_CONTRACT, "bsgd_solve takes device buffers");
        if (P->solver < BSGD_SOLVER_GD || P->solver > BSGD_SOLVER_SVRG) fail(BSGD_E_CONTRACT, "unknown solver");
        if (P->iters < 0 || !isfinite(P->mu0) || P->mu0 <= 0.0) fail(BSGD_E_CONTRACT, "iters < 0 or bad mu0");
        if (!isfinite(P->lambda) || P->lambda < 0.0 || P->tv_iters < 0 || P->svrg_m < 0)
            fail(BSGD_E_CONTRACT, "bad lambda / tv_iters / svrg_m");
        const bool tv = (P->solver == BSGD_SOLVER_ISTA || P->solver == BSGD_SOLVER_FISTA) && P->lambda > 0.0;
        if (tv && !c->tv_shardable())
            fail(BSGD_E_PARTITION, "sharded TV needs whole z-layers of blocks per rank (N/G divisible by bx*by)");
        Ordered order_(c, S(stream));
        c->solve(P->solver, y, x_owned, P->iters, P->mu0, tv ? P->lambda : 0.0, P->tv_iters, P->svrg_m, P->seed,
                 obj, mu, S(stream));
        BSGD_CUDA(cudaStreamSynchronize(S(stream)));
    });
}

bsgd_status bsgd_run(bsgd_ctx c, const float* y_in, float* x_in, const float* xt_in, const bsgd_run_params* P,
                     bsgd_run_log* log, void* stream) {
    return guard(c, [&] {
        if (!c || !y_in || !x_in || !P) fail(BSGD_E_CONTRACT, "NULL");
        if (P->epochs < 0) fail(BSGD_E_CONTRACT, "epochs < 0");
        if (P->total_epochs < 0 || P->is_off_last_epochs < 0)
            fail(BSGD_E_CONTRACT, "total_epochs and is_off_last_epochs must be >= 0");
        if (!isfinite(P->mu0)) fail(BSGD_E_CONTRACT, "mu0 not finite");
        const uint32_t known = BSGD_IS | BSGD_IS_UNIFORM | BSGD_TV | BSGD_AUTO_MU | BSGD_SGD | BSGD_RESUME | BSGD_TIMING |
                               BSGD_STRATIFIED | BSGD_IS_AREA | BSGD_TV_CHAMBOLLE | BSGD_DETERMINISTIC |
                               BSGD_LOG_TRUE_OBJ;
        if (P->flags & ~known) fail(BSGD_E_CONTRACT, "unknown flags");
        const bool sgd = P->flags & BSGD_SGD, im = (P->flags & (BSGD_IS | BSGD_IS_UNIFORM)) && !sgd;
        const bool uni = P->flags & BSGD_IS_UNIFORM, tv = P->flags & BSGD_TV, amu = P->flags & BSGD_AUTO_MU;
        int aM = P->rows_per_epoch, gN = P->cols_per_epoch;
        if (aM == 0 || gN == 0) {
            int a2, g2;
            host::eq8(c->world, c->M, c->N, &a2, &g2);
            if (!aM) aM = a2;
            if (!gN) gN = g2;
        }
        if (aM < 1 || aM > c->M || gN < 1 || gN > c->N) fail(BSGD_E_CONTRACT, "rows/cols per epoch out of range");
        const bool strat = (P->flags & BSGD_STRATIFIED) && !sgd;
        c->det = (P->flags & BSGD_DETERMINISTIC) != 0;
        const int strata = P->strata > 0 ? P->strata : c->world;
        if (strat && (P->strata < 0 || c->N % strata || gN % strata))
            fail(BSGD_E_CONTRACT, "BSGD_STRATIFIED: strata must divide N and cols_per_epoch");
        if (tv && !c->tv_shardable())
            fail(BSGD_E_PARTITION, "sharded TV needs whole z-layers of blocks per rank (N/G divisible by bx*by)");
        if (tv && (P->tv_iters < 0 || !isfinite(P->lambda) || P->lambda < 0.0))
            fail(BSGD_E_CONTRACT, "bad TV parameters (lambda must be finite and >= 0, tv_iters >= 0)");
        if (!(P->mu0 > 0.0)) fail(BSGD_E_CONTRACT, "mu0 must be > 0");
        Ordered order_(c, S(stream));
        cudaStream_t st = S(stream);
        const long long sb = (long long)c->s * c->bsize;
        // host or device buffers.  Host y / x are uploaded on a copy stream that overlaps the
        // first epoch: x block by block ahead of that block's FP, then y ahead of the first
        // residual (epoch_step's Upload hooks); the D2H of x at the end stays in order.
        const float* y = y_in;
        float* x = x_in;
        const float* xt = xt_in;
        const bool y_host = !is_device_ptr(y_in), x_host = !is_device_ptr(x_in);
        bsgd_ctx_s::Upload up;
        if (y_host || x_host) {
            c->ensure_copy_stream();
            BSGD_CUDA(cudaEventRecord(c->up_ev[c->s + 1], st));            // after prior work
            BSGD_CUDA(cudaStreamWaitEvent(c->copy_st, c->up_ev[c->s + 1], 0));
        }
        if (x_host) {
            if (!c->x_dev) c->x_dev = c->dnew<float>(sb, false);
            for (int b = 0; b < c->s; ++b) {
                BSGD_CUDA(cudaMemcpyAsync(c->x_dev + (size_t)b * c->bsize, x_in + (size_t)b * c->bsize,
                                          sizeof(float) * c->bsize, cudaMemcpyHostToDevice, c->copy_st));
                BSGD_CUDA(cudaEventRecord(c->up_ev[b], c->copy_st));
            }
            x = c->x_dev;
            c->x_events.assign(c->up_ev.begin(), c->up_ev.begin() + c->s);
            up.xev = &c->x_events;
        }
        // y in the order of use: the views of the first epoch's selected row blocks (the first
        // residual waits only for them), then the rest (waited for after the first epoch)
        std::vector<int> rows_first(aM), rows_rest;
        if (y_host) {
            if (!c->y_dev) c->y_dev = c->dnew<float>(c->n_rays, false);
            const int eg0 = (P->flags & BSGD_RESUME) ? c->epoch : 0;
            host::select(P->seed, 1, eg0, c->M, aM, rows_first.data());
            std::vector<char> first((size_t)c->n_views, 0);
            for (int i : rows_first)
                for (int v : c->rows[i]) first[(size_t)v] = 1;
            for (int i = 0; i < c->M; ++i)
                if (std::find(rows_first.begin(), rows_first.end(), i) == rows_first.end()) rows_rest.push_back(i);
            const size_t per = (size_t)c->per;
            for (int pass = 1; pass >= 0; --pass) {   // runs of consecutive views of each group
                for (int v = 0; v < c->n_views;) {
                    if (first[(size_t)v] != pass) { ++v; continue; }
                    int w = v;
                    while (w < c->n_views && first[(size_t)w] == pass) ++w;
                    BSGD_CUDA(cudaMemcpyAsync(c->y_dev + (size_t)v * per, y_in + (size_t)v * per,
                                              sizeof(float) * per * (size_t)(w - v), cudaMemcpyHostToDevice,
                                              c->copy_st));
                    v = w;
                }
                BSGD_CUDA(cudaEventRecord(c->up_ev[pass ? c->s : c->s + 2], c->copy_st));
            }
            y = c->y_dev;
            up.yev = c->up_ev[c->s];
        }
        if (xt_in && !is_device_ptr(xt_in)) {
            if (!c->xt_dev) c->xt_dev = c->dnew<float>(sb, false);
            BSGD_CUDA(cudaMemcpyAsync(c->xt_dev, xt_in, sizeof(float) * sb, cudaMemcpyHostToDevice, st));
            xt = c->xt_dev;
        }
        if (amu && !c->eud_cur) {
            c->eud_cur = c->dnew<float>(sb);
            c->eud_prev = c->dnew<float>(sb);
        }
        bool defer_r0 = false;
        if (!(P->flags & BSGD_RESUME)) {
            if (y_host && P->epochs > 0) {   // r = y after the y upload, inside epoch 0
                c->reset_state(st);
                up.y_reset = true;
                defer_r0 = true;
            } else {
                if (y_host) {
                    BSGD_CUDA(cudaStreamWaitEvent(st, up.yev, 0));
                    BSGD_CUDA(cudaStreamWaitEvent(st, c->up_ev[c->s + 2], 0));
                }
                c->reset(y, st);
            }
            c->mu = P->mu0;
            c->rnorm_hist.clear();
        } else if (c->epoch == 0) {
            c->mu = P->mu0;
        }
        auto push_r0 = [&](const double* d_src) {   // ||r||^0 = ||y|| (reading A13/A14)
            BSGD_CUDA(cudaMemcpyAsync(c->h_normsq.data(), d_src, sizeof(double) * c->M, cudaMemcpyDeviceToHost, st));
            BSGD_CUDA(cudaStreamSynchronize(st));
            double s2 = 0;
            for (double v : c->h_normsq) s2 += v;
            c->rnorm_hist.push_back(sqrt(s2));
        };
        if (c->rnorm_hist.empty() && !defer_r0) {
            if (y_host && up.yev) {
                BSGD_CUDA(cudaStreamWaitEvent(st, up.yev, 0));
                BSGD_CUDA(cudaStreamWaitEvent(st, c->up_ev[c->s + 2], 0));
            }
            push_r0(c->d_normsq);
        }
        if (im && !uni) c->ensure_im_table(st, (P->flags & BSGD_IS_AREA) ? 1 : 0);
        std::vector<int> all_slots(c->s);
        for (int b = 0; b < c->s; ++b) all_slots[b] = b;
        if (x_host && P->epochs == 0) {   // no epoch to hide the upload behind
            for (int b = 0; b < c->s; ++b) BSGD_CUDA(cudaStreamWaitEvent(st, c->up_ev[b], 0));
        }
        if (!x_host || P->epochs == 0) c->refresh_xT(x, all_slots, st);
        const int E = P->epochs;
        if (c->d_log_cap < 2LL * E + 2) {
            c->d_log = c->dnew<double>(2LL * E + 2);
            c->d_log_cap = 2LL * E + 2;
        }
        const bool want_visits = log && log->visits;
        if (want_visits) c->ensure_visit_table(st);
        std::vector<unsigned long long> vis_log(E, 0ull);
        BSGD_CUDA(cudaMemsetAsync(c->d_log, 0, sizeof(double) * (2 * E + 2), st));
        std::vector<cudaEvent_t> ev;
        const bool timing = (P->flags & BSGD_TIMING) && log && log->t_ms;
        const bool true_obj = (P->flags & BSGD_LOG_TRUE_OBJ) && log && log->obj_true;
        std::vector<int> all_views;
        if (true_obj) {
            for (int v = 0; v < c->n_views; ++v) all_views.push_back(v);
            if (!c->gap_proj) c->gap_proj = c->dnew<float>(c->n_rays, false);
            if (c->d_gap_n < E) {
                c->d_gap = c->dnew<double>(E);
                c->d_tvv = c->dnew<double>(E);
                c->d_seenlog = c->dnew<double>(2LL * E);
                c->d_gap_n = E;
            }
            if (log->rmse_seen && xt_in) c->ensure_seen(st);
        }
        if (timing) {
            ev.resize((size_t)E * 7);
            for (auto& e : ev) BSGD_CUDA(cudaEventCreate(&e));
        }
        const int period = tv ? (P->tv_period > 0 ? P->tv_period
                                                  : std::max(1, (int)floor((double)c->M * c->N / ((double)aM * gN) + 0.5)))
                              : 0;
        std::vector<double> mu_log(E);
        const long long total = P->total_epochs > 0 ? (long long)P->total_epochs : (long long)c->epoch + E;
        bool downloaded = false;
        std::vector<int> rows(aM), cols(gN);
        for (int e = 0; e < E; ++e) {
            const int eg = c->epoch;          // global 0-based epoch (RNG counter)
            const int k = eg + 1;             // 1-based epoch of Algos 3 and 4
            host::select(P->seed, 1, eg, c->M, aM, rows.data());
            if (strat) host::select_stratified(P->seed, eg, c->N, gN, strata, cols.data());
            else if (!sgd) host::select(P->seed, 2, eg, c->N, gN, cols.data());
            if (log && log->sel_rows) memcpy(log->sel_rows + (size_t)e * aM, rows.data(), sizeof(int) * aM);
            if (log && log->sel_cols && !sgd) memcpy(log->sel_cols + (size_t)e * gN, cols.data(), sizeof(int) * gN);
            std::vector<int> tiles;
            // "the last few iterations without importance sampling", counted in
            // global epochs k against the planned total (the oracle's rule, oracle/bsgd.py)
            const bool use_im = im && !(P->is_off_last_epochs > 0 && k > total - P->is_off_last_epochs);
            if (use_im) {   // Algo 2 line 5: one tile per (selected block, view) by weight
                int V = 0;
                for (int i : rows) V += (int)c->rows[i].size();
                tiles.assign((size_t)V * gN, 0);
                for (int cs = 0; cs < gN; ++cs) {
                    if (!c->owned(cols[cs])) continue;
                    int vs = 0;
                    for (int i : rows)
                        for (int v : c->rows[i]) {
                            const uint32_t* qrow = uni ? nullptr : &c->q[((size_t)(cols[cs] - c->first) * c->n_views + v) * c->T];
                            tiles[(size_t)cs * V + vs] = host::im_draw(P->seed, eg, (uint32_t)(cs * V + vs), qrow, c->T, uni);
                            ++vs;
                        }
                }
            }
            cudaEvent_t* evp = timing ? &ev[(size_t)e * 7] : nullptr;
            // last epoch of a host-x run: overlap the x download with the final BP launches
            // (not when a TV prox follows: it changes x after the updates)
            bsgd_ctx_s::Upload down;
            const bool overlap_down = x_host && !sgd && e + 1 == E && !(tv && k % period == 0);
            bsgd_ctx_s::Upload* hook = e == 0 ? &up : nullptr;
            if (overlap_down) {
                if (hook) down = up;
                down.x_host_out = x_in;
                hook = &down;
                downloaded = true;
            }
            c->epoch_step(y, x, rows, sgd ? std::vector<int>() : cols, tiles, (float)c->mu, sgd, st, evp, false,
                          hook);
            if (e == 0 && y_host) {   // the rest of y: r = y and ||y_I||^2 on the row blocks not selected
                BSGD_CUDA(cudaStreamWaitEvent(st, c->up_ev[c->s + 2], 0));
                if (defer_r0 && !rows_rest.empty()) {
                    c->reset_r(y, st, &rows_rest);
                    if (!c->d_rows_tmp) c->d_rows_tmp = c->dnew<int>(c->M, false);
                    BSGD_CUDA(cudaMemcpyAsync(c->d_rows_tmp, rows_rest.data(), sizeof(int) * rows_rest.size(),
                                              cudaMemcpyHostToDevice, st));
                    launch_copy_rows(c->d_normsq0, c->d_normsq, c->d_rows_tmp, (int)rows_rest.size(), st);
                }
            }
            if (e == 0 && defer_r0) push_r0(c->d_normsq0);
            if (want_visits) {   // FP visits of this epoch on this rank (BP visits are the same segments)
                unsigned long long nvt = 0;
                int V = 0;
                for (int i : rows) V += (int)c->rows[i].size();
                const int ncol = sgd ? c->N : gN;
                for (int cs = 0; cs < ncol; ++cs) {
                    const int j = sgd ? cs : cols[cs];
                    if (!c->owned(j)) continue;
                    int vs = 0;
                    for (int i : rows)
                        for (int v : c->rows[i]) {
                            const unsigned long long* q = &c->vtab[((size_t)(j - c->first) * c->n_views + v) * c->T];
                            if (!tiles.empty()) nvt += q[tiles[(size_t)cs * V + vs]];
                            else for (int t = 0; t < c->T; ++t) nvt += q[t];
                            ++vs;
                        }
                }
                vis_log[e] = nvt;
            }
            mu_log[e] = c->mu;
            launch_obj(c->d_normsq, c->M, c->d_log + 2 * e, st);
            if (amu) launch_axpy_eud(c->eud_cur, c->g, sb, st);            // Algo 3 line 2
            if (tv && k % period == 0) {                                      // Algo 4 lines 15-17
                c->tv_prox(x, c->mu * P->lambda, P->tv_iters, st, (P->flags & BSGD_TV_CHAMBOLLE) ? 1 : 0);
                c->refresh_xT(x, all_slots, st);
            }
            if (evp) BSGD_CUDA(cudaEventRecord(evp[5], st));
            if (true_obj) {   // GAP^2 / 2 = 1/2 |y - A x|^2: FP of every view through every owned block
                BSGD_CUDA(cudaMemsetAsync(c->gap_proj, 0, sizeof(float) * c->n_rays, st));
                for (int b = 0; b < c->s; ++b)
                    c->project(PROJ_FP, all_views, {b}, {}, {c->pN(c->xN, b)}, {c->pT(c->xT, b)}, {}, {},
                               {c->gap_proj}, nullptr, 0.f, 1, st, 0);
                c->allreduce_f(c->gap_proj, (size_t)c->n_rays, st);
                BSGD_CUDA(cudaMemsetAsync(c->d_gap + e, 0, sizeof(double), st));
                launch_sqdiff(y, c->gap_proj, c->n_rays, c->d_gap + e, st);
                if (log->tv) c->tv_value(x, c->d_tvv + e, st);
                if (log->rmse_seen && xt) {
                    BSGD_CUDA(cudaMemsetAsync(c->d_seenlog + 2 * e, 0, 2 * sizeof(double), st));
                    launch_sqdiff_masked(x, xt, c->seen, sb, c->d_seenlog + 2 * e, st);
                    c->allreduce_d(c->d_seenlog + 2 * e, 2, st);
                }
            }
            if (xt) {
                BSGD_CUDA(cudaMemsetAsync(c->d_red + 8, 0, sizeof(double), st));
                launch_sqdiff(x, xt, sb, c->d_red + 8, st);
                c->allreduce_d(c->d_red + 8, 1, st);
                BSGD_CUDA(cudaMemcpyAsync(c->d_log + 2 * e + 1, c->d_red + 8, sizeof(double), cudaMemcpyDeviceToDevice, st));
            }
            if (amu && k % c->M == 0) {                                       // Algo 3 lines 2-12
                double d3[3] = {0, 0, 0};
                bool have_theta = false;
                double theta = 0.0;
                if (c->have_prev_eud) {
                    BSGD_CUDA(cudaMemsetAsync(c->d_red, 0, 3 * sizeof(double), st));
                    launch_dot3(c->eud_cur, c->eud_prev, sb, c->d_red, st);
                    c->allreduce_d(c->d_red, 3, st);
                    BSGD_CUDA(cudaMemcpyAsync(d3, c->d_red, 3 * sizeof(double), cudaMemcpyDeviceToHost, st));
                }
                BSGD_CUDA(cudaMemcpyAsync(c->h_normsq.data(), c->d_normsq, sizeof(double) * c->M, cudaMemcpyDeviceToHost, st));
                BSGD_CUDA(cudaStreamSynchronize(st));
                if (c->have_prev_eud && d3[1] > 0 && d3[2] > 0) {
                    theta = d3[0] / (sqrt(d3[1]) * sqrt(d3[2]));
                    have_theta = true;
                }
                double s2 = 0;
                for (double v : c->h_normsq) s2 += v;
                c->rnorm_hist.push_back(sqrt(s2));
                const size_t h = c->rnorm_hist.size();
                if (k > c->M && h >= 3) {
                    const double rk = c->rnorm_hist[h - 1], rkM = c->rnorm_hist[h - 2], rk2M = c->rnorm_hist[h - 3];
                    if (rk < rkM && rkM < rk2M) c->mu = (1.0 + P->eps) * c->mu;
                    if (rk > rkM && rkM > rk2M) {
                        bool c2 = false;
                        if (have_theta) {
                            if (c->have_theta_prev && fabs(theta - c->theta_prev) > P->t1) c2 = true;
                            if (theta < P->t2) c2 = true;
                        }
                        if (c2) c->mu = (1.0 - P->delta) * c->mu;
                    }
                }
                c->have_theta_prev = have_theta;
                c->theta_prev = theta;
                std::swap(c->eud_cur, c->eud_prev);
                c->have_prev_eud = true;
                BSGD_CUDA(cudaMemsetAsync(c->eud_cur, 0, sizeof(float) * sb, st));
            }
            if (evp) BSGD_CUDA(cudaEventRecord(evp[6], st));
            c->epoch += 1;
        }
        if (downloaded) {   // the per-block downloads on the copy stream
            BSGD_CUDA(cudaEventRecord(c->up_ev[c->s + 1], c->copy_st));
            BSGD_CUDA(cudaStreamWaitEvent(st, c->up_ev[c->s + 1], 0));
        } else if (x_host) {
            BSGD_CUDA(cudaMemcpyAsync(x_in, x, sizeof(float) * sb, cudaMemcpyDeviceToHost, st));
        }
        std::vector<double> hl(2 * (size_t)E + 2), hgap(true_obj ? E : 0);
        BSGD_CUDA(cudaMemcpyAsync(hl.data(), c->d_log, sizeof(double) * hl.size(), cudaMemcpyDeviceToHost, st));
        std::vector<double> htv(true_obj && log->tv ? E : 0);
        std::vector<double> hseen(true_obj && log->rmse_seen && xt ? 2 * E : 0);
        if (!hseen.empty())
            BSGD_CUDA(cudaMemcpyAsync(hseen.data(), c->d_seenlog, sizeof(double) * 2 * E, cudaMemcpyDeviceToHost, st));
        if (true_obj) BSGD_CUDA(cudaMemcpyAsync(hgap.data(), c->d_gap, sizeof(double) * E, cudaMemcpyDeviceToHost, st));
        if (!htv.empty()) BSGD_CUDA(cudaMemcpyAsync(htv.data(), c->d_tvv, sizeof(double) * E, cudaMemcpyDeviceToHost, st));
        BSGD_CUDA(cudaStreamSynchronize(st));
        if (log) {
            const double nvox = (double)c->dims[0] * c->dims[1] * c->dims[2];   // the volume's voxels
            for (int e = 0; e < E; ++e) {
                if (log->obj) log->obj[e] = hl[2 * e];
                if (log->rmse) log->rmse[e] = xt ? sqrt(hl[2 * e + 1] / nvox) : NAN;
                if (true_obj) log->obj_true[e] = 0.5 * hgap[e];
                if (!htv.empty()) log->tv[e] = htv[e];
                if (!hseen.empty()) log->rmse_seen[e] = hseen[2 * e + 1] > 0 ? sqrt(hseen[2 * e] / hseen[2 * e + 1]) : NAN;
                if (log->mu) log->mu[e] = mu_log[e];
                if (log->visits) log->visits[e] = vis_log[e];
                if (timing) {
                    cudaEvent_t* q = &ev[(size_t)e * 7];
                    float t[6];
                    for (int p = 0; p < 4; ++p) BSGD_CUDA(cudaEventElapsedTime(&t[p], q[p], q[p + 1]));
                    BSGD_CUDA(cudaEventElapsedTime(&t[4], q[4], q[6]));
                    BSGD_CUDA(cudaEventElapsedTime(&t[5], q[0], q[6]));
                    for (int p = 0; p < 6; ++p) log->t_ms[(size_t)e * 6 + p] = t[p];
                }
            }
        }
        for (auto& e : ev) cudaEventDestroy(e);
    });
}

bsgd_status bsgd_get_state(bsgd_ctx c, int32_t what, int32_t index, void* dst, size_t bytes) {
    return guard(c, [&] {
        if (!c || !dst) fail(BSGD_E_CONTRACT, "NULL");
        const void* src = nullptr;
        size_t need = 0;
        if (what == 0) {   // z^j of owned slot `index`, expanded from the footprint storage
            if (index < 0 || index >= c->s) fail(BSGD_E_DIMENSION, "slot");
            if (bytes != 4 * (size_t)c->n_rays) fail(BSGD_E_DIMENSION, "size mismatch");
            BSGD_CUDA(cudaDeviceSynchronize());
            float* out = (float*)dst;
            memset(out, 0, bytes);
            for (int v = 0; v < c->n_views; ++v) {
                const ZRect& q = c->h_zr[(size_t)index * c->n_views + v];
                const int w = q.u1 - q.u0;
                if (w <= 0 || q.v1 <= q.v0) continue;
                BSGD_CUDA(cudaMemcpy2D(out + ((size_t)v * c->nv + q.v0) * c->nu + q.u0, sizeof(float) * c->nu,
                                       c->z + q.base, sizeof(float) * w, sizeof(float) * w, q.v1 - q.v0,
                                       cudaMemcpyDeviceToHost));
            }
            return;
        }
        switch (what) {
            case 1: if (index < 0 || index >= c->M * c->s) fail(BSGD_E_DIMENSION, "index"); src = c->ghat_of(index / c->s, index % c->s); need = 4 * c->bsize; break;
            case 2: if (index < 0 || index >= c->s) fail(BSGD_E_DIMENSION, "slot"); src = c->g + index * c->bsize; need = 4 * c->bsize; break;
            case 3: src = c->r; need = 4 * c->n_rays; break;
            case 4: src = c->d_normsq; need = 8 * c->M; break;
            case 5: need = 8; if (bytes != need) fail(BSGD_E_DIMENSION, "size"); memcpy(dst, &c->mu, 8); return;
            default: fail(BSGD_E_CONTRACT, "unknown state item");
        }
        if (bytes != need) fail(BSGD_E_DIMENSION, "size mismatch");
        BSGD_CUDA(cudaDeviceSynchronize());
        BSGD_CUDA(cudaMemcpy(dst, src, need, cudaMemcpyDeviceToHost));
    });
}

bsgd_status bsgd_set_state(bsgd_ctx c, int32_t what, int32_t index, const void* src, size_t bytes) {
    return guard(c, [&] {
        if (!c || !src) fail(BSGD_E_CONTRACT, "NULL");
        void* dst = nullptr;
        size_t need = 0;
        if (what == 0) {   // z^j of owned slot `index`: only its footprint part is stored
            if (index < 0 || index >= c->s) fail(BSGD_E_DIMENSION, "slot");
            if (bytes != 4 * (size_t)c->n_rays) fail(BSGD_E_DIMENSION, "size mismatch");
            BSGD_CUDA(cudaDeviceSynchronize());
            const float* in = (const float*)src;
            for (int v = 0; v < c->n_views; ++v) {
                const ZRect& q = c->h_zr[(size_t)index * c->n_views + v];
                const int w = q.u1 - q.u0;
                if (w <= 0 || q.v1 <= q.v0) continue;
                BSGD_CUDA(cudaMemcpy2D(c->z + q.base, sizeof(float) * w,
                                       in + ((size_t)v * c->nv + q.v0) * c->nu + q.u0, sizeof(float) * c->nu,
                                       sizeof(float) * w, q.v1 - q.v0, cudaMemcpyHostToDevice));
            }
            return;
        }
        switch (what) {
            case 1: if (index < 0 || index >= c->M * c->s) fail(BSGD_E_DIMENSION, "index"); dst = c->ghat_of(index / c->s, index % c->s); need = 4 * c->bsize; break;
            case 2: if (index < 0 || index >= c->s) fail(BSGD_E_DIMENSION, "slot"); dst = c->g + index * c->bsize; need = 4 * c->bsize; break;
            case 3: dst = c->r; need = 4 * c->n_rays; break;
            case 4: dst = c->d_normsq; need = 8 * c->M; break;
            case 5: need = 8; if (bytes != need) fail(BSGD_E_DIMENSION, "size"); memcpy(&c->mu, src, 8); return;
            default: fail(BSGD_E_CONTRACT, "unknown state item");
        }
        if (bytes != need) fail(BSGD_E_DIMENSION, "size mismatch");
        BSGD_CUDA(cudaDeviceSynchronize());
        BSGD_CUDA(cudaMemcpy(dst, src, need, cudaMemcpyHostToDevice));
    });
}

bsgd_status bsgd_tv_prox(bsgd_ctx c, float* x_owned, double w, int32_t iters, int32_t method, void* stream) {
    return guard(c, [&] {
        if (!c || !x_owned || !(w >= 0.0) || !isfinite(w) || iters < 0 || method < 0 || method > 1)
            fail(BSGD_E_CONTRACT, "bad arguments");
        if (!c->tv_shardable())
            fail(BSGD_E_PARTITION, "sharded TV needs whole z-layers of blocks per rank (N/G divisible by bx*by)");
        Ordered order_(c, S(stream));
        c->tv_prox(x_owned, w, iters, S(stream), method);
    });
}

bsgd_status bsgd_tv_value(bsgd_ctx c, const float* x_owned, double* out, void* stream) {
    return guard(c, [&] {
        if (!c || !x_owned || !out) fail(BSGD_E_CONTRACT, "bad arguments");
        Ordered order_(c, S(stream));
        cudaStream_t st = S(stream);
        if (!c->d_tvv1) c->d_tvv1 = c->dnew<double>(1);
        c->tv_value(x_owned, c->d_tvv1, st);
        BSGD_CUDA(cudaMemcpyAsync(out, c->d_tvv1, sizeof(double), cudaMemcpyDeviceToHost, st));
        BSGD_CUDA(cudaStreamSynchronize(st));
    });
}

bsgd_status bsgd_allreduce_time(bsgd_ctx c, int64_t count, int32_t iters, void* stream, double* ms_out) {
    return guard(c, [&] {
        if (!c || !ms_out || iters < 1) fail(BSGD_E_CONTRACT, "bad arguments");
        if (!c->coll || !c->pc) fail(BSGD_E_CONTRACT, "no collective path (world == 1)");
        if (count < 1 || count > c->n_rays) fail(BSGD_E_CONTRACT, "count out of range");
        cudaStream_t st = S(stream);
        Ordered order_(c, st);
        cudaEvent_t e0, e1;
        BSGD_CUDA(cudaEventCreate(&e0));
        BSGD_CUDA(cudaEventCreate(&e1));
        c->allreduce_f(c->pc, (size_t)count, st);   // untimed: first use of the buffers
        BSGD_CUDA(cudaEventRecord(e0, st));
        for (int it = 0; it < iters; ++it) c->allreduce_f(c->pc, (size_t)count, st);
        BSGD_CUDA(cudaEventRecord(e1, st));
        BSGD_CUDA(cudaEventSynchronize(e1));
        float ms = 0.f;
        BSGD_CUDA(cudaEventElapsedTime(&ms, e0, e1));
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        *ms_out = (double)ms / iters;
    });
}

bsgd_status bsgd_exchange_plan(bsgd_ctx c, int32_t world, int32_t n_sel, const int32_t* views,
                               uint64_t* band_bytes, uint64_t* full_bytes) {
    return guard(c, [&] {
        if (!c || world < 1 || n_sel < 0 || (n_sel > 0 && !views) || !band_bytes || !full_bytes)
            fail(BSGD_E_CONTRACT, "bad arguments");
        if (c->N % world) fail(BSGD_E_PARTITION, "N must be divisible by world");
        for (int k = 0; k < n_sel; ++k)
            if (views[k] < 0 || views[k] >= c->n_views) fail(BSGD_E_CONTRACT, "view out of range");
        const std::vector<int2> bd = c->rank_bands(world, c->N / world);
        unsigned long long band = 0;
        for (int g = 0; g < world; ++g)
            for (int h = 0; h < world; ++h) {
                if (h == g) continue;
                for (int k = 0; k < n_sel; ++k) {
                    const int2 o = bsgd_ctx_s::isect(bd[(size_t)g * c->n_views + views[k]], bd[(size_t)h * c->n_views + views[k]]);
                    if (o.x < o.y) band += 4ull * (unsigned long long)(o.y - o.x) * (unsigned long long)c->nu;
                }
            }
        *band_bytes = band;
        *full_bytes = world > 1 ? (uint64_t)(8.0 * (double)n_sel * c->per * (world - 1)) : 0;   // G ranks x 2(G-1)/G
    });
}

bsgd_status bsgd_rank_bands_host(const bsgd_geometry* geom, bsgd_dims dims, bsgd_block_grid blocks, int32_t world,
                                 int32_t rank, int32_t* bands_out) {
    return guard(nullptr, [&] {
        if (!geom || !geom->vecs || !bands_out || world < 1 || rank < 0 || rank >= world)
            fail(BSGD_E_CONTRACT, "bad arguments");
        if (geom->n_views < 1 || geom->det_u < 1 || geom->det_v < 1 || geom->beam < 0 || geom->beam > 2)
            fail(BSGD_E_GEOMETRY, "bad geometry");
        if (blocks.bx < 1 || blocks.by < 1 || blocks.bz < 1 || dims.nx % blocks.bx || dims.ny % blocks.by ||
            dims.nz % blocks.bz)
            fail(BSGD_E_PARTITION, "volume dims must be divisible by the block grid");
        const int N = blocks.bx * blocks.by * blocks.bz;
        if (N % world) fail(BSGD_E_PARTITION, "N must be divisible by world");
        // the host fields the footprint needs (no device state)
        bsgd_ctx_s h;
        h.beam = geom->beam;
        h.n_views = geom->n_views;
        h.nu = geom->det_u;
        h.nv = geom->det_v;
        h.vecs.assign(geom->vecs, geom->vecs + 12LL * geom->n_views);
        h.dims[0] = dims.nx; h.dims[1] = dims.ny; h.dims[2] = dims.nz;
        h.bgrid[0] = blocks.bx; h.bgrid[1] = blocks.by; h.bgrid[2] = blocks.bz;
        for (int k = 0; k < 3; ++k) h.bd[k] = h.dims[k] / h.bgrid[k];
        h.N = N;
        h.world = world;
        h.s = N / world;
        const std::vector<int2> bd = h.rank_bands(world, h.s);
        for (int v = 0; v < h.n_views; ++v) {
            const int2 b = bd[(size_t)rank * h.n_views + v];
            bands_out[2 * v] = b.x;
            bands_out[2 * v + 1] = b.y;
        }
    });
}

bsgd_status bsgd_block_box(bsgd_ctx c, int32_t j, int32_t* lo, int32_t* hi) {
    return guard(c, [&] {
        if (!c || !lo || !hi || j < 0 || j >= c->N) fail(BSGD_E_CONTRACT, "bad arguments");
        int l[3], h[3];
        c->box(j, l, h);
        for (int k = 0; k < 3; ++k) {
            lo[k] = l[k];
            hi[k] = h[k];
        }
    });
}

bsgd_status bsgd_balanced_z_splits(bsgd_ctx c, int32_t n_slabs, int32_t* splits, void* stream) {
    return guard(c, [&] {
        if (!c || !splits || n_slabs < 1) fail(BSGD_E_CONTRACT, "bad arguments");
        if (c->bgrid[0] != 1 || c->bgrid[1] != 1 || c->world != 1)
            fail(BSGD_E_PARTITION, "needs a one-rank z-slab context (its slabs are the candidate boundaries)");
        if (n_slabs > c->N) fail(BSGD_E_PARTITION, "more slabs than the context's slabs");
        cudaStream_t st = S(stream);
        Ordered order_(c, st);
        c->ensure_visit_table(st);
        // visits of every view through each of the context's slabs (the COUNT traversal)
        std::vector<double> cum(c->N + 1, 0.0);
        for (int b = 0; b < c->N; ++b) {
            double v = 0.0;
            for (size_t k = (size_t)b * c->n_views * c->T; k < (size_t)(b + 1) * c->n_views * c->T; ++k)
                v += (double)c->vtab[k];
            cum[b + 1] = cum[b] + v;
        }
        // split k at the slab boundary whose cumulative visit count is nearest to k/n of the
        // total (each slab at least one of the context's slabs)
        int lo_b = 0;
        splits[0] = 0;
        for (int k = 1; k < n_slabs; ++k) {
            const double target = cum[c->N] * k / n_slabs;
            int best = lo_b + 1;
            for (int b = lo_b + 1; b <= c->N - (n_slabs - k); ++b)
                if (fabs(cum[b] - target) < fabs(cum[best] - target)) best = b;
            int l[3], h[3];
            c->box(best, l, h);
            splits[k] = l[2];
            lo_b = best;
        }
        splits[n_slabs] = c->dims[2];
    });
}

bsgd_status bsgd_comm_stats(bsgd_ctx c, uint64_t* bytes_sent, uint64_t* messages, int32_t* band_mode) {
    return guard(c, [&] {
        if (!c || !bytes_sent || !messages) fail(BSGD_E_CONTRACT, "bad arguments");
        *bytes_sent = c->comm_bytes;
        *messages = c->comm_msgs;
        if (band_mode) *band_mode = c->band ? (c->lsa ? 2 : 1) : 0;
    });
}

bsgd_status bsgd_power_iteration(bsgd_ctx c, int32_t iters, uint64_t seed, double* out, void* stream) {
    return guard(c, [&] {
        if (!c || !out || iters < 1) fail(BSGD_E_CONTRACT, "bad arguments");
        Ordered order_(c, S(stream));
        cudaStream_t st = S(stream);
        const long long sb = (long long)c->s * c->bsize;
        if (!c->pw_v) {
            c->pw_v = c->dnew<float>(sb, false);
            c->pw_vT = c->dnew_pad(c->s, true);
            c->pw_vN = c->dnew_pad(c->s, false);
            c->pw_proj = c->dnew<float>(c->n_rays, false);
        }
        launch_fill_random(c->pw_v, sb, seed + 1000003ull * (uint64_t)c->rank, st);
        if (c->zsplit)   // the tails of thinner slabs are not voxels
            for (int b = 0; b < c->s; ++b) {
                const long long nb = c->vox_of(c->first + b);
                if (nb < c->bsize)
                    BSGD_CUDA(cudaMemsetAsync(c->pw_v + b * c->bsize + nb, 0, sizeof(float) * (c->bsize - nb), st));
            }
        BSGD_CUDA(cudaMemsetAsync(c->d_red, 0, 3 * sizeof(double), st));
        launch_dot3(c->pw_v, c->pw_v, sb, c->d_red, st);
        c->allreduce_d(c->d_red, 1, st);
        launch_scale(c->pw_v, sb, c->d_red, st);
        std::vector<int> all(c->n_views);
        for (int v = 0; v < c->n_views; ++v) all[v] = v;
        double lam = 0.0;
        for (int it = 0; it < iters; ++it) {
            BSGD_CUDA(cudaMemsetAsync(c->pw_proj, 0, sizeof(float) * c->n_rays, st));
            for (int b = 0; b < c->s; ++b) {
                c->update(UPD_XT, b, c->pw_v + b * c->bsize, 0.f, 1, nullptr, 0, st, nullptr, nullptr,
                          c->pT(c->pw_vT, b), 0, c->pN(c->pw_vN, b));
                c->project(PROJ_FP, all, {b}, {}, {c->pN(c->pw_vN, b)}, {c->pT(c->pw_vT, b)}, {}, {},
                           {c->pw_proj}, nullptr, 0.f, 1, st, 0);
            }
            c->allreduce_f(c->pw_proj, c->n_rays, st);
            for (int b = 0; b < c->s; ++b) {
                c->project(PROJ_BP, all, {b}, {}, {}, {}, {c->pN(c->accN, b)}, {c->pT(c->accT, b)}, {},
                           c->pw_proj, 1.f, 0, st, 0);
                c->update(UPD_OUT, b, nullptr, 0.f, 0, c->pw_v + b * c->bsize, 0, st);
            }
            BSGD_CUDA(cudaMemsetAsync(c->d_red, 0, 3 * sizeof(double), st));
            launch_dot3(c->pw_v, c->pw_v, sb, c->d_red, st);
            c->allreduce_d(c->d_red, 1, st);
            double nn = 0;
            BSGD_CUDA(cudaMemcpyAsync(&nn, c->d_red, sizeof(double), cudaMemcpyDeviceToHost, st));
            BSGD_CUDA(cudaStreamSynchronize(st));
            lam = sqrt(nn);
            launch_scale(c->pw_v, sb, c->d_red, st);
        }
        *out = lam;
    });
}

}  // extern "C"
#pragma GCC visibility pop
