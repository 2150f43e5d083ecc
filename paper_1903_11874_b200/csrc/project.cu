// Siddon ray-driven projector for sm_100a: FP z = A_I^J x_J (Algo 1 line 5,
// PAPER.md:139), matched BP g = s (A_I^J)^T r (Algo 1 line 9),
// and the ones-pass block masses of BSGD-IM.
//
// Design:
//  * a2 ray setup in fp64 (IEEE round-to-nearest, no FMA contraction, the same
//    parametrisation p(alpha) = a + alpha b, alpha in [0,1], as the problem
//    definition) and slab clipping against the block box;
//  * traversal "slice by slice" along a main in-plane axis: every warp (32 adjacent
//    detector columns of one detector row) walks the planes of that axis in LOCKSTEP, so
//    at every step the 32 lanes touch 32 neighbouring voxels of one image row ->
//    coalesced 128-byte gathers (FP) and coalesced reductions (BP).  Inside a slice the
//    exact Siddon segments are cut by the crossings of the other two axes.
//      k_project3 (default, v3): crossings from 64-bit fixed-point plane distances (no
//        fp64 in the loop); warps with a "steep" ray are left to
//      k_project2 (v2): crossing t kept in fp64, advanced by |1/b|; decisions in fp32 on
//        t-differences (also the whole path under BSGD_PROJECTOR=2, for A/B).
//  * warps whose main axis is x read a transposed copy of the block ([z][x][y]) with
//    x<->y swapped in the ray, so the lockstep axis is always the slow in-plane axis of
//    the layout that is read.
//  * no tensor cores: this is a sparse gather/scatter.
#include <climits>
#include <cstdlib>

#include "internal.h"

namespace bsgd {
#ifndef PROJ3_FP32STEP
#define PROJ3_FP32STEP 1   // FP: 32-bit plane distances (0: the 64-bit stepping, for A/B)
#endif
#if PROJ3_FP32STEP
#define PROJ3_FINE 8192.0
#else
#define PROJ3_FINE 65536.0
#endif
#ifndef PROJ3_MINB
#define PROJ3_MINB 4
#endif

namespace {

__device__ __forceinline__ int cell_enter(double c, int dir, int lo, int hi) {
    double f = floor(c);
    int i = (int)f;
    if (dir < 0 && f == c) i -= 1;   // moving down from a plane: cell below it
    return min(max(i, lo), hi - 1);
}

__device__ __forceinline__ int cell_exit(double c, int dir, int lo, int hi) {
    int i = (dir > 0) ? (int)ceil(c) - 1 : (int)floor(c);
    return min(max(i, lo), hi - 1);
}

__device__ __forceinline__ int sgn(double v) { return (v > 0.0) - (v < 0.0); }

// Fire-and-forget fp32 reduction into GLOBAL memory (REDG.E.ADD.F32 at L2).  atomicAdd on
// a generic pointer compiles to ATOM plus a shared-memory CAS-loop fallback branch.
__device__ __forceinline__ void red_add(float* p, float v) {
    asm volatile("red.global.add.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
}
// BP reduction at element `off` of the target: fp32 RED (PROJ_BP) or, PROJ_BPD, a 64-bit
// integer RED of round(v S) into the int64 accumulator behind the same base (integer
// addition is associative: the result does not depend on the order of the ray threads)
template <int MODE>
__device__ __forceinline__ void red_acc(float* base, int off, float v, float S) {
    if (MODE == PROJ_BPD) {
        const long long q = __float2ll_rn(v * S);
        asm volatile("red.global.add.u64 [%0], %1;" ::"l"(reinterpret_cast<unsigned long long*>(base) + off),
                     "l"((unsigned long long)q) : "memory");
    } else {
        red_add(base + off, v);
    }
}
__device__ __forceinline__ bool lane_steep(const double b[3]) {
    // |b_c / b_1| < 1 with a margin (the v3 increments K = |b_c / b_1| 2^64 stay < 2^64)
    const double lim = fabs(b[1]) * (1.0 - 1.0 / 1073741824.0);
    return b[1] == 0.0 || !(fabs(b[0]) < lim) || !(fabs(b[2]) < lim);
}
// FP: a non-zero minor slope |b_c / b_1| below 1 / PROJ3_FINE (2^-13).  The v3 FP walks
// 32-bit plane distances (2^-32 voxel, see walk3_setup), which move a crossing by < N 2^-33 /
// |k| slices on an N-slice segment: < 2^-31 / |k| of the ray sum per crossing, fine for
// |k| >= 2^-13; warps with a smaller non-zero slope go to the v2 companion like steep ones
// (rare: a ray within 2^-13 rad of a grid axis).  (PROJ3_FP32STEP=0: the 64-bit walk with the
// high-word conversion, whose error 2^-32 / |k| needs only 2^-16.)
__device__ __forceinline__ bool lane_fine(const double b[3]) {
    const double f = fabs(b[1]) * (1.0 / PROJ3_FINE);
    return (b[0] != 0.0 && fabs(b[0]) < f) || (b[2] != 0.0 && fabs(b[2]) < f);
}
// v3 main axis, chosen per WARP (majority of its rays; the lanes must share one layout for
// coalescing): fewer steep lanes than a per-view choice where the fan/cone spans 45 deg.
__device__ __forceinline__ bool warp_main_x(const double b[3], bool inrect) {
    const unsigned vx = __ballot_sync(0xffffffffu, inrect && fabs(b[0]) > fabs(b[1]));
    const unsigned n = __ballot_sync(0xffffffffu, inrect);
    return 2 * __popc(vx) > __popc(n);
}
// the v3 kernel's companion predicate (steep, or FP with a fine slope) evaluated in the v3
// frame of a world-frame direction b
template <int MODE>
__device__ __forceinline__ bool lane_v2_v3(const double b[3], bool mainX) {
    const double f[3] = {mainX ? b[1] : b[0], mainX ? b[0] : b[1], b[2]};
    return lane_steep(f) || (MODE == PROJ_FP && lane_fine(f));
}

// FP output address of ray (view, iu, iv): the full-length vector, or the block's packed
// footprint storage of z^j (the launch rectangles lie inside the footprint)
__device__ __forceinline__ float* zaddr(const BlockDesc& B, const KGeom& g, int view, int iu, int iv) {
    if (!B.zr) return B.z + ((long long)view * g.nv + iv) * g.nu + iu;
    const ZRect q = B.zr[view];
    return B.z + q.base + (long long)(iv - q.v0) * (q.u1 - q.u0) + (iu - q.u0);
}

// Ray (view, iv, iu) in grid coordinates, exactly as the problem defines it.
__device__ __forceinline__ void make_ray(const KGeom& g, const double* vec, int iu, int iv,
                                         double a[3], double b[3]) {
    double ou = (double)iu - (g.nu - 1) / 2.0, ov = (double)iv - (g.nv - 1) / 2.0;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        double d = __dadd_rn(__dadd_rn(vec[3 + c], __dmul_rn(ou, vec[6 + c])), __dmul_rn(ov, vec[9 + c]));
        if (g.beam == BSGD_PARALLEL) {
            a[c] = __dsub_rn(d, __dmul_rn(g.R, vec[c]));
            b[c] = __dmul_rn(__dmul_rn(2.0, g.R), vec[c]);
        } else {
            a[c] = vec[c];
            b[c] = __dsub_rn(d, vec[c]);
        }
        a[c] = __dadd_rn(a[c], g.dims[c] / 2.0);
    }
}

// Clip p(alpha), alpha in [0,1], against [lo, hi); half-open for axes with b = 0.
__device__ __forceinline__ bool clip(const double a[3], const double b[3], const double inv[3],
                                     const int lo[3], const int hi[3], double& amin, double& amax) {
    amin = 0.0;
    amax = 1.0;
    bool ok = true;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        if (b[c] == 0.0) {
            ok = ok && (a[c] >= lo[c]) && (a[c] < hi[c]);
        } else {
            double t0 = (lo[c] - a[c]) * inv[c], t1 = (hi[c] - a[c]) * inv[c];
            amin = fmax(amin, fmin(t0, t1));
            amax = fmin(amax, fmax(t0, t1));
        }
    }
    return ok && amin < amax;
}

// v2 traversal: the same slice-lockstep Siddon, with a straight-line slice body for the
// common case (at most one x and one z plane crossing inside the slice: up to three
// segments, their loads issued together), a rare general loop for further crossings,
// 32-bit voxel offsets and fp32 slice sums flushed into an fp64 accumulator.
// (one warp's work: the warp of CTA (bidx, bidz) whose thread index is tidx; warp-independent)
template <int MODE, bool STEEP_ONLY>
__device__ __forceinline__ void project2_body(const ProjLaunch& L, const unsigned bidx, const unsigned bidz,
                                              const int tidx) {
    // band-major CTA order: blockIdx.x = (band * n_slots + slot) * n_chunks + chunk, so the
    // CTAs resident at any time cover the same detector-row band of consecutive views
    // (rays of one band cross the same z-range of the volume -> L2 reuse across views).
    const BlockDesc& B = L.blocks[bidz];
    unsigned bid = bidx;
    const int chunk = (int)(bid % (unsigned)L.n_chunks);
    bid /= (unsigned)L.n_chunks;
    const int slot = (int)(bid % (unsigned)L.n_slots);
    const int band = B.band_lo + (int)(bid / (unsigned)L.n_slots);
    const int4 rc = L.rects[(size_t)bidz * L.n_slots + slot];
    const int r0 = max(rc.z, band * L.rows_per_band), r1 = min(rc.w, band * L.rows_per_band + L.rows_per_band);
    const int w = rc.y - rc.x;
    if (r0 >= r1 || w <= 0) return;
    const int nrect = (r1 - r0) * w;
    const int base = chunk * 256;
    if (base >= nrect) return;                       // uniform over the CTA
    const int tid = base + tidx;
    const bool inrect = tid < nrect;
    const int iu = rc.x + (inrect ? tid % w : 0);
    const int iv = r0 + (inrect ? tid / w : 0);
    const int view = L.views[slot];
    const double* vec = L.g.vecs + 12 * (size_t)view;
    const double cxv = (L.g.beam == BSGD_PARALLEL) ? vec[0] : vec[3] - vec[0];
    const double cyv = (L.g.beam == BSGD_PARALLEL) ? vec[1] : vec[4] - vec[1];
    const bool mainX = fabs(cxv) > fabs(cyv);

    double a[3], b[3];
    make_ray(L.g, vec, iu, iv, a, b);
    const double blen = sqrt(b[0] * b[0] + b[1] * b[1] + b[2] * b[2]);
    bool steep3 = false;   // STEEP_ONLY: the v3 kernel's predicate, in the v3 kernel's frame
    if (STEEP_ONLY) steep3 = lane_v2_v3<MODE>(b, warp_main_x(b, inrect));
    int lo[3] = {B.lo[0], B.lo[1], B.lo[2]}, hi[3] = {B.hi[0], B.hi[1], B.hi[2]};
    if (mainX) {
        double t = a[0]; a[0] = a[1]; a[1] = t;
        t = b[0]; b[0] = b[1]; b[1] = t;
        int q = lo[0]; lo[0] = lo[1]; lo[1] = q;
        q = hi[0]; hi[0] = hi[1]; hi[1] = q;
    }
    // strides of the padded copy of the frame's layout (BlockDesc)
    const int bdx = mainX ? B.rowT : B.rowN;
    const unsigned plane = (unsigned)(mainX ? B.planeT : B.planeN);
    double inv[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) inv[c] = (b[c] != 0.0) ? 1.0 / b[c] : 0.0;
    double amin, amax;
    bool hit = inrect && clip(a, b, inv, lo, hi, amin, amax);
    // v3 companion mode: only the warps k_project3 leaves (a lane with a steep ray)
    if (STEEP_ONLY && !__any_sync(0xffffffffu, hit && (steep3 || amin == 0.0 || amax == 1.0))) return;
    float rs = 0.f;
    const float S = MODE == PROJ_BPD ? *L.det_scale : 0.f;
    if (is_bp(MODE)) {
        if (inrect) rs = L.scale * L.rproj[((long long)view * L.g.nv + iv) * L.g.nu + iu];
        hit = hit && (rs != 0.f);
    }
    const float* __restrict__ src = mainX ? B.xT : B.xN;
    float* dst = mainX ? B.outT : B.outN;

    const int sx = sgn(b[0]), sy = sgn(b[1]), sz = sgn(b[2]);
    const double INF = __longlong_as_double(0x7ff0000000000000ll);
    // Lane state: voxel (rx, rz) relative to the block origin and its offset o, the current
    // t, the t of the next x / z plane crossing (tx, tz) and of the current slice's exit plane
    // (tpl).  Plane crossings advance by exact-enough fp64 increments (|1/b|: ~1e-13 drift
    // over a whole ray); every in-slice decision runs in fp32 on t-differences.  There are no
    // bounds checks: the only possible out-of-box step is a rounding-induced crossing of the
    // exit face with a ~1e-9-voxel segment, which lands in the zeroed slack the library puts
    // around every image buffer the projector touches (or in a neighbouring voxel).
    int j0 = 0, j1 = -1, rx = 0, rz = 0;
    double t = 0.0, tx = INF, tz = INF, tpl = INF;
    int o = 0;   // signed: an out-of-box step may point one element before the block
    const double dtx = fabs(inv[0]), dtz = fabs(inv[2]), dty = fabs(inv[1]);
    if (hit) {
        j0 = cell_enter(a[1] + amin * b[1], sy, lo[1], hi[1]);
        j1 = cell_exit(a[1] + amax * b[1], sy, lo[1], hi[1]);
        if (sy == 0) j1 = j0;
        const int ix = cell_enter(a[0] + amin * b[0], sx, lo[0], hi[0]);
        const int iz = cell_enter(a[2] + amin * b[2], sz, lo[2], hi[2]);
        rx = ix - lo[0];
        rz = iz - lo[2];
        if (sx) tx = ((double)(ix + (sx > 0)) - a[0]) * inv[0];
        if (sz) tz = ((double)(iz + (sz > 0)) - a[2]) * inv[2];
        if (sy) tpl = ((double)(j0 + (sy > 0)) - a[1]) * inv[1];
        t = amin;
        o = rz * (int)plane + (j0 - lo[1]) * bdx + rx;
    }
    const int pstep = sz * (int)plane;
    const int rowstep = sy * bdx;
    const float wbp = (float)blen * rs;   // BP weight per unit t: |b| * scale * r_ray
    const float cthr = (float)(1e-6 / blen);   // COUNT: segments above 1e-6 voxel (see v3)
    double acc = 0.0;
    float acc32 = 0.f;
    unsigned int nvis = 0;

    for (int pass = 0; pass < 2; ++pass) {
        const int dir = pass == 0 ? 1 : -1;
        const bool mine = hit && (pass == 0 ? sy >= 0 : sy < 0);
        if (__ballot_sync(0xffffffffu, mine) == 0u) continue;
        int jl = mine ? min(j0, j1) : INT_MAX;
        int jh = mine ? max(j0, j1) : INT_MIN;
        jl = __reduce_min_sync(0xffffffffu, jl);
        jh = __reduce_max_sync(0xffffffffu, jh);
        const int jstart = dir > 0 ? jl : jh;
        const int nsl = jh - jl + 1;
        for (int k = 0; k < nsl; ++k) {
            const int j = jstart + dir * k;
            const bool in = mine && (dir > 0 ? (j >= j0 && j <= j1) : (j <= j0 && j >= j1));
            if (in) {
                // (j1 can land one slice late by rounding: never walk past amax)
                const double thi = tpl < amax ? tpl : amax;
                const float dh = (float)(thi - t);
                const float dx = (float)(tx - t);
                const float dz = (float)(tz - t);
                const bool cx = dx < dh, cz = dz < dh;
                const float ex = cx ? dx : dh, ez = cz ? dz : dh;
                const bool xfirst = ex <= ez;
                const float m1 = fmaxf(fminf(ex, ez), 0.f), m2 = fmaxf(fmaxf(ex, ez), 0.f);
                const int dox = cx ? sx : 0, doz = cz ? pstep : 0;
                const int o1 = o + (xfirst ? dox : doz);
                const int o2 = o + dox + doz;
                const double ntx = tx + dtx, ntz = tz + dtz;
                // rare: a second crossing of one axis inside the slice -> commit only the first
                // crossing and let the general loop finish the slice
                const bool more = (cx && ntx < thi) || (cz && ntz < thi);
                // segment 1 exists iff some crossing falls in the slice, segment 2 iff both do
                // (and no second crossing sends the rest to the general loop)
                const bool p1 = !more && (cx || cz), p2 = !more && cx && cz;
                // segment lengths in t units; FP scales the sum by |b| at each flush, BP
                // folds |b| into the ray's weight w = |b| * scale * r
                const float l0 = m1;
                const float l1 = m2 - m1;
                const float l2 = dh - m2;
                if (MODE == PROJ_FP) {
                    const float x0 = __ldg(src + o);
                    const float x1 = p1 ? __ldg(src + o1) : 0.f;
                    const float x2 = p2 ? __ldg(src + o2) : 0.f;
                    acc32 = fmaf(l0, x0, fmaf(l1, x1, fmaf(l2, x2, acc32)));
                }
                if (is_bp(MODE)) {       // zero-length segments (exact-boundary ties) add 0
                    red_acc<MODE>(dst, (int)o, l0 * wbp, S);
                    if (p1) {            // p2 implies p1: one reconvergence region
                        red_acc<MODE>(dst, (int)o1, l1 * wbp, S);
                        if (p2) red_acc<MODE>(dst, (int)o2, l2 * wbp, S);
                    }
                }
                if (MODE == PROJ_COUNT)
                    nvis += (unsigned)(l0 > cthr) + (unsigned)(p1 && l1 > cthr) + (unsigned)(p2 && l2 > cthr);
                if (!more) {
                    o = o2;
                    if (cx) tx = ntx;
                    if (cz) tz = ntz;
                } else {
                    double tt;
                    if (xfirst) { tt = fmax(t, tx); o += sx; tx = ntx; }
                    else { tt = fmax(t, tz); o += pstep; tz = ntz; }
                    for (;;) {      // general loop for the rest of the slice
                        const double tn = fmin(fmin(tx, tz), thi);
                        if (tn > tt) {
                            const float len = (float)(tn - tt);   // t units (see above)
                            if (MODE == PROJ_FP) acc32 = fmaf(len, __ldg(src + o), acc32);
                            if (is_bp(MODE)) red_acc<MODE>(dst, (int)o, len * wbp, S);
                            if (MODE == PROJ_COUNT && len > cthr) ++nvis;
                            tt = tn;
                        }
                        if (tx <= tz) {
                            if (tx < thi) {
                                o += sx;
                                tx += dtx;
                                continue;
                            }
                        } else if (tz < thi) {
                            o += pstep;
                            tz += dtz;
                            continue;
                        }
                        break;
                    }
                }
                t = thi;
                tpl += dty;
                o += rowstep;
            }
            if (MODE == PROJ_FP && (k & 15) == 15) {   // warp-uniform
                acc += (double)acc32;
                acc32 = 0.f;
            }
        }
    }
    if (MODE == PROJ_FP && inrect) {
        acc += (double)acc32;
        acc *= blen;                        // t units -> voxel lengths
        float* zp = zaddr(B, L.g, view, iu, iv);
        *zp = L.accumulate ? (*zp + (float)acc) : (float)acc;
    }
    if (MODE == PROJ_COUNT && L.visits) {   // per (block, slot) counters
        unsigned int s = __reduce_add_sync(0xffffffffu, nvis);
        if ((tidx & 31) == 0 && s) atomicAdd(L.visits + (size_t)bidz * L.n_slots + slot, (unsigned long long)s);
    }
}

template <int MODE, bool STEEP_ONLY = false>
__global__ void __launch_bounds__(256, 4) k_project2(const ProjLaunch L) {
    project2_body<MODE, STEEP_ONLY>(L, blockIdx.x, blockIdx.z, (int)threadIdx.x);
}

// The v2 companion over the warps k_project3 listed (persistent warps striding the list):
// only those warps pay the v2 set-up, instead of every warp of the launch grid.
template <int MODE>
__global__ void __launch_bounds__(256, 4) k_project2_list(const ProjLaunch L) {
    const unsigned n = *L.v2_count;
    const unsigned lane = threadIdx.x & 31;
    const unsigned nw = (gridDim.x * blockDim.x) >> 5;
    for (unsigned e = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; e < n; e += nw) {   // warp-uniform
        const uint2 q = L.v2_list[e];
        project2_body<MODE, true>(L, q.x, q.y >> 3, (int)((q.y & 7u) * 32u + lane));
    }
}

// ---------------------------------------------------------------------------------------
// v3 traversal: the same slice-lockstep Siddon, parametrised by the distance s travelled
// along the main axis instead of by the ray parameter t.  Inside the block the ray is the
// line x(s) = x_p + kx s, z(s) = z_p + kz s (|kx|, |kz| < 1 for "non-steep" rays), so each
// slice holds at most one x- and one z-plane crossing.  Per lane and axis the distance to
// the next plane (of the coordinate mirrored so that it increases) is a 64-bit fixed-point
// integer D in 2^-64 voxel, decremented by K = |k| 2^64 per slice: the plane is crossed
// inside the slice iff the subtraction borrows, at u = D / K of the slice (I2F.U64 + FMUL,
// <= 1.5 ulp).  The integer cell is never stored: the voxel offset o advances by the axis
// stride on a borrow.  No fp64 and no division in the loop; the fp64 ray setup fixes D and
// K to ~1e-16 and the stepping drifts < 2^-54 voxel over 1024 slices.  (A 32-bit fraction
// was too coarse: for a small slope k an error dx in position moves the crossing by dx/k.)
// FP and BP take whole slices: the part of a slice outside the block (entry / exit through
// an x or z face) lies in the padded copies' zero border (BlockDesc); COUNT clamps exactly.
//
// Rays with |kx| or |kz| >= 1 (or parallel to the slices) can cross one axis twice in a
// slice.  A warp containing such a lane is left to the v2 kernel (launched second, it skips
// every warp this kernel handled), so both decide "steep" with the same predicate.

// One slice's three gathers, predicated inside PTX on the lane's slice range
// (rel <= nk, unsigned; no branch).  Without a crossing o1 = o2 = o (an L1 hit) and the
// segment lengths l1 = l2 = 0 exactly, so no crossing masks are needed.
// Outside the range the outputs are left unwritten (undefined): the caller discards the
// slice's contribution with a select on the same predicate (no zero-initialisation).
__device__ __forceinline__ void gather3(unsigned rel, unsigned nk, const float* p0, const float* p1,
                                        const float* p2, float& v0, float& v1, float& v2) {
    asm("{\n\t.reg .pred a;\n\t"
        "setp.le.u32 a, %3, %4;\n\t"
        "@a ld.global.nc.f32 %0, [%5];\n\t"
        "@a ld.global.nc.f32 %1, [%6];\n\t"
        "@a ld.global.nc.f32 %2, [%7];\n\t}"
        : "=f"(v0), "=f"(v1), "=f"(v2)
        : "r"(rel), "r"(nk), "l"(p0), "l"(p1), "l"(p2));
}

// One slice's reductions.  ptxas turns every predicated RED into a BSSY/BRA/BSYNC
// branch, so the rare segments are nested under the common ones (one reconvergence
// region per slice instead of three; measured BP 136 -> 121 ms at cfg5):
// segment 0 iff the lane is in its slice range, segment 1 iff also a plane is crossed
// (m_or != 0), segment 2 iff both planes are (m_and != 0).
template <int MODE>
__device__ __forceinline__ void scatter3(bool in, unsigned m_or, unsigned m_and, float* base, int o0, int o1, int o2,
                                         float v0, float v1, float v2, float S) {
    if (in) {
        red_acc<MODE>(base, o0, v0, S);
        if (m_or) {
            red_acc<MODE>(base, o1, v1, S);
            if (m_and) red_acc<MODE>(base, o2, v2, S);
        }
    }
}

// D -= K on the 64-bit plane distance; returns ~0u when it borrows (a plane is crossed).
// The result goes to a new register (Dn) rather than back into D: the caller still reads D
// (the crossing point D / K), and an in-place subtraction made ptxas copy D every slice.
__device__ __forceinline__ unsigned sub_borrow(unsigned long long& D, unsigned long long K) {
    unsigned m;
    unsigned long long Dn;
    asm("sub.cc.u64 %0, %2, %3;\n\tsubc.u32 %1, 0, 0;" : "=l"(Dn), "=r"(m) : "l"(D), "l"(K));
    D = Dn;
    return m;
}

// 32-bit form: D -= K, ~0u on a borrow
__device__ __forceinline__ unsigned sub_borrow32(unsigned& D, unsigned K) {
    unsigned m, Dn;
    asm("sub.cc.u32 %0, %2, %3;\n\tsubc.u32 %1, 0, 0;" : "=r"(Dn), "=r"(m) : "r"(D), "r"(K));
    D = Dn;
    return m;
}

// Distance from coordinate c (mirrored so that it increases along the ray) to the next
// plane in 2^-64 voxel units, and the cell the walk starts in.  A point exactly on a plane
// with a non-zero slope starts in the cell below with distance 0 (a zero-length segment,
// then the crossing); with zero slope it stays in the cell above (half-open [lo, hi)).
__device__ __forceinline__ unsigned long long plane_dist(double c, unsigned long long K, int& cell) {
    const double f = floor(c);
    cell = (int)f;
    const double rem = 1.0 - (c - f);                         // in (0, 1]
    if (rem >= 1.0) {                                         // on a plane
        if (K) cell -= 1;
        return 0ull;
    }
    return __double2ull_rn(rem * 18446744073709551616.0);
}

// Per-lane state of the v3 / v6 slice walk (see the v3 comment above), set up at the warp's
// first slice plane of each direction group.
struct Walk3 {
    const float* src;          // FP source (the padded copy of the frame's layout)
    float* dst;                // BP target
    unsigned long long DX, DZ, KX, KZ;   // 64-bit plane distances and per-slice decrements
    float ikx, ikz;            // 1 / K (crossing point u = D / K)
    float slo, shi_last;       // COUNT: in-slice entry / exit at the lane's first / last slice
    float Ls;                  // voxel length per unit of main-axis travel
    float wbp;                 // BP weight per unit of main-axis travel
    float S;                   // PROJ_BPD scale
    unsigned o;                // voxel offset at the current slice (wraps outside the range)
    int sxo, pstep, rowstep;   // x step (+-1), z step (+-plane), slice step (+-row)
    int k0, nk;                // the lane's slices [k0, k0 + nk] relative to its group's start
    int jlo_p, jhi_p, jlo_n, jhi_n;   // warp-wide slice ranges of the two direction groups
    bool pos, neg;             // the lane's ray walks the sy > 0 / sy < 0 group
    bool inrect;
    int view, iu, iv;
};

// Ray setup (a2) + v3 walk state.  Returns false when the v2 companion kernel takes this
// warp (a steep ray, or a ray starting / ending inside the box) or the CTA has no rays.
template <int MODE>
__device__ __forceinline__ bool walk3_setup(const ProjLaunch& L, const BlockDesc& B, Walk3& W) {
    unsigned bid = blockIdx.x;
    const int chunk = (int)(bid % (unsigned)L.n_chunks);
    bid /= (unsigned)L.n_chunks;
    const int slot = (int)(bid % (unsigned)L.n_slots);
    const int band = B.band_lo + (int)(bid / (unsigned)L.n_slots);
    const int4 rc = L.rects[(size_t)blockIdx.z * L.n_slots + slot];
    const int r0 = max(rc.z, band * L.rows_per_band), r1 = min(rc.w, band * L.rows_per_band + L.rows_per_band);
    const int w = rc.y - rc.x;
    if (r0 >= r1 || w <= 0) return false;
    const int nrect = (r1 - r0) * w;
    const int base = chunk * (int)blockDim.x;
    if (base >= nrect) return false;                 // uniform over the CTA
    const int tid = base + (int)threadIdx.x;
    const bool inrect = tid < nrect;
    const int iu = rc.x + (inrect ? tid % w : 0);
    const int iv = r0 + (inrect ? tid / w : 0);
    const int view = L.views[slot];
    const double* vec = L.g.vecs + 12 * (size_t)view;
    W.inrect = inrect;
    W.view = view;
    W.iu = iu;
    W.iv = iv;

    double a[3], b[3];
    make_ray(L.g, vec, iu, iv, a, b);
    const bool mainX = warp_main_x(b, inrect);
    int lo[3] = {B.lo[0], B.lo[1], B.lo[2]}, hi[3] = {B.hi[0], B.hi[1], B.hi[2]};
    if (mainX) {
        double t = a[0]; a[0] = a[1]; a[1] = t;
        t = b[0]; b[0] = b[1]; b[1] = t;
        int q = lo[0]; lo[0] = lo[1]; lo[1] = q;
        q = hi[0]; hi[0] = hi[1]; hi[1] = q;
    }
    double inv[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) inv[c] = (b[c] != 0.0) ? 1.0 / b[c] : 0.0;
    double amin, amax;
    bool hit = inrect && clip(a, b, inv, lo, hi, amin, amax);
    // the v2 kernel takes this warp if a lane's ray is steep or starts / ends inside the box
    // (source or detector within the block: no face to exit through, the zero border would
    // not absorb the rest of the slice)
    if (__any_sync(0xffffffffu, hit && (lane_steep(b) || (MODE == PROJ_FP && lane_fine(b)) || amin == 0.0 ||
                                        amax == 1.0))) {
        if (L.v2_list && (threadIdx.x & 31) == 0)   // hand the warp to the list companion
            L.v2_list[atomicAdd(L.v2_count, 1u)] = make_uint2(blockIdx.x, (blockIdx.z << 3) | (threadIdx.x >> 5));
        return false;
    }
    const double blen = sqrt(b[0] * b[0] + b[1] * b[1] + b[2] * b[2]);
    float rs = 0.f;
    W.S = MODE == PROJ_BPD ? *L.det_scale : 0.f;
    if (is_bp(MODE)) {
        if (inrect) rs = L.scale * L.rproj[((long long)view * L.g.nv + iv) * L.g.nu + iu];
        hit = hit && (rs != 0.f);
    }
    W.src = mainX ? B.xT : B.xN;
    W.dst = mainX ? B.outT : B.outN;

    // strides of the padded copy of the frame's layout (BlockDesc): rows carry PAD_X and
    // the block PAD_Z zero cells beyond every face the slice walk can step through
    const int bdx = mainX ? B.rowT : B.rowN;
    const int plane = mainX ? B.planeT : B.planeN;
    const int sy = (b[1] > 0.0) ? 1 : -1;
    const double ainv1 = fabs(inv[1]);
    const double TWO64 = 18446744073709551616.0;
    // The warp walks the slices of each direction group (sy > 0, then sy < 0) in lockstep
    // from the group's first slice jstart.  Every lane's stepping state is set up AT jstart's
    // entry plane by extending its ray (cells outside the block are never dereferenced:
    // loads / reductions are predicated on the lane's own slice range [k0, k0 + nk]), so the
    // loop needs no per-lane freezing of state before the lane's first slice.
    int j0 = 0, j1 = -1;
    if (hit) {
        j0 = cell_enter(a[1] + amin * b[1], sy, lo[1], hi[1]);
        j1 = cell_exit(a[1] + amax * b[1], sy, lo[1], hi[1]);
        if (sy * (j1 - j0) < 0) j1 = j0;              // rounding on a sub-slice chord
    }
    W.pos = hit && sy > 0;
    W.neg = hit && sy < 0;
    W.jlo_p = __reduce_min_sync(0xffffffffu, W.pos ? j0 : INT_MAX);
    W.jhi_p = __reduce_max_sync(0xffffffffu, W.pos ? j1 : INT_MIN);
    W.jlo_n = __reduce_min_sync(0xffffffffu, W.neg ? j1 : INT_MAX);
    W.jhi_n = __reduce_max_sync(0xffffffffu, W.neg ? j0 : INT_MIN);
    W.DX = W.DZ = W.KX = W.KZ = 0ull;
    W.ikx = W.ikz = W.slo = W.Ls = 0.f;
    W.shi_last = 1.f;
    W.o = 0u;
    W.sxo = 1;
    W.pstep = plane;
    W.k0 = INT_MAX;
    W.nk = 0;
    if (hit) {
        const int jstart = sy > 0 ? W.jlo_p : W.jhi_n;
        W.k0 = sy * (j0 - jstart);
        W.nk = sy * (j1 - j0);
        const double ys = (double)(sy > 0 ? jstart : jstart + 1);   // entry plane of jstart
        const double yin0 = (double)(sy > 0 ? j0 : j0 + 1);         // entry plane of slice j0
        const double yin1 = (double)(sy > 0 ? j1 : j1 + 1);
        const double ap = (ys - a[1]) * inv[1];                     // alpha at plane ys
        const double kx = b[0] * ainv1, kz = b[2] * ainv1;          // per unit of main-axis travel
        const bool mx = kx < 0.0, mz = kz < 0.0;
        const double xr = a[0] + ap * b[0] - lo[0], zr = a[2] + ap * b[2] - lo[2];
        const double xm = mx ? -xr : xr, zm = mz ? -zr : zr;
        W.KX = __double2ull_rn(fabs(kx) * TWO64);
        W.KZ = __double2ull_rn(fabs(kz) * TWO64);
        int cxm, czm;
        W.DX = plane_dist(xm, W.KX, cxm);
        W.DZ = plane_dist(zm, W.KZ, czm);
        const int ix = mx ? -cxm - 1 : cxm;                         // frame cell relative to lo
        const int iz = mz ? -czm - 1 : czm;
        // K = 0 (ray parallel to that axis' planes): an infinite distance, never crossed
        if (!W.KX) W.DX = ~0ull;
        if (!W.KZ) W.DZ = ~0ull;
        // (K = 0: D = 2^64 - 1 and 1/K := 2^-63, so D / K = 2 saturates to "no crossing")
        W.ikx = W.KX ? (float)(1.0 / (double)W.KX) : 1.0842022e-19f;
        W.ikz = W.KZ ? (float)(1.0 / (double)W.KZ) : 1.0842022e-19f;
        W.sxo = mx ? -1 : 1;
        W.pstep = mz ? -plane : plane;
        W.o = (unsigned)iz * (unsigned)plane + (unsigned)(jstart - lo[1]) * (unsigned)bdx + (unsigned)ix;
        W.slo = (float)fmin(fmax((amin - (yin0 - a[1]) * inv[1]) * fabs(b[1]), 0.0), 1.0);
        W.shi_last = (float)fmin(fmax((amax - (yin1 - a[1]) * inv[1]) * fabs(b[1]), 0.0), 1.0);
        if (j1 == j0) W.shi_last = fmaxf(W.shi_last, W.slo);
        W.Ls = (float)(blen * ainv1);
#if PROJ3_FP32STEP
        if (MODE == PROJ_FP) {
            // The 32-bit walk (2^-32 voxel distances, K rounded) starts exact at the lane's OWN
            // first slice j0 and is rewound to jstart in modular arithmetic -- D32 + k0 K32, the
            // wraps of that sum are the crossings the k0 steps will count, o backed off by them
            // -- so its drift (< 2^-33 voxel per step) accumulates over the lane's own slices
            // only: a crossing moves by < N 2^-33 / |k| slices on an N-slice segment.
            const double ap0 = (yin0 - a[1]) * inv[1];
            const double xr0 = a[0] + ap0 * b[0] - lo[0], zr0 = a[2] + ap0 * b[2] - lo[2];
            int cx0, cz0;
            unsigned long long DX0 = plane_dist(mx ? -xr0 : xr0, W.KX, cx0);
            unsigned long long DZ0 = plane_dist(mz ? -zr0 : zr0, W.KZ, cz0);
            if (!W.KX) DX0 = ~0ull;
            if (!W.KZ) DZ0 = ~0ull;
            const int ix0 = mx ? -cx0 - 1 : cx0, iz0 = mz ? -cz0 - 1 : cz0;
            const unsigned kx32 = (unsigned)((W.KX >> 32) + ((W.KX >> 31) & 1ull));
            const unsigned kz32 = (unsigned)((W.KZ >> 32) + ((W.KZ >> 31) & 1ull));
            const unsigned long long tx = (DX0 >> 32) + (unsigned long long)(unsigned)W.k0 * kx32;
            const unsigned long long tz = (DZ0 >> 32) + (unsigned long long)(unsigned)W.k0 * kz32;
            W.DX = tx << 32;                                        // the kernel takes the high words
            W.DZ = tz << 32;
            const unsigned o_lane = (unsigned)iz0 * (unsigned)plane + (unsigned)(j0 - lo[1]) * (unsigned)bdx +
                                    (unsigned)ix0;
            W.o = o_lane - (unsigned)W.k0 * (unsigned)(sy * bdx) - (unsigned)(tx >> 32) * (unsigned)W.sxo -
                  (unsigned)(tz >> 32) * (unsigned)W.pstep;
        }
#endif
    }
    W.rowstep = sy * bdx;
    W.wbp = W.Ls * rs;   // BP weight per unit of main-axis travel
    return true;
}

template <int MODE>
__global__ void __launch_bounds__(256, PROJ3_MINB) k_project3(const ProjLaunch L) {
    const BlockDesc& B = L.blocks[blockIdx.z];
    Walk3 W;
    if (!walk3_setup<MODE>(L, B, W)) return;
    const float* __restrict__ src = W.src;
    float* dst = W.dst;
    const bool inrect = W.inrect, pos = W.pos, neg = W.neg;
    const int jlo_p = W.jlo_p, jhi_p = W.jhi_p, jlo_n = W.jlo_n, jhi_n = W.jhi_n;
    unsigned long long DX = W.DX, DZ = W.DZ;
    const unsigned long long KX = W.KX, KZ = W.KZ;
    // FP (PROJ3_FP32STEP): the plane distances in 2^-32 voxel, D truncated, K rounded; the
    // stepping then drifts < N 2^-33 voxel over N slices, a crossing moves by that / |k| --
    // below 2^-32 / |k| slices for |k| >= 2^-13 (lane_fine routes smaller slopes to v2)
    unsigned DX32 = (unsigned)(DX >> 32), DZ32 = (unsigned)(DZ >> 32);
    const unsigned KX32 = (unsigned)((KX >> 32) + ((KX >> 31) & 1ull));
    const unsigned KZ32 = (unsigned)((KZ >> 32) + ((KZ >> 31) & 1ull));
    const float ikx = W.ikx, ikz = W.ikz, slo = W.slo, shi_last = W.shi_last, Ls = W.Ls, S = W.S;
    const float ikxh = ikx * 4294967296.f, ikzh = ikz * 4294967296.f;   // FP: 2^32 / K
    const float ikx32 = KX32 ? (float)(1.0 / (double)KX32) : 4.656613e-10f;   // 1 / K32 (K = 0: 2^-31)
    const float ikz32 = KZ32 ? (float)(1.0 / (double)KZ32) : 4.656613e-10f;
    unsigned o = W.o;
    const int sxo = W.sxo, pstep = W.pstep, k0 = W.k0, nk = W.nk, rowstep = W.rowstep;
    const int view = W.view, iu = W.iu, iv = W.iv;
    const int slot = (int)((blockIdx.x / (unsigned)L.n_chunks) % (unsigned)L.n_slots);

    const float wbp = W.wbp;
    double acc = 0.0;
    float acc32 = 0.f;
    float pv0 = 0.f, pv1 = 0.f, pv2 = 0.f, pl0 = 0.f, pl1 = 0.f, pl2 = 0.f;   // FP: previous slice
    bool pin = false;                                                          // ... and its range flag
    unsigned int nvis = 0;

    for (int pass = 0; pass < 2; ++pass) {
        const int jl = pass == 0 ? jlo_p : jlo_n, jh = pass == 0 ? jhi_p : jhi_n;
        if (jl > jh) continue;                                      // warp-uniform
        const int nsl = jh - jl + 1;
        const int kb = (pass == 0 ? pos : neg) ? k0 : INT_MAX;      // this lane's slices [kb, kb + nk]
        for (int kc = 0; kc < nsl; kc += 16) {     // FP: fp32 sums of 16 slices -> fp64
          const int ke = min(kc + 16, nsl);
#pragma unroll 4
          for (int k = kc; k < ke; ++k) {
            const int rel = k - kb;
            const bool in = (unsigned)rel <= (unsigned)nk;
            // crossing point u = D / K of each axis (round-to-nearest, <= 1.5 ulp) when its
            // plane distance borrows.  FP: the 32-bit walk (I2FP.U32 on the ALU pipe, no 64-bit
            // carries; |k| >= 2^-13 here, see lane_fine and walk3_setup); without a crossing u
            // only has to saturate: the three segments then share voxel o.  (PROJ3_FP32STEP=0:
            // the 64-bit walk with the high-word conversion, for A/B.)
#if PROJ3_FP32STEP
            float fx, fz;
            unsigned bx, bz;
            if (MODE == PROJ_FP) {
                fx = __uint2float_rn(DX32) * ikx32;
                bx = sub_borrow32(DX32, KX32);                      // ~0u on a plane crossing
                fz = __uint2float_rn(DZ32) * ikz32;
                bz = sub_borrow32(DZ32, KZ32);
            } else {
                fx = __ull2float_rn(DX) * ikx;
                bx = sub_borrow(DX, KX);
                fz = __ull2float_rn(DZ) * ikz;
                bz = sub_borrow(DZ, KZ);
            }
#else
            const float fx = MODE == PROJ_FP ? __uint2float_rn((unsigned)(DX >> 32)) * ikxh : __ull2float_rn(DX) * ikx;
            const unsigned bx = sub_borrow(DX, KX);                 // ~0u on a plane crossing
            const float fz = MODE == PROJ_FP ? __uint2float_rn((unsigned)(DZ >> 32)) * ikzh : __ull2float_rn(DZ) * ikz;
            const unsigned bz = sub_borrow(DZ, KZ);
#endif
            float l0, l1, l2, ux, uz;
            if (MODE == PROJ_COUNT) {
                // exact in-block segments: the slice clamped to [s_lo, s_hi] at the lane's
                // first / last slice (entry / exit through an x or z face or the far face)
                const float sl = rel == 0 ? slo : 0.f;
                const float sh = rel == nk ? shi_last : 1.f;
                ux = bx ? fx : 2.f;
                uz = bz ? fz : 2.f;
                const float m1 = fminf(ux, uz), m2 = fmaxf(ux, uz);
                const float c1 = fminf(fmaxf(m1, sl), sh), c2 = fminf(fmaxf(m2, sl), sh);
                l0 = c1 - sl;
                l1 = c2 - c1;
                l2 = sh - c2;
            } else {
                // FP / BP take the whole slice: where the ray enters or leaves inside a slice
                // (through an x or z face) the part outside the block lies in the cell just
                // beyond that face, i.e. in the padded copy's zero border (FP reads 0, BP's
                // reduction lands in the ignored border), so no entry/exit clamping
                // FP: without a crossing D >= K, so the saturated D / K is 1 up to rounding
                // (>= 1 - 2^-23) and the segments it separates share voxel o (no select
                // needed); BP keeps the select (its rare reductions are keyed on the borrows)
                ux = (MODE == PROJ_FP || bx) ? __saturatef(fx) : 1.f;
                uz = (MODE == PROJ_FP || bz) ? __saturatef(fz) : 1.f;
                const float m1 = fminf(ux, uz), m2 = fmaxf(ux, uz);
                l0 = m1;
                l1 = m2 - m1;
                l2 = 1.f - m2;
            }
            // bx, bz are 0 or ~0u: the steps as masks (ALU pipe; the FMA pipe carries the IMADs
            // of the address arithmetic: FP 97.0 -> 96.5 ms)
            const unsigned dox = bx & (unsigned)sxo, doz = bz & (unsigned)pstep;
            const unsigned o1 = o + (ux <= uz ? dox : doz);
            const unsigned o2 = o + dox + doz;
            const unsigned mor = bx | bz, mand = bx & bz;
            if (MODE == PROJ_FP) {
                // software pipeline: this slice's gathers are issued before the previous
                // slice's values are consumed (two slices of loads in flight per warp)
                float v0, v1, v2;
                gather3((unsigned)rel, (unsigned)nk, src + (int)o, src + (int)o1, src + (int)o2, v0, v1, v2);
                const float an = fmaf(pl0, pv0, fmaf(pl1, pv1, fmaf(pl2, pv2, acc32)));
                acc32 = pin ? an : acc32;            // the previous slice was in range
                pv0 = v0; pv1 = v1; pv2 = v2;
                pl0 = l0; pl1 = l1; pl2 = l2;
                pin = in;
            }
            if (is_bp(MODE))
                scatter3<MODE>(in, mor, mand, dst, (int)o, (int)o1, (int)o2, l0 * wbp, l1 * wbp, l2 * wbp, S);
            if (MODE == PROJ_COUNT) {
                const bool p1 = in && mor != 0u, p2 = in && mand != 0u;
                // a segment counts when longer than 1e-6 of the slice: exact ties (a ray through
                // a voxel edge) leave rounding slivers of ~1e-7 that the oracle's exact
                // arithmetic gives as 0 (its zero-length gaps are dropped, reading A18)
                nvis += (unsigned)(in && l0 > 1e-6f) + (unsigned)(p1 && l1 > 1e-6f) + (unsigned)(p2 && l2 > 1e-6f);
            }
            o = o2 + (unsigned)rowstep;
          }
          if (MODE == PROJ_FP) {
              acc += (double)acc32;
              acc32 = 0.f;
          }
        }
    }
    if (MODE == PROJ_FP && inrect) {
        if (pin) acc32 = fmaf(pl0, pv0, fmaf(pl1, pv1, fmaf(pl2, pv2, acc32)));
        acc += (double)acc32;
        acc *= (double)Ls;                  // main-axis units -> voxel lengths
        float* zp = zaddr(B, L.g, view, iu, iv);
        *zp = L.accumulate ? (*zp + (float)acc) : (float)acc;
    }
    if (MODE == PROJ_COUNT && L.visits) {
        unsigned int s = __reduce_add_sync(0xffffffffu, nvis);
        if ((threadIdx.x & 31) == 0 && s) atomicAdd(L.visits + (size_t)blockIdx.z * L.n_slots + slot, (unsigned long long)s);
    }
}

// Ones-pass: w[b][view][t] = sum over tile rays of chord(ray, box_b) = (A_t^{J_b} 1) summed.
__global__ void __launch_bounds__(256) k_im_weights(const ImLaunch I) {
    const int view = blockIdx.y;
    const long long per = (long long)I.g.nu * I.g.nv;
    const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const bool in = tid < per;
    const int iu = in ? (int)(tid % I.g.nu) : 0, iv = in ? (int)(tid / I.g.nu) : 0;
    int tu = 0, tv = 0;
    for (int q = 0; q < I.tiles_u; ++q)
        if (iu >= (int)((long long)q * I.g.nu / I.tiles_u)) tu = q;
    for (int q = 0; q < I.tiles_v; ++q)
        if (iv >= (int)((long long)q * I.g.nv / I.tiles_v)) tv = q;
    const int T = I.tiles_u * I.tiles_v, tile = tv * I.tiles_u + tu;
    double a[3], b[3], inv[3];
    make_ray(I.g, I.g.vecs + 12 * (size_t)view, iu, iv, a, b);
    const double blen = sqrt(b[0] * b[0] + b[1] * b[1] + b[2] * b[2]);
#pragma unroll
    for (int c = 0; c < 3; ++c) inv[c] = (b[c] != 0.0) ? 1.0 / b[c] : 0.0;
    const int key = in ? tile : -1;
    const bool uniform_tile = __reduce_min_sync(0xffffffffu, key < 0 ? INT_MAX : key) ==
                                  __reduce_max_sync(0xffffffffu, key) &&
                              __all_sync(0xffffffffu, in);
    for (int bb = 0; bb < I.n_blocks; ++bb) {
        const BlockDesc& B = I.blocks[bb];
        double amin, amax, c = 0.0;
        if (in && clip(a, b, inv, B.lo, B.hi, amin, amax)) c = (amax - amin) * blen;
        if (I.area) c = c > 1e-6 ? 1.0 : 0.0;   // IS_AREA: rays of the block's shadow (reading A9)
        double* dst = I.w + ((size_t)bb * I.g.n_views + view) * T;
        if (uniform_tile) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
            if ((threadIdx.x & 31) == 0) atomicAdd(dst + tile, c);
        } else if (in && c != 0.0) {
            atomicAdd(dst + tile, c);
        }
    }
}

}  // namespace

void launch_project(int mode, const ProjLaunch& L, cudaStream_t st) {
    if (L.n_slots == 0 || L.n_blocks == 0 || L.max_rect_rays == 0) return;
    static const int version = [] {
        const char* e = getenv("BSGD_PROJECTOR");
        return e ? atoi(e) : 3;
    }();
    const dim3 grid((unsigned)((long long)L.n_bands * L.n_slots * L.n_chunks), 1, (unsigned)L.n_blocks);
    if (grid.x == 0) return;
    if (version == 2) {   // v2 alone (A/B reference)
        if (mode == PROJ_FP) k_project2<PROJ_FP><<<grid, 256, 0, st>>>(L);
        else if (mode == PROJ_BP) k_project2<PROJ_BP><<<grid, 256, 0, st>>>(L);
        else if (mode == PROJ_BPD) k_project2<PROJ_BPD><<<grid, 256, 0, st>>>(L);
        else k_project2<PROJ_COUNT><<<grid, 256, 0, st>>>(L);
        BSGD_CUDA(cudaGetLastError());
        note_launch();
        return;
    }
    // v3 (default), then the v2 traversal for the warps v3 skipped (listed by v3, or the same
    // launch geometry and predicate when no list is given)
    if (L.v2_list) BSGD_CUDA(cudaMemsetAsync(L.v2_count, 0, sizeof(unsigned), st));
    if (mode == PROJ_FP) k_project3<PROJ_FP><<<grid, 256, 0, st>>>(L);
    else if (mode == PROJ_BP) k_project3<PROJ_BP><<<grid, 256, 0, st>>>(L);
    else if (mode == PROJ_BPD) k_project3<PROJ_BPD><<<grid, 256, 0, st>>>(L);
    else k_project3<PROJ_COUNT><<<grid, 256, 0, st>>>(L);
    BSGD_CUDA(cudaGetLastError());
    note_launch();
    if (L.v2_list) {   // only the listed warps
        const dim3 pg(148 * 4);
        if (mode == PROJ_FP) k_project2_list<PROJ_FP><<<pg, 256, 0, st>>>(L);
        else if (mode == PROJ_BP) k_project2_list<PROJ_BP><<<pg, 256, 0, st>>>(L);
        else if (mode == PROJ_BPD) k_project2_list<PROJ_BPD><<<pg, 256, 0, st>>>(L);
        else k_project2_list<PROJ_COUNT><<<pg, 256, 0, st>>>(L);
    } else if (mode == PROJ_FP) k_project2<PROJ_FP, true><<<grid, 256, 0, st>>>(L);
    else if (mode == PROJ_BP) k_project2<PROJ_BP, true><<<grid, 256, 0, st>>>(L);
    else if (mode == PROJ_BPD) k_project2<PROJ_BPD, true><<<grid, 256, 0, st>>>(L);
    else k_project2<PROJ_COUNT, true><<<grid, 256, 0, st>>>(L);
    BSGD_CUDA(cudaGetLastError());
    note_launch();
}

void launch_im_weights(const ImLaunch& I, cudaStream_t st) {
    long long per = (long long)I.g.nu * I.g.nv;
    dim3 grid((unsigned)((per + 255) / 256), (unsigned)I.g.n_views);
    k_im_weights<<<grid, 256, 0, st>>>(I);
    BSGD_CUDA(cudaGetLastError());
    note_launch();
}

}  // namespace bsgd
