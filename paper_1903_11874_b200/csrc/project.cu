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
// v3 main axis, chosen per WARP (majority of its rays; the lanes must share one layout for
// coalescing): fewer steep lanes than a per-view choice where the fan/cone spans 45 deg.
__device__ __forceinline__ bool warp_main_x(const double b[3], bool inrect) {
    const unsigned vx = __ballot_sync(0xffffffffu, inrect && fabs(b[0]) > fabs(b[1]));
    const unsigned n = __ballot_sync(0xffffffffu, inrect);
    return 2 * __popc(vx) > __popc(n);
}
// lane_steep evaluated in the v3 frame of a world-frame direction b
__device__ __forceinline__ bool lane_steep_v3(const double b[3], bool mainX) {
    const double f[3] = {mainX ? b[1] : b[0], mainX ? b[0] : b[1], b[2]};
    return lane_steep(f);
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
template <int MODE, bool STEEP_ONLY = false>
__global__ void __launch_bounds__(256, 4) k_project2(const ProjLaunch L) {
    // band-major CTA order: blockIdx.x = (band * n_slots + slot) * n_chunks + chunk, so the
    // CTAs resident at any time cover the same detector-row band of consecutive views
    // (rays of one band cross the same z-range of the volume -> L2 reuse across views).
    const BlockDesc& B = L.blocks[blockIdx.z];
    unsigned bid = blockIdx.x;
    const int chunk = (int)(bid % (unsigned)L.n_chunks);
    bid /= (unsigned)L.n_chunks;
    const int slot = (int)(bid % (unsigned)L.n_slots);
    const int band = B.band_lo + (int)(bid / (unsigned)L.n_slots);
    const int4 rc = L.rects[(size_t)blockIdx.z * L.n_slots + slot];
    const int r0 = max(rc.z, band * L.rows_per_band), r1 = min(rc.w, band * L.rows_per_band + L.rows_per_band);
    const int w = rc.y - rc.x;
    if (r0 >= r1 || w <= 0) return;
    const int nrect = (r1 - r0) * w;
    const int base = chunk * (int)blockDim.x;
    if (base >= nrect) return;                       // uniform over the CTA
    const int tid = base + (int)threadIdx.x;
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
    if (STEEP_ONLY) steep3 = lane_steep_v3(b, warp_main_x(b, inrect));
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
        if ((threadIdx.x & 31) == 0 && s) atomicAdd(L.visits + (size_t)blockIdx.z * L.n_slots + slot, (unsigned long long)s);
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

// The two gathers of a slice without a z crossing (v4 fast path), predicated like gather3.
__device__ __forceinline__ void gather2(unsigned rel, unsigned nk, const float* p0, const float* p1, float& v0,
                                        float& v1) {
    asm("{\n\t.reg .pred a;\n\t"
        "setp.le.u32 a, %2, %3;\n\t"
        "@a ld.global.nc.f32 %0, [%4];\n\t"
        "@a ld.global.nc.f32 %1, [%5];\n\t}"
        : "=f"(v0), "=f"(v1)
        : "r"(rel), "r"(nk), "l"(p0), "l"(p1));
}

// D -= K on the 64-bit plane distance; returns ~0u when it borrows (a plane is crossed).
__device__ __forceinline__ unsigned sub_borrow(unsigned long long& D, unsigned long long K) {
    unsigned m;
    asm("sub.cc.u64 %0, %0, %2;\n\tsubc.u32 %1, 0, 0;" : "+l"(D), "=r"(m) : "l"(K));
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

template <int MODE, bool FASTZ = false, int PFD = 0>
__global__ void __launch_bounds__(256, 4) k_project3(const ProjLaunch L) {
    const BlockDesc& B = L.blocks[blockIdx.z];
    unsigned bid = blockIdx.x;
    const int chunk = (int)(bid % (unsigned)L.n_chunks);
    bid /= (unsigned)L.n_chunks;
    const int slot = (int)(bid % (unsigned)L.n_slots);
    const int band = B.band_lo + (int)(bid / (unsigned)L.n_slots);
    const int4 rc = L.rects[(size_t)blockIdx.z * L.n_slots + slot];
    const int r0 = max(rc.z, band * L.rows_per_band), r1 = min(rc.w, band * L.rows_per_band + L.rows_per_band);
    const int w = rc.y - rc.x;
    if (r0 >= r1 || w <= 0) return;
    const int nrect = (r1 - r0) * w;
    const int base = chunk * (int)blockDim.x;
    if (base >= nrect) return;                       // uniform over the CTA
    const int tid = base + (int)threadIdx.x;
    const bool inrect = tid < nrect;
    const int iu = rc.x + (inrect ? tid % w : 0);
    const int iv = r0 + (inrect ? tid / w : 0);
    const int view = L.views[slot];
    const double* vec = L.g.vecs + 12 * (size_t)view;

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
    if (__any_sync(0xffffffffu, hit && (lane_steep(b) || amin == 0.0 || amax == 1.0))) return;
    const double blen = sqrt(b[0] * b[0] + b[1] * b[1] + b[2] * b[2]);
    float rs = 0.f;
    const float S = MODE == PROJ_BPD ? *L.det_scale : 0.f;
    if (is_bp(MODE)) {
        if (inrect) rs = L.scale * L.rproj[((long long)view * L.g.nv + iv) * L.g.nu + iu];
        hit = hit && (rs != 0.f);
    }
    const float* __restrict__ src = mainX ? B.xT : B.xN;
    float* dst = mainX ? B.outT : B.outN;

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
    const bool pos = hit && sy > 0, neg = hit && sy < 0;
    const int jlo_p = __reduce_min_sync(0xffffffffu, pos ? j0 : INT_MAX);
    const int jhi_p = __reduce_max_sync(0xffffffffu, pos ? j1 : INT_MIN);
    const int jlo_n = __reduce_min_sync(0xffffffffu, neg ? j1 : INT_MAX);
    const int jhi_n = __reduce_max_sync(0xffffffffu, neg ? j0 : INT_MIN);
    unsigned long long DX = 0ull, DZ = 0ull, KX = 0ull, KZ = 0ull;
    float ikx = 0.f, ikz = 0.f, slo = 0.f, shi_last = 1.f, Ls = 0.f;
    unsigned o = 0u;   // wraps freely outside the lane's range; exact inside it
    int sxo = 1, pstep = plane, k0 = INT_MAX, nk = 0;
    if (hit) {
        const int jstart = sy > 0 ? jlo_p : jhi_n;
        k0 = sy * (j0 - jstart);
        nk = sy * (j1 - j0);
        const double ys = (double)(sy > 0 ? jstart : jstart + 1);   // entry plane of jstart
        const double yin0 = (double)(sy > 0 ? j0 : j0 + 1);         // entry plane of slice j0
        const double yin1 = (double)(sy > 0 ? j1 : j1 + 1);
        const double ap = (ys - a[1]) * inv[1];                     // alpha at plane ys
        const double kx = b[0] * ainv1, kz = b[2] * ainv1;          // per unit of main-axis travel
        const bool mx = kx < 0.0, mz = kz < 0.0;
        const double xr = a[0] + ap * b[0] - lo[0], zr = a[2] + ap * b[2] - lo[2];
        const double xm = mx ? -xr : xr, zm = mz ? -zr : zr;
        KX = __double2ull_rn(fabs(kx) * TWO64);
        KZ = __double2ull_rn(fabs(kz) * TWO64);
        int cxm, czm;
        DX = plane_dist(xm, KX, cxm);
        DZ = plane_dist(zm, KZ, czm);
        const int ix = mx ? -cxm - 1 : cxm;                         // frame cell relative to lo
        const int iz = mz ? -czm - 1 : czm;
        // K = 0 (ray parallel to that axis' planes): an infinite distance, never crossed
        if (!KX) DX = ~0ull;
        if (!KZ) DZ = ~0ull;
        ikx = KX ? (float)(1.0 / (double)KX) : 0.f;
        ikz = KZ ? (float)(1.0 / (double)KZ) : 0.f;
        sxo = mx ? -1 : 1;
        pstep = mz ? -plane : plane;
        o = (unsigned)iz * (unsigned)plane + (unsigned)(jstart - lo[1]) * (unsigned)bdx + (unsigned)ix;
        slo = (float)fmin(fmax((amin - (yin0 - a[1]) * inv[1]) * fabs(b[1]), 0.0), 1.0);
        shi_last = (float)fmin(fmax((amax - (yin1 - a[1]) * inv[1]) * fabs(b[1]), 0.0), 1.0);
        if (j1 == j0) shi_last = fmaxf(shi_last, slo);
        Ls = (float)(blen * ainv1);
    }
    const int rowstep = sy * bdx;
    const unsigned nsxo = (unsigned)(-sxo), npstep = (unsigned)(-pstep);
    const float wbp = Ls * rs;   // BP weight per unit of main-axis travel
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
        if (FASTZ) {
            // v4: z-plane crossings are rare (|kz| <= 0.08 in the cone configs) and coherent
            // across a warp (its lanes trace adjacent pixels of ONE detector row, at nearly the
            // same height), so a slice in which no in-range lane crosses a z plane takes a
            // two-segment body (one gather / reduction less, no z crossing point, no ordering
            // of two crossings); the general three-segment body (the v3 arithmetic) runs only
            // when some lane does (a warp-uniform branch).  FP keeps the fp32 partial sum of
            // 16 slices, then adds it into the fp64 accumulator (an outer loop, not a select).
            const unsigned sxu = (unsigned)sxo;
            for (int kc = 0; kc < nsl; kc += 16) {
                const int kend = min(kc + 16, nsl);
                for (int k = kc; k < kend; ++k) {
                    const unsigned rel = (unsigned)(k - kb);
                    const bool in = rel <= (unsigned)nk;
                    // D >= K without a crossing, so the saturated D / K is 1 up to rounding
                    // (>= 1 - 2^-23); the FP's two segments then share one voxel (o1 = o)
                    const float fx = __saturatef(__ull2float_rn(DX) * ikx);
                    const unsigned bx = sub_borrow(DX, KX);
                    const unsigned bz = sub_borrow(DZ, KZ);
                    const unsigned dox = bx & sxu, doz = bz & (unsigned)pstep;
                    const unsigned o1 = o + dox;
                    if (MODE == PROJ_FP && true) {   // the previous slice's gathers
                        const float an = fmaf(pl0, pv0, fmaf(pl1, pv1, acc32));
                        acc32 = pin ? an : acc32;
                    }
                    if (__any_sync(0xffffffffu, in && bz != 0u)) {
                        const float ux = bx ? fx : 1.f;
                        const float uz = bz ? __saturatef(__ull2float_rn(DZ + KZ) * ikz) : 1.f;
                        const float m1 = fminf(ux, uz), m2 = fmaxf(ux, uz);
                        const float l0 = m1, l1 = m2 - m1, l2 = 1.f - m2;
                        const unsigned oa = ux <= uz ? o1 : o + doz;
                        const unsigned o2 = o1 + doz;
                        if (MODE == PROJ_FP) {
                            float v0, v1, v2;
                            gather3(rel, (unsigned)nk, src + (int)o, src + (int)oa, src + (int)o2, v0, v1, v2);
                            if (true) {
                                if (in) acc32 = fmaf(l2, v2, acc32);   // rare: consumed at once
                                pv0 = v0; pv1 = v1; pl0 = l0; pl1 = l1;
                            } else if (in) {
                                acc32 = fmaf(l0, v0, fmaf(l1, v1, fmaf(l2, v2, acc32)));
                            }
                        }
                        if (is_bp(MODE))
                            scatter3<MODE>(in, bx | bz, bx & bz, dst, (int)o, (int)oa, (int)o2, l0 * wbp, l1 * wbp,
                                           l2 * wbp, S);
                    } else {
                        if (MODE == PROJ_FP) {
                            float v0, v1;
                            gather2(rel, (unsigned)nk, src + (int)o, src + (int)o1, v0, v1);
                            if (true) {
                                pv0 = v0; pv1 = v1; pl0 = fx; pl1 = 1.f - fx;
                            } else if (in) {
                                acc32 = fmaf(fx, v0, fmaf(1.f - fx, v1, acc32));
                            }
                        }
                        if (is_bp(MODE) && in) {
                            const float l0 = bx ? fx : 1.f;
                            red_acc<MODE>(dst, (int)o, l0 * wbp, S);
                            if (bx) red_acc<MODE>(dst, (int)o1, (1.f - l0) * wbp, S);
                        }
                    }
                    if (MODE == PROJ_FP && true) pin = in;
                    o = o1 + doz + (unsigned)rowstep;
                }
                if (MODE == PROJ_FP) {
                    acc += (double)acc32;
                    acc32 = 0.f;
                }
            }
            continue;
        }
        for (int k = 0; k < nsl; ++k) {
            const int rel = k - kb;
            const bool in = (unsigned)rel <= (unsigned)nk;
            // crossing point u = D / K of each axis (round-to-nearest, <= 1.5 ulp) when its
            // plane distance borrows
            const float fx = __ull2float_rn(DX) * ikx;
            const unsigned bx = sub_borrow(DX, KX);                 // ~0u on a plane crossing
            const float fz = __ull2float_rn(DZ) * ikz;
            const unsigned bz = sub_borrow(DZ, KZ);
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
                ux = bx ? __saturatef(fx) : 1.f;
                uz = bz ? __saturatef(fz) : 1.f;
                const float m1 = fminf(ux, uz), m2 = fmaxf(ux, uz);
                l0 = m1;
                l1 = m2 - m1;
                l2 = 1.f - m2;
            }
            // bx, bz are 0 or ~0u (= -1): the steps as multiply-adds (FMA pipe)
            const unsigned dox = bx * nsxo, doz = bz * npstep;
            const unsigned o1 = o + (ux <= uz ? dox : doz);
            const unsigned o2 = bz * npstep + (bx * nsxo + o);
            const unsigned mor = bx | bz, mand = bx & bz;
            if (MODE == PROJ_FP) {
                // software pipeline: this slice's gathers are issued before the previous
                // slice's values are consumed (two slices of loads in flight per warp)
                float v0, v1, v2;
                gather3((unsigned)rel, (unsigned)nk, src + (int)o, src + (int)o1, src + (int)o2, v0, v1, v2);
                // L1 prefetch of the line this lane's ray reaches PFD slices ahead (x / z drift
                // ignored: the warp's lanes cover that line's neighbours anyway), so those
                // gathers hit L1 instead of waiting on L2
                if (PFD > 0 && (unsigned)(rel + PFD) <= (unsigned)nk)
                    asm volatile("prefetch.global.L1 [%0];" ::"l"(src + (int)(o + (unsigned)(PFD * rowstep))));
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
            if (MODE == PROJ_FP && (k & 15) == 15) {               // warp-uniform
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

// ---------------------------------------------------------------------------------------
// v5: two detector rows per thread.  When the detector's v step has no x / y component
// (circular orbits, reading A19: v = pitch_v (0, 0, 1)), the rays of one detector column
// in rows iv and iv + 1 have the same source, the same in-plane direction (b_x, b_y) and so
// the same in-plane path: the same main axis, slice direction, x-plane crossings and x cell
// at every slice.  One thread carries both rays: the x stepping (64-bit plane distance,
// crossing point, x step) is computed once per slice for the pair, the z stepping and the
// three-segment body stay per ray (the v3 arithmetic, bit for bit).  Each ray issues its
// own gathers, so a warp keeps twice the loads in flight per slice.
// The warp / skip decomposition is v3's per detector row (32 adjacent columns of one row;
// the host uses v5 only when no rect width straddles warps), so the v2 companion launch
// with the one-ray mapping takes exactly the 32-ray row groups v5 leaves.
template <int MODE>
__global__ void __launch_bounds__(256, 3) k_project5(const ProjLaunch L) {
    const BlockDesc& B = L.blocks[blockIdx.z];
    unsigned bid = blockIdx.x;
    const int chunk = (int)(bid % (unsigned)L.pair_chunks);
    bid /= (unsigned)L.pair_chunks;
    const int slot = (int)(bid % (unsigned)L.n_slots);
    const int band = B.band_lo + (int)(bid / (unsigned)L.n_slots);
    const int4 rc = L.rects[(size_t)blockIdx.z * L.n_slots + slot];
    const int r0 = max(rc.z, band * L.rows_per_band), r1 = min(rc.w, band * L.rows_per_band + L.rows_per_band);
    const int w = rc.y - rc.x;
    if (r0 >= r1 || w <= 0) return;
    const int npairs = (r1 - r0 + 1) / 2;
    const int nrect = npairs * w;
    const int base = chunk * (int)blockDim.x;
    if (base >= nrect) return;                       // uniform over the CTA
    const int tid = base + (int)threadIdx.x;
    const bool inrect = tid < nrect;
    const int iu = rc.x + (inrect ? tid % w : 0);
    const int ivA = r0 + 2 * (inrect ? tid / w : 0);
    const bool hasB = ivA + 1 < r1;
    const int view = L.views[slot];
    const double* vec = L.g.vecs + 12 * (size_t)view;

    double a[2][3], b[2][3];
    make_ray(L.g, vec, iu, ivA, a[0], b[0]);
    make_ray(L.g, vec, iu, hasB ? ivA + 1 : ivA, a[1], b[1]);
    const bool mainX = warp_main_x(b[0], inrect);    // = v3's choice for either row's warp
    int lo[3] = {B.lo[0], B.lo[1], B.lo[2]}, hi[3] = {B.hi[0], B.hi[1], B.hi[2]};
    if (mainX) {
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            double t = a[r][0]; a[r][0] = a[r][1]; a[r][1] = t;
            t = b[r][0]; b[r][0] = b[r][1]; b[r][1] = t;
        }
        int q = lo[0]; lo[0] = lo[1]; lo[1] = q;
        q = hi[0]; hi[0] = hi[1]; hi[1] = q;
    }
    double inv[2][3], amin[2], amax[2];
    bool hit[2], take[2];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
#pragma unroll
        for (int c = 0; c < 3; ++c) inv[r][c] = (b[r][c] != 0.0) ? 1.0 / b[r][c] : 0.0;
        const bool valid = inrect && (r == 0 || hasB);
        hit[r] = valid && clip(a[r], b[r], inv[r], lo, hi, amin[r], amax[r]);
        // v3's skip rule per 32-ray row group: the v2 companion takes the group
        const bool skip = __any_sync(0xffffffffu, hit[r] && (lane_steep(b[r]) || amin[r] == 0.0 || amax[r] == 1.0));
        take[r] = valid && !skip;
        hit[r] = hit[r] && !skip;
    }
    if (!__any_sync(0xffffffffu, take[0] || take[1])) return;
    float rs[2] = {0.f, 0.f};
    const float S = MODE == PROJ_BPD ? *L.det_scale : 0.f;
    if (is_bp(MODE)) {
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            if (take[r]) rs[r] = L.scale * L.rproj[((long long)view * L.g.nv + ivA + r) * L.g.nu + iu];
            hit[r] = hit[r] && (rs[r] != 0.f);
        }
    }
    const float* __restrict__ src = mainX ? B.xT : B.xN;
    float* dst = mainX ? B.outT : B.outN;
    const int bdx = mainX ? B.rowT : B.rowN;
    const int plane = mainX ? B.planeT : B.planeN;
    // the in-plane direction, and so sy, |1/b_1| and the x stepping, are the pair's
    const int sy = (b[0][1] > 0.0) ? 1 : -1;
    const double ainv1 = fabs(inv[0][1]);
    const double TWO64 = 18446744073709551616.0;
    int j0[2] = {0, 0}, j1[2] = {-1, -1};
#pragma unroll
    for (int r = 0; r < 2; ++r)
        if (hit[r]) {
            j0[r] = cell_enter(a[r][1] + amin[r] * b[r][1], sy, lo[1], hi[1]);
            j1[r] = cell_exit(a[r][1] + amax[r] * b[r][1], sy, lo[1], hi[1]);
            if (sy * (j1[r] - j0[r]) < 0) j1[r] = j0[r];
        }
    const bool pos0 = hit[0] && sy > 0, pos1 = hit[1] && sy > 0;
    const bool neg0 = hit[0] && sy < 0, neg1 = hit[1] && sy < 0;
    const int jlo_p = __reduce_min_sync(0xffffffffu, min(pos0 ? j0[0] : INT_MAX, pos1 ? j0[1] : INT_MAX));
    const int jhi_p = __reduce_max_sync(0xffffffffu, max(pos0 ? j1[0] : INT_MIN, pos1 ? j1[1] : INT_MIN));
    const int jlo_n = __reduce_min_sync(0xffffffffu, min(neg0 ? j1[0] : INT_MAX, neg1 ? j1[1] : INT_MAX));
    const int jhi_n = __reduce_max_sync(0xffffffffu, max(neg0 ? j0[0] : INT_MIN, neg1 ? j0[1] : INT_MIN));
    const bool anyhit = hit[0] || hit[1];
    const int jstart = sy > 0 ? jlo_p : jhi_n;
    // shared x stepping, set up at jstart's entry plane from ray 0 (ray 1 is identical in x)
    unsigned long long DX = 0ull, KX = 0ull;
    float ikx = 0.f;
    int sxo = 1, ix = 0;
    if (anyhit) {
        const double ys = (double)(sy > 0 ? jstart : jstart + 1);
        const double ap = (ys - a[0][1]) * inv[0][1];
        const double kx = b[0][0] * ainv1;
        const bool mx = kx < 0.0;
        const double xr = a[0][0] + ap * b[0][0] - lo[0];
        KX = __double2ull_rn(fabs(kx) * TWO64);
        int cxm;
        DX = plane_dist(mx ? -xr : xr, KX, cxm);
        ix = mx ? -cxm - 1 : cxm;
        if (!KX) DX = ~0ull;
        ikx = KX ? (float)(1.0 / (double)KX) : 0.f;
        sxo = mx ? -1 : 1;
    }
    unsigned long long DZ[2] = {0ull, 0ull}, KZ[2] = {0ull, 0ull};
    float ikz[2] = {0.f, 0.f}, Ls[2] = {0.f, 0.f};
    unsigned o[2] = {0u, 0u};
    int pstep[2] = {plane, plane}, k0[2] = {INT_MAX, INT_MAX}, nk[2] = {0, 0};
#pragma unroll
    for (int r = 0; r < 2; ++r)
        if (hit[r]) {
            k0[r] = sy * (j0[r] - jstart);
            nk[r] = sy * (j1[r] - j0[r]);
            const double ys = (double)(sy > 0 ? jstart : jstart + 1);
            const double ap = (ys - a[r][1]) * inv[r][1];
            const double kz = b[r][2] * ainv1;
            const bool mz = kz < 0.0;
            const double zr = a[r][2] + ap * b[r][2] - lo[2];
            KZ[r] = __double2ull_rn(fabs(kz) * TWO64);
            int czm;
            DZ[r] = plane_dist(mz ? -zr : zr, KZ[r], czm);
            const int iz = mz ? -czm - 1 : czm;
            if (!KZ[r]) DZ[r] = ~0ull;
            ikz[r] = KZ[r] ? (float)(1.0 / (double)KZ[r]) : 0.f;
            pstep[r] = mz ? -plane : plane;
            o[r] = (unsigned)iz * (unsigned)plane + (unsigned)(jstart - lo[1]) * (unsigned)bdx + (unsigned)ix;
            const double blen = sqrt(b[r][0] * b[r][0] + b[r][1] * b[r][1] + b[r][2] * b[r][2]);
            Ls[r] = (float)(blen * ainv1);
        }
    const int rowstep = sy * bdx;
    const unsigned nsxo = (unsigned)(-sxo);
    const unsigned npstep[2] = {(unsigned)(-pstep[0]), (unsigned)(-pstep[1])};
    const float wbp[2] = {Ls[0] * rs[0], Ls[1] * rs[1]};
    double acc[2] = {0.0, 0.0};
    float acc32[2] = {0.f, 0.f};
    float pv[2][3] = {{0.f, 0.f, 0.f}, {0.f, 0.f, 0.f}}, pl[2][3] = {{0.f, 0.f, 0.f}, {0.f, 0.f, 0.f}};
    bool pin[2] = {false, false};
    const int jl = sy > 0 ? jlo_p : jlo_n, jh = sy > 0 ? jhi_p : jhi_n;
    // (one direction group per warp: sy is the pair's, and a warp whose lanes disagree on sy
    // walks each group in its own pass, as in v3)
    for (int pass = 0; pass < 2; ++pass) {
        const int pjl = pass == 0 ? jlo_p : jlo_n, pjh = pass == 0 ? jhi_p : jhi_n;
        if (pjl > pjh) continue;                                    // warp-uniform
        const int nsl = pjh - pjl + 1;
        const bool mine = pass == 0 ? sy > 0 : sy < 0;
        const int kb0 = (mine && hit[0]) ? k0[0] : INT_MAX, kb1 = (mine && hit[1]) ? k0[1] : INT_MAX;
        for (int k = 0; k < nsl; ++k) {
            const float fx = __ull2float_rn(DX) * ikx;
            const unsigned bx = sub_borrow(DX, KX);
            const float ux = bx ? __saturatef(fx) : 1.f;
            const unsigned dox = bx * nsxo;
#pragma unroll
            for (int r = 0; r < 2; ++r) {
                const int rel = k - (r == 0 ? kb0 : kb1);
                const bool in = (unsigned)rel <= (unsigned)nk[r];
                const float fz = __ull2float_rn(DZ[r]) * ikz[r];
                const unsigned bz = sub_borrow(DZ[r], KZ[r]);
                const float uz = bz ? __saturatef(fz) : 1.f;
                const float m1 = fminf(ux, uz), m2 = fmaxf(ux, uz);
                const float l0 = m1, l1 = m2 - m1, l2 = 1.f - m2;
                const unsigned doz = bz * npstep[r];
                const unsigned o1 = o[r] + (ux <= uz ? dox : doz);
                const unsigned o2 = doz + (dox + o[r]);
                if (MODE == PROJ_FP) {
                    float v0, v1, v2;
                    gather3((unsigned)rel, (unsigned)nk[r], src + (int)o[r], src + (int)o1, src + (int)o2, v0, v1, v2);
                    const float an = fmaf(pl[r][0], pv[r][0], fmaf(pl[r][1], pv[r][1], fmaf(pl[r][2], pv[r][2], acc32[r])));
                    acc32[r] = pin[r] ? an : acc32[r];
                    pv[r][0] = v0; pv[r][1] = v1; pv[r][2] = v2;
                    pl[r][0] = l0; pl[r][1] = l1; pl[r][2] = l2;
                    pin[r] = in;
                }
                if (is_bp(MODE))
                    scatter3<MODE>(in, bx | bz, bx & bz, dst, (int)o[r], (int)o1, (int)o2, l0 * wbp[r], l1 * wbp[r],
                                   l2 * wbp[r], S);
                o[r] = o2 + (unsigned)rowstep;
            }
            if (MODE == PROJ_FP && (k & 15) == 15) {                // warp-uniform
#pragma unroll
                for (int r = 0; r < 2; ++r) {
                    acc[r] += (double)acc32[r];
                    acc32[r] = 0.f;
                }
            }
        }
    }
    (void)jl; (void)jh;
    if (MODE == PROJ_FP) {
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            if (!take[r]) continue;
            if (pin[r]) acc32[r] = fmaf(pl[r][0], pv[r][0], fmaf(pl[r][1], pv[r][1], fmaf(pl[r][2], pv[r][2], acc32[r])));
            double v = (acc[r] + (double)acc32[r]) * (double)Ls[r];
            float* zp = zaddr(B, L.g, view, iu, ivA + r);
            *zp = L.accumulate ? (*zp + (float)v) : (float)v;
        }
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
        return e ? atoi(e) : 5;
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
    // v4 (default): the v3 traversal with the two-segment fast path for slices without a z
    // crossing (FASTZ); v3 (BSGD_PROJECTOR=3): the three-segment body throughout.  Then the
    // v2 traversal for the warps either skipped (same launch geometry, same predicate).
    // The COUNT traversal (visit table) always takes the v3 body (exact clamps).
    if (version >= 5 && L.pair_chunks > 0 && mode != PROJ_COUNT) {
        const dim3 g5((unsigned)((long long)L.n_bands * L.n_slots * L.pair_chunks), 1, (unsigned)L.n_blocks);
        if (mode == PROJ_FP) k_project5<PROJ_FP><<<g5, 256, 0, st>>>(L);
        else if (mode == PROJ_BP) k_project5<PROJ_BP><<<g5, 256, 0, st>>>(L);
        else k_project5<PROJ_BPD><<<g5, 256, 0, st>>>(L);
    } else if (version >= 4 && mode != PROJ_COUNT) {
        static const int pfd = [] {
            const char* e = getenv("BSGD_FP_PREFETCH");
            return e ? atoi(e) : 0;
        }();
        if (mode == PROJ_FP && pfd == 4) k_project3<PROJ_FP, false, 4><<<grid, 256, 0, st>>>(L);
        else if (mode == PROJ_FP && pfd == 8) k_project3<PROJ_FP, false, 8><<<grid, 256, 0, st>>>(L);
        else if (mode == PROJ_FP && pfd == 16) k_project3<PROJ_FP, false, 16><<<grid, 256, 0, st>>>(L);
        else if (mode == PROJ_FP && pfd == -1) k_project3<PROJ_FP, true><<<grid, 256, 0, st>>>(L);
        else if (mode == PROJ_FP) k_project3<PROJ_FP><<<grid, 256, 0, st>>>(L);
        else if (mode == PROJ_BP) k_project3<PROJ_BP, true><<<grid, 256, 0, st>>>(L);
        else k_project3<PROJ_BPD, true><<<grid, 256, 0, st>>>(L);
    } else {
        if (mode == PROJ_FP) k_project3<PROJ_FP><<<grid, 256, 0, st>>>(L);
        else if (mode == PROJ_BP) k_project3<PROJ_BP><<<grid, 256, 0, st>>>(L);
        else if (mode == PROJ_BPD) k_project3<PROJ_BPD><<<grid, 256, 0, st>>>(L);
        else k_project3<PROJ_COUNT><<<grid, 256, 0, st>>>(L);
    }
    BSGD_CUDA(cudaGetLastError());
    note_launch();
    if (mode == PROJ_FP) k_project2<PROJ_FP, true><<<grid, 256, 0, st>>>(L);
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
