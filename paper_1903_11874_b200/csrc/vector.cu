// HBM-streaming kernels of the hot path:
//  * k_block_update: g_hat / g / x step of Algo 1 lines 11-14
//    fused with the combination of the two BP accumulators (normal + transposed
//    layout) and the refresh of the transposed image copy used by the FP;
//  * k_residual: r_I = y_I - sum_j z^j_I (Algo 1 line 7) with the
//    per-row-block ||r_I||^2 (fp64) that Algo 3 and the log need;
//  * small reductions (EUD of Algo 3, dot products, RMSE) and the FGP TV prox
//    stencil of Algo 4 line 16 (Eq. 6 backward differences).
#include <algorithm>
#include <cstdlib>

#include <nccl.h>
#include <nccl_device.h>

#include "internal.h"

namespace bsgd {

namespace {

__device__ __forceinline__ double block_sum(double v) {
    __shared__ double red[32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    __syncthreads();
    if (lane == 0) red[wid] = v;
    __syncthreads();
    const int nw = (blockDim.x + 31) >> 5;
    v = (threadIdx.x < nw) ? red[threadIdx.x] : 0.0;
    if (wid == 0) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    }
    return v;   // valid in thread 0
}

// Vectorised variant for block dims that are multiples of 32: thread (q, r) of an
// 8 x 32 CTA owns the float4 x = x0+4q..+3 at y = y0+r of the normal layout and the
// float4 y = y0+4q..+3 at x = x0+r of the transposed layout; both 32x33 shared-memory
// transposes are bank-conflict free.  All loads are issued before any store.
template <int MODE>
__global__ void __launch_bounds__(256) k_block_update4(const UpdLaunch U) {
    __shared__ float tT[32][33];
    __shared__ float tX[32][33];
    const int bdx = U.bd[0], bdy = U.bd[1];
    const int x0 = blockIdx.x * 32, y0 = blockIdx.y * 32;
    const long long zoff = (long long)blockIdx.z * bdx * bdy;
    const int q = threadIdx.x, r = threadIdx.y;
    constexpr bool use_acc = MODE != UPD_XT;
    const bool final_ = U.final_ != 0;
    const bool writes_x = (MODE == UPD_XT) || ((MODE == UPD_BSGD || MODE == UPD_SGD) && final_);
    const bool needs_x = (MODE == UPD_BSGD && final_) || MODE == UPD_SGD || MODE == UPD_XT;
    const long long in_ = zoff + (long long)(y0 + r) * bdx + x0 + 4 * q;     // normal layout
    // the padded copies (accN / xN normal, accT / xT transposed; see BlockDesc)
    const long long inP = (long long)blockIdx.z * U.planeN + (long long)(y0 + r) * U.rowN + x0 + 4 * q;
    const long long itP = (long long)blockIdx.z * U.planeT + (long long)(x0 + r) * U.rowT + y0 + 4 * q;
    const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
    float4 vT = z4, vN = z4, vgh = z4, vg = z4, vx = z4, vo = z4;
    if (use_acc) {
        vT = *reinterpret_cast<const float4*>(U.accT + itP);
        vN = *reinterpret_cast<const float4*>(U.accN + inP);
    }
    if (MODE == UPD_BSGD) {
        vgh = *reinterpret_cast<const float4*>(U.ghat + in_);
        vg = *reinterpret_cast<const float4*>(U.g + in_);
    }
    if (needs_x) vx = *reinterpret_cast<const float4*>(U.x + in_);
    if (MODE == UPD_OUT && U.accumulate) vo = *reinterpret_cast<const float4*>(U.out + in_);
    if (use_acc) {
        tT[r][4 * q + 0] = vT.x; tT[r][4 * q + 1] = vT.y; tT[r][4 * q + 2] = vT.z; tT[r][4 * q + 3] = vT.w;
        *reinterpret_cast<float4*>(U.accT + itP) = z4;
        *reinterpret_cast<float4*>(U.accN + inP) = z4;
    }
    __syncthreads();
    float nv[4] = {vN.x, vN.y, vN.z, vN.w};
    if (use_acc) {
#pragma unroll
        for (int e = 0; e < 4; ++e) nv[e] += tT[4 * q + e][r];
    }
    const float gh[4] = {vgh.x, vgh.y, vgh.z, vgh.w}, gg[4] = {vg.x, vg.y, vg.z, vg.w};
    const float xx[4] = {vx.x, vx.y, vx.z, vx.w}, oo[4] = {vo.x, vo.y, vo.z, vo.w};
    float ng[4], nx[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        if (MODE == UPD_BSGD) {
            ng[e] = gg[e] + (nv[e] - gh[e]);
            nx[e] = final_ ? xx[e] + U.mu * ng[e] : 0.f;
        } else if (MODE == UPD_SGD) {
            ng[e] = nv[e];
            nx[e] = xx[e] + U.mu * nv[e];
        } else if (MODE == UPD_OUT) {
            ng[e] = oo[e] + nv[e];
            nx[e] = 0.f;
        } else {
            ng[e] = 0.f;
            nx[e] = xx[e];
        }
        tX[4 * q + e][r] = nx[e];
    }
    if (MODE == UPD_BSGD) {
        *reinterpret_cast<float4*>(U.ghat + in_) = make_float4(nv[0], nv[1], nv[2], nv[3]);
        *reinterpret_cast<float4*>(U.g + in_) = make_float4(ng[0], ng[1], ng[2], ng[3]);
        if (final_) *reinterpret_cast<float4*>(U.x + in_) = make_float4(nx[0], nx[1], nx[2], nx[3]);
    } else if (MODE == UPD_SGD) {
        *reinterpret_cast<float4*>(U.g + in_) = make_float4(ng[0], ng[1], ng[2], ng[3]);
        *reinterpret_cast<float4*>(U.x + in_) = make_float4(nx[0], nx[1], nx[2], nx[3]);
    } else if (MODE == UPD_OUT) {
        *reinterpret_cast<float4*>(U.out + in_) = make_float4(ng[0], ng[1], ng[2], ng[3]);
    }
    if (!writes_x) return;
    if (U.xN) *reinterpret_cast<float4*>(U.xN + inP) = make_float4(nx[0], nx[1], nx[2], nx[3]);
    __syncthreads();
    *reinterpret_cast<float4*>(U.xT + itP) =
        make_float4(tX[r][4 * q + 0], tX[r][4 * q + 1], tX[r][4 * q + 2], tX[r][4 * q + 3]);
}

// One 32x32 tile of one z-plane per CTA (32 x 8 threads, 4 elements each).  All global
// loads of the tile are issued before any store (the arrays are distinct; the
// compiler cannot prove it, so the code makes the order explicit) -> 5 loads in
// flight per element instead of a dependent load/store chain.
template <int MODE>
__global__ void __launch_bounds__(256) k_block_update(const UpdLaunch U) {
    __shared__ float tT[32][33];
    __shared__ float tX[32][33];
    const int bdx = U.bd[0], bdy = U.bd[1];
    const int x0 = blockIdx.x * 32, y0 = blockIdx.y * 32;
    const long long zoff = (long long)blockIdx.z * bdx * bdy;
    const int tx = threadIdx.x, ty = threadIdx.y;
    constexpr bool use_acc = MODE != UPD_XT;
    const bool final_ = U.final_ != 0;
    const bool writes_x = (MODE == UPD_XT) || ((MODE == UPD_BSGD || MODE == UPD_SGD) && final_);
    float* __restrict__ accN = U.accN;
    float* __restrict__ accT = U.accT;
    float* __restrict__ ghat = U.ghat;
    float* __restrict__ g = U.g;
    float* __restrict__ x = U.x;
    float* __restrict__ out = U.out;
    float vT[4], vN[4], vgh[4], vg[4], vx[4], vo[4];
    bool okT[4], ok[4];
    long long iT[4], idx[4], iP[4];   // iT: padded transposed; idx: plain normal; iP: padded normal
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const int xxT = x0 + ty + 8 * k, yyT = y0 + tx;
        okT[k] = xxT < bdx && yyT < bdy;
        iT[k] = (long long)blockIdx.z * U.planeT + (long long)xxT * U.rowT + yyT;
        const int xx = x0 + tx, yy = y0 + ty + 8 * k;
        ok[k] = xx < bdx && yy < bdy;
        idx[k] = zoff + (long long)yy * bdx + xx;
        iP[k] = (long long)blockIdx.z * U.planeN + (long long)yy * U.rowN + xx;
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        vT[k] = (use_acc && okT[k]) ? accT[iT[k]] : 0.f;
        vN[k] = (use_acc && ok[k]) ? accN[iP[k]] : 0.f;
        vgh[k] = (MODE == UPD_BSGD && ok[k]) ? ghat[idx[k]] : 0.f;
        vg[k] = (MODE == UPD_BSGD && ok[k]) ? g[idx[k]] : 0.f;
        vx[k] = (((MODE == UPD_BSGD && final_) || MODE == UPD_SGD || MODE == UPD_XT) && ok[k]) ? x[idx[k]] : 0.f;
        vo[k] = (MODE == UPD_OUT && U.accumulate && ok[k]) ? out[idx[k]] : 0.f;
    }
    if (use_acc) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            tT[ty + 8 * k][tx] = vT[k];
            if (okT[k]) accT[iT[k]] = 0.f;
        }
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        float xv = 0.f;
        if (ok[k]) {
            const long long i = idx[k];
            const float nv = use_acc ? vN[k] + tT[tx][ty + 8 * k] : 0.f;
            if (use_acc) accN[iP[k]] = 0.f;
            if (MODE == UPD_BSGD) {
                ghat[i] = nv;
                const float gv = vg[k] + (nv - vgh[k]);
                g[i] = gv;
                if (final_) {
                    xv = vx[k] + U.mu * gv;
                    x[i] = xv;
                }
            } else if (MODE == UPD_SGD) {
                g[i] = nv;
                xv = vx[k] + U.mu * nv;
                x[i] = xv;
            } else if (MODE == UPD_OUT) {
                out[i] = vo[k] + nv;
            } else if (MODE == UPD_XT) {
                xv = vx[k];
            }
            if (writes_x && U.xN) U.xN[iP[k]] = xv;
        }
        tX[ty + 8 * k][tx] = xv;
    }
    if (!writes_x) return;
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 4; ++k)
        if (okT[k]) U.xT[iT[k]] = tX[tx][ty + 8 * k];
}

// sum_j z^j over the owned blocks whose footprint holds the ray (packed storage, ZRect)
__device__ __forceinline__ const float* zrow(const ResLaunch& R, int j, int view, int iu, int iv) {
    const ZRect q = R.zr[(size_t)j * R.n_views + view];
    if (iu < q.u0 || iu >= q.u1 || iv < q.v0 || iv >= q.v1) return nullptr;
    return R.z + q.base + (long long)(iv - q.v0) * (q.u1 - q.u0) + (iu - q.u0);
}

__global__ void __launch_bounds__(256) k_residual(const ResLaunch R) {
    const int slot = blockIdx.y;
    const int view = R.views[slot];
    const long long base = (long long)view * R.per;
    const long long cbase = (long long)slot * R.per;
    double ss = 0.0;
    // float4 along u: footprint rectangles start and end on multiples of 32 columns (or nu)
    const bool v4 = (R.per & 3) == 0 && (R.nu & 3) == 0;
    const long long nvec = v4 ? R.per / 4 : R.per;
    for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < nvec;
         q += (long long)gridDim.x * blockDim.x) {
        if (v4) {
            const long long e = base + 4 * q;
            const int iv = (int)((4 * q) / R.nu), iu = (int)((4 * q) % R.nu);
            float4 acc;
            if (R.mode == 2) {
                acc = *reinterpret_cast<const float4*>(R.pc + cbase + 4 * q);
            } else {
                acc = make_float4(0.f, 0.f, 0.f, 0.f);
                for (int j = 0; j < R.s; ++j) {   // sum over owned blocks in ascending order
                    const float* zp = zrow(R, j, view, iu, iv);
                    if (!zp) continue;
                    const float4 zz = __ldg(reinterpret_cast<const float4*>(zp));
                    acc.x += zz.x; acc.y += zz.y; acc.z += zz.z; acc.w += zz.w;
                }
            }
            if (R.mode == 1) {
                *reinterpret_cast<float4*>(R.pc + cbase + 4 * q) = acc;
            } else {
                const float4 yy = __ldg(reinterpret_cast<const float4*>(R.y + e));
                float4 rr = make_float4(yy.x - acc.x, yy.y - acc.y, yy.z - acc.z, yy.w - acc.w);
                *reinterpret_cast<float4*>(R.r + e) = rr;
                ss += (double)rr.x * rr.x + (double)rr.y * rr.y + (double)rr.z * rr.z + (double)rr.w * rr.w;
            }
        } else {
            const long long e = base + q;
            const int iv = (int)(q / R.nu), iu = (int)(q % R.nu);
            float acc = 0.f;
            if (R.mode == 2) acc = R.pc[cbase + q];
            else
                for (int j = 0; j < R.s; ++j) {
                    const float* zp = zrow(R, j, view, iu, iv);
                    if (zp) acc += __ldg(zp);
                }
            if (R.mode == 1) {
                R.pc[cbase + q] = acc;
            } else {
                const float rr = R.y[e] - acc;
                R.r[e] = rr;
                ss += (double)rr * rr;
            }
        }
    }
    if (R.mode != 1) {   // per-CTA partial; k_normsq_final sums them in a fixed order so
        ss = block_sum(ss);  // that ||r_I||^2 (Algo 3's decisions) is bit-identical on every rank
        if (threadIdx.x == 0) R.part[(size_t)slot * RES_GX + blockIdx.x] = ss;
    }
}

// N2 band residual (BandLaunch): r = y - sum over the ranks whose band covers the row, in
// ascending rank order; fp64 ||r||^2 partials of the rows this rank owns (per CTA)
__global__ void __launch_bounds__(256) k_residual_band(const BandLaunch B) {
    const int slot = blockIdx.y;
    const int view = B.views[slot];
    const int2 rg = B.range[slot];
    const int2* bd = B.bands + (size_t)slot * B.G;
    const long long base = (long long)view * B.per, cbase = (long long)slot * B.per;
    double ss = 0.0;
    const bool v4 = (B.nu & 3) == 0;
    const int W = v4 ? B.nu / 4 : B.nu;
    const long long n = (long long)(rg.y - rg.x) * W;
    for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < n;
         q += (long long)gridDim.x * blockDim.x) {
        const int v = rg.x + (int)(q / W), u = (int)(q % W) * (v4 ? 4 : 1);
        int first = -1;
        bool mine = false;
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
        const long long e = (long long)v * B.nu + u;
        for (int h = 0; h < B.G; ++h) {          // ascending ranks: one order everywhere
            const int2 b = bd[h];
            if (v < b.x || v >= b.y) continue;
            if (first < 0) first = h;
            mine |= h == B.me;
            const float* d = B.data[h];
            if (!d) continue;                    // a band not overlapping this rank's
            const long long a = cbase + e + B.adj[(size_t)slot * B.G + h];
            if (v4) {
                const float4 t = *reinterpret_cast<const float4*>(d + a);
                acc.x += t.x; acc.y += t.y; acc.z += t.z; acc.w += t.w;
            } else {
                acc.x += d[a];
            }
        }
        if (mine) {
            if (v4) {
                const float4 yy = __ldg(reinterpret_cast<const float4*>(B.y + base + e));
                const float4 rr = make_float4(yy.x - acc.x, yy.y - acc.y, yy.z - acc.z, yy.w - acc.w);
                *reinterpret_cast<float4*>(B.r + base + e) = rr;
                if (first == B.me)
                    ss += (double)rr.x * rr.x + (double)rr.y * rr.y + (double)rr.z * rr.z + (double)rr.w * rr.w;
            } else {
                const float rr = B.y[base + e] - acc.x;
                B.r[base + e] = rr;
                if (first == B.me) ss += (double)rr * rr;
            }
        } else if (first < 0 && B.me == 0) {     // no band: r = y, never changed
            if (v4) {
                const float4 yy = __ldg(reinterpret_cast<const float4*>(B.y + base + e));
                ss += (double)yy.x * yy.x + (double)yy.y * yy.y + (double)yy.z * yy.z + (double)yy.w * yy.w;
            } else {
                const float yy = B.y[base + e];
                ss += (double)yy * yy;
            }
        }
    }
    ss = block_sum(ss);
    if (threadIdx.x == 0) B.part[(size_t)slot * RES_GX + blockIdx.x] = ss;
}

__global__ void __launch_bounds__(256) k_copy_chunks(const float* src, float* dst, const long long* t) {
    const long long s0 = t[3 * blockIdx.y], d0 = t[3 * blockIdx.y + 1], n = t[3 * blockIdx.y + 2];
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        dst[d0 + i] = src[s0 + i];
}

__global__ void k_copy_rows(double* dst, const double* src, const int* rows, int n) {
    const int i = threadIdx.x;
    if (i < n) dst[rows[i]] = src[rows[i]];
}

// normsq[i] = sum of the partials of the slots of row block i (CTA i; fixed assignment of
// partials to threads and a fixed reduction tree: deterministic).  Rows without slots keep
// their value.
__global__ void __launch_bounds__(256) k_normsq_final(const ResLaunch R, int gx) {
    const int i = blockIdx.x;
    double ss = 0.0;
    int hit = 0;
    for (long long q = threadIdx.x; q < (long long)R.n_slots * gx; q += blockDim.x) {
        const int slot = (int)(q / gx), b = (int)(q % gx);
        if (R.slot_row[slot] == i) {
            ss += R.part[(size_t)slot * RES_GX + b];
            hit = 1;
        }
    }
    ss = block_sum(ss);
    hit = __syncthreads_or(hit);
    if (threadIdx.x == 0 && hit) R.normsq[i] = ss;
}

__global__ void __launch_bounds__(256) k_zero_rects(float* proj, const int* views, const int4* rects, int nu,
                                                    int nv) {
    const int slot = blockIdx.y;
    const int4 rc = rects[slot];
    const int w = rc.y - rc.x, h = rc.w - rc.z;
    const long long base = (long long)views[slot] * nv * nu;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < w * h; i += gridDim.x * blockDim.x)
        proj[base + (long long)(rc.z + i / w) * nu + rc.x + i % w] = 0.f;
}

__global__ void k_zero_rows(double* normsq, const int* rows, int n) {
    int i = threadIdx.x;
    if (i < n) normsq[rows[i]] = 0.0;
}

__global__ void k_obj(const double* normsq, int M, double* out) {
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int i = 0; i < M; ++i) s += normsq[i];
        *out = 0.5 * s;
    }
}

__global__ void __launch_bounds__(256) k_axpy(float* eud, const float* g, long long n) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        eud[i] += g[i];
}

__global__ void __launch_bounds__(256) k_dot3(const float* a, const float* b, long long n, double* out) {
    double ab = 0, aa = 0, bb = 0;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        double x = a[i], y = b[i];
        ab += x * y; aa += x * x; bb += y * y;
    }
    ab = block_sum(ab);
    if (threadIdx.x == 0) atomicAdd(out, ab);
    aa = block_sum(aa);
    if (threadIdx.x == 0) atomicAdd(out + 1, aa);
    bb = block_sum(bb);
    if (threadIdx.x == 0) atomicAdd(out + 2, bb);
}

__global__ void __launch_bounds__(256) k_sqdiff(const float* a, const float* b, long long n, double* out) {
    double s = 0;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        double d = (double)a[i] - (double)b[i];
        s += d * d;
    }
    s = block_sum(s);
    if (threadIdx.x == 0) atomicAdd(out, s);
}

// out[0] += sum (a - b)^2 and out[1] += count over the voxels with mask > 0 (RMSE over the
// voxels some ray sees, reading A32)
__global__ void __launch_bounds__(256) k_sqdiff_masked(const float* a, const float* b, const float* mask,
                                                       long long n, double* out) {
    double s = 0, c = 0;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        if (mask[i] > 0.f) {
            const double d = (double)a[i] - (double)b[i];
            s += d * d;
            c += 1.0;
        }
    }
    s = block_sum(s);
    if (threadIdx.x == 0) atomicAdd(out, s);
    c = block_sum(c);
    if (threadIdx.x == 0) atomicAdd(out + 1, c);
}

__global__ void __launch_bounds__(256) k_fill(float* v, long long n, float val) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        v[i] = val;
}

// out = a x + b y (+ c z): the comparison solvers' vector updates.
// Plain fp32 streaming (HBM-bound: 12-16 B per element).
__global__ void __launch_bounds__(256) k_lincomb(float* out, float a, const float* x, float b,
                                                 const float* y, float c, const float* z, long long n) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        float v = fmaf(a, x[i], b * y[i]);
        if (z) v = fmaf(c, z[i], v);
        out[i] = v;
    }
}

// Barzilai-Borwein dots: s = x - xp, w = gp - g  ->  out[0] += <s,s>, out[1] += <s,w> (fp64).
__global__ void __launch_bounds__(256) k_bb_dots(const float* x, const float* xp, const float* gp,
                                                 const float* g, long long n, double* out) {
    double ss = 0, sw = 0;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const double s = (double)x[i] - (double)xp[i], w = (double)gp[i] - (double)g[i];
        ss += s * s;
        sw += s * w;
    }
    ss = block_sum(ss);
    if (threadIdx.x == 0) atomicAdd(out, ss);
    sw = block_sum(sw);
    if (threadIdx.x == 0) atomicAdd(out + 1, sw);
}

__device__ __forceinline__ uint64_t dmix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__global__ void k_fill_random(float* v, long long n, uint64_t seed) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        v[i] = (float)((dmix(seed + (uint64_t)(i + 1) * 0x9E3779B97F4A7C15ull) >> 40) * (1.0 / 16777216.0)) - 0.5f;
}

__global__ void k_scale(float* v, long long n, const double* nrm) {
    const float s = (float)(1.0 / sqrt(*nrm));
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        v[i] *= s;
}

// ------------------------------------------------------------------ TV prox
struct Vox {
    int x, y, z;
};

__device__ __forceinline__ Vox owned_coords(const TvLaunch& T, long long o) {
    if (T.bgrid[0] == 1 && T.bgrid[1] == 1) {   // z-slabs (any thicknesses): planes z0.. back to back
        const long long plane = (long long)T.dims[0] * T.dims[1];
        const long long l = o % plane;
        return {(int)(l % T.dims[0]), (int)(l / T.dims[0]), T.z0 + (int)(o / plane)};
    }
    const long long bs = (long long)T.bdims[0] * T.bdims[1] * T.bdims[2];
    const long long blk = T.block0 + o / bs;
    const long long l = o % bs;
    const int lx = (int)(l % T.bdims[0]), ly = (int)((l / T.bdims[0]) % T.bdims[1]),
              lz = (int)(l / ((long long)T.bdims[0] * T.bdims[1]));
    const int jx = (int)(blk % T.bgrid[0]), jy = (int)((blk / T.bgrid[0]) % T.bgrid[1]),
              jz = (int)(blk / ((long long)T.bgrid[0] * T.bgrid[1]));
    return {jx * T.bdims[0] + lx, jy * T.bdims[1] + ly, jz * T.bdims[2] + lz};
}

// owned index of global voxel (x,y,z); -1 if outside the owned range
__device__ __forceinline__ long long owned_index(const TvLaunch& T, int x, int y, int z) {
    if (T.bgrid[0] == 1 && T.bgrid[1] == 1) {   // z-slabs: the owned planes [z0, z1) back to back
        if (z < T.z0 || z >= T.z1) return -1;
        return ((long long)(z - T.z0) * T.dims[1] + y) * T.dims[0] + x;
    }
    const int jx = x / T.bdims[0], jy = y / T.bdims[1], jz = z / T.bdims[2];
    const long long blk = ((long long)jz * T.bgrid[1] + jy) * T.bgrid[0] + jx;
    const long long rel = blk - T.block0;
    const long long bs = (long long)T.bdims[0] * T.bdims[1] * T.bdims[2];
    if (rel < 0 || rel * bs >= T.n) return -1;
    const int lx = x - jx * T.bdims[0], ly = y - jy * T.bdims[1], lz = z - jz * T.bdims[2];
    return rel * bs + ((long long)lz * T.bdims[1] + ly) * T.bdims[0] + lx;
}

// dst = b - w * grad^T(src)  (src = 3 component fields, component stride T.n)
__global__ void __launch_bounds__(256) k_tv_u(const TvLaunch T, const float* src, float* dst) {
    for (long long o = (long long)blockIdx.x * blockDim.x + threadIdx.x; o < T.n;
         o += (long long)gridDim.x * blockDim.x) {
        const Vox v = owned_coords(T, o);
        double div = 0.0;
        const int c[3] = {v.x, v.y, v.z};
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            if (c[a] >= 1) div += src[a * T.n + o];
            if (c[a] + 1 <= T.dims[a] - 1) {
                const int nx = v.x + (a == 0), ny = v.y + (a == 1), nz = v.z + (a == 2);
                const long long on = owned_index(T, nx, ny, nz);
                float q;
                if (on >= 0) q = src[a * T.n + on];
                else q = T.halo_q_next[(long long)ny * T.dims[0] + nx];   // z comp of plane z1
                div -= q;
            }
        }
        dst[o] = (float)((double)T.b[o] - T.w * div);
    }
}

// TV(x) = sum_i |(grad x)_i|_2 (isotropic, backward differences, zero at index 0; Eq. 6)
// over the owned voxels; x of plane z0-1 comes from T.halo_u_prev when sharded
__global__ void __launch_bounds__(256) k_tv_value(const TvLaunch T, const float* x, double* out) {
    double acc = 0.0;
    for (long long o = (long long)blockIdx.x * blockDim.x + threadIdx.x; o < T.n;
         o += (long long)gridDim.x * blockDim.x) {
        const Vox v = owned_coords(T, o);
        const int c[3] = {v.x, v.y, v.z};
        const double xo = x[o];
        double s2 = 0.0;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            if (c[a] < 1) continue;
            const int nx = v.x - (a == 0), ny = v.y - (a == 1), nz = v.z - (a == 2);
            const long long on = owned_index(T, nx, ny, nz);
            const double xn = on >= 0 ? (double)x[on] : (double)T.halo_u_prev[(long long)ny * T.dims[0] + nx];
            s2 += (xo - xn) * (xo - xn);
        }
        acc += sqrt(s2);
    }
    acc = block_sum(acc);
    if (threadIdx.x == 0) atomicAdd(out, acc);
}

// one global z-plane of an owned block-major field, gathered into [y][x] (halo exchange of
// block grids whose ranks own whole z-layers of blocks)
__global__ void __launch_bounds__(256) k_pack_plane(const TvLaunch T, const float* owned, int z, float* out) {
    const long long plane = (long long)T.dims[0] * T.dims[1];
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < plane;
         i += (long long)gridDim.x * blockDim.x) {
        const int x = (int)(i % T.dims[0]), y = (int)(i / T.dims[0]);
        const long long o = owned_index(T, x, y, z);
        out[i] = o >= 0 ? owned[o] : 0.f;
    }
}

// p_new = P(q + grad(u)/(L w)); q = p_new + beta (p_new - p); p = p_new
__global__ void __launch_bounds__(256) k_tv_pq(const TvLaunch T) {
    const double s = 1.0 / (T.L * T.w);
    for (long long o = (long long)blockIdx.x * blockDim.x + threadIdx.x; o < T.n;
         o += (long long)gridDim.x * blockDim.x) {
        const Vox v = owned_coords(T, o);
        const int c[3] = {v.x, v.y, v.z};
        const double uo = T.u[o];
        double pn[3];
        double nrm = 0.0;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            double gr = 0.0;
            if (c[a] >= 1) {
                const int nx = v.x - (a == 0), ny = v.y - (a == 1), nz = v.z - (a == 2);
                const long long on = owned_index(T, nx, ny, nz);
                const float un = on >= 0 ? T.u[on] : T.halo_u_prev[(long long)ny * T.dims[0] + nx];
                gr = uo - (double)un;
            }
            pn[a] = (double)T.q[a * T.n + o] + gr * s;
            nrm += pn[a] * pn[a];
        }
        if (T.chambolle) {   // pn = q + s g: p <- (q + s g) / (1 + s |g|), in place on q
            double g2 = 0.0;
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                const double ga = pn[a] - (double)T.q[a * T.n + o];
                g2 += ga * ga;
            }
            const double d = 1.0 + sqrt(g2);
#pragma unroll
            for (int a = 0; a < 3; ++a) T.q[a * T.n + o] = (float)(pn[a] / d);
            continue;
        }
        const double d = fmax(1.0, sqrt(nrm));
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            const double p1 = pn[a] / d;
            const double p0 = T.p[a * T.n + o];
            T.q[a * T.n + o] = (float)(p1 + T.beta * (p1 - p0));
            T.p[a * T.n + o] = (float)p1;
        }
    }
}

// Fused FGP iteration for z-slab layouts (the owned volume is one [z][y][x] array of planes
// z0..z1-1).  Same arithmetic as k_tv_u + k_tv_pq (Beck-Teboulle FGP):
//   u = b - w grad^T q;  p1 = P(q + grad(u) / (L w));  q_out = p1 + beta (p1 - p);  p = p1
// without storing u: one thread per voxel, a 32 x 8 CTA per plane tile; u of x-1 comes from
// the neighbouring lane (shuffle), of y-1 from the row above (shared memory), and u of z-1 is
// evaluated directly (its q / b planes are L2 hits: the CTAs of plane z-1 just read them);
// tile-edge threads evaluate their halo u directly.  All loads of a thread are independent
// and issued together (a z-marching variant with one barrier per plane was latency-bound at
// 2.1 TB/s).  HBM per voxel: read q (3), p (3), b; write q_out (3), p (3) = 52 B.  q is
// double-buffered (q -> q_out) because neighbouring tiles read q around their edges.
constexpr int TV_TX = 32, TV_TY = 16;

struct TvPlane {
    const float *qx, *qy, *qz, *b;   // plane z (qx, qy, qz, b), indexed y * nx + x
    const float* qz1;                // q_z of plane z + 1
};

__device__ __forceinline__ TvPlane tv_plane(const TvLaunch& T, int z) {
    const long long plane = (long long)T.dims[0] * T.dims[1];
    TvPlane P;
    if (z < T.z0) {                  // previous rank's last plane (only read when z >= 0)
        P.qx = T.halo_prev;
        P.qy = T.halo_prev + plane;
        P.qz = T.halo_prev + 2 * plane;
        P.b = T.halo_prev + 3 * plane;
        P.qz1 = T.q + 2 * T.n;       // own first plane (z + 1 = z0)
    } else {
        const long long off = (long long)(z - T.z0) * plane;
        P.qx = T.q + off;
        P.qy = T.q + T.n + off;
        P.qz = T.q + 2 * T.n + off;
        P.b = T.b + off;
        P.qz1 = (z + 1 < T.z1) ? P.qz + plane : T.halo_q_next;   // next rank's first plane
    }
    return P;
}

// u at (x, y) of plane z: b - w grad^T q with the zero-boundary adjoint of Eq. 6 (fp32: the
// dual fields are stored in fp32 anyway; the oracle parity margin is ~100x)
__device__ __forceinline__ float tv_u_at(const TvLaunch& T, const TvPlane& P, int x, int y, int z, float w) {
    const int i = y * T.dims[0] + x;
    if (T.first) return P.b[i];
    float t = 0.f;
    if (x >= 1) t += P.qx[i];
    if (x + 1 < T.dims[0]) t -= P.qx[i + 1];
    if (y >= 1) t += P.qy[i];
    if (y + 1 < T.dims[1]) t -= P.qy[i + T.dims[0]];
    if (z >= 1) t += P.qz[i];
    if (z + 1 < T.dims[2]) t -= P.qz1[i];
    return fmaf(-w, t, P.b[i]);
}

// CTA = a TV_TX x TV_TY output tile of one plane plus helper threads for the u halo
// (row y0-1 and column x0-1), so that no output warp diverges on a halo evaluation.
constexpr int TV_OUT = TV_TX * TV_TY, TV_HALO = TV_TX + TV_TY;
constexpr int TV_THREADS = (TV_OUT + TV_HALO + 31) / 32 * 32;

template <int ZT>
__global__ void __launch_bounds__(TV_THREADS, ZT == 1 ? 3 : (ZT == 2 ? 2 : 1)) k_tv_fgp(const TvLaunch T) {
    __shared__ float su[ZT][TV_TY + 1][TV_TX + 1];
    const int t = threadIdx.x;
    int tx, ty;                              // slot in su: (ty + 1, tx + 1) <-> voxel (x0 + tx, y0 + ty)
    if (t < TV_OUT) { tx = t % TV_TX; ty = t / TV_TX; }
    else if (t < TV_OUT + TV_TX) { tx = t - TV_OUT; ty = -1; }
    else if (t < TV_OUT + TV_HALO) { tx = -1; ty = t - TV_OUT - TV_TX; }
    else { tx = TV_TX; ty = TV_TY; }         // idle padding thread (outside the tile, x or y invalid)
    const int x = blockIdx.x * TV_TX + tx, y = blockIdx.y * TV_TY + ty, zb = T.z0 + blockIdx.z * ZT;
    const bool inside = x >= 0 && y >= 0 && x < T.dims[0] && y < T.dims[1] && tx < TV_TX && ty < TV_TY;
    const bool out = inside && t < TV_OUT;
    const float w = T.wf;
    const long long plane = (long long)T.dims[0] * T.dims[1];
    const long long i0 = (long long)(zb - T.z0) * plane + (long long)y * T.dims[0] + x;
    // every load of the thread is independent: issue all of them before the barrier
    float u[ZT + 1], qx[ZT], qy[ZT], qz[ZT], ox[ZT], oy[ZT], oz[ZT];
    u[0] = 0.f;
    if (out && zb >= 1) u[0] = tv_u_at(T, tv_plane(T, zb - 1), x, y, zb - 1, w);
#pragma unroll
    for (int k = 0; k < ZT; ++k) {
        const bool pin = zb + k < T.z1;
        u[k + 1] = 0.f;
        if (inside && pin) u[k + 1] = tv_u_at(T, tv_plane(T, zb + k), x, y, zb + k, w);
        const long long i = i0 + k * plane;
        if (out && pin && T.first) {
            qx[k] = qy[k] = qz[k] = ox[k] = oy[k] = oz[k] = 0.f;
        } else if (out && pin) {
            qx[k] = T.q[i];
            qy[k] = T.q[T.n + i];
            qz[k] = T.q[2 * T.n + i];
            if (!T.chambolle) {
                ox[k] = T.p[i];
                oy[k] = T.p[T.n + i];
                oz[k] = T.p[2 * T.n + i];
            }
        }
        if (inside) su[k][ty + 1][tx + 1] = u[k + 1];
    }
    __syncthreads();
    if (!out) return;
    const float s = T.sf, beta = T.betaf;
#pragma unroll
    for (int k = 0; k < ZT; ++k) {
        const int z = zb + k;
        if (z >= T.z1) break;
        const float uo = u[k + 1];
        const float gx = (x >= 1 ? uo - su[k][ty + 1][tx] : 0.f) * s;
        const float gy = (y >= 1 ? uo - su[k][ty][tx + 1] : 0.f) * s;
        const float gz = (z >= 1 ? uo - u[k] : 0.f) * s;
        const long long i = i0 + k * plane;
        if (T.chambolle) {       // p <- (p + s g) / (1 + s |g|)
            const float d = 1.f / (1.f + sqrtf(gx * gx + gy * gy + gz * gz));
            T.q_out[i] = (qx[k] + gx) * d;
            T.q_out[T.n + i] = (qy[k] + gy) * d;
            T.q_out[2 * T.n + i] = (qz[k] + gz) * d;
            continue;
        }
        const float p0x = qx[k] + gx, p0y = qy[k] + gy, p0z = qz[k] + gz;
        const float n2 = p0x * p0x + p0y * p0y + p0z * p0z;
        const float inv = n2 > 1.f ? rsqrtf(n2) : 1.f;      // projection onto |p| <= 1
        const float px = p0x * inv, py = p0y * inv, pz = p0z * inv;
        T.q_out[i] = px + beta * (px - ox[k]);
        T.q_out[T.n + i] = py + beta * (py - oy[k]);
        T.q_out[2 * T.n + i] = pz + beta * (pz - oz[k]);
        T.p[i] = px;
        T.p[T.n + i] = py;
        T.p[2 * T.n + i] = pz;
    }
}

// Vectorised fused FGP iteration (nx % 4 == 0): each thread owns 4 consecutive x voxels and
// moves them with 16-byte loads / stores (the scalar kernel above tops out near 3.5 TB/s on
// request count).  CTA = TV4_TY rows x 128 x of one plane + one warp for the halo row y0-1
// (vectors) + TV4_TY lanes for the halo column x0-1 (scalars).  Within a vector the x
// difference is local; across lanes it comes by shuffle, at lane 0 from the halo column.
constexpr int TV4_TX = 128;

__device__ __forceinline__ float4 ld4(const float* p) { return *reinterpret_cast<const float4*>(p); }
__device__ __forceinline__ void st4(float* p, float a, float b, float c, float d) {
    *reinterpret_cast<float4*>(p) = make_float4(a, b, c, d);
}

// u at the 4 voxels (x..x+3, y) of plane z (x % 4 == 0); all lanes of the warp must call it
// (the qx(x+4) neighbour comes from the next lane)
__device__ __forceinline__ void tv_u4(const TvLaunch& T, const TvPlane& P, int x, int y, int z, bool act,
                                      float w, float u[4]) {
    const int nx = T.dims[0];
    const int i = y * nx + x;
    float4 qx = make_float4(0.f, 0.f, 0.f, 0.f), qy = qx, qyn = qx, qz = qx, qz1 = qx, b = qx;
    float qxe = 0.f;
    if (T.first) {                 // q = 0: u = b
        if (act) {
            b = ld4(P.b + i);
            u[0] = b.x; u[1] = b.y; u[2] = b.z; u[3] = b.w;
        }
        return;
    }
    if (act) {
        qx = ld4(P.qx + i);
        qy = ld4(P.qy + i);
        if (y + 1 < T.dims[1]) qyn = ld4(P.qy + i + nx);
        qz = ld4(P.qz + i);
        if (z + 1 < T.dims[2]) qz1 = ld4(P.qz1 + i);
        b = ld4(P.b + i);
    }
    float qx4 = __shfl_down_sync(0xffffffffu, qx.x, 1);
    if ((threadIdx.x & 31) == 31 && act && x + 4 < nx) qxe = P.qx[i + 4];
    if ((threadIdx.x & 31) == 31) qx4 = qxe;
    if (!act) return;
    const float qxa[5] = {qx.x, qx.y, qx.z, qx.w, x + 4 < nx ? qx4 : 0.f};
    const float qya[4] = {qy.x, qy.y, qy.z, qy.w}, qyb[4] = {qyn.x, qyn.y, qyn.z, qyn.w};
    const float qza[4] = {qz.x, qz.y, qz.z, qz.w}, qzb[4] = {qz1.x, qz1.y, qz1.z, qz1.w};
    const float ba[4] = {b.x, b.y, b.z, b.w};
    const float cy = y >= 1 ? 1.f : 0.f, cz = z >= 1 ? 1.f : 0.f;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        float t = (x + k >= 1 ? qxa[k] : 0.f) - qxa[k + 1];   // qxa[4] is 0 at the last column
        t += cy * qya[k] - qyb[k] + cz * qza[k] - qzb[k];     // qyb / qzb are 0 past the boundary
        u[k] = fmaf(-w, t, ba[k]);
    }
}

template <int TV4_TY, int MINB>
__global__ void __launch_bounds__((TV4_TY + 2) * 32, MINB) k_tv_fgp4(const TvLaunch T) {
    constexpr int RS = TV4_TX + 8;                 // row stride (16-byte aligned rows)
    __shared__ __align__(16) float su[TV4_TY + 1][RS];   // slot 4 + (x - x0) <-> x; slot 3 <-> x0 - 1
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int x0 = blockIdx.x * TV4_TX, y0 = blockIdx.y * TV4_TY, z = T.z0 + blockIdx.z;
    const int nx = T.dims[0], ny = T.dims[1];
    const float w = T.wf;
    const TvPlane P = tv_plane(T, z);
    // the last warp is the helper of the halo column x0 - 1 (scalars, rows y0 .. y0+TY-1);
    // every thread of the CTA reaches the one barrier below (no divergent barriers)
    const bool helper = warp > TV4_TY;
    const int row = helper ? 0 : warp;             // 0 = halo row y0 - 1, 1.. = output rows
    const int y = helper ? y0 + lane : y0 + row - 1, x = x0 + 4 * lane;
    const bool act = !helper && y >= 0 && y < ny && x < nx;
    const bool out = act && row >= 1;
    float u[4] = {0.f, 0.f, 0.f, 0.f}, uz[4] = {0.f, 0.f, 0.f, 0.f};
    const long long plane = (long long)nx * ny;
    const long long i = (long long)(z - T.z0) * plane + (long long)y * nx + x;
    float4 q0 = make_float4(0.f, 0.f, 0.f, 0.f), q1 = q0, q2 = q0, p0 = q0, p1 = q0, p2 = q0;
    float ul = 0.f;
    if (helper) {
        if (lane < TV4_TY && x0 >= 1 && y < ny) su[lane + 1][3] = tv_u_at(T, P, x0 - 1, y, z, w);
    } else {                                       // warp-uniform branch: whole warps
        tv_u4(T, P, x, y, z, act, w, u);
        if (row >= 1) {
            if (z >= 1) tv_u4(T, tv_plane(T, z - 1), x, y, z - 1, out, w, uz);
            if (out && !T.first) {
                q0 = ld4(T.q + i);
                q1 = ld4(T.q + T.n + i);
                q2 = ld4(T.q + 2 * T.n + i);
                if (!T.chambolle) {
                    p0 = ld4(T.p + i);
                    p1 = ld4(T.p + T.n + i);
                    p2 = ld4(T.p + 2 * T.n + i);
                }
            }
        }
        if (act) *reinterpret_cast<float4*>(&su[row][4 + 4 * lane]) = make_float4(u[0], u[1], u[2], u[3]);
        ul = __shfl_up_sync(0xffffffffu, u[3], 1);
    }
    __syncthreads();
    if (!out) return;
    const float uxm = lane > 0 ? ul : su[row][3];   // u(x - 1)
    const float4 up = *reinterpret_cast<const float4*>(&su[row - 1][4 + 4 * lane]);
    const float upa[4] = {up.x, up.y, up.z, up.w};
    const float qa[3][4] = {{q0.x, q0.y, q0.z, q0.w}, {q1.x, q1.y, q1.z, q1.w}, {q2.x, q2.y, q2.z, q2.w}};
    const float pa[3][4] = {{p0.x, p0.y, p0.z, p0.w}, {p1.x, p1.y, p1.z, p1.w}, {p2.x, p2.y, p2.z, p2.w}};
    const float s = T.sf, beta = T.betaf;
    float qo[3][4], po[3][4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const float left = k == 0 ? uxm : u[k - 1];
        const float gx = x + k >= 1 ? u[k] - left : 0.f;
        const float gy = y >= 1 ? u[k] - upa[k] : 0.f;
        const float gz = z >= 1 ? u[k] - uz[k] : 0.f;
        const float a0 = qa[0][k] + gx * s, a1 = qa[1][k] + gy * s, a2 = qa[2][k] + gz * s;
        if (T.chambolle) {       // p <- (p + s g) / (1 + s |g|); qo = the new p
            const float d = 1.f / (1.f + s * sqrtf(gx * gx + gy * gy + gz * gz));
            qo[0][k] = a0 * d;
            qo[1][k] = a1 * d;
            qo[2][k] = a2 * d;
            continue;
        }
        const float n2 = a0 * a0 + a1 * a1 + a2 * a2;
        const float inv = n2 > 1.f ? rsqrtf(n2) : 1.f;
        po[0][k] = a0 * inv;
        po[1][k] = a1 * inv;
        po[2][k] = a2 * inv;
#pragma unroll
        for (int c = 0; c < 3; ++c) qo[c][k] = po[c][k] + beta * (po[c][k] - pa[c][k]);
    }
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        st4(T.q_out + c * T.n + i, qo[c][0], qo[c][1], qo[c][2], qo[c][3]);
        if (!T.chambolle) st4(T.p + c * T.n + i, po[c][0], po[c][1], po[c][2], po[c][3]);
    }
}

// ---- z-marching FGP (TvzLaunch) -------------------------------------------------------
// Per plane z, component c (0..2) of P1 / P2 and b: owned planes from the buffers, plane
// z0-1 from halo_prev, plane z1 (z components only) from halo_next.
struct ZPlane {
    const float* p1[3];
    const float* p2[3];
    const float* b;
};
__device__ __forceinline__ ZPlane zplane(const TvzLaunch& T, int z) {
    const long long plane = (long long)T.nx * T.ny;
    ZPlane P;
    if (z < T.z0) {
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            P.p1[c] = T.halo_prev + c * plane;
            P.p2[c] = T.halo_prev + (3 + c) * plane;
        }
        P.b = T.halo_prev + 6 * plane;
    } else if (z >= T.z1) {           // only the z components are read there
        P.p1[0] = P.p1[1] = P.p1[2] = T.halo_next;
        P.p2[0] = P.p2[1] = P.p2[2] = T.halo_next + plane;
        P.b = nullptr;
    } else {
        const long long off = (long long)(z - T.z0) * plane;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            P.p1[c] = T.P1 + c * T.n + off;
            P.p2[c] = T.P2 + c * T.n + off;
        }
        P.b = T.b + off;
    }
    return P;
}
// q = p1 + beta (p1 - p2) as the fused kernel formed it (stage 1: q = 0, stage 2: q = p1)
__device__ __forceinline__ float4 zq4(const TvzLaunch& T, const float* p1, const float* p2, long long i) {
    if (T.stage == 1) return make_float4(0.f, 0.f, 0.f, 0.f);
    const float4 a = ld4(p1 + i);
    if (T.stage == 2) return a;
    const float4 c = ld4(p2 + i);
    return make_float4(a.x + T.beta * (a.x - c.x), a.y + T.beta * (a.y - c.y), a.z + T.beta * (a.z - c.z),
                       a.w + T.beta * (a.w - c.w));
}
__device__ __forceinline__ float zq1(const TvzLaunch& T, const float* p1, const float* p2, long long i) {
    if (T.stage == 1) return 0.f;
    const float a = p1[i];
    if (T.stage == 2) return a;
    return a + T.beta * (a - p2[i]);
}

// u = b - w grad^T q at (x..x+3, y) of plane z (x % 4 == 0; all lanes of the warp call it),
// with q own (3 components) returned for the p update
__device__ __forceinline__ void zu4(const TvzLaunch& T, int x, int y, int z, bool act, float u[4], float4 q[3]) {
    const int nx = T.nx;
    const long long i = (long long)y * nx + x;
    const ZPlane P = zplane(T, z);
    float4 qyn = make_float4(0.f, 0.f, 0.f, 0.f), qz1 = qyn, b = qyn;
    q[0] = q[1] = q[2] = qyn;
    float qxe = 0.f;
    if (act) {
        q[0] = zq4(T, P.p1[0], P.p2[0], i);
        q[1] = zq4(T, P.p1[1], P.p2[1], i);
        q[2] = zq4(T, P.p1[2], P.p2[2], i);
        if (y + 1 < T.ny) qyn = zq4(T, P.p1[1], P.p2[1], i + nx);
        if (z + 1 < T.nz) {
            const ZPlane Q = zplane(T, z + 1);
            qz1 = zq4(T, Q.p1[2], Q.p2[2], i);
        }
        b = ld4(P.b + i);
        if ((threadIdx.x & 31) == 31 && x + 4 < nx) qxe = zq1(T, P.p1[0], P.p2[0], i + 4);
    }
    float qx4 = __shfl_down_sync(0xffffffffu, q[0].x, 1);
    if ((threadIdx.x & 31) == 31) qx4 = qxe;
    if (!act) {
        u[0] = u[1] = u[2] = u[3] = 0.f;
        return;
    }
    const float qxa[5] = {q[0].x, q[0].y, q[0].z, q[0].w, x + 4 < nx ? qx4 : 0.f};
    const float qya[4] = {q[1].x, q[1].y, q[1].z, q[1].w}, qyb[4] = {qyn.x, qyn.y, qyn.z, qyn.w};
    const float qza[4] = {q[2].x, q[2].y, q[2].z, q[2].w}, qzb[4] = {qz1.x, qz1.y, qz1.z, qz1.w};
    const float ba[4] = {b.x, b.y, b.z, b.w};
    const float cy = y >= 1 ? 1.f : 0.f, cz = z >= 1 ? 1.f : 0.f;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        float t = (x + k >= 1 ? qxa[k] : 0.f) - qxa[k + 1];
        t += cy * qya[k] - qyb[k] + cz * qza[k] - qzb[k];
        u[k] = fmaf(-T.w, t, ba[k]);
    }
}
// scalar u at (x, y) of plane z (the helper lanes' halo column x0 - 1)
__device__ __forceinline__ float zu1(const TvzLaunch& T, int x, int y, int z) {
    const int nx = T.nx;
    const long long i = (long long)y * nx + x;
    const ZPlane P = zplane(T, z);
    float t = 0.f;
    if (x >= 1) t += zq1(T, P.p1[0], P.p2[0], i);
    if (x + 1 < nx) t -= zq1(T, P.p1[0], P.p2[0], i + 1);
    if (y >= 1) t += zq1(T, P.p1[1], P.p2[1], i);
    if (y + 1 < T.ny) t -= zq1(T, P.p1[1], P.p2[1], i + nx);
    if (z >= 1) t += zq1(T, P.p1[2], P.p2[2], i);
    if (z + 1 < T.nz) {
        const ZPlane Q = zplane(T, z + 1);
        t -= zq1(T, Q.p1[2], Q.p2[2], i);
    }
    return fmaf(-T.w, t, P.b[i]);
}

// CTA: warp 0 = the halo row y0 - 1, warps 1..TY = output rows y0..y0+TY-1 (4 x voxels per
// lane, 128 per row), warp TY + 1 = helper lanes for the halo column x0 - 1; the CTA walks
// planes zs..zs+zc-1 with u(z-1) of its output rows in registers (a prologue evaluates
// u(zs-1)).  Per plane: every warp evaluates u on its row, one barrier, the output rows
// project q + s grad u onto the unit ball and write p_k, a second barrier before the shared
// u rows are overwritten.
template <int TY, int MINB>
__global__ void __launch_bounds__((TY + 2) * 32, MINB) k_tv_fgp_z(const TvzLaunch T) {
    constexpr int RS = TV4_TX + 8;
    __shared__ __align__(16) float su[TY + 1][RS];   // slot 4 + (x - x0) <-> x; slot 3 <-> x0 - 1
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int x0 = blockIdx.x * TV4_TX, y0 = blockIdx.y * TY;
    const int zs = T.z0 + blockIdx.z * T.zc, ze = min(zs + T.zc, T.z1);
    const bool helper = warp > TY;
    const int row = helper ? 0 : warp;
    const int y = helper ? y0 + lane : y0 + row - 1, x = x0 + 4 * lane;
    const bool act = !helper && y >= 0 && y < T.ny && x < T.nx;
    const bool out = act && row >= 1;
    const long long plane = (long long)T.nx * T.ny;
    float uprev[4] = {0.f, 0.f, 0.f, 0.f};
    if (!helper && row >= 1 && zs >= 1) {          // u(zs - 1) of the output rows
        float4 qd[3];
        zu4(T, x, y, zs - 1, out, uprev, qd);
    }
    for (int z = zs; z < ze; ++z) {
        float u[4] = {0.f, 0.f, 0.f, 0.f};
        float4 q[3];
        float ul = 0.f;
        // L2 prefetch of this thread's lines of plane z + pf (the DRAM latency of the next
        // planes overlaps this plane's work; each plane's own loads then hit L2)
        const int zp = z + T.pf;
        if (T.pf > 0 && act && zp < T.z1) {
            const ZPlane Q = zplane(T, zp);
            const long long ip = (long long)y * T.nx + x;
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                if (T.stage != 1) asm volatile("prefetch.global.L2 [%0];" ::"l"(Q.p1[c] + ip));
                if (T.stage == 0) asm volatile("prefetch.global.L2 [%0];" ::"l"(Q.p2[c] + ip));
            }
            asm volatile("prefetch.global.L2 [%0];" ::"l"(Q.b + ip));
        }
        if (helper) {
            if (lane < TY && x0 >= 1 && y < T.ny) su[lane + 1][3] = zu1(T, x0 - 1, y, z);
        } else {
            zu4(T, x, y, z, act, u, q);
            if (act) *reinterpret_cast<float4*>(&su[row][4 + 4 * lane]) = make_float4(u[0], u[1], u[2], u[3]);
            ul = __shfl_up_sync(0xffffffffu, u[3], 1);
        }
        __syncthreads();
        if (out) {
            const float uxm = lane > 0 ? ul : su[row][3];
            const float4 up = *reinterpret_cast<const float4*>(&su[row - 1][4 + 4 * lane]);
            const float upa[4] = {up.x, up.y, up.z, up.w};
            const float qa[3][4] = {{q[0].x, q[0].y, q[0].z, q[0].w}, {q[1].x, q[1].y, q[1].z, q[1].w},
                                    {q[2].x, q[2].y, q[2].z, q[2].w}};
            float po[3][4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const float left = k == 0 ? uxm : u[k - 1];
                const float gx = x + k >= 1 ? u[k] - left : 0.f;
                const float gy = y >= 1 ? u[k] - upa[k] : 0.f;
                const float gz = z >= 1 ? u[k] - uprev[k] : 0.f;
                const float a0 = qa[0][k] + gx * T.s, a1 = qa[1][k] + gy * T.s, a2 = qa[2][k] + gz * T.s;
                const float n2 = a0 * a0 + a1 * a1 + a2 * a2;
                const float inv = n2 > 1.f ? rsqrtf(n2) : 1.f;
                po[0][k] = a0 * inv;
                po[1][k] = a1 * inv;
                po[2][k] = a2 * inv;
            }
            const long long i = (long long)(z - T.z0) * plane + (long long)y * T.nx + x;
#pragma unroll
            for (int c = 0; c < 3; ++c) st4(T.Pn + c * T.n + i, po[c][0], po[c][1], po[c][2], po[c][3]);
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) uprev[k] = u[k];
        __syncthreads();
    }
}

// ---- two FGP iterations per pass (k_tv_fgp_z2, Tvz2Launch; nx % 4 == 0) ---------------
// Region coordinates (rx, ry) in [0, 64) x [0, 16) <-> voxel (x0 - 4 + rx, y0 - 2 + ry) of a
// 56 x 12 output tile (x0, y0): a thread owns the 4 x-consecutive voxels of one region row
// (float4 in global and shared memory; x0 - 4 keeps the quads 16-byte aligned).  Iteration k
// needs u_k on [-2, W] (the backward gradient of p_k's 1-voxel halo), hence q_k on
// [-2, W + 1]; p_k / q_{k+1} live on [-1, W], u_{k+1} on [-1, W - 1], p_{k+1} on the tile
// (the same in y, where the halo is exactly 2).  Values beyond these ranges are computed from
// whatever the region holds and never read.
// Step z of the march: L loads plane z + 1 (q_k = p_{k-1} + beta_{k-1} (p_{k-1} - p_{k-2}) to
// shared memory; p_{k-1} and b, which only the loading thread reads, in registers), U1 evaluates u_k(z) = b - w grad^T q_k, P1 projects p_k(z) and forms
// q_{k+1}(z) = p_k + beta_k (p_k - p_{k-1}), U2 evaluates u_{k+1}(z - 1), P2 projects
// p_{k+1}(z - 1).  Four barriers per plane (two per iteration, as k_tv_fgp_z).
constexpr int Z2_W = 56, Z2_RW = 64;
constexpr int Z2_FIELDS = 16;   // sq 2x3, su 2, sq1 2x3, su1 2 (p_{k-1} and b stay in registers)
template <int RH> constexpr int z2_threads() { return Z2_RW / 4 * RH; }
template <int RH> constexpr size_t z2_smem() { return sizeof(float) * Z2_FIELDS * Z2_RW * RH; }

__device__ __forceinline__ float4 lds4(const float* p) { return *reinterpret_cast<const float4*>(p); }
__device__ __forceinline__ void sts4(float* p, float4 v) { *reinterpret_cast<float4*>(p) = v; }
__device__ __forceinline__ void f4a(float4 v, float a[4]) {
    a[0] = v.x;
    a[1] = v.y;
    a[2] = v.z;
    a[3] = v.w;
}

// u = b - w grad^T q on the quad at offset o of row gy, plane zq (q: 3 component fields of
// plane zq, qzn: z component of plane zq + 1; zero differences at index 0 and beyond the
// last index, Eq. 6 adjoint)
__device__ __forceinline__ float4 z2_u(const float* qx, const float* qy, const float* qz, const float* qzn,
                                       float4 bb, int o, int gx0, int gy, int zq, int nx, int ny, int nz, float w) {
    float ax[5], ay[4], ayn[4], az[4], azn[4], b[4];
    f4a(lds4(qx + o), ax);
    ax[4] = qx[o + 4];
    f4a(lds4(qy + o), ay);
    f4a(lds4(qy + o + Z2_RW), ayn);
    f4a(lds4(qz + o), az);
    f4a(lds4(qzn + o), azn);
    f4a(bb, b);
    const float cy = gy >= 1 ? 1.f : 0.f, cyn = gy + 1 < ny ? 1.f : 0.f;
    const float cz = zq >= 1 ? 1.f : 0.f, czn = zq + 1 < nz ? 1.f : 0.f;
    float u[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        float t = (gx0 + e >= 1 ? ax[e] : 0.f) - (gx0 + e + 1 < nx ? ax[e + 1] : 0.f);
        t += cy * ay[e] - cyn * ayn[e] + cz * az[e] - czn * azn[e];
        u[e] = fmaf(-w, t, b[e]);
    }
    return make_float4(u[0], u[1], u[2], u[3]);
}

// p = P_{|p| <= 1}(q + s grad u) on the quad at offset o (uu: u of the plane, uprev: u of the
// plane below; backward differences, zero at index 0)
__device__ __forceinline__ void z2_p(const float* uu, const float* uprev, const float* qx, const float* qy,
                                     const float* qz, int o, int gx0, int gy, int zq, float s, float p[3][4]) {
    float u[4], uup[4], upr[4], q[3][4];
    f4a(lds4(uu + o), u);
    const float ul = uu[o - 1];
    f4a(lds4(uu + o - Z2_RW), uup);
    f4a(lds4(uprev + o), upr);
    f4a(lds4(qx + o), q[0]);
    f4a(lds4(qy + o), q[1]);
    f4a(lds4(qz + o), q[2]);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        const float left = e == 0 ? ul : u[e - 1];
        const float gx = gx0 + e >= 1 ? u[e] - left : 0.f;
        const float gy_ = gy >= 1 ? u[e] - uup[e] : 0.f;
        const float gz = zq >= 1 ? u[e] - upr[e] : 0.f;
        const float a0 = q[0][e] + gx * s, a1 = q[1][e] + gy_ * s, a2 = q[2][e] + gz * s;
        const float n2 = a0 * a0 + a1 * a1 + a2 * a2;
        const float iv = n2 > 1.f ? rsqrtf(n2) : 1.f;
        p[0][e] = a0 * iv;
        p[1][e] = a1 * iv;
        p[2][e] = a2 * iv;
    }
}

template <int Z2_RH>
__global__ void __launch_bounds__(Z2_RW / 4 * Z2_RH, Z2_RH <= 16 ? 3 : 2) k_tv_fgp_z2(const Tvz2Launch T) {
    constexpr int Z2_H = Z2_RH - 4, Z2_F = Z2_RW * Z2_RH;
    extern __shared__ __align__(16) float sm[];
    float* const sq = sm;                       // [2][3][F]  q_k of planes z, z + 1
    float* const su = sq + 6 * Z2_F;            // [2][F]     u_k of planes z - 1, z
    float* const sq1 = su + 2 * Z2_F;           // [2][3][F]  q_{k+1} of planes z - 1, z
    float* const su1 = sq1 + 6 * Z2_F;          // [2][F]     u_{k+1} of planes z - 2, z - 1
    const int nx = T.nx, ny = T.ny, nz = T.nz;
    const long long plane = (long long)nx * ny;
    const int tq = threadIdx.x & 15, ty = threadIdx.x >> 4;
    const int rx0 = 4 * tq, o = ty * Z2_RW + rx0;
    const int gx0 = blockIdx.x * Z2_W - 4 + rx0, gy = blockIdx.y * Z2_H - 2 + ty;
    const int zs = blockIdx.z * T.zc, ze = min(zs + T.zc, nz);
    const bool qin = gy >= 0 && gy < ny && gx0 >= 0 && gx0 < nx;   // nx % 4 == 0: whole quads
    const bool tile_x = tq >= 1 && tq < 15, tile = tile_x && ty >= 2 && ty < Z2_RH - 2 && qin;
    const long long gi = (long long)gy * nx + gx0;
    const float w = T.w, s = T.s, be0 = T.beta0, be1 = T.beta1;
    const int stage = T.stage;
    const float4 zero4 = make_float4(0.f, 0.f, 0.f, 0.f);
    // a thread always owns the same quad, so what only its own quad reads stays in registers:
    // p_{k-1} of plane z (P1's momentum) and b of planes z - 1, z (U2, U1), loaded one step ahead
    float4 p1n[3] = {zero4, zero4, zero4}, bn = zero4, bz = zero4, bzm = zero4;

    for (int z = max(zs - 3, -1); z <= ze; ++z) {
        const float4 p1z[3] = {p1n[0], p1n[1], p1n[2]};   // p_{k-1}(z)
        bzm = bz;                                         // b(z - 1)
        bz = bn;                                          // b(z)
        // ---- L: plane z + 1 -> sq (+ p_{k-1}, b in registers)
        {
            const int zl = z + 1, a = zl & 1;
            const int zp = zl + T.pf;
            if (T.pf > 0 && qin && zp >= 0 && zp < nz && (tq == 0 || (gx0 & 31) == 0)) {   // once per line
                const long long ip = (long long)zp * plane + gi;
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    if (stage != 1) asm volatile("prefetch.global.L2 [%0];" ::"l"(T.P1 + c * T.n + ip));
                    if (stage == 0) asm volatile("prefetch.global.L2 [%0];" ::"l"(T.P2 + c * T.n + ip));
                }
                asm volatile("prefetch.global.L2 [%0];" ::"l"(T.b + ip));
            }
            float4 p1[3] = {zero4, zero4, zero4}, p2[3] = {zero4, zero4, zero4}, bb = zero4;
            if (qin && zl >= 0 && zl < nz) {
                const long long i = (long long)zl * plane + gi;
                if (stage != 1) {
#pragma unroll
                    for (int c = 0; c < 3; ++c) p1[c] = __ldg(reinterpret_cast<const float4*>(T.P1 + c * T.n + i));
                }
                if (stage == 0) {
#pragma unroll
                    for (int c = 0; c < 3; ++c) p2[c] = __ldg(reinterpret_cast<const float4*>(T.P2 + c * T.n + i));
                }
                bb = __ldg(reinterpret_cast<const float4*>(T.b + i));
            }
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                // q_k as k_tv_fgp_z forms it (stage 1: 0; stage 2: p_1)
                float4 q = p1[c];
                if (stage == 0)
                    q = make_float4(p1[c].x + be0 * (p1[c].x - p2[c].x), p1[c].y + be0 * (p1[c].y - p2[c].y),
                                    p1[c].z + be0 * (p1[c].z - p2[c].z), p1[c].w + be0 * (p1[c].w - p2[c].w));
                sts4(sq + (a * 3 + c) * Z2_F + o, q);
                p1n[c] = p1[c];
            }
            bn = bb;
        }
        __syncthreads();
        // ---- U1: u_k(z) on region rows [0, 15)
        if (z >= 0 && z < nz && ty < Z2_RH - 1) {
            const int a = z & 1, an = (z + 1) & 1;
            sts4(su + a * Z2_F + o, z2_u(sq + (a * 3 + 0) * Z2_F, sq + (a * 3 + 1) * Z2_F, sq + (a * 3 + 2) * Z2_F,
                                         sq + (an * 3 + 2) * Z2_F, bz, o, gx0, gy, z, nx, ny, nz, w));
        }
        __syncthreads();
        // ---- P1: p_k(z) on rows [1, 15); q_{k+1}(z); p_k written on the output tile
        if (z >= 0 && z < nz && ty >= 1 && ty < Z2_RH - 1) {
            const int a = z & 1, ap = (z + 1) & 1;   // ap = (z - 1) & 1
            float pk[3][4];
            z2_p(su + a * Z2_F, su + ap * Z2_F, sq + (a * 3 + 0) * Z2_F, sq + (a * 3 + 1) * Z2_F,
                 sq + (a * 3 + 2) * Z2_F, o, gx0, gy, z, s, pk);
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                float pm[4];
                f4a(p1z[c], pm);
                float4 qn = zero4;
                if (qin)
                    qn = make_float4(pk[c][0] + be1 * (pk[c][0] - pm[0]), pk[c][1] + be1 * (pk[c][1] - pm[1]),
                                     pk[c][2] + be1 * (pk[c][2] - pm[2]), pk[c][3] + be1 * (pk[c][3] - pm[3]));
                sts4(sq1 + (a * 3 + c) * Z2_F + o, qn);
            }
            if (tile && z >= zs && z < ze) {
                const long long i = (long long)z * plane + gi;
#pragma unroll
                for (int c = 0; c < 3; ++c) st4(T.Pa + c * T.n + i, pk[c][0], pk[c][1], pk[c][2], pk[c][3]);
            }
        }
        __syncthreads();
        // ---- U2: u_{k+1}(z - 1) on rows [1, 14)
        const int zz = z - 1;
        if (zz >= 0 && zz < nz && ty >= 1 && ty < Z2_RH - 2) {
            const int a = zz & 1, an = z & 1;
            sts4(su1 + a * Z2_F + o, z2_u(sq1 + (a * 3 + 0) * Z2_F, sq1 + (a * 3 + 1) * Z2_F, sq1 + (a * 3 + 2) * Z2_F,
                                          sq1 + (an * 3 + 2) * Z2_F, bzm, o, gx0, gy, zz, nx, ny, nz, w));
        }
        __syncthreads();
        // ---- P2: p_{k+1}(z - 1) on the output tile
        if (tile && zz >= zs && zz < ze) {
            const int a = zz & 1, ap = (zz + 1) & 1;   // ap = (zz - 1) & 1
            float pk[3][4];
            z2_p(su1 + a * Z2_F, su1 + ap * Z2_F, sq1 + (a * 3 + 0) * Z2_F, sq1 + (a * 3 + 1) * Z2_F,
                 sq1 + (a * 3 + 2) * Z2_F, o, gx0, gy, zz, s, pk);
            const long long i = (long long)zz * plane + gi;
#pragma unroll
            for (int c = 0; c < 3; ++c) st4(T.Pb + c * T.n + i, pk[c][0], pk[c][1], pk[c][2], pk[c][3]);
        }
    }
}

// float4 form of k_tv_out (nx % 4 == 0): 4 x voxels per lane, in place (b = x is read only at
// the lane's own voxels)
__global__ void __launch_bounds__(256) k_tv_out4(const TvLaunch T, float* out) {
    const int lane = threadIdx.x & 31, row = threadIdx.x >> 5;
    const int x = blockIdx.x * TV4_TX + 4 * lane, y = blockIdx.y * 8 + row, z = T.z0 + blockIdx.z;
    const bool act = x < T.dims[0] && y < T.dims[1];
    float u[4];
    tv_u4(T, tv_plane(T, z), x, y, z, act, T.wf, u);
    if (!act) return;
    const long long i = (long long)blockIdx.z * T.dims[0] * T.dims[1] + (long long)y * T.dims[0] + x;
    st4(out + i, u[0], u[1], u[2], u[3]);
}

// x = b - w grad^T p on a z-slab layout (the final step of the prox): one thread per voxel
__global__ void __launch_bounds__(TV_TX * TV_TY) k_tv_out(const TvLaunch T, float* out) {
    const int x = blockIdx.x * TV_TX + threadIdx.x, y = blockIdx.y * TV_TY + threadIdx.y,
              z = T.z0 + blockIdx.z;
    if (x >= T.dims[0] || y >= T.dims[1]) return;
    const long long i = (long long)blockIdx.z * T.dims[0] * T.dims[1] + (long long)y * T.dims[0] + x;
    out[i] = tv_u_at(T, tv_plane(T, z), x, y, z, T.wf);
}

struct PtrPack {
    const void* p[8];
};

template <class T>
__global__ void __launch_bounds__(256) k_sum_ptrs(T* out, const PtrPack P, int G, long long n) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        T s = static_cast<const T*>(P.p[0])[i];
        for (int g = 1; g < G; ++g) s += static_cast<const T*>(P.p[g])[i];
        out[i] = s;
    }
}

unsigned grid_for(long long n, int per_thread = 1) {
    long long b = (n / per_thread + 255) / 256;
    if (b < 1) b = 1;
    if (b > 148LL * 16) b = 148LL * 16;
    return (unsigned)b;
}

}  // namespace

void launch_block_update(int mode, const UpdLaunch& U, cudaStream_t st) {
    dim3 grid((unsigned)((U.bd[0] + 31) / 32), (unsigned)((U.bd[1] + 31) / 32), (unsigned)U.bd[2]);
    const bool vec = (U.bd[0] % 32 == 0) && (U.bd[1] % 32 == 0) && !(U.out && ((uintptr_t)U.out & 15));
    if (vec) {
        switch (mode) {
            case UPD_BSGD: k_block_update4<UPD_BSGD><<<grid, dim3(8, 32), 0, st>>>(U); break;
            case UPD_SGD: k_block_update4<UPD_SGD><<<grid, dim3(8, 32), 0, st>>>(U); break;
            case UPD_OUT: k_block_update4<UPD_OUT><<<grid, dim3(8, 32), 0, st>>>(U); break;
            default: k_block_update4<UPD_XT><<<grid, dim3(8, 32), 0, st>>>(U); break;
        }
        BSGD_CUDA(cudaGetLastError());
        note_launch();
        return;
    }
    switch (mode) {
        case UPD_BSGD: k_block_update<UPD_BSGD><<<grid, dim3(32, 8), 0, st>>>(U); break;
        case UPD_SGD: k_block_update<UPD_SGD><<<grid, dim3(32, 8), 0, st>>>(U); break;
        case UPD_OUT: k_block_update<UPD_OUT><<<grid, dim3(32, 8), 0, st>>>(U); break;
        default: k_block_update<UPD_XT><<<grid, dim3(32, 8), 0, st>>>(U); break;
    }
    BSGD_CUDA(cudaGetLastError());
    note_launch();
}

void launch_residual(const ResLaunch& R, cudaStream_t st) {
    if (R.n_slots == 0) return;
    long long nvec = (R.per % 4 == 0) ? R.per / 4 : R.per;
    unsigned gx = (unsigned)std::min<long long>((nvec + 255) / 256, RES_GX);
    k_residual<<<dim3(gx, (unsigned)R.n_slots), 256, 0, st>>>(R);
    BSGD_CUDA(cudaGetLastError());
    note_launch();
    if (R.mode != 1) {
        k_normsq_final<<<R.M, 256, 0, st>>>(R, (int)gx);
        BSGD_CUDA(cudaGetLastError());
        note_launch();
    }
}

void launch_normsq_final(const ResLaunch& R, int gx, cudaStream_t st) {
    k_normsq_final<<<R.M, 256, 0, st>>>(R, gx);
    BSGD_CUDA(cudaGetLastError());
    note_launch();
}

void launch_zero_rects(float* proj, const int* views, const int4* rects, int n, int nu, int nv, cudaStream_t st) {
    if (n == 0) return;
    k_zero_rects<<<dim3(64, (unsigned)n), 256, 0, st>>>(proj, views, rects, nu, nv);
    BSGD_CUDA(cudaGetLastError());
    note_launch();
}

void launch_zero_rows(double* normsq, const int* rows, int n, cudaStream_t st) {
    k_zero_rows<<<1, 1024, 0, st>>>(normsq, rows, n);
    BSGD_CUDA(cudaGetLastError());
    note_launch();
}

void launch_obj(const double* normsq, int M, double* out, cudaStream_t st) {
    k_obj<<<1, 32, 0, st>>>(normsq, M, out);
    BSGD_CUDA(cudaGetLastError());
    note_launch();
}

void launch_axpy_eud(float* eud, const float* g, long long n, cudaStream_t st) {
    k_axpy<<<grid_for(n, 4), 256, 0, st>>>(eud, g, n);
    BSGD_CUDA(cudaGetLastError());
    note_launch();
}

void launch_dot3(const float* a, const float* b, long long n, double* out3, cudaStream_t st) {
    k_dot3<<<grid_for(n, 8), 256, 0, st>>>(a, b, n, out3);
    BSGD_CUDA(cudaGetLastError());
    note_launch();
}

void launch_sqdiff(const float* a, const float* b, long long n, double* out, cudaStream_t st) {
    k_sqdiff<<<grid_for(n, 8), 256, 0, st>>>(a, b, n, out);
    BSGD_CUDA(cudaGetLastError());
    note_launch();
}

void launch_lincomb(float* out, float a, const float* x, float b, const float* y, float c, const float* z,
                    long long n, cudaStream_t st) {
    k_lincomb<<<grid_for(n, 4), 256, 0, st>>>(out, a, x, b, y, c, z, n);
    BSGD_CUDA(cudaGetLastError());
    note_launch();
}

void launch_bb_dots(const float* x, const float* xp, const float* gp, const float* g, long long n, double* out2,
                    cudaStream_t st) {
    k_bb_dots<<<grid_for(n, 8), 256, 0, st>>>(x, xp, gp, g, n, out2);
    BSGD_CUDA(cudaGetLastError());
    note_launch();
}

void launch_sqdiff_masked(const float* a, const float* b, const float* mask, long long n, double* out,
                          cudaStream_t st) {
    k_sqdiff_masked<<<grid_for(n, 8), 256, 0, st>>>(a, b, mask, n, out);
    BSGD_CUDA(cudaGetLastError());
    note_launch();
}

void launch_fill(float* v, long long n, float val, cudaStream_t st) {
    k_fill<<<grid_for(n, 4), 256, 0, st>>>(v, n, val);
    BSGD_CUDA(cudaGetLastError());
    note_launch();
}

void launch_fill_random(float* v, long long n, uint64_t seed, cudaStream_t st) {
    k_fill_random<<<grid_for(n, 4), 256, 0, st>>>(v, n, seed);
    BSGD_CUDA(cudaGetLastError());
    note_launch();
}

void launch_scale(float* v, long long n, const double* nrm, cudaStream_t st) {
    k_scale<<<grid_for(n, 4), 256, 0, st>>>(v, n, nrm);
    BSGD_CUDA(cudaGetLastError());
    note_launch();
}

void launch_residual_band(const BandLaunch& B, cudaStream_t st) {
    if (B.n_slots == 0) return;
    k_residual_band<<<dim3(RES_GX, (unsigned)B.n_slots), 256, 0, st>>>(B);
    BSGD_CUDA(cudaGetLastError());
    note_launch();
}

void launch_copy_chunks(const float* src, float* dst, const long long* t, int n, cudaStream_t st) {
    if (n <= 0) return;
    k_copy_chunks<<<dim3(32, (unsigned)n), 256, 0, st>>>(src, dst, t);
    BSGD_CUDA(cudaGetLastError());
    note_launch();
}

void launch_copy_rows(double* dst, const double* src, const int* rows, int n, cudaStream_t st) {
    if (n <= 0) return;
    k_copy_rows<<<1, 1024, 0, st>>>(dst, src, rows, n);
    BSGD_CUDA(cudaGetLastError());
    note_launch();
}

void launch_pack_plane(const TvLaunch& T, const float* owned, int z, float* out, cudaStream_t st) {
    k_pack_plane<<<grid_for((long long)T.dims[0] * T.dims[1], 1), 256, 0, st>>>(T, owned, z, out);
    BSGD_CUDA(cudaGetLastError());
    note_launch();
}

void launch_tv_value(const TvLaunch& T, const float* x, double* out, cudaStream_t st) {
    k_tv_value<<<grid_for(T.n, 4), 256, 0, st>>>(T, x, out);
    BSGD_CUDA(cudaGetLastError());
    note_launch();
}

void launch_tv_u(const TvLaunch& T, const float* src, float* dst, cudaStream_t st) {
    k_tv_u<<<grid_for(T.n, 2), 256, 0, st>>>(T, src, dst);
    BSGD_CUDA(cudaGetLastError());
    note_launch();
}

void launch_sum_ptrs(void* out, const void* const* ptrs, int G, long long n, bool dbl, cudaStream_t st) {
    PtrPack P;
    for (int g = 0; g < 8; ++g) P.p[g] = g < G ? ptrs[g] : nullptr;
    if (dbl) k_sum_ptrs<double><<<grid_for(n, 4), 256, 0, st>>>(static_cast<double*>(out), P, G, n);
    else k_sum_ptrs<float><<<grid_for(n, 4), 256, 0, st>>>(static_cast<float*>(out), P, G, n);
    BSGD_CUDA(cudaGetLastError());
    note_launch();
}

// ---- deterministic BP (PROJ_BPD): the fixed-point scale and the int64 -> fp32 conversion
__global__ void __launch_bounds__(256) k_absmax(const float* r, long long n, unsigned* out) {
    unsigned m = 0;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        m = max(m, __float_as_uint(fabsf(r[i])));          // non-negative floats order as integers
    m = __reduce_max_sync(0xffffffffu, m);
    if ((threadIdx.x & 31) == 0) atomicMax(out, m);         // max is order-independent
}

// S = 2^e with e = floor(log2(2^62 / bound)), bound = V * rpc * sqrt(3) * scale * max|r| >= any
// per-cell sum of |l w r|: at most rpc rays of one view cross a cell (the host's geometric bound,
// bsgd_ctx_s::rays_per_cell), each with a length <= sqrt(3)
__global__ void k_det_scale(const unsigned* mx, int V, double rpc, float scale, float* S) {
    const double rmax = (double)__uint_as_float(*mx);
    const double bound = (double)V * rpc * 1.7320508075688772 * (double)scale * rmax;
    int e = 40;
    if (bound > 0.0 && isfinite(bound)) e = (int)floor(log2(4.611686018427388e18 / bound));
    e = max(-60, min(120, e));
    *S = ldexpf(1.f, e);
}

__global__ void __launch_bounds__(256) k_acc64_to_f32(const long long* a, float* out, long long n, const float* S) {
    const double inv = 1.0 / (double)*S;                    // exact: S is a power of two
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        out[i] += (float)((double)a[i] * inv);
}

void launch_det_scale(const float* r, long long n, int V, double rpc, float scale, unsigned* mx, float* S,
                      cudaStream_t st) {
    BSGD_CUDA(cudaMemsetAsync(mx, 0, sizeof(unsigned), st));
    k_absmax<<<grid_for(n, 8), 256, 0, st>>>(r, n, mx);
    BSGD_CUDA(cudaGetLastError());
    k_det_scale<<<1, 1, 0, st>>>(mx, V, rpc, scale, S);
    BSGD_CUDA(cudaGetLastError());
    note_launch();
    note_launch();
}

void launch_acc64_to_f32(const long long* a, float* out, long long n, const float* S, cudaStream_t st) {
    k_acc64_to_f32<<<grid_for(n, 4), 256, 0, st>>>(a, out, n, S);
    BSGD_CUDA(cudaGetLastError());
    note_launch();
}

void launch_tv_fgp(const TvLaunch& T, cudaStream_t st) {
    if (T.dims[0] % 4 == 0) {   // float4 kernel: 4 x 128 tiles, 6 CTAs per SM (56 registers, no spills)
        constexpr int TY = 4;
        const dim3 g4((unsigned)((T.dims[0] + TV4_TX - 1) / TV4_TX), (unsigned)((T.dims[1] + TY - 1) / TY),
                      (unsigned)(T.z1 - T.z0));
        k_tv_fgp4<TY, 6><<<g4, (TY + 2) * 32, 0, st>>>(T);
    } else {
        const dim3 grid((unsigned)((T.dims[0] + TV_TX - 1) / TV_TX), (unsigned)((T.dims[1] + TV_TY - 1) / TV_TY),
                        (unsigned)(T.z1 - T.z0));
        k_tv_fgp<1><<<grid, TV_THREADS, 0, st>>>(T);
    }
    BSGD_CUDA(cudaGetLastError());
    note_launch();
}

void launch_tv_fgp_z(const TvzLaunch& T, cudaStream_t st) {
    constexpr int TY = 4;
    const int nzl = T.z1 - T.z0;
    const dim3 g((unsigned)((T.nx + TV4_TX - 1) / TV4_TX), (unsigned)((T.ny + TY - 1) / TY),
                 (unsigned)((nzl + T.zc - 1) / T.zc));
    static const int minb = [] {
        const char* e = getenv("BSGD_TV_MINB");
        return e ? atoi(e) : 4;
    }();
    if (minb >= 6) k_tv_fgp_z<TY, 6><<<g, (TY + 2) * 32, 0, st>>>(T);
    else k_tv_fgp_z<TY, 4><<<g, (TY + 2) * 32, 0, st>>>(T);
    BSGD_CUDA(cudaGetLastError());
    note_launch();
}

template <int RH>
static void launch_z2(const Tvz2Launch& T, cudaStream_t st) {
    static const bool attr = [] {
        BSGD_CUDA(cudaFuncSetAttribute(k_tv_fgp_z2<RH>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)z2_smem<RH>()));
        return true;
    }();
    (void)attr;
    const dim3 g((unsigned)((T.nx + Z2_W - 1) / Z2_W), (unsigned)((T.ny + RH - 5) / (RH - 4)),
                 (unsigned)((T.nz + T.zc - 1) / T.zc));
    k_tv_fgp_z2<RH><<<g, z2_threads<RH>(), z2_smem<RH>(), st>>>(T);
    BSGD_CUDA(cudaGetLastError());
    note_launch();
}

void launch_tv_fgp_z2(const Tvz2Launch& T, cudaStream_t st) {
    // region height (output rows + 4 halo rows); A/B hook BSGD_TV_Z2H
    static const int rh = [] {
        const char* e = getenv("BSGD_TV_Z2H");
        return e ? atoi(e) : 16;
    }();
    if (rh >= 24) launch_z2<24>(T, st);
    else launch_z2<16>(T, st);
}

__global__ void k_lsa_ptrs(ncclWindow_t w, int n, void** out) {
    const int h = threadIdx.x;
    if (h < n) out[h] = ncclGetPeerPointer(w, 0, h);
}

void launch_lsa_ptrs(void* w, int n, void** out, cudaStream_t st) {
    k_lsa_ptrs<<<1, 32, 0, st>>>((ncclWindow_t)w, n, out);
    BSGD_CUDA(cudaGetLastError());
    note_launch();
}

void launch_tv_out(const TvLaunch& T, float* out, cudaStream_t st) {
    const dim3 grid((unsigned)((T.dims[0] + TV_TX - 1) / TV_TX), (unsigned)((T.dims[1] + TV_TY - 1) / TV_TY),
                    (unsigned)(T.z1 - T.z0));
    if (T.dims[0] % 4 == 0) {
        const dim3 g4((unsigned)((T.dims[0] + TV4_TX - 1) / TV4_TX), (unsigned)((T.dims[1] + 7) / 8),
                      (unsigned)(T.z1 - T.z0));
        k_tv_out4<<<g4, 256, 0, st>>>(T, out);
    } else {
        k_tv_out<<<grid, dim3(TV_TX, TV_TY), 0, st>>>(T, out);
    }
    BSGD_CUDA(cudaGetLastError());
    note_launch();
}

void launch_tv_pq(const TvLaunch& T, cudaStream_t st) {
    k_tv_pq<<<grid_for(T.n, 2), 256, 0, st>>>(T);
    BSGD_CUDA(cudaGetLastError());
    note_launch();
}

}  // namespace bsgd
