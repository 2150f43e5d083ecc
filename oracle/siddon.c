/*
 * ORACLE — test infrastructure only.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.  It
 * shares no code with the CUDA path (paper_1903_11874_b200/) and never calls it.
 *
 * Plain, slow, fp64 implementation of the system matrix A of the paper,
 *   y = A x + e, "A ... has non-negative elements, which can be computed using
 *   Siddon's method"                       (§I, Eq. 1 `yax`)
 * applied "on the fly" (never stored at scale)   (§I)
 * to the sub-matrices A_I^J of the block partition  (§II, Eq. 3).
 *
 * Siddon is written in its ORIGINAL merged-alpha form (Siddon 1985, cited by the
 * paper through jacobs1998fast): the ray p(alpha) = a + alpha*b,
 * alpha in [0,1], is clipped against the block box; the alpha values of every
 * voxel-plane crossing strictly inside the clip interval are generated per axis
 * and merged in increasing order; each gap between consecutive alphas is one
 * voxel segment whose voxel is floor(p(midpoint)) (this midpoint rule makes the
 * voxel intervals half-open [lo, hi)) and whose length is
 * (alpha_{k+1} - alpha_k) * |b|.  Zero-length gaps are dropped.
 * Coordinates are GRID coordinates: voxel (ix,iy,iz) = [ix,ix+1)x[iy,iy+1)x[iz,iz+1).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define PARALLEL 0

/* Ray (view, iv, iu) in grid coordinates.  Pixel centre
 *   d = det + (iu - (nu-1)/2) u + (iv - (nv-1)/2) v
 * fan/cone: a = src, b = d - src; parallel: a = d - R dir, b = 2 R dir with
 * R = |volume diagonal|/2 + 1.  Grid = world + n/2.     */
void oracle_ray(int beam, const double *vec, int nu, int nv, int iu, int iv,
                const int *dims, double *a, double *b)
{
    double ou = (double)iu - (nu - 1) / 2.0, ov = (double)iv - (nv - 1) / 2.0;
    double d[3];
    for (int c = 0; c < 3; ++c)
        d[c] = vec[3 + c] + ou * vec[6 + c] + ov * vec[9 + c];
    if (beam == PARALLEL) {
        double R = 0.5 * sqrt((double)dims[0] * dims[0] + (double)dims[1] * dims[1] +
                              (double)dims[2] * dims[2]) + 1.0;
        for (int c = 0; c < 3; ++c) {
            a[c] = d[c] - R * vec[c];
            b[c] = 2.0 * R * vec[c];
        }
    } else {
        for (int c = 0; c < 3; ++c) {
            a[c] = vec[c];
            b[c] = d[c] - vec[c];
        }
    }
    for (int c = 0; c < 3; ++c) a[c] += dims[c] / 2.0;
}

/* Merged-alpha Siddon through the box [lo, hi) (grid coords).  Writes up to
 * `cap` segments (block-local voxel index z-y-x, length) and returns how many
 * (or the count needed if it exceeds cap; callers size cap generously).     */
int oracle_trace(const double *a, const double *b, const int *lo, const int *hi,
                 int64_t *idx, double *len, int cap)
{
    double amin = 0.0, amax = 1.0;
    for (int c = 0; c < 3; ++c) {
        if (b[c] == 0.0) {
            if (!(a[c] >= lo[c] && a[c] < hi[c])) return 0;  /* half-open in-plane rule */
        } else {
            double t0 = (lo[c] - a[c]) / b[c], t1 = (hi[c] - a[c]) / b[c];
            if (t0 > t1) { double t = t0; t0 = t1; t1 = t; }
            if (t0 > amin) amin = t0;
            if (t1 < amax) amax = t1;
        }
    }
    if (!(amin < amax)) return 0;

    /* per-axis arithmetic sequence of plane crossings, increasing in alpha */
    long k[3], kend[3], kstep[3];
    int active[3];
    for (int c = 0; c < 3; ++c) {
        active[c] = 0;
        if (b[c] == 0.0) continue;
        double c0 = a[c] + amin * b[c], c1 = a[c] + amax * b[c];
        double lo_c = fmin(c0, c1), hi_c = fmax(c0, c1);
        long kl = (long)floor(lo_c) - 1, kh = (long)ceil(hi_c) + 1;
        if (b[c] > 0) { k[c] = kl; kend[c] = kh + 1; kstep[c] = 1; }
        else          { k[c] = kh; kend[c] = kl - 1; kstep[c] = -1; }
        active[c] = 1;
    }
    double blen = sqrt(b[0] * b[0] + b[1] * b[1] + b[2] * b[2]);
    int bx = hi[0] - lo[0], by = hi[1] - lo[1];
    int n = 0;
    double prev = amin;
    for (;;) {
        /* next crossing alpha strictly greater than prev on each axis */
        double nxt = amax;
        for (int c = 0; c < 3; ++c) {
            if (!active[c]) continue;
            while (k[c] != kend[c] && (k[c] - a[c]) / b[c] <= prev) k[c] += kstep[c];
            if (k[c] == kend[c]) { active[c] = 0; continue; }
            double al = (k[c] - a[c]) / b[c];
            if (al < nxt) nxt = al;
        }
        if (nxt > prev) {
            double mid = 0.5 * (prev + nxt);
            long ii[3];
            for (int c = 0; c < 3; ++c) {
                long i = (long)floor(a[c] + mid * b[c]);
                if (i < lo[c]) i = lo[c];          /* rounding guard for sub-1e-12 segments */
                if (i > hi[c] - 1) i = hi[c] - 1;
                ii[c] = i - lo[c];
            }
            if (n < cap) {
                idx[n] = ((int64_t)ii[2] * by + ii[1]) * bx + ii[0];
                len[n] = (nxt - prev) * blen;
            }
            ++n;
            prev = nxt;
        }
        if (nxt >= amax) break;
    }
    return n;
}

/* ---- helpers over a list of views and optional per-view detector rects ----
 * rects: per listed view (u0, u1, v0, v1) half-open, or NULL for the whole
 * detector.  proj arrays are FULL length (n_views_total * nv * nu) indexed by
 * the global ray id (view*nv + iv)*nu + iu.                                 */
typedef struct {
    int beam, nu, nv;
    const double *vecs;
    const int *dims;
    const int *lo, *hi;
} og_t;

#define SEGCAP 16384

static void rect_of(const int *rects, int s, int nu, int nv, int *r)
{
    if (rects) { r[0] = rects[4 * s]; r[1] = rects[4 * s + 1]; r[2] = rects[4 * s + 2]; r[3] = rects[4 * s + 3]; }
    else { r[0] = 0; r[1] = nu; r[2] = 0; r[3] = nv; }
}

/* z_I^J = A_I^J x_J   (Algo 1 line 5).  Writes (or adds) to proj. */
void oracle_fp(int beam, const double *vecs, int nu, int nv, const int *dims,
               const int *lo, const int *hi, const int *views, int n_sel, const int *rects,
               const double *xblk, double *proj, int accumulate)
{
    for (int s = 0; s < n_sel; ++s) {
        int r[4];
        rect_of(rects, s, nu, nv, r);
        int view = views[s];
        int w = r[1] - r[0], h = r[3] - r[2];
        #pragma omp parallel for schedule(dynamic, 64)
        for (long q = 0; q < (long)w * h; ++q) {
            int iu = r[0] + (int)(q % w), iv = r[2] + (int)(q / w);
            double a[3], b[3];
            int64_t idx[SEGCAP];
            double len[SEGCAP];
            oracle_ray(beam, vecs + 12 * (long)view, nu, nv, iu, iv, dims, a, b);
            int n = oracle_trace(a, b, lo, hi, idx, len, SEGCAP);
            if (n > SEGCAP) abort();
            double acc = 0.0;
            for (int t = 0; t < n; ++t) acc += len[t] * xblk[idx[t]];
            long ray = ((long)view * nv + iv) * nu + iu;
            if (accumulate) proj[ray] += acc; else proj[ray] = acc;
        }
    }
}

/* g_J += (A_I^J)^T r_I   (Algo 1 line 9, without the factor 2,
 * which the caller applies).  Scatter with fp64 atomics (order-independent up
 * to fp64 rounding).                                                         */
void oracle_bp(int beam, const double *vecs, int nu, int nv, const int *dims,
               const int *lo, const int *hi, const int *views, int n_sel, const int *rects,
               const double *proj, double *gblk)
{
    for (int s = 0; s < n_sel; ++s) {
        int r[4];
        rect_of(rects, s, nu, nv, r);
        int view = views[s];
        int w = r[1] - r[0], h = r[3] - r[2];
        #pragma omp parallel for schedule(dynamic, 64)
        for (long q = 0; q < (long)w * h; ++q) {
            int iu = r[0] + (int)(q % w), iv = r[2] + (int)(q / w);
            double a[3], b[3];
            int64_t idx[SEGCAP];
            double len[SEGCAP];
            long ray = ((long)view * nv + iv) * nu + iu;
            double rv = proj[ray];
            if (rv == 0.0) continue;
            oracle_ray(beam, vecs + 12 * (long)view, nu, nv, iu, iv, dims, a, b);
            int n = oracle_trace(a, b, lo, hi, idx, len, SEGCAP);
            if (n > SEGCAP) abort();
            for (int t = 0; t < n; ++t) {
                #pragma omp atomic
                gblk[idx[t]] += len[t] * rv;
            }
        }
    }
}

/* Ones-pass per detector tile: w[s*T + t] = sum over rays of tile t of
 * sum of segment lengths through the box (= (A_tile^J 1) summed), the block
 * weight of BSGD-IM (§II-A; SURVEY §8c A9 reading).  With
 * area != 0: the number of tile rays whose chord through the box exceeds 1e-6
 * (the "fraction of a volume block's projection area", IS_AREA).           */
void oracle_tile_mass(int beam, const double *vecs, int nu, int nv, const int *dims,
                      const int *lo, const int *hi, const int *views, int n_sel,
                      int tiles_u, int tiles_v, int area, double *w)
{
    int T = tiles_u * tiles_v;
    for (int s = 0; s < n_sel; ++s) {
        int view = views[s];
        for (int t = 0; t < T; ++t) {
            int tu = t % tiles_u, tv = t / tiles_u;
            int u0 = (int)((long)tu * nu / tiles_u), u1 = (int)((long)(tu + 1) * nu / tiles_u);
            int v0 = (int)((long)tv * nv / tiles_v), v1 = (int)((long)(tv + 1) * nv / tiles_v);
            double sum = 0.0;
            #pragma omp parallel for reduction(+:sum) schedule(dynamic, 64)
            for (long q = 0; q < (long)(u1 - u0) * (v1 - v0); ++q) {
                int iu = u0 + (int)(q % (u1 - u0)), iv = v0 + (int)(q / (u1 - u0));
                double a[3], b[3];
                int64_t idx[SEGCAP];
                double len[SEGCAP];
                oracle_ray(beam, vecs + 12 * (long)view, nu, nv, iu, iv, dims, a, b);
                int n = oracle_trace(a, b, lo, hi, idx, len, SEGCAP);
                double chord = 0.0;
                for (int k = 0; k < n; ++k) chord += len[k];
                /* area mode: the ray belongs to the block's shadow (reading A9, threshold
                 * 1e-6 voxel so that corner touches do not count)                        */
                sum += area ? (chord > 1e-6 ? 1.0 : 0.0) : chord;
            }
            w[(long)s * T + t] = sum;
        }
    }
}

/* Explicit CSR of A_I^J: rows = every ray of the listed views (view order,
 * then iv, iu), columns = block-local voxel index.  Two passes.            */
void oracle_csr_count(int beam, const double *vecs, int nu, int nv, const int *dims,
                      const int *lo, const int *hi, const int *views, int n_sel, int64_t *rowcnt)
{
    long per = (long)nu * nv;
    #pragma omp parallel for schedule(dynamic, 64)
    for (long q = 0; q < per * n_sel; ++q) {
        int s = (int)(q / per);
        long p = q % per;
        int iu = (int)(p % nu), iv = (int)(p / nu);
        double a[3], b[3];
        int64_t idx[SEGCAP];
        double len[SEGCAP];
        oracle_ray(beam, vecs + 12 * (long)views[s], nu, nv, iu, iv, dims, a, b);
        rowcnt[q] = oracle_trace(a, b, lo, hi, idx, len, SEGCAP);
    }
}

void oracle_csr_fill(int beam, const double *vecs, int nu, int nv, const int *dims,
                     const int *lo, const int *hi, const int *views, int n_sel,
                     const int64_t *indptr, int64_t *indices, double *data)
{
    long per = (long)nu * nv;
    #pragma omp parallel for schedule(dynamic, 64)
    for (long q = 0; q < per * n_sel; ++q) {
        int s = (int)(q / per);
        long p = q % per;
        int iu = (int)(p % nu), iv = (int)(p / nu);
        double a[3], b[3];
        oracle_ray(beam, vecs + 12 * (long)views[s], nu, nv, iu, iv, dims, a, b);
        int cap = (int)(indptr[q + 1] - indptr[q]);
        oracle_trace(a, b, lo, hi, indices + indptr[q], data + indptr[q], cap);
    }
}

/* Count of segments (non-zeros a_ij) over the listed views, optional rects. */
int64_t oracle_count(int beam, const double *vecs, int nu, int nv, const int *dims,
                     const int *lo, const int *hi, const int *views, int n_sel, const int *rects)
{
    int64_t total = 0;
    for (int s = 0; s < n_sel; ++s) {
        int r[4];
        rect_of(rects, s, nu, nv, r);
        int w = r[1] - r[0], h = r[3] - r[2];
        int64_t sub = 0;
        #pragma omp parallel for reduction(+:sub) schedule(dynamic, 64)
        for (long q = 0; q < (long)w * h; ++q) {
            int iu = r[0] + (int)(q % w), iv = r[2] + (int)(q / w);
            double a[3], b[3];
            int64_t idx[SEGCAP];
            double len[SEGCAP];
            oracle_ray(beam, vecs + 12 * (long)views[s], nu, nv, iu, iv, dims, a, b);
            sub += oracle_trace(a, b, lo, hi, idx, len, SEGCAP);
        }
        total += sub;
    }
    return total;
}
