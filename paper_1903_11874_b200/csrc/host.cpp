// Host-side pieces of the hot path: scan geometry, the counter RNG and the
// block selection (Algo 1 line 3), the row-block partition
// (PAPER.md:449), Eq. 8 and the importance draw (Algo 2
// line 5).  Integer work; bit-exact with the oracle's
// independent Python implementation (tests/test_capi_host.py).
#include <math.h>
#include <string.h>

#include <algorithm>
#include <numeric>
#include <vector>

#include "internal.h"

namespace bsgd {
namespace host {

// cos/sin in degrees, exact at multiples of 90 degrees.
void cos_sin_deg(double theta, double* c, double* s) {
    double t = fmod(theta, 360.0);
    if (t < 0.0) t += 360.0;
    int k = (int)floor(t / 90.0);
    double r = t - 90.0 * k;
    if (r < 0.0) { k -= 1; r = t - 90.0 * k; }
    if (r >= 90.0) { k += 1; r = t - 90.0 * k; }
    double cc, ss;
    if (r == 0.0) {
        cc = 1.0;
        ss = 0.0;
    } else {
        double rad = r * (M_PI / 180.0);
        cc = cos(rad);
        ss = sin(rad);
    }
    for (int q = 0; q < k; ++q) {
        double nc = -ss, ns = cc;
        cc = nc;
        ss = ns;
    }
    *c = cc;
    *s = ss;
}

void circular(int beam, int n_views, double arc, double OP, double OD, int nu, int nv, double pu,
              double pv, double* out) {
    (void)nu;
    (void)nv;
    for (int v = 0; v < n_views; ++v) {
        double th = v * arc / n_views, c, s;
        cos_sin_deg(th, &c, &s);
        double* o = out + 12 * (size_t)v;
        if (beam == BSGD_PARALLEL) {
            o[0] = -c; o[1] = -s; o[2] = 0.0;
            o[3] = 0.0; o[4] = 0.0; o[5] = 0.0;
        } else {
            o[0] = OP * c; o[1] = OP * s; o[2] = 0.0;
            o[3] = -OD * c; o[4] = -OD * s; o[5] = 0.0;
        }
        o[6] = pu * -s; o[7] = pu * c; o[8] = 0.0;
        o[9] = 0.0; o[10] = 0.0; o[11] = pv;
    }
}

uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

uint64_t rnd(uint64_t seed, uint32_t stream, uint32_t epoch, uint32_t k) {
    uint64_t ctr = ((uint64_t)stream << 48) | ((uint64_t)epoch << 24) | (uint64_t)k;
    return mix64(seed + (ctr + 1) * 0x9E3779B97F4A7C15ull);
}

uint32_t bounded(uint64_t u, uint32_t n) { return (uint32_t)(((u >> 32) * (uint64_t)n) >> 32); }

void select(uint64_t seed, int stream, int epoch, int n, int m, int32_t* out) {
    std::vector<int32_t> a(n);
    std::iota(a.begin(), a.end(), 0);
    for (int i = 0; i < m; ++i) {
        int j = i + (int)bounded(rnd(seed, stream, epoch, i), (uint32_t)(n - i));
        std::swap(a[i], a[j]);
    }
    std::sort(a.begin(), a.begin() + m);
    memcpy(out, a.data(), sizeof(int32_t) * m);
}

void select_stratified(uint64_t seed, int epoch, int n, int m, int strata, int32_t* out) {
    const int ns = n / strata, ms = m / strata;
    std::vector<int32_t> a(ns);
    for (int s = 0; s < strata; ++s) {
        std::iota(a.begin(), a.end(), 0);
        for (int i = 0; i < ms; ++i) {
            int j = i + (int)bounded(rnd(seed, 2, epoch, s * ns + i), (uint32_t)(ns - i));
            std::swap(a[i], a[j]);
        }
        std::sort(a.begin(), a.begin() + ms);
        for (int i = 0; i < ms; ++i) out[s * ms + i] = s * ns + a[i];
    }
}

void view_partition(int n_views, int M, int kind, uint64_t seed, int32_t* views, int32_t* offsets) {
    std::vector<int32_t> order(n_views);
    std::iota(order.begin(), order.end(), 0);
    if (kind == 0) {
        for (int i = 0; i < n_views; ++i) {
            int j = i + (int)bounded(rnd(seed, 0, 0, i), (uint32_t)(n_views - i));
            std::swap(order[i], order[j]);
        }
    }
    int pos = 0;
    offsets[0] = 0;
    if (kind == 2) {  // interleaved
        for (int i = 0; i < M; ++i) {
            for (int v = i; v < n_views; v += M) views[pos++] = v;
            offsets[i + 1] = pos;
        }
        return;
    }
    int base = n_views / M, extra = n_views % M, s = 0;
    for (int i = 0; i < M; ++i) {
        int c = base + (i < extra ? 1 : 0);
        std::vector<int32_t> chunk(order.begin() + s, order.begin() + s + c);
        std::sort(chunk.begin(), chunk.end());
        for (int v : chunk) views[pos++] = v;
        s += c;
        offsets[i + 1] = pos;
    }
}

void eq8(int nodes, int M, int N, int* aM, int* gN) {
    double gamma = std::min(1.0, (double)nodes / N);
    double alpha = (double)nodes / (M * N * gamma);
    int a = std::max(1, (int)floor(alpha * M + 0.5));
    int g = std::max(1, (int)floor(gamma * N + 0.5));
    *aM = std::min(a, M);
    *gN = std::min(g, N);
}

int im_draw(uint64_t seed, int epoch, uint32_t k, const uint32_t* q, int T, bool uniform) {
    uint64_t u = rnd(seed, 3, (uint32_t)epoch, k);
    uint64_t S = 0;
    if (!uniform)
        for (int t = 0; t < T; ++t) S += q[t];
    if (uniform || S == 0) return (int)bounded(u, (uint32_t)T);
    uint32_t x = bounded(u, (uint32_t)S);
    uint64_t c = 0;
    for (int t = 0; t < T; ++t) {
        c += q[t];
        if (x < c) return t;
    }
    return T - 1;
}

}  // namespace host
}  // namespace bsgd
