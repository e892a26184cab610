// update.cu — K14: the squared-Hellinger trust-region step.
//
// K14a, one thread per splat, reads its 14 coordinates of x, g, g-hat, D-hat
// (and z.w on refresh steps) once and writes g-hat, D-hat and, for the ten
// non-rotation coordinates, the clamped x:
//   g     = g_acc * M/(m|S1|)                     (optimizer.cpp:58-59)
//   g_hat = theta1 g_hat + (1-theta1) g           (optimizer.hpp:119-122)
//   D_hat = theta2 D_hat + (1-theta2) d  [refresh] (optimizer.cpp:212)
//   dx    = -g_hat / max(D_hat, gamma)            (optimizer.cpp:106-112)
//   eta   = shd_radii(x, eps)                     (trust_region.cpp:236-252)
//   x'    = clamp(x + clip(dx, eta))              (optimizer.cpp:124-142,
//                                                  scene.cpp:49-57)
// The four rotation coordinates wait for their certified radii (K14a' per
// (splat, axis), K14b's bisections of the failures) and are clipped and
// applied by K14c.  The step diagnostics are deterministic block partials.
// Compiled with --fmad=false so every expression rounds like the oracle.
#include <math_constants.h>

#include <cfloat>
#include <climits>

#include "common.cuh"
#include "geometry.cuh"
#include "launch.h"

namespace sgtr {
namespace {

constexpr int kThreads = 128;

__device__ __forceinline__ double cap_radius(double r, double cap) {
    if (!(r > 0.0) || !isfinite(r)) return cap;
    return cap < r ? cap : r;  // std::min(r, cap)
}

__device__ __forceinline__ double log_factor(double eps, double alpha) {
    const double u = eps / alpha;
    if (u >= 1.0 - 1e-12) return -1.0;
    return -8.0 * log1p(-u);
}

__device__ __forceinline__ double det3(const double* m) {
    return m[0] * (m[4] * m[8] - m[5] * m[7]) - m[1] * (m[3] * m[8] - m[5] * m[6]) +
           m[2] * (m[3] * m[7] - m[4] * m[6]);
}

struct Prim {
    double mu[3], s[3], q[4], alpha, c[3];
};

__device__ __forceinline__ void set9(double* d, double a0, double a1, double a2, double a3,
                                     double a4, double a5, double a6, double a7, double a8) {
    d[0] = a0; d[1] = a1; d[2] = a2; d[3] = a3; d[4] = a4;
    d[5] = a5; d[6] = a6; d[7] = a7; d[8] = a8;
}

// dR~/dq_c (trust_region.cpp:95-117)
__device__ __forceinline__ void quat_drt(double x, double y, double z, double w, int axis,
                                         double* d) {
    switch (axis) {
        case 0: set9(d, 2 * x, 2 * y, 2 * z, 2 * y, -2 * x, -2 * w, 2 * z, 2 * w, -2 * x); break;
        case 1: set9(d, -2 * y, 2 * x, 2 * w, 2 * x, 2 * y, 2 * z, -2 * w, 2 * z, -2 * y); break;
        case 2: set9(d, -2 * z, -2 * w, 2 * x, 2 * w, -2 * z, 2 * y, 2 * x, 2 * y, 2 * z); break;
        default: set9(d, 2 * w, -2 * z, 2 * y, 2 * z, 2 * w, -2 * x, -2 * y, 2 * x, 2 * w); break;
    }
}

// trust_region.cpp:54-69 (inverse diagonal by cofactors)
__device__ void radius_mean(const Prim& p, double eps, double cap, double* out) {
    const double lf = log_factor(eps, p.alpha);
    if (lf <= 0.0) {
        out[0] = out[1] = out[2] = cap;
        return;
    }
    double m[9];
    if (!covariance(p.s, p.q, m)) {
        out[0] = out[1] = out[2] = cap;
        return;
    }
    const double c00 = m[4] * m[8] - m[5] * m[7];
    const double c10 = m[7] * m[2] - m[8] * m[1];
    const double c20 = m[1] * m[5] - m[2] * m[4];
    const double det = c00 * m[0] + c10 * m[3] + c20 * m[6];
    const double invdet = 1.0 / det;
    const double c11 = m[8] * m[0] - m[6] * m[2];
    const double c22 = m[0] * m[4] - m[1] * m[3];
    out[0] = cap_radius(sqrt(lf / (c00 * invdet)), cap);
    out[1] = cap_radius(sqrt(lf / (c11 * invdet)), cap);
    out[2] = cap_radius(sqrt(lf / (c22 * invdet)), cap);
}

// trust_region.cpp:95-155
__device__ double beta_rotation(const Prim& p, int axis) {
    const double x = p.q[0], y = p.q[1], z = p.q[2], w = p.q[3];
    const double r2 = x * x + y * y + z * z + w * w;
    const double qc = axis == 0 ? x : (axis == 1 ? y : (axis == 2 ? z : w));
    const double rt[9] = {r2 - 2.0 * (y * y + z * z), 2.0 * (x * y - w * z),
                          2.0 * (x * z + w * y),      2.0 * (x * y + w * z),
                          r2 - 2.0 * (z * z + x * x), 2.0 * (y * z - w * x),
                          2.0 * (x * z - w * y),      2.0 * (y * z + w * x),
                          r2 - 2.0 * (x * x + y * y)};
    double drt[9];
    quat_drt(x, y, z, w, axis, drt);
    double d2rt[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    d2rt[0] = (axis == 0 || axis == 3) ? 2.0 : -2.0;
    d2rt[4] = (axis == 1 || axis == 3) ? 2.0 : -2.0;
    d2rt[8] = (axis == 2 || axis == 3) ? 2.0 : -2.0;
    // reciprocals instead of the reference's per-entry divisions (same
    // quantities; rounding-level differences only)
    const double ir2 = 1.0 / r2, ir4 = ir2 * ir2;
    double r[9];
    for (int i = 0; i < 9; ++i) r[i] = rt[i] * ir2;
    const double k1 = 2.0 * qc * ir4;
    const double k2 = 4.0 * qc * ir4;
    const double k3 = 8.0 * qc * qc * ir4 * ir2 - 2.0 * ir4;
    double in1[9], in2[9];
    for (int i = 0; i < 9; ++i) {
        in1[i] = drt[i] * ir2 - k1 * rt[i];
        in2[i] = d2rt[i] * ir2 - k2 * drt[i] + k3 * rt[i];
    }
    const double is[3] = {1.0 / p.s[0], 1.0 / p.s[1], 1.0 / p.s[2]};
    double frob = 0.0, tr = 0.0;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            const double de = r[i] * in1[j] + r[3 + i] * in1[3 + j] + r[6 + i] * in1[6 + j];
            const double v = p.s[i] * de * is[j];
            frob += v * v;
        }
    // trace of r^T in2, summed over the diagonal in order
    for (int i = 0; i < 3; ++i)
        tr += r[i] * in2[i] + r[3 + i] * in2[3 + i] + r[6 + i] * in2[6 + i];
    return 2.0 * frob + 2.0 * tr;
}

// Rotation-only squared Hellinger (trust_region.cpp:183-194) as a function of
// dq along axis c, evaluated from per-axis precomputed terms: R~(q + dq e_c)
// = R~(q) + dq dR~/dq_c + dq^2 diag(d2R~/dq_c^2)/2 exactly (R~ is quadratic),
// and R^T S^2 R = R~^T S^2 R~ / |q'|^4.  Same quantity as the reference's
// covariance() path with one division instead of nine; differences are at the
// rounding level of the 1 - det_s/sqrt(det) cancellation the reference has too.
struct RotAxis {
    double rt[9], drt[9], h[3];
    double r2, qc, s2[3], sigma[9], det_s, alpha;
};

__device__ void rot_axis_setup(const Prim& p, const double* sigma, int axis, RotAxis& ra) {
    const double x = p.q[0], y = p.q[1], z = p.q[2], w = p.q[3];
    ra.r2 = x * x + y * y + z * z + w * w;
    ra.qc = axis == 0 ? x : (axis == 1 ? y : (axis == 2 ? z : w));
    const double rt[9] = {ra.r2 - 2.0 * (y * y + z * z), 2.0 * (x * y - w * z),
                          2.0 * (x * z + w * y),         2.0 * (x * y + w * z),
                          ra.r2 - 2.0 * (z * z + x * x), 2.0 * (y * z - w * x),
                          2.0 * (x * z - w * y),         2.0 * (y * z + w * x),
                          ra.r2 - 2.0 * (x * x + y * y)};
    for (int i = 0; i < 9; ++i) ra.rt[i] = rt[i];
    quat_drt(x, y, z, w, axis, ra.drt);
    // diag(d2R~/dq_c^2) / 2 (trust_region.cpp:119-128)
    ra.h[0] = (axis == 0 || axis == 3) ? 1.0 : -1.0;
    ra.h[1] = (axis == 1 || axis == 3) ? 1.0 : -1.0;
    ra.h[2] = (axis == 2 || axis == 3) ? 1.0 : -1.0;
    for (int i = 0; i < 3; ++i) ra.s2[i] = p.s[i] * p.s[i];
    for (int i = 0; i < 9; ++i) ra.sigma[i] = sigma[i];
    ra.det_s = p.s[0] * p.s[1] * p.s[2];
    ra.alpha = p.alpha;
}

// rotation-only H^2 at quaternion offset dq along the axis.  This TU is
// compiled without FMA contraction (bit-exact projection-side arithmetic);
// here the products are fused explicitly: the certification and the 60-step
// bisection evaluate it ~100 times per queued axis, and its ~1e-8 relative
// floor (the 1 - det_s / sqrt(det) cancellation) is far above the rounding
// the fusion changes.
__device__ double rot_h2(const RotAxis& ra, double dq) {
    const double r2p = __fma_rn(dq, 2.0 * ra.qc + dq, ra.r2);
    if (r2p < 1e-24) return CUDART_INF;
    const double dq2 = dq * dq;
    double m[9];
#pragma unroll
    for (int i = 0; i < 9; ++i) m[i] = __fma_rn(dq, ra.drt[i], ra.rt[i]);
    m[0] = __fma_rn(dq2, ra.h[0], m[0]);
    m[4] = __fma_rn(dq2, ra.h[1], m[4]);
    m[8] = __fma_rn(dq2, ra.h[2], m[8]);
    const double inv = 1.0 / (r2p * r2p);
    double ms[9];  // m[3a + i] * s_a^2
#pragma unroll
    for (int a3 = 0; a3 < 3; ++a3)
#pragma unroll
        for (int i = 0; i < 3; ++i) ms[3 * a3 + i] = m[3 * a3 + i] * ra.s2[a3];
    double c[6];  // (R~^T S^2 R~)_{00,01,02,11,12,22}
    const int ij[6][2] = {{0, 0}, {0, 1}, {0, 2}, {1, 1}, {1, 2}, {2, 2}};
#pragma unroll
    for (int e = 0; e < 6; ++e) {
        const int i = ij[e][0], j = ij[e][1];
        double t = ms[i] * m[j];
        t = __fma_rn(ms[3 + i], m[3 + j], t);
        t = __fma_rn(ms[6 + i], m[6 + j], t);
        c[e] = t * inv;
    }
    const double mid[9] = {0.5 * (ra.sigma[0] + c[0]), 0.5 * (ra.sigma[1] + c[1]),
                           0.5 * (ra.sigma[2] + c[2]), 0.5 * (ra.sigma[3] + c[1]),
                           0.5 * (ra.sigma[4] + c[3]), 0.5 * (ra.sigma[5] + c[4]),
                           0.5 * (ra.sigma[6] + c[2]), 0.5 * (ra.sigma[7] + c[4]),
                           0.5 * (ra.sigma[8] + c[5])};
    const double d0 = __fma_rn(mid[4], mid[8], -(mid[5] * mid[7]));
    const double d1 = __fma_rn(mid[3], mid[8], -(mid[5] * mid[6]));
    const double d2 = __fma_rn(mid[3], mid[7], -(mid[4] * mid[6]));
    const double dm = __fma_rn(mid[2], d2, __fma_rn(mid[0], d0, -(mid[1] * d1)));
    if (!(dm > 0.0)) return CUDART_INF;
    return ra.alpha * (1.0 - ra.det_s * rsqrt(dm));
}

// Sigma = R^T diag(s^2) R with R = R~(q) * (1/|q|^2): the covariance of
// geometry.cuh with one division instead of nine (rotation certification only)
__device__ bool cov_fast(const double* s, const double* q, double* cov) {
    const double x = q[0], y = q[1], z = q[2], w = q[3];
    const double r2 = x * x + y * y + z * z + w * w;
    if (r2 < 1e-24) return false;
    const double ir2 = 1.0 / r2;
    const double r[9] = {(r2 - 2.0 * (y * y + z * z)) * ir2, 2.0 * (x * y - w * z) * ir2,
                         2.0 * (x * z + w * y) * ir2,         2.0 * (x * y + w * z) * ir2,
                         (r2 - 2.0 * (z * z + x * x)) * ir2, 2.0 * (y * z - w * x) * ir2,
                         2.0 * (x * z - w * y) * ir2,         2.0 * (y * z + w * x) * ir2,
                         (r2 - 2.0 * (x * x + y * y)) * ir2};
    const double s2[3] = {s[0] * s[0], s[1] * s[1], s[2] * s[2]};
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j)
            cov[3 * i + j] = r[i] * s2[0] * r[j] + r[3 + i] * s2[1] * r[3 + j] +
                             r[6 + i] * s2[2] * r[6 + j];
    return true;
}

__device__ __forceinline__ bool rot_within(const RotAxis& ra, double st, double tol) {
    return rot_h2(ra, st) <= tol && rot_h2(ra, -st) <= tol;
}

// the reference's 60-step bisection down to the constraint boundary
__device__ double rot_bisect(const RotAxis& ra, double r, double tol) {
    double lo = 0.0, hi = r;
    for (int it = 0; it < 60; ++it) {
        const double mid = 0.5 * (lo + hi);
        // once mid rounds onto an endpoint the remaining iterations cannot
        // move lo: the reference's 60-step result is reached
        if (mid == lo || mid == hi) break;
        if (rot_within(ra, mid, tol))
            lo = mid;
        else
            hi = mid;
    }
    return lo > 0.0 ? lo : r * 0x1.0p-60;
}

__device__ void radii(const Prim& p, double eps, const double* caps, double* eta) {
    radius_mean(p, eps, caps[0], eta);
    for (int c = 0; c < 3; ++c) {
        eta[3 + c] = cap_radius(sqrt(2.0 * p.s[c] * p.s[c] * eps / p.alpha), caps[1]);
        eta[11 + c] = cap_radius(sqrt(4.0 * p.c[c] * eps / p.alpha), caps[4]);
    }
    eta[10] = cap_radius(sqrt(4.0 * p.alpha * eps), caps[3]);
    // rotation (trust_region.cpp:198-234)
    const double lf = log_factor(eps, p.alpha);
    double sigma[9];
    if (lf <= 0.0 || !cov_fast(p.s, p.q, sigma)) {
        for (int c = 0; c < 4; ++c) eta[6 + c] = caps[2];
        return;
    }
    const double tol = eps * (1.0 + 1e-9);
    for (int c = 0; c < 4; ++c) {
        const double beta = beta_rotation(p, c);
        double r = beta <= 1e-12 ? caps[2] : cap_radius(sqrt(lf / beta), caps[2]);
        RotAxis ra;
        rot_axis_setup(p, sigma, c, ra);
        if (!rot_within(ra, r, tol)) r = rot_bisect(ra, r, tol);
        eta[6 + c] = r;
    }
}

// flat index of local coordinate j (0..13) of splat i in the group-major layout
__device__ __forceinline__ long long flat_index(long long K, int i, int j) {
    if (j < 3) return 3LL * i + j;
    if (j < 6) return 3 * K + 3LL * i + (j - 3);
    if (j < 10) return 6 * K + 4LL * i + (j - 6);
    if (j == 10) return 10 * K + i;
    return 11 * K + 3LL * i + (j - 11);
}

// flat index of coordinate j (0..13 reference groups, 14.. the SH group of
// 3 * nb coefficients) of splat i
__device__ __forceinline__ long long coord_index(long long K, int nb, int i, int j) {
    return j < 14 ? flat_index(K, i, j) : 14 * K + 3LL * nb * i + (j - 14);
}

__device__ __forceinline__ Prim load_prim(const double* __restrict__ x, long long K, int i) {
    Prim p;
    for (int a = 0; a < 3; ++a) {
        p.mu[a] = x[3LL * i + a];
        p.s[a] = x[3 * K + 3LL * i + a];
        p.c[a] = x[11 * K + 3LL * i + a];
    }
    for (int a = 0; a < 4; ++a) p.q[a] = x[6 * K + 4LL * i + a];
    p.alpha = x[10 * K + i];
    return p;
}

// deterministic block reduction of up to 5 values (sums, with value 4 a max)
// and a min index; thread 0 stores them at out[0..4] and folds bad into *bad
__device__ void block_reduce5(double* v, int bad, double* out, int* bad_out) {
    __shared__ double s_red[5][kThreads / 32];
    __shared__ int s_bad[kThreads / 32];
    for (int o = 16; o > 0; o >>= 1) {
        for (int q = 0; q < 4; ++q) v[q] += __shfl_xor_sync(0xffffffffu, v[q], o);
        const double m = __shfl_xor_sync(0xffffffffu, v[4], o);
        v[4] = v[4] < m ? m : v[4];
        bad = min(bad, __shfl_xor_sync(0xffffffffu, bad, o));
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) {
        for (int q = 0; q < 5; ++q) s_red[q][warp] = v[q];
        s_bad[warp] = bad;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double r[5] = {0, 0, 0, 0, 0};
        int b = INT_MAX;
        for (int w = 0; w < kThreads / 32; ++w) {
            for (int q = 0; q < 4; ++q) r[q] += s_red[q][w];
            r[4] = r[4] < s_red[4][w] ? s_red[4][w] : r[4];
            b = min(b, s_bad[w]);
        }
        for (int q = 0; q < 5; ++q) out[q] = r[q];
        if (bad_out && b != INT_MAX) atomicMin(bad_out, b);
    }
}

// K14a, one thread per splat over all K: EMAs (or the ADAM moments), the
// direction, and for every coordinate but the four rotation ones the radius,
// clip, step statistics, apply and clamp (optimizer.cpp:124-142,
// scene.cpp:49-57) -- those coordinates never touch a dx or eta buffer.  The
// rotation coordinates' directions go to dx_buf for K14c, which clips them
// against the certified rotation radii of K14a'/K14b.  (ADAM applies every
// coordinate here, unclipped.)
__device__ __forceinline__ double clamp_coord(int j, double v, const double* b) {
    if (j >= 3 && j < 6) return v < b[0] ? b[0] : v;  // scales >= s_min
    if (j == 10) {                                      // alpha in [alpha_min, alpha_max]
        v = v < b[1] ? b[1] : v;
        return b[2] < v ? b[2] : v;
    }
    if (j >= 11 && j < 14) {  // colours in [c_min, c_max]
        v = v < b[3] ? b[3] : v;
        return b[4] < v ? b[4] : v;
    }
    return v;  // means, rotation, SH coefficients
}

__global__ void __launch_bounds__(kThreads, 8) k_tr_prepare(TrArgs a) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const long long K = a.K;
    // sum g^2, sum dx^2, sum clipped^2, n clipped, max ratio
    double s_g2 = 0.0, s_dx2 = 0.0, s_c2 = 0.0, n_clip = 0.0, max_ratio = 0.0;
    int bad = INT_MAX;
    if (i < a.K) {
        const Prim p = load_prim(a.x, K, i);
        const bool degenerate =
            p.q[0] * p.q[0] + p.q[1] * p.q[1] + p.q[2] * p.q[2] + p.q[3] * p.q[3] < 1e-24;
        const bool clipped = a.kind != 1;
        // shd_radii (and its degenerate-quaternion throw) runs for the
        // trust-region kinds only
        if (!a.ghat_only && clipped && degenerate) atomicOr(a.degenerate_flag, 1);
        // the non-rotation radii (trust_region.cpp:236-252); a degenerate
        // splat fails the step, its radii are never used
        double eta[14] = {};
        if (!a.ghat_only && clipped && !degenerate) {
            radius_mean(p, a.eps, a.caps[0], eta);
            for (int c = 0; c < 3; ++c) {
                eta[3 + c] = cap_radius(sqrt(2.0 * p.s[c] * p.s[c] * a.eps / p.alpha), a.caps[1]);
                eta[11 + c] = cap_radius(sqrt(4.0 * p.c[c] * a.eps / p.alpha), a.caps[4]);
            }
            eta[10] = cap_radius(sqrt(4.0 * p.alpha * a.eps), a.caps[3]);
        }
        // one coordinate: direction, then (but for rotation) clip, apply, clamp;
        // e is its radius
        auto coord = [&](int j, double e) {
            const long long k = coord_index(K, a.nb, i, j);
            const double g = a.g_acc[k] * a.gscale;
            s_g2 += g * g;
            double dx;
            if (a.kind != 0) {
                // adam_direction (optimizer.cpp:153-185); SH coefficients at
                // the colour rate / 20 (extension)
                const double m = a.beta1 * a.adam_m[k] + (1.0 - a.beta1) * g;
                const double vv = a.beta2 * a.adam_v[k] + (1.0 - a.beta2) * (g * g);
                a.adam_m[k] = m;
                a.adam_v[k] = vv;
                const int grp = j < 3 ? 0 : j < 6 ? 1 : j < 10 ? 2 : j == 10 ? 3 : 4;
                const double lr = j < 14 ? a.lr[grp] : a.lr[4] / 20.0;
                const double mhat = m / a.bc1;
                const double vhat = vv / a.bc2;
                dx = -lr * mhat / (sqrt(vhat) + a.adam_eps);
            } else {
                const double gh = a.theta1 * a.g_hat[k] + (1.0 - a.theta1) * g;
                a.g_hat[k] = gh;
                if (a.ghat_only) return;
                double dh = a.d_hat[k];
                if (a.refresh) {
                    const double d = a.w_acc[k] * a.dscale;
                    dh = a.theta2 * dh + (1.0 - a.theta2) * d;
                    a.d_hat[k] = dh;
                }
                // std::max(d, gamma) returns d unless d < gamma (NaN d -> d)
                dx = -gh / ((dh < a.gamma_d) ? a.gamma_d : dh);
            }
            s_dx2 += dx * dx;
            if (clipped && j >= 6 && j < 10) {  // rotation: clipped by K14c
                a.dx_buf[k] = dx;
                return;
            }
            double c = dx;
            if (clipped) {
                // cwiseMax(-eta).cwiseMin(eta) with std::max/std::min semantics
                c = dx < -e ? -e : dx;
                c = e < c ? e : c;
                if (fabs(dx) > e) n_clip += 1.0;
                const double ratio = fabs(c) / e;
                max_ratio = max_ratio < ratio ? ratio : max_ratio;
            }
            if (!isfinite(c)) bad = min(bad, (int)min(k, (long long)INT_MAX));
            s_c2 += c * c;
            if (a.applied) a.applied[k] = c;
            a.x_out[k] = clamp_coord(j, a.x[k] + c, a.bounds);
        };
#pragma unroll
        for (int j = 0; j < 14; ++j) coord(j, eta[j]);
        // SH extension: colour radius / max|Y_m|
        for (int j = 14; j < 14 + 3 * a.nb; ++j) {
            const int ch = (j - 14) % 3;
            coord(j, (ch == 0 ? eta[11] : ch == 1 ? eta[12] : eta[13]) / sh_max((j - 14) / 3));
        }
    }
    double v[5] = {s_g2, s_dx2, s_c2, n_clip, max_ratio};
    block_reduce5(v, bad, a.partials + 5LL * blockIdx.x, a.bad_index);
}

// K14a': one thread per (splat, rotation axis) (trust_region.cpp:198-234):
// curvature beta_c, Taylor radius, certification against the exact
// rotation-only H^2; axes failing certification are queued for K14b
__global__ void __launch_bounds__(kThreads, 5) k_tr_rot(TrArgs a) {
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= 4LL * a.n) return;
    const int i = a.i0 + (int)(t >> 2), c = (int)(t & 3);
    const long long K = a.K;
    const Prim p = load_prim(a.x, K, i);
    const long long k = 6 * K + 4LL * i + c;
    const double lf = log_factor(a.eps, p.alpha);
    double sigma[9];
    if (lf <= 0.0 || !cov_fast(p.s, p.q, sigma)) {
        a.eta_buf[k] = a.caps[2];
        return;
    }
    const double beta = beta_rotation(p, c);
    const double r = beta <= 1e-12 ? a.caps[2] : cap_radius(sqrt(lf / beta), a.caps[2]);
    a.eta_buf[k] = r;
    RotAxis ra;
    rot_axis_setup(p, sigma, c, ra);
    if (!rot_within(ra, r, a.eps * (1.0 + 1e-9))) {
        const int slot = atomicAdd(a.queue_count, 1);
        a.queue[slot] = 4 * i + c;
    }
}

// K14b: one thread per queued (splat, rotation axis): the 60-step bisection
__global__ void __launch_bounds__(kThreads) k_tr_bisect(TrArgs a) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= *a.queue_count) return;
    const int i = a.queue[t] >> 2, c = a.queue[t] & 3;
    const long long K = a.K;
    const Prim p = load_prim(a.x, K, i);
    double sigma[9];
    cov_fast(p.s, p.q, sigma);
    RotAxis ra;
    rot_axis_setup(p, sigma, c, ra);
    const long long k = 6 * K + 4LL * i + c;
    a.eta_buf[k] = rot_bisect(ra, a.eta_buf[k], a.eps * (1.0 + 1e-9));
}

// K14c: the rotation coordinates' clip against their certified radii, step
// statistics and apply (optimizer.cpp:124-142; Scene::clamp leaves q alone)
__global__ void __launch_bounds__(kThreads) k_tr_apply(TrArgs a) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;  // all K splats
    const long long K = a.K;
    double v[5] = {0, 0, 0, 0, 0};  // -, -, sum clipped^2, n clipped, max ratio
    int bad = INT_MAX;
    if (i < a.K && a.kind != 1) {
#pragma unroll
        for (int cq = 0; cq < 4; ++cq) {
            const long long k = 6 * K + 4LL * i + cq;
            const double dx = a.dx_buf[k];
            const double eta = a.eta_buf[k];
            double c = dx < -eta ? -eta : dx;
            c = eta < c ? eta : c;
            if (fabs(dx) > eta) v[3] += 1.0;
            const double ratio = fabs(c) / eta;
            v[4] = v[4] < ratio ? ratio : v[4];
            if (!isfinite(c)) bad = min(bad, (int)min(k, (long long)INT_MAX));
            v[2] += c * c;
            if (a.applied) a.applied[k] = c;
            a.x_out[k] = a.x[k] + c;
        }
    }
    block_reduce5(v, bad, a.partials + 5LL * (gridDim.x + blockIdx.x), a.bad_index);
}

__global__ void k_tr_finalize(const double* __restrict__ partials, int nblocks, double* out) {
    __shared__ double s[5][256];
    double r[5] = {0, 0, 0, 0, 0};
    for (int b = threadIdx.x; b < nblocks; b += 256) {
        for (int q = 0; q < 4; ++q) r[q] += partials[5LL * b + q];
        const double m = partials[5LL * b + 4];
        r[4] = r[4] < m ? m : r[4];
    }
    for (int q = 0; q < 5; ++q) s[q][threadIdx.x] = r[q];
    __syncthreads();
    if (threadIdx.x == 0) {
        double t[5] = {0, 0, 0, 0, 0};
        for (int w = 0; w < 256; ++w) {
            for (int q = 0; q < 4; ++q) t[q] += s[q][w];
            t[4] = t[4] < s[4][w] ? s[4][w] : t[4];
        }
        for (int q = 0; q < 5; ++q) out[q] = t[q];
    }
}

__global__ void k_shd_radii(int K, int nb, const double* __restrict__ x, double eps, double c0,
                            double c1, double c2, double c3, double c4,
                            double* __restrict__ eta) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= K) return;
    const double caps[5] = {c0, c1, c2, c3, c4};
    const Prim p = load_prim(x, K, i);
    double e[14];
    radii(p, eps, caps, e);
    for (int j = 0; j < 14; ++j) eta[flat_index(K, i, j)] = e[j];
    for (int m = 0; m < nb; ++m)
        for (int c = 0; c < 3; ++c)
            eta[14LL * K + 3LL * nb * i + 3 * m + c] = e[11 + c] / sh_max(m);
}

__global__ void k_scale(double* v, long long n, double s) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) v[i] = v[i] * s;
}

__global__ void k_add(double* __restrict__ dst, const double* __restrict__ src, long long n) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) dst[i] = dst[i] + src[i];
}

__global__ void k_fill_int(int* p, long long n, int v) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) p[i] = v;
}

}  // namespace

int tr_num_blocks(int K) { return ceil_div(K, kThreads); }

void launch_tr_update(cudaStream_t st, const TrArgs& a, int phase) {
    if (a.K == 0) return;
    const int nbK = tr_num_blocks(a.K);
    if (phase == 0) {
        SGTR_CUDA(cudaMemsetAsync(a.queue_count, 0, sizeof(int), st));
        if (a.elementwise) {  // (further shards only add rotation radii)
            k_tr_prepare<<<nbK, kThreads, 0, st>>>(a);
            SGTR_CUDA(cudaGetLastError());
        }
        if (a.ghat_only && a.elementwise)
            SGTR_CUDA(cudaMemsetAsync(a.partials + 5LL * nbK, 0, sizeof(double) * 5 * nbK, st));
    } else if (phase == 3 && !a.ghat_only && a.kind != 1 && a.n > 0) {
        k_tr_rot<<<ceil_div(4LL * a.n, kThreads), kThreads, 0, st>>>(a);
        SGTR_CUDA(cudaGetLastError());
    } else if (phase == 1 && !a.ghat_only && a.kind != 1 && a.n > 0) {
        k_tr_bisect<<<ceil_div(4LL * a.n, kThreads), kThreads, 0, st>>>(a);
        SGTR_CUDA(cudaGetLastError());
    } else if (phase == 2 && !a.ghat_only) {
        k_tr_apply<<<nbK, kThreads, 0, st>>>(a);
        SGTR_CUDA(cudaGetLastError());
    }
}

// partials: [nblocks][5] from K14a (sums of g^2, dx^2 and the non-rotation
// coordinates' clipped^2, their clip count and max ratio) then [nblocks][5]
// from K14c (the same three for the rotation coordinates)
void launch_tr_finalize(cudaStream_t st, const double* partials, int nblocks, double* out5) {
    k_tr_finalize<<<1, 256, 0, st>>>(partials, 2 * nblocks, out5);
    SGTR_CUDA(cudaGetLastError());
}

void launch_shd_radii(cudaStream_t st, int K, int nb, const double* x, double eps,
                      const double caps[5], double* eta) {
    if (K == 0) return;
    k_shd_radii<<<ceil_div(K, 128), 128, 0, st>>>(K, nb, x, eps, caps[0], caps[1], caps[2],
                                                  caps[3], caps[4], eta);
    SGTR_CUDA(cudaGetLastError());
}

void launch_scale(cudaStream_t st, double* v, long long n, double s) {
    if (n == 0) return;
    k_scale<<<ceil_div(n, 256), 256, 0, st>>>(v, n, s);
    SGTR_CUDA(cudaGetLastError());
}

void launch_add(cudaStream_t st, double* dst, const double* src, long long n) {
    if (n == 0) return;
    k_add<<<ceil_div(n, 256), 256, 0, st>>>(dst, src, n);
    SGTR_CUDA(cudaGetLastError());
}

void launch_fill_int(cudaStream_t st, int* p, long long n, int v) {
    if (n == 0) return;
    k_fill_int<<<ceil_div(n, 256), 256, 0, st>>>(p, n, v);
    SGTR_CUDA(cudaGetLastError());
}

}  // namespace sgtr
