// geometry.cuh — forward-mode dual scalar and the EWA projection chain.
//
// Included only by translation units compiled with --fmad=false (and the
// host side with -ffp-contract=off), so each expression below rounds exactly
// like the oracle's restatement: projection keys, screen-space means and
// bounding boxes come out bit-identical, which is what makes the depth order
// and the tile lists bit-exact.
//   Dual semantics:        dual.hpp:14-96
//   rotation/covariance:   geometry.hpp:25-65
//   projection:            render.hpp:34-63
//   invert2x2:             render.cpp:42-49
#pragma once
#include <math.h>

#define SGTR_HD __host__ __device__ __forceinline__

namespace sgtr {

struct Dual {
    double v, d;
    SGTR_HD Dual() : v(0.0), d(0.0) {}
    SGTR_HD Dual(double a) : v(a), d(0.0) {}
    SGTR_HD Dual(double a, double b) : v(a), d(b) {}
};
SGTR_HD Dual operator-(const Dual& a) { return Dual(-a.v, -a.d); }
SGTR_HD Dual operator+(const Dual& a, const Dual& b) { return Dual(a.v + b.v, a.d + b.d); }
SGTR_HD Dual operator-(const Dual& a, const Dual& b) { return Dual(a.v - b.v, a.d - b.d); }
SGTR_HD Dual operator*(const Dual& a, const Dual& b) {
    return Dual(a.v * b.v, a.d * b.v + a.v * b.d);
}
SGTR_HD Dual operator/(const Dual& a, const Dual& b) {
    return Dual(a.v / b.v, (a.d * b.v - a.v * b.d) / (b.v * b.v));
}
SGTR_HD Dual operator+(const Dual& a, double b) { return Dual(a.v + b, a.d); }
SGTR_HD Dual operator+(double a, const Dual& b) { return Dual(a + b.v, b.d); }
SGTR_HD Dual operator-(const Dual& a, double b) { return Dual(a.v - b, a.d); }
SGTR_HD Dual operator-(double a, const Dual& b) { return Dual(a - b.v, -b.d); }
SGTR_HD Dual operator*(const Dual& a, double b) { return Dual(a.v * b, a.d * b); }
SGTR_HD Dual operator*(double a, const Dual& b) { return Dual(a * b.v, a * b.d); }
SGTR_HD Dual operator/(const Dual& a, double b) { return Dual(a.v / b, a.d / b); }
SGTR_HD Dual operator/(double a, const Dual& b) {
    return Dual(a / b.v, -a * b.d / (b.v * b.v));
}
SGTR_HD Dual dsqrt(const Dual& a) {
    const double r = sqrt(a.v);
    return Dual(r, a.d / (2.0 * r));
}
SGTR_HD double dsqrt(double a) { return sqrt(a); }
SGTR_HD double primal(double a) { return a; }
SGTR_HD double primal(const Dual& a) { return a.v; }
SGTR_HD double tangent(double) { return 0.0; }
SGTR_HD double tangent(const Dual& a) { return a.d; }

// R = R~(q)/|q|^2; returns false on a degenerate quaternion (|q|^2 < 1e-24),
// where the reference throws std::invalid_argument
template <typename T>
SGTR_HD bool quat_rot(const T* q, T* m) {
    const T x = q[0], y = q[1], z = q[2], w = q[3];
    const T r2 = x * x + y * y + z * z + w * w;
    if (primal(r2) < 1e-24) return false;
    m[0] = r2 - 2.0 * (y * y + z * z);
    m[1] = 2.0 * (x * y - w * z);
    m[2] = 2.0 * (x * z + w * y);
    m[3] = 2.0 * (x * y + w * z);
    m[4] = r2 - 2.0 * (z * z + x * x);
    m[5] = 2.0 * (y * z - w * x);
    m[6] = 2.0 * (x * z - w * y);
    m[7] = 2.0 * (y * z + w * x);
    m[8] = r2 - 2.0 * (x * x + y * y);
#pragma unroll
    for (int i = 0; i < 9; ++i) m[i] = m[i] / r2;
    return true;
}

// The reference's Eigen 3.4 build sums a small product coefficient with a
// column-major lhs in halves, a0 b0 + (a1 b1 + a2 b2) (oracle/refshim/Eigen/Core
// documents the model and its evidence); this TU is built without FMA
// contraction, so the projection is bit-identical to the reference's.
template <typename T>
SGTR_HD T tree3(const T& a, const T& b, const T& c) {
    return a + (b + c);
}

// Sigma = (R^T diag(s^2)) R: one non-zero term per coefficient in the first
// product, the second summed in halves
template <typename T>
SGTR_HD bool covariance(const T* s, const T* q, T* cov) {
    T r[9];
    if (!quat_rot(q, r)) return false;
    const T s2[3] = {s[0] * s[0], s[1] * s[1], s[2] * s[2]};
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j)
            cov[3 * i + j] = tree3<T>(r[i] * s2[0] * r[j], r[3 + i] * s2[1] * r[3 + j],
                                      r[6 + i] * s2[2] * r[6 + j]);
    return true;
}

template <typename T>
struct Proj {
    bool culled;
    bool degenerate;
    double depth;
    T mx, my, c00, c01, c11;
};

template <typename T>
SGTR_HD Proj<T> project(const T* mu, const T* s, const T* q, const double* w,
                        const double* t, double fx, double fy, double cx, double cy,
                        double z_near, double lowpass) {
    Proj<T> out;
    out.culled = true;
    out.degenerate = false;
    T pc[3];
#pragma unroll
    for (int i = 0; i < 3; ++i)
        pc[i] = tree3<T>(w[3 * i] * mu[0], w[3 * i + 1] * mu[1], w[3 * i + 2] * mu[2]) + t[i];
    out.depth = primal(pc[2]);
    if (out.depth <= z_near) return out;
    out.culled = false;
    const T inv_z = 1.0 / pc[2];
    out.mx = fx * pc[0] * inv_z + cx;
    out.my = fy * pc[1] * inv_z + cy;
    T sig[9];
    if (!covariance(s, q, sig)) {
        out.degenerate = true;
        return out;
    }
    T ws[9], sc[9];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j)
            ws[3 * i + j] = tree3<T>(w[3 * i] * sig[j], w[3 * i + 1] * sig[3 + j],
                                     w[3 * i + 2] * sig[6 + j]);
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j)
            sc[3 * i + j] = tree3<T>(ws[3 * i] * w[3 * j], ws[3 * i + 1] * w[3 * j + 1],
                                     ws[3 * i + 2] * w[3 * j + 2]);
    const T j00 = fx * inv_z;
    const T j02 = -fx * pc[0] * inv_z * inv_z;
    const T j11 = fy * inv_z;
    const T j12 = -fy * pc[1] * inv_z * inv_z;
    // J's structural zeros at (0,1), (1,0) are omitted (same as the oracle)
    const T a0 = j00 * sc[0] + j02 * sc[6];
    const T a1 = j00 * sc[1] + j02 * sc[7];
    const T a2 = j00 * sc[2] + j02 * sc[8];
    const T b1 = j11 * sc[4] + j12 * sc[7];
    const T b2 = j11 * sc[5] + j12 * sc[8];
    out.c00 = a0 * j00 + a2 * j02 + lowpass;
    out.c01 = a1 * j11 + a2 * j12;
    out.c11 = b1 * j11 + b2 * j12 + lowpass;
    return out;
}

template <typename T>
SGTR_HD void invert2x2(const T& c00, const T& c01, const T& c11, T& i00, T& i01,
                       T& i11) {
    const T det = c00 * c11 - c01 * c01;
    i00 = c11 / det;
    i01 = -c01 / det;
    i11 = c00 / det;
}

// Reverse-mode chain of the 5 screen-space adjoints (mu2d, inverse 2d
// covariance) through invert2x2 and project() to (mu, s, q): the transpose of
// the 5x10 Jacobian the reference evaluates with 10 dual seeds
// (render.cpp:297-329), one backward sweep over the same computational graph.
SGTR_HD void chain_reverse(const double* mu, const double* s, const double* q,
                           const double* w, const double* t, double fx, double fy,
                           double lowpass, const double* a, double* gmu, double* gs,
                           double* gq) {
    // ---- forward recompute (the graph of project() + invert2x2)
    double pc[3];
#pragma unroll
    for (int i = 0; i < 3; ++i)
        pc[i] = tree3(w[3 * i] * mu[0], w[3 * i + 1] * mu[1], w[3 * i + 2] * mu[2]) + t[i];
    const double iz = 1.0 / pc[2];
    const double x = q[0], y = q[1], z = q[2], qw = q[3];
    const double r2 = x * x + y * y + z * z + qw * qw;
    const double rt[9] = {r2 - 2.0 * (y * y + z * z), 2.0 * (x * y - qw * z),
                          2.0 * (x * z + qw * y),      2.0 * (x * y + qw * z),
                          r2 - 2.0 * (z * z + x * x), 2.0 * (y * z - qw * x),
                          2.0 * (x * z - qw * y),      2.0 * (y * z + qw * x),
                          r2 - 2.0 * (x * x + y * y)};
    const double ir2 = 1.0 / r2;
    double R[9];
#pragma unroll
    for (int i = 0; i < 9; ++i) R[i] = rt[i] * ir2;
    const double s2[3] = {s[0] * s[0], s[1] * s[1], s[2] * s[2]};
    double sig[9], ws[9], sc[9];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j)
            sig[3 * i + j] = tree3(R[i] * s2[0] * R[j], R[3 + i] * s2[1] * R[3 + j],
                                   R[6 + i] * s2[2] * R[6 + j]);
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j)
            ws[3 * i + j] = tree3(w[3 * i] * sig[j], w[3 * i + 1] * sig[3 + j], w[3 * i + 2] * sig[6 + j]);
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j)
            sc[3 * i + j] = tree3(ws[3 * i] * w[3 * j], ws[3 * i + 1] * w[3 * j + 1],
                                  ws[3 * i + 2] * w[3 * j + 2]);
    const double j00 = fx * iz, j02 = -fx * pc[0] * iz * iz;
    const double j11 = fy * iz, j12 = -fy * pc[1] * iz * iz;
    const double js00 = j00 * sc[0] + j02 * sc[6], js01 = j00 * sc[1] + j02 * sc[7];
    const double js02 = j00 * sc[2] + j02 * sc[8];
    const double js11 = j11 * sc[4] + j12 * sc[7], js12 = j11 * sc[5] + j12 * sc[8];
    const double c00 = js00 * j00 + js02 * j02 + lowpass;
    const double c01 = js01 * j11 + js02 * j12;
    const double c11 = js11 * j11 + js12 * j12 + lowpass;
    const double det = c00 * c11 - c01 * c01;
    const double idet = 1.0 / det;
    const double i00 = c11 * idet, i01 = -c01 * idet, i11 = c00 * idet;
    // ---- invert2x2 backward
    const double a_det = -(a[2] * i00 + a[3] * i01 + a[4] * i11) * idet;
    const double a_c00 = a[4] * idet + a_det * c11;
    const double a_c11 = a[2] * idet + a_det * c00;
    const double a_c01 = -a[3] * idet - 2.0 * a_det * c01;
    // ---- J SC J^T backward
    const double a_js00 = a_c00 * j00, a_js02 = a_c00 * j02 + a_c01 * j12;
    const double a_js01 = a_c01 * j11, a_js11 = a_c11 * j11, a_js12 = a_c11 * j12;
    double a_j00 = a_c00 * js00 + a_js00 * sc[0] + a_js01 * sc[1] + a_js02 * sc[2];
    double a_j02 = a_c00 * js02 + a_js00 * sc[6] + a_js01 * sc[7] + a_js02 * sc[8];
    double a_j11 = a_c01 * js01 + a_c11 * js11 + a_js11 * sc[4] + a_js12 * sc[5];
    double a_j12 = a_c01 * js02 + a_c11 * js12 + a_js11 * sc[7] + a_js12 * sc[8];
    double a_sc[9] = {a_js00 * j00, a_js01 * j00, a_js02 * j00,
                      0.0,          a_js11 * j11, a_js12 * j11,
                      a_js00 * j02, a_js01 * j02 + a_js11 * j12, a_js02 * j02 + a_js12 * j12};
    // ---- SC = (W Sigma) W^T, WS = W Sigma backward
    double a_ws[9], a_sig[9];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int k = 0; k < 3; ++k)
            a_ws[3 * i + k] = a_sc[3 * i] * w[k] + a_sc[3 * i + 1] * w[3 + k] + a_sc[3 * i + 2] * w[6 + k];
#pragma unroll
    for (int k = 0; k < 3; ++k)
#pragma unroll
        for (int j = 0; j < 3; ++j)
            a_sig[3 * k + j] = w[k] * a_ws[j] + w[3 + k] * a_ws[3 + j] + w[6 + k] * a_ws[6 + j];
    // ---- Sigma = R^T diag(s^2) R backward
    double a_R[9];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        double as2 = 0.0;
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            double acc = 0.0;
#pragma unroll
            for (int j = 0; j < 3; ++j) {
                acc += (a_sig[3 * i + j] + a_sig[3 * j + i]) * R[3 * k + j];
                as2 += a_sig[3 * i + j] * R[3 * k + i] * R[3 * k + j];
            }
            a_R[3 * k + i] = s2[k] * acc;
        }
        gs[k] = 2.0 * s[k] * as2;
    }
    // ---- R = R~(q) / |q|^2 backward (dR~/dq_c as trust_region.cpp:95-117)
    double a_r2 = 0.0;
#pragma unroll
    for (int i = 0; i < 9; ++i) a_r2 -= a_R[i] * R[i];
    a_r2 *= ir2;
    double art[9];
#pragma unroll
    for (int i = 0; i < 9; ++i) art[i] = a_R[i] * ir2;
    gq[0] = 2.0 * (x * (art[0] - art[4] - art[8]) + y * (art[1] + art[3]) +
                   z * (art[2] + art[6]) + qw * (art[7] - art[5])) + 2.0 * x * a_r2;
    gq[1] = 2.0 * (-y * (art[0] - art[4] + art[8]) + x * (art[1] + art[3]) +
                   qw * (art[2] - art[6]) + z * (art[5] + art[7])) + 2.0 * y * a_r2;
    gq[2] = 2.0 * (-z * (art[0] + art[4] - art[8]) + qw * (art[3] - art[1]) +
                   x * (art[2] + art[6]) + y * (art[5] + art[7])) + 2.0 * z * a_r2;
    gq[3] = 2.0 * (qw * (art[0] + art[4] + art[8]) + z * (art[3] - art[1]) +
                   y * (art[2] - art[6]) + x * (art[7] - art[5])) + 2.0 * qw * a_r2;
    // ---- J, mu2d, inverse depth, pc = W mu + t backward
    double a_pc0 = a[0] * fx * iz - a_j02 * fx * iz * iz;
    double a_pc1 = a[1] * fy * iz - a_j12 * fy * iz * iz;
    const double a_iz = a[0] * fx * pc[0] + a[1] * fy * pc[1] + a_j00 * fx + a_j11 * fy -
                        2.0 * a_j02 * fx * pc[0] * iz - 2.0 * a_j12 * fy * pc[1] * iz;
    const double a_pc2 = -a_iz * iz * iz;
#pragma unroll
    for (int k = 0; k < 3; ++k) gmu[k] = w[k] * a_pc0 + w[3 + k] * a_pc1 + w[6 + k] * a_pc2;
}

// rho2 = 2 ln(alpha / alpha_skip): the fragment can contribute at a pixel
// only where d^T Sigma^-1 d <= rho2 (alpha_bar = alpha exp(-q/2) >=
// alpha_skip, render.cpp:132-137).  Negative: it never contributes.
// Infinite: no culling (alpha_skip <= 0).
SGTR_HD double contrib_rho2(double alpha, double alpha_skip) {
    if (!(alpha_skip > 0.0)) return INFINITY;
    if (alpha < alpha_skip) return -1.0;
    return 2.0 * log(alpha / alpha_skip);
}

// Conservative culling of a fragment against the pixel centres
// [x0+0.5, x1+0.5] x [y0+0.5, y1+0.5]: false only when every centre has
// q = d^T Sigma^-1 d certainly above rho2 (the minimum of the convex q over
// the rectangle, with a margin far above the rounding of the reference's own
// exponent), i.e. when the reference would skip every one of these pairs.
// k11 = i01 / i11 and k00 = i01 / i00 are the edge-minimiser slopes.
SGTR_HD bool ellipse_may_hit(double mx, double my, double i00, double i01, double i11,
                             double k11, double k00, double rho2, int x0, int x1, int y0,
                             int y1) {
    if (!(rho2 < INFINITY)) return true;
    if (rho2 < 0.0) return false;
    const double ax = (x0 + 0.5) - mx, bx = (x1 + 0.5) - mx;
    const double ay = (y0 + 0.5) - my, by = (y1 + 0.5) - my;
    if (ax <= 0.0 && bx >= 0.0 && ay <= 0.0 && by >= 0.0) return true;
    auto q = [&](double dx, double dy) {
        return i00 * dx * dx + 2.0 * i01 * dx * dy + i11 * dy * dy;
    };
    auto clampd = [](double v, double lo, double hi) { return v < lo ? lo : (v > hi ? hi : v); };
    double qmin = q(ax, clampd(-(k11 * ax), ay, by));
    qmin = fmin(qmin, q(bx, clampd(-(k11 * bx), ay, by)));
    qmin = fmin(qmin, q(clampd(-(k00 * ay), ax, bx), ay));
    qmin = fmin(qmin, q(clampd(-(k00 * by), ax, bx), by));
    const double mxd = fmax(fabs(ax), fabs(bx)), myd = fmax(fabs(ay), fabs(by));
    const double bound = fabs(i00) * mxd * mxd + fabs(i11) * myd * myd + 2.0 * fabs(i01) * mxd * myd;
    // NaN (a degenerate conic) keeps the fragment: the reference evaluates every
    // pair whose bbox test passes, and a NaN alpha_bar is not skipped (render.cpp:136)
    return !(qmin > rho2 + 1e-9 * rho2 + 1e-12 * bound + 1e-12);
}

// pixel-centre range [p0, p1] inside the closed interval [lo, hi], clipped
// to [0, n-1]; p0 > p1 means empty.  Exact: every comparison is between
// p + 0.5 (exactly representable) and the FP64 bound itself.
SGTR_HD void pixel_range(double lo, double hi, int n, int& p0, int& p1) {
    if (isnan(lo) || isnan(hi)) {
        p0 = 0;
        p1 = n - 1;
        return;
    }
    if (!(hi >= 0.5) || !(lo <= n - 0.5)) {
        p0 = 1;
        p1 = 0;
        return;
    }
    p0 = lo <= 0.5 ? 0 : (int)ceil(lo - 0.5);
    while (p0 > 0 && (p0 - 1) + 0.5 >= lo) --p0;
    while (p0 + 0.5 < lo) ++p0;
    p1 = hi >= n - 0.5 ? n - 1 : (int)floor(hi - 0.5);
    while (p1 < n - 1 && (p1 + 1) + 0.5 <= hi) ++p1;
    while (p1 + 0.5 > hi) --p1;
}

// ---------------------------------------------------------------- SH colour
// Extension beyond the reference (SH degree 0, parity unpinned,
// restated identically in oracle/oracle.cpp): nb = (d+1)^2 - 1 real-SH
// coefficients per channel appended after the 14 reference groups as a
// splat-major group, and
//   c_view = c + sum_j Y_j(dir) k_j,  dir = normalize(mu - camera centre)
// with the reference's linear RGB as the DC term (degree 0 is the reference
// bit for bit), no offset and no clamp.  3DGS basis constants and signs.
template <typename T>
SGTR_HD void sh_basis(const T& x, const T& y, const T& z, int nb, T* Y) {
    if (nb >= 3) {
        Y[0] = -0.4886025119029199 * y;
        Y[1] = 0.4886025119029199 * z;
        Y[2] = -0.4886025119029199 * x;
    }
    if (nb >= 8) {
        const T xx = x * x, yy = y * y, zz = z * z;
        Y[3] = 1.0925484305920792 * (x * y);
        Y[4] = -1.0925484305920792 * (y * z);
        Y[5] = 0.31539156525252005 * (2.0 * zz - xx - yy);
        Y[6] = -1.0925484305920792 * (x * z);
        Y[7] = 0.5462742152960396 * (xx - yy);
        if (nb >= 15) {
            Y[8] = -0.5900435899266435 * y * (3.0 * xx - yy);
            Y[9] = 2.890611442640554 * (x * y) * z;
            Y[10] = -0.4570457994644658 * y * (4.0 * zz - xx - yy);
            Y[11] = 0.3731763325901154 * z * (2.0 * zz - 3.0 * xx - 3.0 * yy);
            Y[12] = -0.4570457994644658 * x * (4.0 * zz - xx - yy);
            Y[13] = 1.445305721320277 * z * (xx - yy);
            Y[14] = -0.5900435899266435 * x * (xx - 3.0 * yy);
        }
    }
}

// max over unit directions of |Y_j| (the SH trust-region radius divisor)
SGTR_HD double sh_max(int j) {
    switch (j) {
        case 0: case 1: case 2: return 0.4886025119029199;
        case 3: case 4: case 6: return 0.5462742152960397;
        case 5: return 0.6307831305050401;
        case 7: return 0.5462742152960396;
        case 8: case 14: return 0.5900435899266437;
        case 9: return 0.5562984315103788;
        case 10: return 0.6293798292550865;
        case 11: return 0.7463526651802308;
        case 12: return 0.6293798292550866;
        default: return 0.5562984315103789;  // 13
    }
}

template <typename T>
SGTR_HD void sh_dir(const T* mu, const double* cen, T* d) {
    const T vx = mu[0] - cen[0], vy = mu[1] - cen[1], vz = mu[2] - cen[2];
    const T inv = 1.0 / dsqrt(vx * vx + vy * vy + vz * vz);
    d[0] = vx * inv;
    d[1] = vy * inv;
    d[2] = vz * inv;
}

// view colour; k points at the splat's 3 * nb coefficients (rgb interleaved)
template <typename T, typename KT>
SGTR_HD void sh_color(const T* mu, const T* c, const KT* k, int nb, const double* cen, T* out) {
    if (nb == 0) {
        for (int a = 0; a < 3; ++a) out[a] = c[a];
        return;
    }
    T d[3], Y[15];
    sh_dir(mu, cen, d);
    sh_basis(d[0], d[1], d[2], nb, Y);
    for (int a = 0; a < 3; ++a) {
        T acc = Y[0] * k[a];
        for (int j = 1; j < nb; ++j) acc = acc + Y[j] * k[3 * j + a];
        out[a] = c[a] + acc;
    }
}

}  // namespace sgtr
