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

// Sigma = R^T diag(s^2) R, each entry summed over k left to right
template <typename T>
SGTR_HD bool covariance(const T* s, const T* q, T* cov) {
    T r[9];
    if (!quat_rot(q, r)) return false;
    const T s2[3] = {s[0] * s[0], s[1] * s[1], s[2] * s[2]};
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j)
            cov[3 * i + j] = r[i] * s2[0] * r[j] + r[3 + i] * s2[1] * r[3 + j] +
                             r[6 + i] * s2[2] * r[6 + j];
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
        pc[i] = w[3 * i] * mu[0] + w[3 * i + 1] * mu[1] + w[3 * i + 2] * mu[2] + t[i];
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
            ws[3 * i + j] = w[3 * i] * sig[j] + w[3 * i + 1] * sig[3 + j] +
                            w[3 * i + 2] * sig[6 + j];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j)
            sc[3 * i + j] = ws[3 * i] * w[3 * j] + ws[3 * i + 1] * w[3 * j + 1] +
                            ws[3 * i + 2] * w[3 * j + 2];
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

}  // namespace sgtr
