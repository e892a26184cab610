// oracle.cpp — CPU restatement of the reference 3DGS²-TR hot path.
//
// TEST INFRASTRUCTURE ONLY (see oracle.h for the pinning statement).  Each
// function names the reference file:line it restates; reference paths are
// relative to /root/reference/proj.  Arithmetic is FP64 with an explicit,
// left-to-right operation order and no FMA contraction (built with
// -ffp-contract=off) so that the GPU build's bit-exact stages (projection
// keys, bounding boxes, binning) can be compared with memcmp.
#include "oracle.h"

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <functional>
#include <memory>
#include <limits>
#include <mutex>
#include <random>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

namespace {

thread_local std::string g_err;

struct InvalidArg : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct NumericErr : std::runtime_error {
    using std::runtime_error::runtime_error;
};

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const InvalidArg& e) {
        g_err = e.what();
        return 1;
    } catch (const NumericErr& e) {
        g_err = e.what();
        return 2;
    } catch (const std::out_of_range& e) {
        g_err = e.what();
        return 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 3;
    }
}

// ---------------------------------------------------------------- Dual
// forward-mode scalar, semantics of dual.hpp:14-96 (branches on primal)
struct Dual {
    double v = 0.0, d = 0.0;
    Dual() = default;
    Dual(double a) : v(a) {}
    Dual(double a, double b) : v(a), d(b) {}
};
inline Dual operator-(const Dual& a) { return {-a.v, -a.d}; }
inline Dual operator+(const Dual& a, const Dual& b) { return {a.v + b.v, a.d + b.d}; }
inline Dual operator-(const Dual& a, const Dual& b) { return {a.v - b.v, a.d - b.d}; }
inline Dual operator*(const Dual& a, const Dual& b) {
    return {a.v * b.v, a.d * b.v + a.v * b.d};
}
inline Dual operator/(const Dual& a, const Dual& b) {
    return {a.v / b.v, (a.d * b.v - a.v * b.d) / (b.v * b.v)};
}
inline Dual operator+(const Dual& a, double b) { return {a.v + b, a.d}; }
inline Dual operator+(double a, const Dual& b) { return {a + b.v, b.d}; }
inline Dual operator-(const Dual& a, double b) { return {a.v - b, a.d}; }
inline Dual operator-(double a, const Dual& b) { return {a - b.v, -b.d}; }
inline Dual operator*(const Dual& a, double b) { return {a.v * b, a.d * b}; }
inline Dual operator*(double a, const Dual& b) { return {a * b.v, a * b.d}; }
inline Dual operator/(const Dual& a, double b) { return {a.v / b, a.d / b}; }
inline Dual operator/(double a, const Dual& b) {
    return {a / b.v, -a * b.d / (b.v * b.v)};
}
inline Dual& operator+=(Dual& a, const Dual& b) { return a = a + b; }
inline Dual dexp(const Dual& a) {
    const double e = std::exp(a.v);
    return {e, e * a.d};
}
inline double dexp(double a) { return std::exp(a); }
inline Dual dsqrt(const Dual& a) {
    const double r = std::sqrt(a.v);
    return {r, a.d / (2.0 * r)};
}
inline double dsqrt(double a) { return std::sqrt(a); }
inline double P(double a) { return a; }
inline double P(const Dual& a) { return a.v; }

// ---------------------------------------------------------------- Rng
// rng.hpp:15-72: mt19937_64 with hand-rolled variates
struct Rng {
    std::mt19937_64 gen;
    bool have_spare = false;
    double spare = 0.0;
    explicit Rng(uint64_t seed) : gen(seed) {}
    uint64_t raw() { return gen(); }
    double uniform() { return static_cast<double>(gen() >> 11) * 0x1.0p-53; }
    double uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }
    double log_uniform(double lo, double hi) {
        return std::exp(uniform(std::log(lo), std::log(hi)));
    }
    double normal() {
        if (have_spare) {
            have_spare = false;
            return spare;
        }
        double u1 = uniform();
        while (u1 <= 0.0) u1 = uniform();
        const double u2 = uniform();
        const double r = std::sqrt(-2.0 * std::log(u1));
        spare = r * std::sin(2.0 * M_PI * u2);
        have_spare = true;
        return r * std::cos(2.0 * M_PI * u2);
    }
    double rademacher() { return (gen() & 1u) ? 1.0 : -1.0; }
    uint64_t below(uint64_t n) { return gen() % n; }
    std::vector<int> sample(int n, int k) {
        std::vector<int> idx(n);
        for (int i = 0; i < n; ++i) idx[i] = i;
        const int m = std::min(k, n);
        for (int i = 0; i < m; ++i) {
            const int j = i + static_cast<int>(below(n - i));
            std::swap(idx[i], idx[j]);
        }
        idx.resize(m);
        return idx;
    }
};

// ---------------------------------------------------------------- scene view
// SH extension (parity unpinned: the reference is SH degree 0).
// Degree d adds nb = (d+1)^2 - 1 real-SH coefficients per colour channel,
// stored after the reference's 14 groups as one more splat-major group
// [k_1..k_nb (rgb interleaved) x K]; the view colour is
//   c_view = c + sum_j Y_j(dir) k_j,  dir = normalize(mu - camera centre),
// with the DC term the reference's linear RGB (degree 0 is the reference
// bit for bit), no offset and no clamp.  Set per process with
// orc_set_sh_degree (test infrastructure).
int g_sh_nb = 0;

// group-major layout, scene.hpp:37-52
struct SceneView {
    const double* x;
    int64_t k;
    int nb = g_sh_nb;
    const double* mu(int64_t i) const { return x + 3 * i; }
    const double* s(int64_t i) const { return x + 3 * k + 3 * i; }
    const double* q(int64_t i) const { return x + 6 * k + 4 * i; }
    double alpha(int64_t i) const { return x[10 * k + i]; }
    const double* c(int64_t i) const { return x + 11 * k + 3 * i; }
    const double* sh(int64_t i) const { return x + 14 * k + 3LL * nb * i; }
    int64_t sh_off(int64_t i) const { return 14 * k + 3LL * nb * i; }
    int64_t dim() const { return (14 + 3LL * nb) * k; }
};

// real SH basis of degrees 1..3 at a unit direction (3DGS constants and
// sign conventions), and max over the sphere of |Y_j| (numerically
// maximised; used for the SH trust-region radii)
const double kShC1 = 0.4886025119029199;
const double kShC2[5] = {1.0925484305920792, -1.0925484305920792, 0.31539156525252005,
                         -1.0925484305920792, 0.5462742152960396};
const double kShC3[7] = {-0.5900435899266435, 2.890611442640554, -0.4570457994644658,
                         0.3731763325901154,  -0.4570457994644658, 1.445305721320277,
                         -0.5900435899266435};
const double kShMax[15] = {0.4886025119029199, 0.4886025119029199, 0.4886025119029199,
                           0.5462742152960397, 0.5462742152960397, 0.6307831305050401,
                           0.5462742152960397, 0.5462742152960396, 0.5900435899266437,
                           0.5562984315103788, 0.6293798292550865, 0.7463526651802308,
                           0.6293798292550866, 0.5562984315103789, 0.5900435899266437};

template <typename T>
void sh_basis(const T& x, const T& y, const T& z, int nb, T* Y) {
    if (nb >= 3) {
        Y[0] = -kShC1 * y;
        Y[1] = kShC1 * z;
        Y[2] = -kShC1 * x;
    }
    if (nb >= 8) {
        const T xx = x * x, yy = y * y, zz = z * z;
        Y[3] = kShC2[0] * (x * y);
        Y[4] = kShC2[1] * (y * z);
        Y[5] = kShC2[2] * (2.0 * zz - xx - yy);
        Y[6] = kShC2[3] * (x * z);
        Y[7] = kShC2[4] * (xx - yy);
        if (nb >= 15) {
            Y[8] = kShC3[0] * y * (3.0 * xx - yy);
            Y[9] = kShC3[1] * (x * y) * z;
            Y[10] = kShC3[2] * y * (4.0 * zz - xx - yy);
            Y[11] = kShC3[3] * z * (2.0 * zz - 3.0 * xx - 3.0 * yy);
            Y[12] = kShC3[4] * x * (4.0 * zz - xx - yy);
            Y[13] = kShC3[5] * z * (xx - yy);
            Y[14] = kShC3[6] * x * (xx - 3.0 * yy);
        }
    }
}

// unit direction from the camera centre to mu
template <typename T>
void sh_dir(const T mu[3], const double cen[3], T d[3]) {
    const T vx = mu[0] - cen[0], vy = mu[1] - cen[1], vz = mu[2] - cen[2];
    const T inv = 1.0 / dsqrt(vx * vx + vy * vy + vz * vz);
    d[0] = vx * inv;
    d[1] = vy * inv;
    d[2] = vz * inv;
}

// c_view = c + sum_j Y_j k_j, the sum accumulated in j order per channel
template <typename T>
void sh_color(const T mu[3], const T c[3], const T* k, int nb, const double cen[3], T out[3]) {
    if (nb == 0) {
        for (int a = 0; a < 3; ++a) out[a] = c[a];
        return;
    }
    T d[3], Y[15] = {};
    sh_dir(mu, cen, d);
    sh_basis(d[0], d[1], d[2], nb, Y);
    for (int a = 0; a < 3; ++a) {
        T acc = Y[0] * k[a];
        for (int j = 1; j < nb; ++j) acc = acc + Y[j] * k[3 * j + a];
        out[a] = c[a] + acc;
    }
}

const char* const kGroup[5] = {"position", "scale", "rotation", "opacity",
                               "color"};
int group_of(int64_t k, int64_t idx) {  // scene.cpp:41-47
    if (idx < 3 * k) return 0;
    if (idx < 6 * k) return 1;
    if (idx < 10 * k) return 2;
    if (idx < 11 * k) return 3;
    return 4;
}

// ---------------------------------------------------------------- Eigen order
// The reference's Eigen 3.4 (x86-64, SSE2) reduction orders, as modelled by
// oracle/refshim/Eigen/Core (which documents the evidence):
//  * a small product coefficient over k = 0..2 with a column-major lhs is
//    split in halves, a0 b0 + (a1 b1 + a2 b2) (W mu, W Sigma, (W Sigma) W^T,
//    (R^T S^2) R); with a transposed lhs it is vectorised: left to right;
//  * a trace is d0 + (d1 + d2); a 4-vector's squaredNorm / norm is
//    (q0^2 + q2^2) + (q1^2 + q3^2); a 3-vector's is left to right;
//  * a VectorXd squaredNorm / norm runs two SSE2 packet accumulators.
template <typename T>
inline T tree3(const T& a, const T& b, const T& c) {
    return a + (b + c);
}
inline double sqnorm4(const double q[4]) {
    return (q[0] * q[0] + q[2] * q[2]) + (q[1] * q[1] + q[3] * q[3]);
}

// ---------------------------------------------------------------- geometry
// geometry.hpp:25-54: R = R~(q)/|q|^2; throws on |q|^2 < 1e-24
template <typename T>
void quat_rot(const T q[4], T m[9]) {
    const T x = q[0], y = q[1], z = q[2], w = q[3];
    const T r2 = x * x + y * y + z * z + w * w;
    if (P(r2) < 1e-24)
        throw InvalidArg("quat_to_rotation: degenerate quaternion");
    m[0] = r2 - 2.0 * (y * y + z * z);
    m[1] = 2.0 * (x * y - w * z);
    m[2] = 2.0 * (x * z + w * y);
    m[3] = 2.0 * (x * y + w * z);
    m[4] = r2 - 2.0 * (z * z + x * x);
    m[5] = 2.0 * (y * z - w * x);
    m[6] = 2.0 * (x * z - w * y);
    m[7] = 2.0 * (y * z + w * x);
    m[8] = r2 - 2.0 * (x * x + y * y);
    for (int i = 0; i < 9; ++i) m[i] = m[i] / r2;
}

// geometry.hpp:57-65: Sigma = (R^T diag(s^2)) R.  The first product has one
// non-zero term per coefficient (exact); the second sums in halves.
template <typename T>
void covariance(const T s[3], const T q[4], T cov[9]) {
    T r[9];
    quat_rot(q, r);
    const T s2[3] = {s[0] * s[0], s[1] * s[1], s[2] * s[2]};
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
            cov[3 * i + j] = tree3<T>(r[i] * s2[0] * r[j], r[3 + i] * s2[1] * r[3 + j],
                                      r[6 + i] * s2[2] * r[6 + j]);
}

struct Cam {
    orc_camera c;
    double w[9];    // world->camera rotation, quat_to_rotation(q_wc)
    double cen[3];  // camera centre -W^T t (scene.hpp:80)
};

Cam make_cam(const orc_camera& c) {
    Cam out;
    out.c = c;
    quat_rot(c.q_wc, out.w);
    for (int a = 0; a < 3; ++a)
        out.cen[a] = -(out.w[a] * c.t_wc[0] + out.w[3 + a] * c.t_wc[1] + out.w[6 + a] * c.t_wc[2]);
    return out;
}

template <typename T>
struct Proj {
    bool culled = true;
    double depth = 0.0;
    T mx{}, my{}, c00{}, c01{}, c11{};
};

// render.hpp:34-63: EWA local-affine projection (no frustum clamp)
template <typename T>
Proj<T> project(const T mu[3], const T s[3], const T q[4], const Cam& cam,
                const orc_render_opts& o) {
    Proj<T> out;
    const double* w = cam.w;
    T pc[3];
    for (int i = 0; i < 3; ++i)
        pc[i] = tree3<T>(w[3 * i] * mu[0], w[3 * i + 1] * mu[1], w[3 * i + 2] * mu[2]) +
                cam.c.t_wc[i];
    out.depth = P(pc[2]);
    if (out.depth <= o.z_near) return out;
    out.culled = false;
    const T inv_z = 1.0 / pc[2];
    out.mx = cam.c.fx * pc[0] * inv_z + cam.c.cx;
    out.my = cam.c.fy * pc[1] * inv_z + cam.c.cy;
    T sig[9];
    covariance(s, q, sig);
    T ws[9], sc[9];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
            ws[3 * i + j] = tree3<T>(w[3 * i] * sig[j], w[3 * i + 1] * sig[3 + j],
                                     w[3 * i + 2] * sig[6 + j]);
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
            sc[3 * i + j] = tree3<T>(ws[3 * i] * w[3 * j], ws[3 * i + 1] * w[3 * j + 1],
                                     ws[3 * i + 2] * w[3 * j + 2]);
    const T j00 = cam.c.fx * inv_z;
    const T j02 = -cam.c.fx * pc[0] * inv_z * inv_z;
    const T j11 = cam.c.fy * inv_z;
    const T j12 = -cam.c.fy * pc[1] * inv_z * inv_z;
    // J has structural zeros at (0,1) and (1,0); those terms are omitted
    const T a0 = j00 * sc[0] + j02 * sc[6];
    const T a1 = j00 * sc[1] + j02 * sc[7];
    const T a2 = j00 * sc[2] + j02 * sc[8];
    const T b1 = j11 * sc[4] + j12 * sc[7];
    const T b2 = j11 * sc[5] + j12 * sc[8];
    out.c00 = a0 * j00 + a2 * j02 + o.lowpass;
    out.c01 = a1 * j11 + a2 * j12;
    out.c11 = b1 * j11 + b2 * j12 + o.lowpass;
    return out;
}

// render.cpp:42-49
template <typename T>
void invert2x2(const T& c00, const T& c01, const T& c11, T& i00, T& i01,
               T& i11) {
    const T det = c00 * c11 - c01 * c01;
    i00 = c11 / det;
    i01 = -c01 / det;
    i11 = c00 / det;
}

template <typename T>
struct Frag {
    int64_t splat = -1;
    double depth = 0.0;
    double bx0 = 0, bx1 = 0, by0 = 0, by1 = 0;  // px -/+ rx, py -/+ ry
    T mx{}, my{}, i00{}, i01{}, i11{}, alpha{};
    T col[3];
};

// render.cpp:29-39
void check_finite(const SceneView& sc) {
    for (int64_t i = 0; i < sc.k; ++i) {
        bool ok = std::isfinite(sc.alpha(i));
        for (int a = 0; a < 3; ++a)
            ok = ok && std::isfinite(sc.mu(i)[a]) && std::isfinite(sc.s(i)[a]) &&
                 std::isfinite(sc.c(i)[a]);
        for (int a = 0; a < 4; ++a) ok = ok && std::isfinite(sc.q(i)[a]);
        for (int a = 0; a < 3 * sc.nb; ++a) ok = ok && std::isfinite(sc.sh(i)[a]);
        if (!ok)
            throw NumericErr("rasterize: non-finite parameter in splat " +
                             std::to_string(i));
    }
}

// render.cpp:51-69 (make_fragment) with the bbox bounds precomputed
template <typename T>
bool make_frag(int64_t i, const T mu[3], const T s[3], const T q[4],
               const T& alpha, const T col[3], const Cam& cam,
               const orc_render_opts& o, Frag<T>& f) {
    const Proj<T> pr = project<T>(mu, s, q, cam, o);
    if (pr.culled) return false;
    f.splat = i;
    f.depth = pr.depth;
    f.mx = pr.mx;
    f.my = pr.my;
    const double px = P(pr.mx), py = P(pr.my);
    const double rx = o.cutoff_sigma * std::sqrt(P(pr.c00));
    const double ry = o.cutoff_sigma * std::sqrt(P(pr.c11));
    f.bx0 = px - rx;
    f.bx1 = px + rx;
    f.by0 = py - ry;
    f.by1 = py + ry;
    invert2x2(pr.c00, pr.c01, pr.c11, f.i00, f.i01, f.i11);
    f.alpha = alpha;
    for (int a = 0; a < 3; ++a) f.col[a] = col[a];
    return true;
}

template <typename T>
void sort_frags(std::vector<Frag<T>>& fr) {  // render.cpp:83-87
    std::sort(fr.begin(), fr.end(), [](const Frag<T>& a, const Frag<T>& b) {
        return a.depth != b.depth ? a.depth < b.depth : a.splat < b.splat;
    });
}

std::vector<Frag<double>> build_frags(const SceneView& sc, const Cam& cam,
                                      const orc_render_opts& o) {
    std::vector<Frag<double>> fr;
    fr.reserve(sc.k);
    for (int64_t i = 0; i < sc.k; ++i) {
        Frag<double> f;
        double col[3];
        sh_color<double>(sc.mu(i), sc.c(i), sc.sh(i), sc.nb, cam.cen, col);
        if (make_frag<double>(i, sc.mu(i), sc.s(i), sc.q(i), sc.alpha(i), col, cam, o, f))
            fr.push_back(f);
    }
    sort_frags(fr);
    return fr;
}

std::vector<Frag<Dual>> build_frags_dual(const SceneView& sc, const Cam& cam,
                                         const double* v,
                                         const orc_render_opts& o) {
    const int64_t k = sc.k;
    std::vector<Frag<Dual>> fr;
    fr.reserve(k);
    for (int64_t i = 0; i < k; ++i) {
        Dual mu[3], s[3], q[4], col[3];
        for (int a = 0; a < 3; ++a) {
            mu[a] = Dual(sc.mu(i)[a], v[3 * i + a]);
            s[a] = Dual(sc.s(i)[a], v[3 * k + 3 * i + a]);
            col[a] = Dual(sc.c(i)[a], v[11 * k + 3 * i + a]);
        }
        for (int a = 0; a < 4; ++a) q[a] = Dual(sc.q(i)[a], v[6 * k + 4 * i + a]);
        const Dual alpha(sc.alpha(i), v[10 * k + i]);
        Dual shk[45], vcol[3];
        for (int a = 0; a < 3 * sc.nb; ++a) shk[a] = Dual(sc.sh(i)[a], v[sc.sh_off(i) + a]);
        sh_color<Dual>(mu, col, shk, sc.nb, cam.cen, vcol);
        Frag<Dual> f;
        if (make_frag<Dual>(i, mu, s, q, alpha, vcol, cam, o, f)) fr.push_back(f);
    }
    sort_frags(fr);
    return fr;
}

inline bool outside(const Frag<double>& f, double px, double py) {
    return px < f.bx0 || px > f.bx1 || py < f.by0 || py > f.by1;
}
inline bool outside(const Frag<Dual>& f, double px, double py) {
    return px < f.bx0 || px > f.bx1 || py < f.by0 || py > f.by1;
}

struct BlendCount {
    int64_t evaluated = 0, contributing = 0;
    std::vector<int32_t>* contrib = nullptr;  // splat ids of the contributing pairs
};

// render.cpp:122-151: front-to-back blend of one pixel
template <typename T>
void blend(const std::vector<Frag<T>>& fr, double px, double py,
           const orc_render_opts& o, T out[3], T& out_t,
           BlendCount* cnt = nullptr) {
    T tr(1.0);
    T acc[3] = {T(0.0), T(0.0), T(0.0)};
    for (const Frag<T>& f : fr) {
        if (outside(f, px, py)) continue;
        const T dx = px - f.mx;
        const T dy = py - f.my;
        const T expo = -0.5 * (dx * dx * f.i00 + dy * dy * f.i11) - dx * dy * f.i01;
        T abar = f.alpha * dexp(expo);
        if (cnt) ++cnt->evaluated;
        if (P(abar) >= o.alpha_clamp) abar = T(o.alpha_clamp);
        if (P(abar) < o.alpha_skip) continue;
        if (cnt) {
            ++cnt->contributing;
            if (cnt->contrib) cnt->contrib->push_back(static_cast<int32_t>(f.splat));
        }
        const T w = abar * tr;
        acc[0] += f.col[0] * w;
        acc[1] += f.col[1] * w;
        acc[2] += f.col[2] * w;
        tr = tr * (1.0 - abar);
        if (P(tr) < o.t_stop) break;
    }
    for (int c = 0; c < 3; ++c) out[c] = acc[c] + o.background[c] * tr;
    out_t = tr;
}

// parallel.hpp:12-44: round-robin rows over hardware_concurrency threads
void parallel_rows(int count, int workers, const std::function<void(int)>& fn) {
    if (workers <= 0) {
        const unsigned hw = std::thread::hardware_concurrency();
        workers = hw == 0 ? 1 : static_cast<int>(hw);
    }
    if (workers <= 1 || count <= 1) {
        for (int i = 0; i < count; ++i) fn(i);
        return;
    }
    const int n = std::min(workers, count);
    std::vector<std::thread> pool;
    std::mutex mu;
    std::exception_ptr err;
    for (int t = 0; t < n; ++t)
        pool.emplace_back([&, t]() {
            try {
                for (int i = t; i < count; i += n) fn(i);
            } catch (...) {
                std::lock_guard<std::mutex> g(mu);
                if (!err) err = std::current_exception();
            }
        });
    for (auto& th : pool) th.join();
    if (err) std::rethrow_exception(err);
}

// render.cpp:155-173
void rasterize(const SceneView& sc, const Cam& cam, const orc_render_opts& o,
               int workers, double* color, double* tfin) {
    check_finite(sc);
    const auto fr = build_frags(sc, cam, o);
    const int W = cam.c.width, H = cam.c.height;
    parallel_rows(H, workers, [&](int y) {
        for (int x = 0; x < W; ++x) {
            double c[3], t;
            blend<double>(fr, x + 0.5, y + 0.5, o, c, t);
            for (int ch = 0; ch < 3; ++ch) color[3 * (y * W + x) + ch] = c[ch];
            if (tfin) tfin[y * W + x] = t;
        }
    });
}

// render.cpp:175-192
void rasterize_jvp(const SceneView& sc, const Cam& cam,
                   const orc_render_opts& o, int workers, const double* v,
                   double* out) {
    check_finite(sc);
    const auto fr = build_frags_dual(sc, cam, v, o);
    const int W = cam.c.width, H = cam.c.height;
    parallel_rows(H, workers, [&](int y) {
        for (int x = 0; x < W; ++x) {
            Dual c[3], t;
            blend<Dual>(fr, x + 0.5, y + 0.5, o, c, t);
            for (int ch = 0; ch < 3; ++ch) out[3 * (y * W + x) + ch] = c[ch].d;
        }
    });
}

struct Processed {
    int fi;
    double abar, gauss, t_in;
    bool clamped;
    double dx, dy;
};

// render.cpp:210-258: forward replay then reverse sweep for one pixel;
// adj accumulates 9 slots per splat (mu2d 2, inverse cov 3, alpha, rgb)
void pixel_vjp(const std::vector<Frag<double>>& fr, double px, double py,
               const double* ub, const orc_render_opts& o,
               std::vector<Processed>& scr, double* adj,
               std::vector<int64_t>& touched, std::vector<char>& mark) {
    scr.clear();
    double tr = 1.0;
    for (int fi = 0; fi < static_cast<int>(fr.size()); ++fi) {
        const Frag<double>& f = fr[fi];
        if (outside(f, px, py)) continue;
        const double dx = px - f.mx, dy = py - f.my;
        const double expo =
            -0.5 * (dx * dx * f.i00 + dy * dy * f.i11) - dx * dy * f.i01;
        const double gauss = std::exp(expo);
        double abar = f.alpha * gauss;
        const bool clamped = abar >= o.alpha_clamp;
        if (clamped) abar = o.alpha_clamp;
        if (abar < o.alpha_skip) continue;
        scr.push_back({fi, abar, gauss, tr, clamped, dx, dy});
        tr = tr * (1.0 - abar);
        if (tr < o.t_stop) break;
    }
    double behind[3] = {o.background[0] * tr, o.background[1] * tr,
                        o.background[2] * tr};
    for (int i = static_cast<int>(scr.size()) - 1; i >= 0; --i) {
        const Processed& p = scr[i];
        const Frag<double>& f = fr[p.fi];
        if (!mark[f.splat]) {
            mark[f.splat] = 1;
            touched.push_back(f.splat);
        }
        double* a = adj + 9 * f.splat;
        double dab = 0.0;
        for (int ch = 0; ch < 3; ++ch) {
            a[6 + ch] += ub[ch] * p.abar * p.t_in;
            dab += ub[ch] * (f.col[ch] * p.t_in - behind[ch] / (1.0 - p.abar));
            behind[ch] += f.col[ch] * p.abar * p.t_in;
        }
        if (p.clamped) continue;
        a[5] += p.gauss * dab;
        const double de = p.abar * dab;
        a[2] += de * (-0.5 * p.dx * p.dx);
        a[3] += de * (-p.dx * p.dy);
        a[4] += de * (-0.5 * p.dy * p.dy);
        a[0] += de * (f.i00 * p.dx + f.i01 * p.dy);
        a[1] += de * (f.i01 * p.dx + f.i11 * p.dy);
    }
}

// chain of the 9 per-splat adjoints through project + invert2x2 with 10
// dual seeds (render.cpp:294-329)
void chain_splat(const SceneView& sc, const Cam& cam, const orc_render_opts& o,
                 int64_t i, const double* a, double* grad) {
    const int64_t k = sc.k;
    grad[10 * k + i] += a[5];
    for (int ch = 0; ch < 3; ++ch) grad[11 * k + 3 * i + ch] += a[6 + ch];
    if (sc.nb > 0 && (a[6] != 0.0 || a[7] != 0.0 || a[8] != 0.0)) {
        // SH extension: dL/dk_j = Y_j a_rgb, and the colour's dependence on
        // mu through the view direction (3 dual seeds)
        double d[3], Y[15];
        sh_dir<double>(sc.mu(i), cam.cen, d);
        sh_basis<double>(d[0], d[1], d[2], sc.nb, Y);
        for (int j = 0; j < sc.nb; ++j)
            for (int ch = 0; ch < 3; ++ch) grad[sc.sh_off(i) + 3 * j + ch] += Y[j] * a[6 + ch];
        Dual shk[45], c0[3], col[3];
        for (int t = 0; t < 3 * sc.nb; ++t) shk[t] = Dual(sc.sh(i)[t]);
        for (int ch = 0; ch < 3; ++ch) c0[ch] = Dual(sc.c(i)[ch]);
        for (int seed = 0; seed < 3; ++seed) {
            Dual mu[3];
            for (int c = 0; c < 3; ++c) mu[c] = Dual(sc.mu(i)[c], seed == c ? 1.0 : 0.0);
            sh_color<Dual>(mu, c0, shk, sc.nb, cam.cen, col);
            grad[3 * i + seed] += a[6] * col[0].d + a[7] * col[1].d + a[8] * col[2].d;
        }
    }
    bool any = false;
    for (int j = 0; j < 5; ++j) any = any || a[j] != 0.0;
    if (!any) return;
    for (int seed = 0; seed < 10; ++seed) {
        Dual mu[3], s[3], q[4];
        for (int c = 0; c < 3; ++c) {
            mu[c] = Dual(sc.mu(i)[c], seed == c ? 1.0 : 0.0);
            s[c] = Dual(sc.s(i)[c], seed == 3 + c ? 1.0 : 0.0);
        }
        for (int c = 0; c < 4; ++c) q[c] = Dual(sc.q(i)[c], seed == 6 + c ? 1.0 : 0.0);
        const Proj<Dual> pr = project<Dual>(mu, s, q, cam, o);
        if (pr.culled) break;
        Dual i00, i01, i11;
        invert2x2(pr.c00, pr.c01, pr.c11, i00, i01, i11);
        const double dot = a[0] * pr.mx.d + a[1] * pr.my.d + a[2] * i00.d +
                           a[3] * i01.d + a[4] * i11.d;
        const int64_t off = seed < 3 ? 3 * i + seed
                                     : (seed < 6 ? 3 * k + 3 * i + (seed - 3)
                                                 : 6 * k + 4 * i + (seed - 6));
        grad[off] += dot;
    }
}

// render.cpp:262-331.  Per-row partials are kept sparse (touched splats only)
// and reduced in row order, the reference's order, without its H*9*K buffer.
void rasterize_vjp(const SceneView& sc, const Cam& cam,
                   const orc_render_opts& o, int workers, const double* adjimg,
                   double* grad) {
    check_finite(sc);
    const auto fr = build_frags(sc, cam, o);
    const int W = cam.c.width, H = cam.c.height;
    const int64_t k = sc.k;
    struct RowPart {
        std::vector<int64_t> idx;
        std::vector<double> val;
    };
    std::vector<RowPart> rows(H);
    // one dense scratch per worker thread
    std::mutex pool_mu;
    std::vector<std::vector<double>*> pool;
    std::vector<std::unique_ptr<std::vector<double>>> owners;
    parallel_rows(H, workers, [&](int y) {
        std::vector<double>* buf = nullptr;
        {
            std::lock_guard<std::mutex> g(pool_mu);
            if (!pool.empty()) {
                buf = pool.back();
                pool.pop_back();
            } else {
                owners.emplace_back(new std::vector<double>(9 * k, 0.0));
                buf = owners.back().get();
            }
        }
        std::vector<double>& adj = *buf;
        std::vector<Processed> scr;
        std::vector<int64_t> touched;
        std::vector<char> mark(k, 0);
        for (int x = 0; x < W; ++x) {
            const double* ub = adjimg + 3 * (y * W + x);
            if (ub[0] == 0.0 && ub[1] == 0.0 && ub[2] == 0.0) continue;
            pixel_vjp(fr, x + 0.5, y + 0.5, ub, o, scr, adj.data(), touched, mark);
        }
        std::sort(touched.begin(), touched.end());
        RowPart& rp = rows[y];
        rp.idx = touched;
        rp.val.resize(9 * touched.size());
        for (size_t t = 0; t < touched.size(); ++t)
            for (int j = 0; j < 9; ++j) {
                rp.val[9 * t + j] = adj[9 * touched[t] + j];
                adj[9 * touched[t] + j] = 0.0;
            }
        std::lock_guard<std::mutex> g(pool_mu);
        pool.push_back(buf);
    });
    std::vector<double> adj(9 * k, 0.0);
    for (int y = 0; y < H; ++y) {
        const RowPart& rp = rows[y];
        for (size_t t = 0; t < rp.idx.size(); ++t)
            for (int j = 0; j < 9; ++j) adj[9 * rp.idx[t] + j] += rp.val[9 * t + j];
    }
    std::fill(grad, grad + sc.dim(), 0.0);
    for (int64_t i = 0; i < k; ++i) chain_splat(sc, cam, o, i, adj.data() + 9 * i, grad);
}

// ---------------------------------------------------------------- SSIM
// ssim.cpp:15-58
constexpr int kWin = 11, kHalf = 5;
constexpr double kC1 = 0.01 * 0.01, kC2 = 0.03 * 0.03;

const double* kernel1d() {
    static const std::vector<double> k = [] {
        std::vector<double> w(kWin);
        double sum = 0.0;
        for (int i = 0; i < kWin; ++i) {
            const double d = i - kHalf;
            w[i] = std::exp(-d * d / (2.0 * 1.5 * 1.5));
            sum += w[i];
        }
        for (double& v : w) v /= sum;
        return w;
    }();
    return k.data();
}

inline int reflect(int i, int n) {
    if (i < 0) return -i;
    if (i >= n) return 2 * n - 2 - i;
    return i;
}

void check_ssim_shape(int w, int h) {
    if (w < kHalf + 1 || h < kHalf + 1)
        throw InvalidArg("ssim: image smaller than the window");
}

template <typename T>
T ssim_moments(const T& mu_a, double mu_b, const T& maa, double mbb,
               const T& mab) {
    const T n1 = 2.0 * mu_a * mu_b + kC1;
    const T d1 = mu_a * mu_a + mu_b * mu_b + kC1;
    const T n2 = 2.0 * (mab - mu_a * mu_b) + kC2;
    const T d2 = (maa - mu_a * mu_a) + (mbb - mu_b * mu_b) + kC2;
    return (n1 * n2) / (d1 * d2);
}

// ssim.cpp:60-86: direct 121-tap gather
template <typename T, typename GetA, typename Put>
void ssim_generic(const double* b, int W, int H, GetA get_a, Put put) {
    const double* k = kernel1d();
    for (int y = 0; y < H; ++y)
        for (int x = 0; x < W; ++x)
            for (int c = 0; c < 3; ++c) {
                T mu_a(0.0), maa(0.0), mab(0.0);
                double mu_b = 0.0, mbb = 0.0;
                for (int dy = -kHalf; dy <= kHalf; ++dy) {
                    const int yy = reflect(y + dy, H);
                    const double wy = k[dy + kHalf];
                    for (int dx = -kHalf; dx <= kHalf; ++dx) {
                        const int xx = reflect(x + dx, W);
                        const double w = wy * k[dx + kHalf];
                        const T av = get_a(xx, yy, c);
                        const double bv = b[3 * (yy * W + xx) + c];
                        mu_a += w * av;
                        maa += w * av * av;
                        mab += (w * bv) * av;
                        mu_b += w * bv;
                        mbb += w * bv * bv;
                    }
                }
                put(x, y, c, ssim_moments<T>(mu_a, mu_b, maa, mbb, mab));
            }
}

void ssim_map(const double* a, const double* b, int W, int H, double* out) {
    check_ssim_shape(W, H);
    ssim_generic<double>(
        b, W, H, [&](int x, int y, int c) { return a[3 * (y * W + x) + c]; },
        [&](int x, int y, int c, double s) { out[3 * (y * W + x) + c] = s; });
}

void ssim_jvp(const double* a, const double* da, const double* b, int W, int H,
              double* s, double* ds) {
    check_ssim_shape(W, H);
    ssim_generic<Dual>(
        b, W, H,
        [&](int x, int y, int c) {
            const int64_t i = 3 * (y * W + x) + c;
            return Dual(a[i], da[i]);
        },
        [&](int x, int y, int c, const Dual& v) {
            const int64_t i = 3 * (y * W + x) + c;
            s[i] = v.v;
            ds[i] = v.d;
        });
}

// ssim.cpp:115-168: scatter-form adjoint
void ssim_vjp(const double* a, const double* b, const double* up, int W, int H,
              double* grad) {
    check_ssim_shape(W, H);
    const double* k = kernel1d();
    std::fill(grad, grad + 3 * (int64_t)W * H, 0.0);
    auto at = [&](const double* img, int x, int y, int c) {
        return img[3 * (y * W + x) + c];
    };
    for (int y = 0; y < H; ++y)
        for (int x = 0; x < W; ++x)
            for (int c = 0; c < 3; ++c) {
                const double u = at(up, x, y, c);
                if (u == 0.0) continue;
                double mu_a = 0, mu_b = 0, maa = 0, mbb = 0, mab = 0;
                for (int dy = -kHalf; dy <= kHalf; ++dy) {
                    const int yy = reflect(y + dy, H);
                    const double wy = k[dy + kHalf];
                    for (int dx = -kHalf; dx <= kHalf; ++dx) {
                        const int xx = reflect(x + dx, W);
                        const double w = wy * k[dx + kHalf];
                        const double av = at(a, xx, yy, c), bv = at(b, xx, yy, c);
                        mu_a += w * av;
                        mu_b += w * bv;
                        maa += w * av * av;
                        mbb += w * bv * bv;
                        mab += w * av * bv;
                    }
                }
                const double n1 = 2.0 * mu_a * mu_b + kC1;
                const double d1 = mu_a * mu_a + mu_b * mu_b + kC1;
                const double n2 = 2.0 * (mab - mu_a * mu_b) + kC2;
                const double d2 = (maa - mu_a * mu_a) + (mbb - mu_b * mu_b) + kC2;
                const double p = n1 / d1, q = n2 / d2;
                const double ds_dmu =
                    q * (2.0 * mu_b * d1 - 2.0 * mu_a * n1) / (d1 * d1) +
                    p * (2.0 * mu_a * n2 - 2.0 * mu_b * d2) / (d2 * d2);
                const double ds_dmaa = -p * n2 / (d2 * d2);
                const double ds_dmab = p * 2.0 / d2;
                for (int dy = -kHalf; dy <= kHalf; ++dy) {
                    const int yy = reflect(y + dy, H);
                    const double wy = k[dy + kHalf];
                    for (int dx = -kHalf; dx <= kHalf; ++dx) {
                        const int xx = reflect(x + dx, W);
                        const double w = wy * k[dx + kHalf];
                        grad[3 * (yy * W + xx) + c] +=
                            u * w *
                            (ds_dmu + ds_dmaa * 2.0 * at(a, xx, yy, c) +
                             ds_dmab * at(b, xx, yy, c));
                    }
                }
            }
}

// ---------------------------------------------------------------- residuals
inline double sgn(double v) { return v > 0.0 ? 1.0 : (v < 0.0 ? -1.0 : 0.0); }

// residuals.cpp:27-45
void residual_vector(const double* img, const double* gt, int W, int H,
                     const orc_residual_opts& o, double* r) {
    const int64_t P = (int64_t)W * H, n = 3 * P;
    std::vector<double> ss(n);
    ssim_map(img, gt, W, H, ss.data());
    for (int y = 0; y < H; ++y)
        for (int x = 0; x < W; ++x)
            for (int c = 0; c < 3; ++c) {
                const int64_t i = c * P + (int64_t)y * W + x;
                const int64_t p = 3 * ((int64_t)y * W + x) + c;
                const double d = img[p] - gt[p];
                r[i] = std::sqrt(std::max((1.0 - o.lambda) * std::abs(d), o.floor_));
                const double dssim = o.lambda * (1.0 - ss[p]) / 2.0;
                r[n + i] = std::sqrt(std::max(dssim, o.floor_));
            }
}

// residuals.cpp:47-79
void residual_jvp(const double* img, const double* tan, const double* gt,
                  int W, int H, const orc_residual_opts& o, double* dr) {
    const int64_t P = (int64_t)W * H, n = 3 * P;
    std::vector<double> ss(n), dss(n);
    ssim_jvp(img, tan, gt, W, H, ss.data(), dss.data());
    for (int y = 0; y < H; ++y)
        for (int x = 0; x < W; ++x)
            for (int c = 0; c < 3; ++c) {
                const int64_t i = c * P + (int64_t)y * W + x;
                const int64_t p = 3 * ((int64_t)y * W + x) + c;
                const double d = img[p] - gt[p];
                const double u1 = (1.0 - o.lambda) * std::abs(d);
                if (u1 > o.floor_) {
                    const double r = std::sqrt(u1);
                    dr[i] = (1.0 - o.lambda) * sgn(d) * tan[p] / (2.0 * r);
                } else {
                    dr[i] = 0.0;
                }
                const double u2 = o.lambda * (1.0 - ss[p]) / 2.0;
                if (u2 > o.floor_) {
                    const double r = std::sqrt(u2);
                    dr[n + i] = -o.lambda * dss[p] / (4.0 * r);
                } else {
                    dr[n + i] = 0.0;
                }
            }
}

// residuals.cpp:81-117
void residual_vjp(const double* img, const double* gt, int W, int H,
                  const double* u, const orc_residual_opts& o, double* adj) {
    const int64_t P = (int64_t)W * H, n = 3 * P;
    std::vector<double> ss(n), up(n, 0.0);
    ssim_map(img, gt, W, H, ss.data());
    std::fill(adj, adj + n, 0.0);
    for (int y = 0; y < H; ++y)
        for (int x = 0; x < W; ++x)
            for (int c = 0; c < 3; ++c) {
                const int64_t i = c * P + (int64_t)y * W + x;
                const int64_t p = 3 * ((int64_t)y * W + x) + c;
                const double d = img[p] - gt[p];
                const double u1 = (1.0 - o.lambda) * std::abs(d);
                if (u1 > o.floor_)
                    adj[p] += u[i] * (1.0 - o.lambda) * sgn(d) / (2.0 * std::sqrt(u1));
                const double u2 = o.lambda * (1.0 - ss[p]) / 2.0;
                if (u2 > o.floor_) up[p] = u[n + i] * (-o.lambda / (4.0 * std::sqrt(u2)));
            }
    bool any = false;
    for (double v : up)
        if (v != 0.0) {
            any = true;
            break;
        }
    if (any) {
        std::vector<double> g(n);
        ssim_vjp(img, gt, up.data(), W, H, g.data());
        for (int64_t i = 0; i < n; ++i) adj[i] += g[i];
    }
}

// VectorXd::squaredNorm(): two SSE2 packet accumulators over the aligned
// body, lanes added, scalar tail (Redux.h, LinearVectorized/NoUnrolling)
double sq_norm(const std::vector<double>& v) {
    const size_t n = v.size(), n4 = n / 4 * 4, n2 = n / 2 * 2;
    if (n2 == 0) return n ? v[0] * v[0] : 0.0;
    double a0 = v[0] * v[0], a1 = v[1] * v[1];
    if (n2 > 2) {
        double b0 = v[2] * v[2], b1 = v[3] * v[3];
        for (size_t k = 4; k < n4; k += 4) {
            a0 += v[k] * v[k];
            a1 += v[k + 1] * v[k + 1];
            b0 += v[k + 2] * v[k + 2];
            b1 += v[k + 3] * v[k + 3];
        }
        a0 += b0;
        a1 += b1;
        if (n2 > n4) {
            a0 += v[n4] * v[n4];
            a1 += v[n4 + 1] * v[n4 + 1];
        }
    }
    double s = a0 + a1;
    for (size_t k = n2; k < n; ++k) s += v[k] * v[k];
    return s;
}

// ---------------------------------------------------------------- optimizer
struct Problem {
    SceneView sc;
    std::vector<Cam> cams;
    std::vector<const double*> gts;
    orc_residual_opts rs;
    orc_render_opts ro;
    int workers;
    int W() const { return cams[0].c.width; }
    int H() const { return cams[0].c.height; }
};

Problem make_problem(const double* x, int64_t k, const orc_camera* cams,
                     const double* const* gts, int n, const orc_residual_opts* rs,
                     const orc_render_opts* ro, int workers) {
    Problem p{{x, k}, {}, {}, *rs, *ro, workers};
    for (int i = 0; i < n; ++i) {
        p.cams.push_back(make_cam(cams[i]));
        p.gts.push_back(gts ? gts[i] : nullptr);
    }
    return p;
}

// optimizer.cpp:18-25
std::vector<double> jac_apply(const Problem& pb, int vi, const double* v) {
    const Cam& cam = pb.cams.at(vi);
    const int W = cam.c.width, H = cam.c.height;
    const int64_t n = 3LL * W * H;
    std::vector<double> img(n), tan(n), out(2 * n);
    rasterize(pb.sc, cam, pb.ro, pb.workers, img.data(), nullptr);
    rasterize_jvp(pb.sc, cam, pb.ro, pb.workers, v, tan.data());
    residual_jvp(img.data(), tan.data(), pb.gts[vi], W, H, pb.rs, out.data());
    return out;
}

// optimizer.cpp:27-34
std::vector<double> jac_applyT(const Problem& pb, int vi, const double* u) {
    const Cam& cam = pb.cams.at(vi);
    const int W = cam.c.width, H = cam.c.height;
    const int64_t n = 3LL * W * H;
    std::vector<double> img(n), adj(n), g(pb.sc.dim());
    rasterize(pb.sc, cam, pb.ro, pb.workers, img.data(), nullptr);
    residual_vjp(img.data(), pb.gts[vi], W, H, u, pb.rs, adj.data());
    rasterize_vjp(pb.sc, cam, pb.ro, pb.workers, adj.data(), g.data());
    return g;
}

// optimizer.cpp:36-65
std::vector<double> stochastic_gradient(const Problem& pb,
                                        const std::vector<int>& batch,
                                        double* batch_loss) {
    if (batch.empty()) throw InvalidArg("stochastic_gradient: empty batch");
    const int64_t M = pb.cams.size();
    const long m = 6L * pb.W() * pb.H() * M;
    const int64_t dim = pb.sc.dim();
    std::vector<double> g(dim, 0.0), gv(dim);
    double loss = 0.0;
    for (int vi : batch) {
        const Cam& cam = pb.cams.at(vi);
        const int W = cam.c.width, H = cam.c.height;
        const int64_t n = 3LL * W * H;
        std::vector<double> img(n), f(2 * n), adj(n);
        rasterize(pb.sc, cam, pb.ro, pb.workers, img.data(), nullptr);
        residual_vector(img.data(), pb.gts[vi], W, H, pb.rs, f.data());
        residual_vjp(img.data(), pb.gts[vi], W, H, f.data(), pb.rs, adj.data());
        rasterize_vjp(pb.sc, cam, pb.ro, pb.workers, adj.data(), gv.data());
        bool finite = true;
        for (int64_t i = 0; i < dim; ++i) {
            g[i] += gv[i];
            finite = finite && std::isfinite(g[i]);
        }
        loss += sq_norm(f);
        if (!finite)
            throw NumericErr("stochastic_gradient: non-finite gradient from view " +
                             std::to_string(cam.c.id));
    }
    const double scale = static_cast<double>(M) /
                         (static_cast<double>(m) * batch.size());
    for (double& v : g) v *= scale;
    if (batch_loss)
        *batch_loss = loss * static_cast<double>(M) /
                      (2.0 * static_cast<double>(m) * batch.size());
    return g;
}

// optimizer.cpp:75-104
template <typename ProbeFn>
std::vector<double> hutchinson_diag(const Problem& pb,
                                    const std::vector<int>& batch, int nu,
                                    ProbeFn probes) {
    if (nu < 1) throw InvalidArg("hutchinson_diag: nu must be >= 1");
    if (batch.empty()) throw InvalidArg("hutchinson_diag: empty batch");
    const int64_t M = pb.cams.size();
    const long m = 6L * pb.W() * pb.H() * M;
    const int64_t dim = pb.sc.dim();
    std::vector<double> acc(dim, 0.0);
    for (int s = 0; s < nu; ++s) {
        const std::vector<double> z = probes(s);
        std::vector<double> w(dim, 0.0);
        for (int vi : batch) {
            const std::vector<double> jz = jac_apply(pb, vi, z.data());
            const std::vector<double> wv = jac_applyT(pb, vi, jz.data());
            for (int64_t i = 0; i < dim; ++i) w[i] += wv[i];
        }
        for (double v : w)
            if (!std::isfinite(v)) throw NumericErr("hutchinson_diag: non-finite sample");
        for (int64_t i = 0; i < dim; ++i) acc[i] += z[i] * w[i];
    }
    const double scale = static_cast<double>(M) /
                         (static_cast<double>(m) * batch.size() * nu);
    for (double& v : acc) v *= scale;
    return acc;
}

// ---------------------------------------------------------------- trust region
inline double cap_radius(double r, double cap) {  // trust_region.cpp:39-42
    if (!(r > 0.0) || !std::isfinite(r)) return cap;
    return std::min(r, cap);
}

inline double log_factor(double eps, double alpha) {  // trust_region.cpp:46-50
    const double u = eps / alpha;
    if (u >= 1.0 - 1e-12) return -1.0;
    return -8.0 * std::log1p(-u);
}

// 3x3 determinant by first-row cofactors
inline double det3(const double m[9]) {
    return m[0] * (m[4] * m[8] - m[5] * m[7]) - m[1] * (m[3] * m[8] - m[5] * m[6]) +
           m[2] * (m[3] * m[7] - m[4] * m[6]);
}

struct Prim {
    double mu[3], s[3], q[4], alpha, c[3];
};

Prim prim_at(const SceneView& sc, int64_t i) {
    Prim p;
    for (int a = 0; a < 3; ++a) {
        p.mu[a] = sc.mu(i)[a];
        p.s[a] = sc.s(i)[a];
        p.c[a] = sc.c(i)[a];
    }
    for (int a = 0; a < 4; ++a) p.q[a] = sc.q(i)[a];
    p.alpha = sc.alpha(i);
    return p;
}

// trust_region.cpp:54-69 (inverse diagonal via cofactors)
void radius_mean(const Prim& p, double eps, double cap, double out[3]) {
    const double lf = log_factor(eps, p.alpha);
    if (lf <= 0.0) {
        out[0] = out[1] = out[2] = cap;
        return;
    }
    double m[9];
    covariance(p.s, p.q, m);
    const double c00 = m[4] * m[8] - m[5] * m[7];
    const double c10 = m[7] * m[2] - m[8] * m[1];
    const double c20 = m[1] * m[5] - m[2] * m[4];
    const double det = c00 * m[0] + c10 * m[3] + c20 * m[6];
    const double invdet = 1.0 / det;
    const double c11 = m[8] * m[0] - m[6] * m[2];
    const double c22 = m[0] * m[4] - m[1] * m[3];
    const double inv[3] = {c00 * invdet, c11 * invdet, c22 * invdet};
    for (int c = 0; c < 3; ++c) out[c] = cap_radius(std::sqrt(lf / inv[c]), cap);
}

// trust_region.cpp:95-128
void quat_dR(const double q[4], int axis, double d[9]) {
    const double x = q[0], y = q[1], z = q[2], w = q[3];
    const double t0[9] = {2 * x, 2 * y, 2 * z, 2 * y, -2 * x, -2 * w, 2 * z, 2 * w, -2 * x};
    const double t1[9] = {-2 * y, 2 * x, 2 * w, 2 * x, 2 * y, 2 * z, -2 * w, 2 * z, -2 * y};
    const double t2[9] = {-2 * z, -2 * w, 2 * x, 2 * w, -2 * z, 2 * y, 2 * x, 2 * y, 2 * z};
    const double t3[9] = {2 * w, -2 * z, 2 * y, 2 * z, 2 * w, -2 * x, -2 * y, 2 * x, 2 * w};
    const double* t = axis == 0 ? t0 : axis == 1 ? t1 : axis == 2 ? t2 : t3;
    for (int i = 0; i < 9; ++i) d[i] = t[i];
}

void quat_d2R(int axis, double d[9]) {
    static const double diag[4][3] = {{2, -2, -2}, {-2, 2, -2}, {-2, -2, 2}, {2, 2, 2}};
    for (int i = 0; i < 9; ++i) d[i] = 0.0;
    for (int i = 0; i < 3; ++i) d[4 * i] = diag[axis][i];
}

// trust_region.cpp:132-155
double beta_rotation(const Prim& p, int axis) {
    const double* q = p.q;
    const double r2 = sqnorm4(q);  // q.squaredNorm()
    if (r2 < 1e-24) throw InvalidArg("beta_rotation: degenerate quaternion");
    const double qc = q[axis];
    const double x = q[0], y = q[1], z = q[2], w = q[3];
    const double ru = x * x + y * y + z * z + w * w;  // quat_rotation_unnormalized's own
    const double rt[9] = {ru - 2.0 * (y * y + z * z), 2.0 * (x * y - w * z),
                          2.0 * (x * z + w * y),      2.0 * (x * y + w * z),
                          ru - 2.0 * (z * z + x * x), 2.0 * (y * z - w * x),
                          2.0 * (x * z - w * y),      2.0 * (y * z + w * x),
                          ru - 2.0 * (x * x + y * y)};
    double r[9], drt[9], d2rt[9];
    for (int i = 0; i < 9; ++i) r[i] = rt[i] / r2;
    quat_dR(q, axis, drt);
    quat_d2R(axis, d2rt);
    const double k1 = 2.0 * qc / (r2 * r2);
    const double k2 = 4.0 * qc / (r2 * r2);
    const double k3 = 8.0 * qc * qc / (r2 * r2 * r2) - 2.0 / (r2 * r2);
    double in1[9], in2[9], de[9], d2e[9];
    for (int i = 0; i < 9; ++i) {
        in1[i] = drt[i] / r2 - k1 * rt[i];
        in2[i] = d2rt[i] / r2 - k2 * drt[i] + k3 * rt[i];
    }
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            de[3 * i + j] = r[i] * in1[j] + r[3 + i] * in1[3 + j] + r[6 + i] * in1[6 + j];
            d2e[3 * i + j] = r[i] * in2[j] + r[3 + i] * in2[3 + j] + r[6 + i] * in2[6 + j];
        }
    double frob = 0.0;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            const double v = p.s[i] * de[3 * i + j] / p.s[j];
            frob += v * v;
        }
    return 2.0 * frob + 2.0 * tree3(d2e[0], d2e[4], d2e[8]);
}

// trust_region.cpp:183-194
double rotation_h2(const Prim& p, const double sigma[9], double det_s, int axis,
                   double dq) {
    double q2[4] = {p.q[0], p.q[1], p.q[2], p.q[3]};
    q2[axis] += dq;
    if (q2[0] * q2[0] + q2[1] * q2[1] + q2[2] * q2[2] + q2[3] * q2[3] < 1e-24)
        return std::numeric_limits<double>::infinity();
    double c2[9], mid[9];
    covariance(p.s, q2, c2);
    for (int i = 0; i < 9; ++i) mid[i] = 0.5 * (sigma[i] + c2[i]);
    const double dm = det3(mid);
    if (!(dm > 0.0)) return std::numeric_limits<double>::infinity();
    return p.alpha * (1.0 - det_s / std::sqrt(dm));
}

// trust_region.cpp:198-234
void radius_rotation(const Prim& p, double eps, double cap, double out[4]) {
    const double lf = log_factor(eps, p.alpha);
    if (lf <= 0.0) {
        for (int c = 0; c < 4; ++c) out[c] = cap;
        return;
    }
    double sigma[9];
    covariance(p.s, p.q, sigma);
    const double det_s = p.s[0] * p.s[1] * p.s[2];
    for (int c = 0; c < 4; ++c) {
        const double beta = beta_rotation(p, c);
        double r = beta <= 1e-12 ? cap : cap_radius(std::sqrt(lf / beta), cap);
        const double tol = eps * (1.0 + 1e-9);
        auto within = [&](double st) {
            return rotation_h2(p, sigma, det_s, c, st) <= tol &&
                   rotation_h2(p, sigma, det_s, c, -st) <= tol;
        };
        if (!within(r)) {
            double lo = 0.0, hi = r;
            for (int it = 0; it < 60; ++it) {
                const double mid = 0.5 * (lo + hi);
                if (within(mid))
                    lo = mid;
                else
                    hi = mid;
            }
            r = lo > 0.0 ? lo : r * 0x1.0p-60;
        }
        out[c] = r;
    }
}

// trust_region.cpp:236-252
void shd_radii(const SceneView& sc, double eps, const double caps[5], double* eta) {
    const int64_t k = sc.k;
    for (int64_t i = 0; i < k; ++i) {
        const Prim p = prim_at(sc, i);
        double rm[3], rq[4];
        radius_mean(p, eps, caps[0], rm);
        radius_rotation(p, eps, caps[2], rq);
        for (int c = 0; c < 3; ++c) {
            eta[3 * i + c] = rm[c];
            eta[3 * k + 3 * i + c] =
                cap_radius(std::sqrt(2.0 * p.s[c] * p.s[c] * eps / p.alpha), caps[1]);
            eta[11 * k + 3 * i + c] =
                cap_radius(std::sqrt(4.0 * p.c[c] * eps / p.alpha), caps[4]);
        }
        for (int c = 0; c < 4; ++c) eta[6 * k + 4 * i + c] = rq[c];
        eta[10 * k + i] = cap_radius(std::sqrt(4.0 * p.alpha * eps), caps[3]);
        // SH extension: a single-coefficient step moves the view colour by
        // at most the reference's colour radius in any direction
        for (int j = 0; j < sc.nb; ++j)
            for (int c = 0; c < 3; ++c)
                eta[sc.sh_off(i) + 3 * j + c] = eta[11 * k + 3 * i + c] / kShMax[j];
    }
}

double eps_at(double e0, double e1, int total, int t) {  // trust_region.cpp:261-268
    if (!(e0 >= e1) || !(e1 > 0.0)) throw InvalidArg("eps_at: bad schedule");
    if (total <= 0 || t <= 0) return e0;
    if (t >= total) return e1;
    const double frac = static_cast<double>(t) / total;
    return e0 * std::pow(e1 / e0, frac);
}

// ---------------------------------------------------------------- Algorithm 1
}  // namespace

struct orc_state {
    std::vector<double> g_hat, d_hat, adam_m, adam_v;
    int64_t t = 0;
    Rng rng;
    orc_state(int64_t dim, uint64_t seed)
        : g_hat(dim, 0.0), d_hat(dim, 0.0), adam_m(dim, 0.0), adam_v(dim, 0.0), rng(seed) {}
};

struct orc_rng {
    Rng r;
    explicit orc_rng(uint64_t s) : r(s) {}
};

namespace {

double vnorm(const std::vector<double>& v) { return std::sqrt(sq_norm(v)); }

void apply_clipped(orc_state* st, double* x, const Problem& pb, const orc_tr_opts& o,
                   const std::vector<double>& dx, orc_diag& dg, double* applied);

// optimizer.cpp:189-220 with the draws either taken from the state's Rng
// (reference order: S1, then on refresh S2 and nu probes coordinate-
// ascending) or supplied explicitly (teacher forcing)
void step_tr(orc_state* st, double* x, const Problem& pb, const orc_tr_opts& o,
             const std::vector<int>* s1_in, const std::vector<int>* s2_in,
             const double* probes_in, orc_diag* diag, double* applied) {
    const int64_t dim = pb.sc.dim();
    orc_diag dg{0, 0, 0, 0, -1, -1, 0};
    st->t += 1;
    const int mv = static_cast<int>(pb.cams.size());
    const std::vector<int> s1 = s1_in ? *s1_in : st->rng.sample(mv, o.batch_size);
    const std::vector<double> g = stochastic_gradient(pb, s1, &dg.batch_loss);
    dg.gnorm = vnorm(g);
    for (int64_t i = 0; i < dim; ++i)
        st->g_hat[i] = o.theta1 * st->g_hat[i] + (1.0 - o.theta1) * g[i];
    const bool refresh = o.hess_interval <= 1 || st->t % o.hess_interval == 1;
    if (refresh) {
        const std::vector<int> s2 =
            s2_in ? *s2_in : st->rng.sample(mv, o.hutch_batch_size);
        auto probe = [&](int s) {
            std::vector<double> z(dim);
            if (probes_in)
                std::copy(probes_in + s * dim, probes_in + (s + 1) * dim, z.begin());
            else
                for (int64_t i = 0; i < dim; ++i) z[i] = st->rng.rademacher();
            return z;
        };
        const std::vector<double> d = hutchinson_diag(pb, s2, o.hutch_samples, probe);
        for (int64_t i = 0; i < dim; ++i)
            st->d_hat[i] = o.theta2 * st->d_hat[i] + (1.0 - o.theta2) * d[i];
    }
    std::vector<double> dx(dim);
    for (int64_t i = 0; i < dim; ++i)
        dx[i] = -st->g_hat[i] / std::max(st->d_hat[i], o.gamma_d);
    dg.step_pre = vnorm(dx);
    apply_clipped(st, x, pb, o, dx, dg, applied);
    *diag = dg;
}

// Scene::clamp, scene.cpp:49-57
void clamp_scene(double* x, int64_t k, const orc_tr_opts& o) {
    for (int64_t i = 0; i < k; ++i) {
        for (int a = 0; a < 3; ++a) {
            double& s = x[3 * k + 3 * i + a];
            s = std::max(s, o.s_min);
            double& c = x[11 * k + 3 * i + a];
            c = std::min(std::max(c, o.c_min), o.c_max);
        }
        double& al = x[10 * k + i];
        al = std::min(std::max(al, o.alpha_min), o.alpha_max);
    }
}

// apply_clipped, optimizer.cpp:124-142
void apply_clipped(orc_state* st, double* x, const Problem& pb, const orc_tr_opts& o,
                   const std::vector<double>& dx, orc_diag& dg, double* applied) {
    const int64_t k = pb.sc.k, dim = pb.sc.dim();
    const double eps = eps_at(o.eps_start, o.eps_end, o.total_steps, (int)st->t);
    const double caps[5] = {o.cap_mean, o.cap_scale, o.cap_rotation, o.cap_opacity,
                            o.cap_color};
    std::vector<double> eta(dim), cl(dim);
    shd_radii(pb.sc, eps, caps, eta.data());
    for (int64_t i = 0; i < dim; ++i) cl[i] = std::min(std::max(dx[i], -eta[i]), eta[i]);
    for (int64_t i = 0; i < dim; ++i)
        if (!std::isfinite(cl[i]))
            throw NumericErr(std::string("non-finite update in group ") +
                             kGroup[group_of(k, i)]);
    int64_t nclip = 0;
    double mr = 0.0;
    for (int64_t i = 0; i < dim; ++i) {
        if (std::abs(dx[i]) > eta[i]) ++nclip;
        mr = std::max(mr, std::abs(cl[i]) / eta[i]);
    }
    dg.eps = eps;
    dg.clip_frac = static_cast<double>(nclip) / dim;
    dg.step_post = vnorm(cl);
    dg.max_step_over_radius = mr;
    if (applied) std::copy(cl.begin(), cl.end(), applied);
    for (int64_t i = 0; i < dim; ++i) x[i] = x[i] + cl[i];
    clamp_scene(x, k, o);
}

// apply_unclipped, optimizer.cpp:145-151
void apply_unclipped(double* x, int64_t k, const orc_tr_opts& o, const std::vector<double>& dx,
                     orc_diag& dg, double* applied) {
    const int64_t dim = (14 + 3LL * g_sh_nb) * k;
    for (int64_t i = 0; i < dim; ++i)
        if (!std::isfinite(dx[i]))
            throw NumericErr(std::string("non-finite update in group ") + kGroup[group_of(k, i)]);
    dg.step_post = vnorm(dx);
    if (applied) std::copy(dx.begin(), dx.end(), applied);
    for (int64_t i = 0; i < dim; ++i) x[i] = x[i] + dx[i];
    clamp_scene(x, k, o);
}

// adam_direction, optimizer.cpp:153-185: bias-corrected moments, per-group
// rates, the position rate scaled by the scene extent and decayed
// geometrically over lr_position_decay_steps
std::vector<double> adam_direction(orc_state* st, int64_t k, const std::vector<double>& g,
                                   const orc_adam_opts& a) {
    const int64_t dim = (14 + 3LL * g_sh_nb) * k;
    for (int64_t i = 0; i < dim; ++i) {
        st->adam_m[i] = a.beta1 * st->adam_m[i] + (1.0 - a.beta1) * g[i];
        st->adam_v[i] = a.beta2 * st->adam_v[i] + (1.0 - a.beta2) * (g[i] * g[i]);
    }
    const double c1 = 1.0 - std::pow(a.beta1, static_cast<double>(st->t));
    const double c2 = 1.0 - std::pow(a.beta2, static_cast<double>(st->t));
    const double span = std::max(1, a.lr_position_decay_steps);
    const double frac = std::min(1.0, static_cast<double>(st->t) / span);
    const double lr_pos =
        a.scene_extent * a.lr_position * std::pow(a.lr_position_final / a.lr_position, frac);
    const double lrs[5] = {lr_pos, a.lr_scale, a.lr_rotation, a.lr_opacity, a.lr_color};
    std::vector<double> dx(dim);
    for (int64_t i = 0; i < dim; ++i) {
        // SH coefficients (extension) at the colour rate / 20 (3DGS's
        // feature_rest convention)
        const double lr = i >= 14 * k ? a.lr_color / 20.0 : lrs[group_of(k, i)];
        const double mhat = st->adam_m[i] / c1;
        const double vhat = st->adam_v[i] / c2;
        dx[i] = -lr * mhat / (std::sqrt(vhat) + a.eps);
    }
    return dx;
}

// step_adam / step_adam_tr, optimizer.cpp:222-253: one S1 draw, gradient,
// ADAM direction, then the plain or the trust-region-clipped update
void step_adam(orc_state* st, double* x, const Problem& pb, const orc_tr_opts& o,
               const orc_adam_opts& a, bool trust_region, const std::vector<int>* s1_in,
               orc_diag* diag, double* applied) {
    const int64_t k = pb.sc.k;
    orc_diag dg{0, 0, 0, 0, -1, -1, 0};
    st->t += 1;
    const int mv = static_cast<int>(pb.cams.size());
    const std::vector<int> s1 = s1_in ? *s1_in : st->rng.sample(mv, o.batch_size);
    const std::vector<double> g = stochastic_gradient(pb, s1, &dg.batch_loss);
    dg.gnorm = vnorm(g);
    const std::vector<double> dx = adam_direction(st, k, g, a);
    dg.step_pre = vnorm(dx);
    if (trust_region)
        apply_clipped(st, x, pb, o, dx, dg, applied);
    else
        apply_unclipped(x, k, o, dx, dg, applied);
    *diag = dg;
}

// ---------------------------------------------------------------- datasets
// scene.cpp:94-128 (Shepperd), returns unit (x, y, z, w)
void rotation_to_quat(const double r[9], double q[4]) {
    const double tr = tree3(r[0], r[4], r[8]);
    if (tr > 0.0) {
        const double s = std::sqrt(tr + 1.0) * 2.0;
        q[3] = 0.25 * s;
        q[0] = (r[7] - r[5]) / s;
        q[1] = (r[2] - r[6]) / s;
        q[2] = (r[3] - r[1]) / s;
    } else if (r[0] > r[4] && r[0] > r[8]) {
        const double s = std::sqrt(1.0 + r[0] - r[4] - r[8]) * 2.0;
        q[3] = (r[7] - r[5]) / s;
        q[0] = 0.25 * s;
        q[1] = (r[1] + r[3]) / s;
        q[2] = (r[2] + r[6]) / s;
    } else if (r[4] > r[8]) {
        const double s = std::sqrt(1.0 + r[4] - r[0] - r[8]) * 2.0;
        q[3] = (r[2] - r[6]) / s;
        q[0] = (r[1] + r[3]) / s;
        q[1] = 0.25 * s;
        q[2] = (r[5] + r[7]) / s;
    } else {
        const double s = std::sqrt(1.0 + r[8] - r[0] - r[4]) * 2.0;
        q[3] = (r[3] - r[1]) / s;
        q[0] = (r[2] + r[6]) / s;
        q[1] = (r[5] + r[7]) / s;
        q[2] = 0.25 * s;
    }
    const double n = std::sqrt(sqnorm4(q));
    for (int i = 0; i < 4; ++i) q[i] = q[i] / n;
}

void normalize3(double v[3]) {
    const double z = v[0] * v[0] + v[1] * v[1] + v[2] * v[2];
    if (z > 0.0) {
        const double s = std::sqrt(z);
        for (int i = 0; i < 3; ++i) v[i] = v[i] / s;
    }
}

void cross3(const double a[3], const double b[3], double o[3]) {
    o[0] = a[1] * b[2] - a[2] * b[1];
    o[1] = a[2] * b[0] - a[0] * b[2];
    o[2] = a[0] * b[1] - a[1] * b[0];
}

// scene.cpp:130-147
orc_camera look_at(const double eye[3], const double tgt[3], double fx, double fy,
                   int w, int h) {
    double z[3] = {tgt[0] - eye[0], tgt[1] - eye[1], tgt[2] - eye[2]};
    normalize3(z);
    double up[3] = {0, 0, 1};
    if (std::abs(z[0] * up[0] + z[1] * up[1] + z[2] * up[2]) > 0.999) {
        up[1] = 1;
        up[2] = 0;
    }
    double xa[3], ya[3];
    cross3(z, up, xa);
    normalize3(xa);
    cross3(z, xa, ya);
    const double r[9] = {xa[0], xa[1], xa[2], ya[0], ya[1], ya[2], z[0], z[1], z[2]};
    orc_camera c{};
    c.fx = fx;
    c.fy = fy;
    c.cx = w / 2.0;
    c.cy = h / 2.0;
    c.width = w;
    c.height = h;
    rotation_to_quat(r, c.q_wc);
    for (int i = 0; i < 3; ++i)
        c.t_wc[i] = tree3(-r[3 * i] * eye[0], -r[3 * i + 1] * eye[1], -r[3 * i + 2] * eye[2]);
    return c;
}

void quantize8(const double* in, int64_t n, double* out) {  // image.cpp:13-20
    for (int64_t i = 0; i < n; ++i) {
        const double c = in[i] < 0.0 ? 0.0 : (in[i] > 1.0 ? 1.0 : in[i]);
        out[i] = std::round(c * 255.0) / 255.0;
    }
}

void set_prim(double* x, int64_t k, int64_t i, const Prim& p) {
    for (int a = 0; a < 3; ++a) {
        x[3 * i + a] = p.mu[a];
        x[3 * k + 3 * i + a] = p.s[a];
        x[11 * k + 3 * i + a] = p.c[a];
    }
    for (int a = 0; a < 4; ++a) x[6 * k + 4 * i + a] = p.q[a];
    x[10 * k + i] = p.alpha;
}

const orc_render_opts kDefaultRender = {0.01, 0.3, 0.99, 1.0 / 255.0, 1e-4, 3.0, {0, 0, 0}};

}  // namespace

// ====================================================================== C-ABI
extern "C" {

const char* orc_last_error(void) { return g_err.c_str(); }

int orc_set_sh_degree(int32_t degree) {
    if (degree < 0 || degree > 3) return 1;
    g_sh_nb = (degree + 1) * (degree + 1) - 1;
    return 0;
}

int orc_rasterize(const double* x, int64_t k, const orc_camera* cam,
                  const orc_render_opts* ro, int workers, double* color,
                  double* t_final) {
    return guarded([&] { rasterize({x, k}, make_cam(*cam), *ro, workers, color, t_final); });
}

int orc_rasterize_jvp(const double* x, int64_t k, const orc_camera* cam,
                      const orc_render_opts* ro, int workers, const double* v,
                      int64_t v_len, double* tangent) {
    return guarded([&] {
        if (v_len != (14 + 3LL * g_sh_nb) * k)
            throw InvalidArg("rasterize_jvp: direction length mismatch");
        rasterize_jvp({x, k}, make_cam(*cam), *ro, workers, v, tangent);
    });
}

int orc_rasterize_vjp(const double* x, int64_t k, const orc_camera* cam,
                      const orc_render_opts* ro, int workers, const double* adjoint,
                      int32_t adj_w, int32_t adj_h, double* grad) {
    return guarded([&] {
        if (adj_w != cam->width || adj_h != cam->height)
            throw InvalidArg("rasterize_vjp: adjoint shape mismatch");
        rasterize_vjp({x, k}, make_cam(*cam), *ro, workers, adjoint, grad);
    });
}

int orc_blend_pairs(const double* x, int64_t k, const orc_camera* cam,
                    const orc_render_opts* ro, int workers, int32_t x0, int32_t y0,
                    int32_t w, int32_t h, int64_t* offsets, int32_t* ids, int64_t cap) {
    return guarded([&] {
        const SceneView sc{x, k};
        check_finite(sc);
        const Cam c = make_cam(*cam);
        const auto fr = build_frags(sc, c, *ro);
        if (x0 < 0 || y0 < 0 || x0 + w > c.c.width || y0 + h > c.c.height || w < 1 || h < 1)
            throw InvalidArg("blend_pairs: window outside the image");
        std::vector<std::vector<int32_t>> rows(h);
        std::vector<std::vector<int64_t>> cnts(h);
        parallel_rows(h, workers, [&](int r) {
            BlendCount bc;
            bc.contrib = &rows[r];
            cnts[r].resize(w);
            for (int xx = 0; xx < w; ++xx) {
                double col[3], t;
                const size_t before = rows[r].size();
                blend<double>(fr, x0 + xx + 0.5, y0 + r + 0.5, *ro, col, t, &bc);
                cnts[r][xx] = static_cast<int64_t>(rows[r].size() - before);
            }
        });
        int64_t n = 0;
        offsets[0] = 0;
        for (int r = 0; r < h; ++r)
            for (int xx = 0; xx < w; ++xx) {
                n += cnts[r][xx];
                offsets[static_cast<int64_t>(r) * w + xx + 1] = n;
            }
        if (ids && n <= cap) {
            int64_t o = 0;
            for (int r = 0; r < h; ++r)
                for (int32_t id : rows[r]) ids[o++] = id;
        }
    });
}

int orc_blend_stats(const double* x, int64_t k, const orc_camera* cam,
                    const orc_render_opts* ro, int workers, int64_t* evaluated,
                    int64_t* contributing) {
    return guarded([&] {
        const SceneView sc{x, k};
        check_finite(sc);
        const Cam c = make_cam(*cam);
        const auto fr = build_frags(sc, c, *ro);
        const int W = c.c.width, H = c.c.height;
        std::vector<BlendCount> rows(H);
        parallel_rows(H, workers, [&](int y) {
            for (int xx = 0; xx < W; ++xx) {
                double col[3], t;
                blend<double>(fr, xx + 0.5, y + 0.5, *ro, col, t, &rows[y]);
            }
        });
        int64_t e = 0, cc = 0;
        for (const auto& r : rows) {
            e += r.evaluated;
            cc += r.contributing;
        }
        *evaluated = e;
        *contributing = cc;
    });
}

int orc_project(const double* x, int64_t k, const orc_camera* cam,
                const orc_render_opts* ro, double* out) {
    return guarded([&] {
        const SceneView sc{x, k};
        const Cam c = make_cam(*cam);
        for (int64_t i = 0; i < k; ++i) {
            double* o = out + 12 * i;
            std::fill(o, o + 12, 0.0);
            Frag<double> f;
            if (!make_frag<double>(i, sc.mu(i), sc.s(i), sc.q(i), sc.alpha(i), sc.c(i), c,
                                   *ro, f)) {
                o[0] = 1.0;
                continue;
            }
            const double v[12] = {0.0,   f.depth, f.mx,  f.my,  f.bx0, f.bx1,
                                  f.by0, f.by1,   f.i00, f.i01, f.i11, 0.0};
            std::copy(v, v + 12, o);
        }
    });
}

// Conservative contribution test of the GPU binning (restated from
// geometry.cuh): can any pixel centre of [x0..x1] x [y0..y1] reach
// alpha_bar = alpha exp(-q/2) >= alpha_skip?  False only when the minimum of
// q = d^T Sigma^-1 d over the rectangle is certainly above
// rho2 = 2 ln(alpha/alpha_skip), i.e. when blend() skips every such pair
// (render.cpp:132-137).
static double contrib_rho2(double alpha, double alpha_skip) {
    if (!(alpha_skip > 0.0)) return INFINITY;
    if (alpha < alpha_skip) return -1.0;
    return 2.0 * std::log(alpha / alpha_skip);
}

static bool ellipse_may_hit(double mx, double my, double i00, double i01, double i11,
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
    qmin = std::fmin(qmin, q(bx, clampd(-(k11 * bx), ay, by)));
    qmin = std::fmin(qmin, q(clampd(-(k00 * ay), ax, bx), ay));
    qmin = std::fmin(qmin, q(clampd(-(k00 * by), ax, bx), by));
    const double mxd = std::fmax(std::fabs(ax), std::fabs(bx));
    const double myd = std::fmax(std::fabs(ay), std::fabs(by));
    const double bound = std::fabs(i00) * mxd * mxd + std::fabs(i11) * myd * myd +
                         2.0 * std::fabs(i01) * mxd * myd;
    // NaN (a degenerate conic) keeps the fragment: the reference evaluates every
    // pair whose bbox test passes, and a NaN alpha_bar is not skipped (render.cpp:136)
    return !(qmin > rho2 + 1e-9 * rho2 + 1e-12 * bound + 1e-12);
}

// Restated tile binning of the GPU build.  A visible fragment belongs to tile
// (tx, ty) iff its closed bbox contains at least one pixel centre
// (x+0.5, y+0.5) of that tile inside the image — exactly the pixels whose
// bbox test in blend() passes (render.cpp:129-131) — and ellipse_may_hit
// admits those centres.  Lists are in (depth, index) order.
int orc_binning(const double* x, int64_t k, const orc_camera* cam,
                const orc_render_opts* ro, int32_t tile, int32_t* n_visible,
                int32_t* order, int64_t* n_dup, int64_t* tile_start,
                int64_t* tile_end, int32_t* lists) {
    return guarded([&] {
        const SceneView sc{x, k};
        check_finite(sc);
        const Cam c = make_cam(*cam);
        const auto fr = build_frags(sc, c, *ro);
        const int W = c.c.width, H = c.c.height;
        const int tw = (W + tile - 1) / tile, th = (H + tile - 1) / tile;
        *n_visible = static_cast<int32_t>(fr.size());
        if (order)
            for (size_t i = 0; i < fr.size(); ++i) order[i] = (int32_t)fr[i].splat;
        // pixel range of centres inside [lo, hi]: smallest/largest integer p
        // with lo <= p + 0.5 <= hi, clipped to [0, n-1]
        auto prange = [](double lo, double hi, int n, int& p0, int& p1) {
            if (std::isnan(lo) || std::isnan(hi)) {
                p0 = 0;
                p1 = n - 1;
                return;
            }
            if (!(hi >= 0.5) || !(lo <= n - 0.5)) {
                p0 = 1;
                p1 = 0;
                return;
            }
            p0 = lo <= 0.5 ? 0 : (int)std::ceil(lo - 0.5);
            while (p0 > 0 && (p0 - 1) + 0.5 >= lo) --p0;
            while (p0 + 0.5 < lo) ++p0;
            p1 = hi >= n - 0.5 ? n - 1 : (int)std::floor(hi - 0.5);
            while (p1 < n - 1 && (p1 + 1) + 0.5 <= hi) ++p1;
            while (p1 + 0.5 > hi) --p1;
        };
        std::vector<std::vector<int32_t>> per(static_cast<size_t>(tw) * th);
        for (const auto& f : fr) {
            int x0, x1, y0, y1;
            prange(f.bx0, f.bx1, W, x0, x1);
            prange(f.by0, f.by1, H, y0, y1);
            if (x0 > x1 || y0 > y1) continue;
            const double rho2 = contrib_rho2(f.alpha, ro->alpha_skip);
            const double k11 = f.i01 / f.i11, k00 = f.i01 / f.i00;
            for (int ty = y0 / tile; ty <= y1 / tile; ++ty)
                for (int tx = x0 / tile; tx <= x1 / tile; ++tx)
                    if (ellipse_may_hit(f.mx, f.my, f.i00, f.i01, f.i11, k11, k00, rho2,
                                        std::max(x0, tx * tile), std::min(x1, tx * tile + tile - 1),
                                        std::max(y0, ty * tile), std::min(y1, ty * tile + tile - 1)))
                        per[(size_t)ty * tw + tx].push_back((int32_t)f.splat);
        }
        // empty tiles are reported as [0, 0) (the GPU leaves their range
        // unset); non-empty ones as their [start, end) in the tile-major list
        int64_t total = 0;
        for (size_t t = 0; t < per.size(); ++t) {
            const bool empty = per[t].empty();
            if (tile_start) tile_start[t] = empty ? 0 : total;
            if (lists)
                std::copy(per[t].begin(), per[t].end(), lists + total);
            total += (int64_t)per[t].size();
            if (tile_end) tile_end[t] = empty ? 0 : total;
        }
        *n_dup = total;
    });
}

int orc_ssim_map(const double* a, const double* b, int32_t w, int32_t h, double* out) {
    return guarded([&] { ssim_map(a, b, w, h, out); });
}

int orc_ssim_jvp(const double* a, const double* da, const double* b, int32_t w,
                 int32_t h, double* s, double* ds) {
    return guarded([&] { ssim_jvp(a, da, b, w, h, s, ds); });
}

int orc_ssim_vjp(const double* a, const double* b, const double* up, int32_t w,
                 int32_t h, double* grad) {
    return guarded([&] { ssim_vjp(a, b, up, w, h, grad); });
}

double orc_mean_ssim(const double* a, const double* b, int32_t w, int32_t h) {
    std::vector<double> s(3LL * w * h);
    if (guarded([&] { ssim_map(a, b, w, h, s.data()); }) != 0)
        return std::numeric_limits<double>::quiet_NaN();
    double sum = 0.0;
    for (double v : s) sum += v;
    return sum / static_cast<double>(s.size());
}

int orc_residual_vector(const double* rendered, const double* gt, int32_t w,
                        int32_t h, const orc_residual_opts* o, double* r) {
    return guarded([&] { residual_vector(rendered, gt, w, h, *o, r); });
}

int orc_residual_jvp(const double* rendered, const double* tangent, const double* gt,
                     int32_t w, int32_t h, const orc_residual_opts* o, double* dr) {
    return guarded([&] { residual_jvp(rendered, tangent, gt, w, h, *o, dr); });
}

int orc_residual_vjp(const double* rendered, const double* gt, int32_t w, int32_t h,
                     const double* u, int64_t u_len, const orc_residual_opts* o,
                     double* adj) {
    return guarded([&] {
        if (u_len != 6LL * w * h) throw InvalidArg("residual_vjp: adjoint length mismatch");
        residual_vjp(rendered, gt, w, h, u, *o, adj);
    });
}

double orc_psnr(const double* a, const double* b, int64_t n) {  // residuals.cpp:133-144
    double mse = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        const double d = a[i] - b[i];
        mse += d * d;
    }
    mse /= static_cast<double>(n);
    if (mse < 1e-10) return 100.0;
    return 10.0 * std::log10(1.0 / mse);
}

void orc_quantize8(const double* in, int64_t n, double* out) { quantize8(in, n, out); }

int orc_view_jacobian_apply(const double* x, int64_t k, const orc_camera* cam,
                            const double* gt, const double* v,
                            const orc_residual_opts* rs, const orc_render_opts* ro,
                            int workers, double* out) {
    return guarded([&] {
        const Problem pb = make_problem(x, k, cam, &gt, 1, rs, ro, workers);
        const auto r = jac_apply(pb, 0, v);
        std::copy(r.begin(), r.end(), out);
    });
}

int orc_view_jacobian_applyT(const double* x, int64_t k, const orc_camera* cam,
                             const double* gt, const double* u,
                             const orc_residual_opts* rs, const orc_render_opts* ro,
                             int workers, double* grad) {
    return guarded([&] {
        const Problem pb = make_problem(x, k, cam, &gt, 1, rs, ro, workers);
        const auto g = jac_applyT(pb, 0, u);
        std::copy(g.begin(), g.end(), grad);
    });
}

int orc_stochastic_gradient(const double* x, int64_t k, const orc_camera* cams,
                            const double* const* gts, int32_t n_views,
                            const int32_t* batch, int32_t n_batch,
                            const orc_residual_opts* rs, const orc_render_opts* ro,
                            int workers, double* g, double* batch_loss) {
    return guarded([&] {
        const Problem pb = make_problem(x, k, cams, gts, n_views, rs, ro, workers);
        const std::vector<int> b(batch, batch + n_batch);
        const auto r = stochastic_gradient(pb, b, batch_loss);
        std::copy(r.begin(), r.end(), g);
    });
}

int orc_hutchinson_diag(const double* x, int64_t k, const orc_camera* cams,
                        const double* const* gts, int32_t n_views, const int32_t* batch,
                        int32_t n_batch, int32_t nu, const double* probes,
                        const orc_residual_opts* rs, const orc_render_opts* ro,
                        int workers, double* d) {
    return guarded([&] {
        const Problem pb = make_problem(x, k, cams, gts, n_views, rs, ro, workers);
        const std::vector<int> b(batch, batch + n_batch);
        const int64_t dim = (14 + 3LL * g_sh_nb) * k;
        const auto r = hutchinson_diag(pb, b, nu, [&](int s) {
            return std::vector<double>(probes + s * dim, probes + (s + 1) * dim);
        });
        std::copy(r.begin(), r.end(), d);
    });
}

double orc_objective(const double* x, int64_t k, const orc_camera* cams,
                     const double* const* gts, int32_t n_views,
                     const orc_residual_opts* rs, const orc_render_opts* ro,
                     int workers) {
    double out = std::numeric_limits<double>::quiet_NaN();
    guarded([&] {  // residuals.cpp:119-131
        const Problem pb = make_problem(x, k, cams, gts, n_views, rs, ro, workers);
        double sum = 0.0;
        long m = 0;
        for (int v = 0; v < n_views; ++v) {
            const Cam& c = pb.cams[v];
            const int64_t n = 3LL * c.c.width * c.c.height;
            std::vector<double> img(n), f(2 * n);
            rasterize(pb.sc, c, *ro, workers, img.data(), nullptr);
            residual_vector(img.data(), gts[v], c.c.width, c.c.height, *rs, f.data());
            sum += sq_norm(f);
            m += (long)f.size();
        }
        out = sum / (2.0 * static_cast<double>(m));
    });
    return out;
}

int orc_exact_gn_diagonal(const double* x, int64_t k, const orc_camera* cams,
                          const double* const* gts, int32_t n_views,
                          const orc_residual_opts* rs, const orc_render_opts* ro,
                          int workers, double* d) {
    return guarded([&] {  // checks.cpp:127-141
        const Problem pb = make_problem(x, k, cams, gts, n_views, rs, ro, workers);
        const int64_t dim = (14 + 3LL * g_sh_nb) * k;
        const long m = 6L * pb.W() * pb.H() * n_views;
        std::vector<double> e(dim, 0.0);
        for (int64_t j = 0; j < dim; ++j) {
            e[j] = 1.0;
            double acc = 0.0;
            for (int v = 0; v < n_views; ++v) acc += sq_norm(jac_apply(pb, v, e.data()));
            d[j] = acc / static_cast<double>(m);
            e[j] = 0.0;
        }
    });
}

int orc_shd_radii(const double* x, int64_t k, double eps, const double caps[5],
                  double* eta) {
    return guarded([&] { shd_radii({x, k}, eps, caps, eta); });
}

double orc_beta_rotation(const double* prim14, int32_t axis) {
    double out = std::numeric_limits<double>::quiet_NaN();
    guarded([&] { out = beta_rotation(prim_at({prim14, 1}, 0), axis); });
    return out;
}

double orc_eps_at(double eps_start, double eps_end, int32_t total, int32_t t) {
    double out = std::numeric_limits<double>::quiet_NaN();
    guarded([&] { out = eps_at(eps_start, eps_end, total, t); });
    return out;
}

// trust_region.cpp:20-35 via Cholesky-free closed form (SPD checked by
// leading minors); used only by the KAT tests of the radii
double orc_hellinger_sq(double ma, const double* mua, const double* sa, double mb,
                        const double* mub, const double* sb) {
    double mid[9];
    for (int i = 0; i < 9; ++i) mid[i] = 0.5 * (sa[i] + sb[i]);
    auto spd = [](const double* m) {
        return m[0] > 0 && (m[0] * m[4] - m[1] * m[3]) > 0 && det3(m) > 0;
    };
    if (!spd(sa) || !spd(sb) || !spd(mid)) {
        g_err = "hellinger_sq: covariance is not SPD";
        return std::numeric_limits<double>::quiet_NaN();
    }
    const double da = det3(sa), db = det3(sb), dm = det3(mid);
    const double shape = std::pow(da, 0.25) * std::pow(db, 0.25) / std::sqrt(dm);
    const double dmu[3] = {mua[0] - mub[0], mua[1] - mub[1], mua[2] - mub[2]};
    // solve mid * y = dmu by cofactors
    double inv[9];
    const double id = 1.0 / dm;
    inv[0] = (mid[4] * mid[8] - mid[5] * mid[7]) * id;
    inv[1] = (mid[2] * mid[7] - mid[1] * mid[8]) * id;
    inv[2] = (mid[1] * mid[5] - mid[2] * mid[4]) * id;
    inv[3] = (mid[5] * mid[6] - mid[3] * mid[8]) * id;
    inv[4] = (mid[0] * mid[8] - mid[2] * mid[6]) * id;
    inv[5] = (mid[2] * mid[3] - mid[0] * mid[5]) * id;
    inv[6] = (mid[3] * mid[7] - mid[4] * mid[6]) * id;
    inv[7] = (mid[1] * mid[6] - mid[0] * mid[7]) * id;
    inv[8] = (mid[0] * mid[4] - mid[1] * mid[3]) * id;
    double md = 0.0;
    for (int i = 0; i < 3; ++i)
        md += dmu[i] * (inv[3 * i] * dmu[0] + inv[3 * i + 1] * dmu[1] + inv[3 * i + 2] * dmu[2]);
    return 0.5 * (ma + mb) - std::sqrt(ma * mb) * shape * std::exp(-md / 8.0);
}

orc_state* orc_state_create(int64_t dim, uint64_t seed) { return new orc_state(dim, seed); }
void orc_state_rng_raw(orc_state* s, int64_t n, uint64_t* out) {
    for (int64_t i = 0; i < n; ++i) out[i] = s->rng.raw();
}
void orc_state_destroy(orc_state* s) { delete s; }

int orc_state_get(const orc_state* s, double* g_hat, double* d_hat, int64_t* t) {
    if (g_hat) std::copy(s->g_hat.begin(), s->g_hat.end(), g_hat);
    if (d_hat) std::copy(s->d_hat.begin(), s->d_hat.end(), d_hat);
    if (t) *t = s->t;
    return 0;
}

int orc_state_set(orc_state* s, const double* g_hat, const double* d_hat, int64_t t) {
    if (g_hat) std::copy(g_hat, g_hat + s->g_hat.size(), s->g_hat.begin());
    if (d_hat) std::copy(d_hat, d_hat + s->d_hat.size(), s->d_hat.begin());
    s->t = t;
    return 0;
}

int orc_step_3dgs2tr(orc_state* s, double* x, int64_t k, const orc_camera* cams,
                     const double* const* gts, int32_t n_views, const orc_tr_opts* o,
                     const orc_residual_opts* rs, const orc_render_opts* ro,
                     int workers, orc_diag* diag, double* applied_step) {
    return guarded([&] {
        const Problem pb = make_problem(x, k, cams, gts, n_views, rs, ro, workers);
        step_tr(s, x, pb, *o, nullptr, nullptr, nullptr, diag, applied_step);
    });
}

int orc_step_3dgs2tr_explicit(orc_state* s, double* x, int64_t k, const orc_camera* cams,
                              const double* const* gts, int32_t n_views,
                              const orc_tr_opts* o, const orc_residual_opts* rs,
                              const orc_render_opts* ro, int workers, const int32_t* s1,
                              int32_t n1, const int32_t* s2, int32_t n2,
                              const double* probes, orc_diag* diag,
                              double* applied_step) {
    return guarded([&] {
        const Problem pb = make_problem(x, k, cams, gts, n_views, rs, ro, workers);
        const std::vector<int> v1(s1, s1 + n1), v2(s2, s2 + n2);
        step_tr(s, x, pb, *o, &v1, &v2, probes, diag, applied_step);
    });
}

int orc_state_get_adam(const orc_state* s, double* m, double* v) {
    if (m) std::copy(s->adam_m.begin(), s->adam_m.end(), m);
    if (v) std::copy(s->adam_v.begin(), s->adam_v.end(), v);
    return 0;
}

int orc_state_set_adam(orc_state* s, const double* m, const double* v) {
    if (m) std::copy(m, m + s->adam_m.size(), s->adam_m.begin());
    if (v) std::copy(v, v + s->adam_v.size(), s->adam_v.begin());
    return 0;
}

int orc_step_adam(orc_state* s, double* x, int64_t k, const orc_camera* cams,
                  const double* const* gts, int32_t n_views, const orc_tr_opts* o,
                  const orc_adam_opts* a, int32_t trust_region, const orc_residual_opts* rs,
                  const orc_render_opts* ro, int workers, const int32_t* s1, int32_t n1,
                  orc_diag* diag, double* applied_step) {
    return guarded([&] {
        const Problem pb = make_problem(x, k, cams, gts, n_views, rs, ro, workers);
        if (s1) {
            const std::vector<int> v1(s1, s1 + n1);
            step_adam(s, x, pb, *o, *a, trust_region != 0, &v1, diag, applied_step);
        } else {
            step_adam(s, x, pb, *o, *a, trust_region != 0, nullptr, diag, applied_step);
        }
    });
}

orc_rng* orc_rng_create(uint64_t seed) { return new orc_rng(seed); }
void orc_rng_destroy(orc_rng* r) { delete r; }
void orc_rng_raw(orc_rng* r, int64_t n, uint64_t* out) {
    for (int64_t i = 0; i < n; ++i) out[i] = r->r.raw();
}
void orc_rng_normal(orc_rng* r, int64_t n, double* out) {
    for (int64_t i = 0; i < n; ++i) out[i] = r->r.normal();
}
void orc_rng_uniform(orc_rng* r, int64_t n, double lo, double hi, double* out) {
    for (int64_t i = 0; i < n; ++i) out[i] = r->r.uniform(lo, hi);
}
void orc_rng_sample(orc_rng* r, int32_t n, int32_t k, int32_t* out) {
    const auto v = r->r.sample(n, k);
    std::copy(v.begin(), v.end(), out);
}
void orc_rng_rademacher(orc_rng* r, int64_t n, double* out) {
    for (int64_t i = 0; i < n; ++i) out[i] = r->r.rademacher();
}

// dataset.cpp:25-67
int orc_make_synthetic(const orc_synth_cfg* cfg, const orc_render_opts* ro, int workers,
                       double* gt_x, double* init_x, orc_camera* cams,
                       double* const* gts) {
    return guarded([&] {
        Rng rng(cfg->seed);
        const int64_t kg = cfg->gt_splats, ki = cfg->init_splats;
        const double ss = cfg->size_scale > 0.0 ? cfg->size_scale : 1.0;
        const int W = cfg->width > 0 ? cfg->width : cfg->image_size;
        const int H = cfg->height > 0 ? cfg->height : cfg->image_size;
        std::vector<Prim> gt(kg);
        for (Prim& p : gt) {
            for (int a = 0; a < 3; ++a) p.mu[a] = rng.uniform(-0.5, 0.5);
            for (int a = 0; a < 3; ++a) p.s[a] = rng.log_uniform(0.02 * ss, 0.2 * ss);
            double q[4];
            for (int a = 0; a < 4; ++a) q[a] = rng.normal();
            const double n = std::sqrt(sqnorm4(q));  // random_unit_quat: q.norm()
            if (n > 1e-9)
                for (int a = 0; a < 4; ++a) p.q[a] = q[a] / n;
            else
                p.q[0] = p.q[1] = p.q[2] = 0.0, p.q[3] = 1.0;
            p.alpha = rng.uniform(0.3, 0.9);
            for (int a = 0; a < 3; ++a) p.c[a] = rng.uniform(0.1, 1.0);
        }
        for (int64_t i = 0; i < kg; ++i) set_prim(gt_x, kg, i, gt[i]);
        for (int64_t i = 0; i < ki; ++i) {
            const Prim& src = gt[i % kg];
            Prim p{};
            for (int a = 0; a < 3; ++a) p.mu[a] = src.mu[a] + cfg->sigma_init * ss * rng.normal();
            for (int a = 0; a < 3; ++a) p.s[a] = cfg->init_scale * ss;
            p.q[0] = p.q[1] = p.q[2] = 0.0;
            p.q[3] = 1.0;
            p.alpha = cfg->init_opacity;
            for (int a = 0; a < 3; ++a) p.c[a] = 0.5;
            set_prim(init_x, ki, i, p);
        }
        if ((cfg->sh_degree + 1) * (cfg->sh_degree + 1) - 1 != g_sh_nb)
            throw InvalidArg("make_synthetic: sh_degree differs from orc_set_sh_degree");
        if (g_sh_nb > 0) {
            Rng rs(cfg->seed + 0x5348ULL);
            const int64_t nsh = 3LL * g_sh_nb;
            for (int64_t t = 0; t < nsh * kg; ++t) gt_x[14 * kg + t] = 0.1 * rs.normal();
            for (int64_t t = 0; t < nsh * ki; ++t) init_x[14 * ki + t] = 0.0;
        }
        const double focal = cfg->focal_factor * H;
        const int64_t n = 3LL * W * H;
        std::vector<double> img(n);
        for (int v = 0; v < cfg->views; ++v) {
            const double ang = 2.0 * M_PI * v / cfg->views;
            const double eye[3] = {cfg->camera_radius * std::cos(ang),
                                   cfg->camera_radius * std::sin(ang), cfg->camera_height};
            const double tgt[3] = {0, 0, 0};
            orc_camera c = look_at(eye, tgt, focal, focal, W, H);
            c.id = v;
            cams[v] = c;
            if (gts) {
                rasterize({gt_x, kg}, make_cam(c), *ro, workers, img.data(), nullptr);
                quantize8(img.data(), n, gts[v]);
            }
        }
    });
}

// checks.cpp:52-102
int orc_make_check_scene(int32_t splats, int32_t image_size, int32_t n_views,
                         uint64_t seed, double* x, orc_camera* cams,
                         double* const* gts) {
    return guarded([&] {
        for (int attempt = 0; attempt < 100; ++attempt) {
            Rng rng(seed + attempt);
            std::vector<Prim> target(splats);
            for (Prim& p : target) {
                for (int a = 0; a < 3; ++a) p.mu[a] = rng.uniform(-0.4, 0.4);
                for (int a = 0; a < 3; ++a) p.s[a] = rng.log_uniform(0.06, 0.22);
                double q[4];
                for (int a = 0; a < 4; ++a) q[a] = rng.normal();
                double n = std::sqrt(sqnorm4(q));  // q.normalized()
                for (int a = 0; a < 4; ++a) p.q[a] = q[a] / n;
                p.alpha = rng.uniform(0.3, 0.8);
                for (int a = 0; a < 3; ++a) p.c[a] = rng.uniform(0.15, 1.0);
            }
            std::vector<Prim> sc = target;
            for (Prim& p : sc) {
                for (int a = 0; a < 3; ++a) {
                    p.mu[a] += 0.03 * rng.normal();
                    p.s[a] *= std::exp(0.1 * rng.normal());
                    p.c[a] = std::min(1.2, std::max(0.1, p.c[a] + 0.1 * rng.normal()));
                }
                p.alpha = std::min(0.9, std::max(0.2, p.alpha + 0.05 * rng.normal()));
            }
            std::vector<double> tx(14 * (int64_t)splats);
            for (int i = 0; i < splats; ++i) {
                set_prim(tx.data(), splats, i, target[i]);
                set_prim(x, splats, i, sc[i]);
            }
            const double focal = 2.0 * image_size;
            bool ok = true;
            for (int v = 0; v < n_views; ++v) {
                const double ang = 2.0 * M_PI * v / n_views + 0.4;
                const double eye[3] = {1.9 * std::cos(ang), 1.9 * std::sin(ang), 0.7};
                const double tgt[3] = {0, 0, 0};
                orc_camera c = look_at(eye, tgt, focal, focal, image_size, image_size);
                c.id = v;
                cams[v] = c;
                const Cam cc = make_cam(c);
                // the check scenes are degree-0 scenes whatever orc_set_sh_degree says
                if (gts)
                    rasterize({tx.data(), splats, 0}, cc, kDefaultRender, 0, gts[v], nullptr);
                std::vector<double> depths;
                for (const Prim& p : sc)
                    depths.push_back(cc.w[6] * p.mu[0] + cc.w[7] * p.mu[1] +
                                     cc.w[8] * p.mu[2] + c.t_wc[2]);
                std::sort(depths.begin(), depths.end());
                for (size_t i = 1; i < depths.size(); ++i)
                    if (depths[i] - depths[i - 1] < 1e-3) ok = false;
            }
            if (ok) return;
        }
        throw std::runtime_error("make_check_scene: no tie-free seed found");
    });
}

int orc_look_at_camera(const double eye[3], const double target[3], double fx, double fy,
                       int32_t width, int32_t height, orc_camera* out) {
    return guarded([&] { *out = look_at(eye, target, fx, fy, width, height); });
}

}  // extern "C"
