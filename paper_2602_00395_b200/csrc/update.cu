// update.cu — K14: the fused squared-Hellinger trust-region step.
//
// One thread per splat reads its 14 coordinates of x, g, g-hat, D-hat (and
// z.w on refresh steps) once and writes g-hat, D-hat and the clamped x once:
//   g     = g_acc * M/(m|S1|)                     (optimizer.cpp:58-59)
//   g_hat = theta1 g_hat + (1-theta1) g           (optimizer.hpp:119-122)
//   D_hat = theta2 D_hat + (1-theta2) d  [refresh] (optimizer.cpp:212)
//   dx    = -g_hat / max(D_hat, gamma)            (optimizer.cpp:106-112)
//   eta   = shd_radii(x, eps)                     (trust_region.cpp:236-252)
//   x'    = clamp(x + clip(dx, eta))              (optimizer.cpp:124-142,
//                                                  scene.cpp:49-57)
// with the step diagnostics as deterministic block partials.  Compiled with
// --fmad=false so every expression rounds like the oracle.
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
    const double qc = p.q[axis];
    const double rt[9] = {r2 - 2.0 * (y * y + z * z), 2.0 * (x * y - w * z),
                          2.0 * (x * z + w * y),      2.0 * (x * y + w * z),
                          r2 - 2.0 * (z * z + x * x), 2.0 * (y * z - w * x),
                          2.0 * (x * z - w * y),      2.0 * (y * z + w * x),
                          r2 - 2.0 * (x * x + y * y)};
    double drt[9];
    switch (axis) {
        case 0: {
            const double t[9] = {2 * x, 2 * y, 2 * z, 2 * y, -2 * x, -2 * w, 2 * z, 2 * w, -2 * x};
            for (int i = 0; i < 9; ++i) drt[i] = t[i];
        } break;
        case 1: {
            const double t[9] = {-2 * y, 2 * x, 2 * w, 2 * x, 2 * y, 2 * z, -2 * w, 2 * z, -2 * y};
            for (int i = 0; i < 9; ++i) drt[i] = t[i];
        } break;
        case 2: {
            const double t[9] = {-2 * z, -2 * w, 2 * x, 2 * w, -2 * z, 2 * y, 2 * x, 2 * y, 2 * z};
            for (int i = 0; i < 9; ++i) drt[i] = t[i];
        } break;
        default: {
            const double t[9] = {2 * w, -2 * z, 2 * y, 2 * z, 2 * w, -2 * x, -2 * y, 2 * x, 2 * w};
            for (int i = 0; i < 9; ++i) drt[i] = t[i];
        } break;
    }
    const double dg[4][3] = {{2, -2, -2}, {-2, 2, -2}, {-2, -2, 2}, {2, 2, 2}};
    double d2rt[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    d2rt[0] = dg[axis][0];
    d2rt[4] = dg[axis][1];
    d2rt[8] = dg[axis][2];
    double r[9];
    for (int i = 0; i < 9; ++i) r[i] = rt[i] / r2;
    const double k1 = 2.0 * qc / (r2 * r2);
    const double k2 = 4.0 * qc / (r2 * r2);
    const double k3 = 8.0 * qc * qc / (r2 * r2 * r2) - 2.0 / (r2 * r2);
    double in1[9], in2[9];
    for (int i = 0; i < 9; ++i) {
        in1[i] = drt[i] / r2 - k1 * rt[i];
        in2[i] = d2rt[i] / r2 - k2 * drt[i] + k3 * rt[i];
    }
    double frob = 0.0, tr = 0.0;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            const double de = r[i] * in1[j] + r[3 + i] * in1[3 + j] + r[6 + i] * in1[6 + j];
            const double v = p.s[i] * de / p.s[j];
            frob += v * v;
        }
    // trace of r^T in2, summed over the diagonal in order
    for (int i = 0; i < 3; ++i)
        tr += r[i] * in2[i] + r[3 + i] * in2[3 + i] + r[6 + i] * in2[6 + i];
    return 2.0 * frob + 2.0 * tr;
}

// trust_region.cpp:183-194
__device__ double rotation_h2(const Prim& p, const double* sigma, double det_s, int axis,
                              double dq) {
    double q2[4] = {p.q[0], p.q[1], p.q[2], p.q[3]};
    q2[axis] += dq;
    if (q2[0] * q2[0] + q2[1] * q2[1] + q2[2] * q2[2] + q2[3] * q2[3] < 1e-24) return CUDART_INF;
    double c2[9], mid[9];
    covariance(p.s, q2, c2);
    for (int i = 0; i < 9; ++i) mid[i] = 0.5 * (sigma[i] + c2[i]);
    const double dm = det3(mid);
    if (!(dm > 0.0)) return CUDART_INF;
    return p.alpha * (1.0 - det_s / sqrt(dm));
}

// trust_region.cpp:198-234 (Taylor radius, certified, bisected if needed)
__device__ void radius_rotation(const Prim& p, double eps, double cap, double* out) {
    const double lf = log_factor(eps, p.alpha);
    if (lf <= 0.0) {
        out[0] = out[1] = out[2] = out[3] = cap;
        return;
    }
    double sigma[9];
    if (!covariance(p.s, p.q, sigma)) {
        out[0] = out[1] = out[2] = out[3] = cap;
        return;
    }
    const double det_s = p.s[0] * p.s[1] * p.s[2];
    const double tol = eps * (1.0 + 1e-9);
    for (int c = 0; c < 4; ++c) {
        const double beta = beta_rotation(p, c);
        double r = beta <= 1e-12 ? cap : cap_radius(sqrt(lf / beta), cap);
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

__device__ void radii(const Prim& p, double eps, const double* caps, double* eta) {
    radius_mean(p, eps, caps[0], eta);
    for (int c = 0; c < 3; ++c) {
        eta[3 + c] = cap_radius(sqrt(2.0 * p.s[c] * p.s[c] * eps / p.alpha), caps[1]);
        eta[11 + c] = cap_radius(sqrt(4.0 * p.c[c] * eps / p.alpha), caps[4]);
    }
    radius_rotation(p, eps, caps[2], eta + 6);
    eta[10] = cap_radius(sqrt(4.0 * p.alpha * eps), caps[3]);
}

// flat index of local coordinate j (0..13) of splat i in the group-major layout
__device__ __forceinline__ long long flat_index(long long K, int i, int j) {
    if (j < 3) return 3LL * i + j;
    if (j < 6) return 3 * K + 3LL * i + (j - 3);
    if (j < 10) return 6 * K + 4LL * i + (j - 6);
    if (j == 10) return 10 * K + i;
    return 11 * K + 3LL * i + (j - 11);
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

__global__ void __launch_bounds__(kThreads) k_tr_update(TrArgs a) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const long long K = a.K;
    double sg = 0.0, sdx = 0.0, scl = 0.0, nclip = 0.0, mr = 0.0;
    int bad = INT_MAX;
    if (i < a.K) {
        const Prim p = load_prim(a.x, K, i);
        if (!a.ghat_only && p.q[0] * p.q[0] + p.q[1] * p.q[1] + p.q[2] * p.q[2] +
                                    p.q[3] * p.q[3] < 1e-24)
            atomicOr(a.degenerate_flag, 1);  // quat_to_rotation throws in shd_radii
        double dx[14];
        for (int j = 0; j < 14; ++j) {
            const long long k = flat_index(K, i, j);
            const double g = a.g_acc[k] * a.gscale;
            sg += g * g;
            const double gh = a.theta1 * a.g_hat[k] + (1.0 - a.theta1) * g;
            a.g_hat[k] = gh;
            if (a.ghat_only) continue;
            double dh = a.d_hat[k];
            if (a.refresh) {
                const double d = a.w_acc[k] * a.dscale;
                dh = a.theta2 * dh + (1.0 - a.theta2) * d;
                a.d_hat[k] = dh;
            }
            // std::max(d, gamma) returns d unless d < gamma (NaN d -> d)
            dx[j] = -gh / ((dh < a.gamma_d) ? a.gamma_d : dh);
            sdx += dx[j] * dx[j];
        }
        if (!a.ghat_only) {
            double eta[14];
            radii(p, a.eps, a.caps, eta);
            double xo[14];
            for (int j = 0; j < 14; ++j) {
                const long long k = flat_index(K, i, j);
                // cwiseMax(-eta).cwiseMin(eta) with std::max/std::min semantics
                double c = dx[j] < -eta[j] ? -eta[j] : dx[j];
                c = eta[j] < c ? eta[j] : c;
                if (!isfinite(c)) bad = min(bad, (int)min(k, (long long)INT_MAX));
                if (fabs(dx[j]) > eta[j]) nclip += 1.0;
                const double ratio = fabs(c) / eta[j];
                mr = mr < ratio ? ratio : mr;
                scl += c * c;
                if (a.applied) a.applied[k] = c;
                xo[j] = a.x[k] + c;
            }
            // Scene::clamp (scene.cpp:49-57)
            for (int c = 0; c < 3; ++c) {
                double& s = xo[3 + c];
                s = s < a.bounds[0] ? a.bounds[0] : s;
                double& col = xo[11 + c];
                col = col < a.bounds[3] ? a.bounds[3] : col;
                col = a.bounds[4] < col ? a.bounds[4] : col;
            }
            double& al = xo[10];
            al = al < a.bounds[1] ? a.bounds[1] : al;
            al = a.bounds[2] < al ? a.bounds[2] : al;
            for (int j = 0; j < 14; ++j) a.x_out[flat_index(K, i, j)] = xo[j];
        }
    }
    // deterministic block reduction of the diagnostics
    __shared__ double s_red[5][kThreads / 32];
    __shared__ int s_bad[kThreads / 32];
    double v[5] = {sg, sdx, scl, nclip, mr};
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
        for (int q = 0; q < 5; ++q) a.partials[5LL * blockIdx.x + q] = r[q];
        if (b != INT_MAX) atomicMin(a.bad_index, b);
    }
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

__global__ void k_shd_radii(int K, const double* __restrict__ x, double eps, double c0,
                            double c1, double c2, double c3, double c4,
                            double* __restrict__ eta) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= K) return;
    const double caps[5] = {c0, c1, c2, c3, c4};
    const Prim p = load_prim(x, K, i);
    double e[14];
    radii(p, eps, caps, e);
    for (int j = 0; j < 14; ++j) eta[flat_index(K, i, j)] = e[j];
}

__global__ void k_scale(double* v, long long n, double s) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) v[i] = v[i] * s;
}

__global__ void k_fill_int(int* p, long long n, int v) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) p[i] = v;
}

}  // namespace

int tr_num_blocks(int K) { return ceil_div(K, kThreads); }

void launch_tr_update(cudaStream_t st, const TrArgs& a) {
    if (a.K == 0) return;
    k_tr_update<<<tr_num_blocks(a.K), kThreads, 0, st>>>(a);
    SGTR_CUDA(cudaGetLastError());
}

void launch_tr_finalize(cudaStream_t st, const double* partials, int nblocks, double* out5) {
    k_tr_finalize<<<1, 256, 0, st>>>(partials, nblocks, out5);
    SGTR_CUDA(cudaGetLastError());
}

void launch_shd_radii(cudaStream_t st, int K, const double* x, double eps, const double caps[5],
                      double* eta) {
    if (K == 0) return;
    k_shd_radii<<<ceil_div(K, 128), 128, 0, st>>>(K, x, eps, caps[0], caps[1], caps[2], caps[3],
                                                  caps[4], eta);
    SGTR_CUDA(cudaGetLastError());
}

void launch_scale(cudaStream_t st, double* v, long long n, double s) {
    if (n == 0) return;
    k_scale<<<ceil_div(n, 256), 256, 0, st>>>(v, n, s);
    SGTR_CUDA(cudaGetLastError());
}

void launch_fill_int(cudaStream_t st, int* p, long long n, int v) {
    if (n == 0) return;
    k_fill_int<<<ceil_div(n, 256), 256, 0, st>>>(p, n, v);
    SGTR_CUDA(cudaGetLastError());
}

}  // namespace sgtr
