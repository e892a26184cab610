// ssim.cu — K8 SSIM + residual + residual-VJP fields, K13 (its JVP form),
// K9 reflection-aware transposed-window gather.
//
// The reference evaluates SSIM with a direct 121-tap gather per pixel and
// its adjoint as a 121-tap scatter (ssim.cpp:60-168), single-threaded.  The
// window weight is k[dy]*k[dx] and the reflection is per axis, so both are
// separable: K8 runs a horizontal then a vertical 11-tap pass over a tile
// staged in shared memory with a 5-pixel reflected halo, and K9 turns the
// scatter into a gather: with P = u*dS/dmu_a, Q = 2u*dS/dmaa, R = u*dS/dmab
// at each window centre,
//     grad[p] = (W^T P)[p] + a[p] (W^T Q)[p] + b[p] (W^T R)[p]
// where per axis (W^T X)(p) = B0(p) + [1<=p<=5] B0(-p)
//                              + [n-6<=p<=n-2] B0(2n-2-p)
// and B0(i) = sum_d k[d] X[i+d] with zero padding (k is symmetric), i.e. the
// preimages of p under reflect() over [-5, n+4].
//
// Images are planar (3, H, W); for a planar image the residual block index
// c*H*W + y*W + x (residuals.cpp:19-22) is the plane index itself.
#include <cmath>
#include <type_traits>

#include "common.cuh"
#include "geometry.cuh"
#include "launch.h"

namespace sgtr {
namespace {

constexpr int TX = 32, TY = 16, HALO = 5;
constexpr int kThreads = 256;  // TX * TY / 2: two output rows per thread
constexpr int kHC = 4;         // horizontal pass: output columns per thread
constexpr int SX = TX + 2 * HALO, SY = TY + 2 * HALO;  // 42 x 26
// Shared-memory layout, bank-conflict free for FP64 (a half-warp's 16
// doubles fill the 32 banks once when their indices are distinct mod 16):
// * staging walks each staged row in 16-column segments, one half-warp per
//   segment, so a half-warp never straddles two rows (kSegs segments per row);
// * the horizontal passes give lane l of warp w staged row l and column group
//   w: row stride 43 doubles (11 mod 16) makes 16 consecutive rows distinct;
// * the filtered rows are written and read at stride 33 doubles (1 mod 16).
constexpr int SXP = SX + 1, TXP = TX + 1;
constexpr int kSegs = (SX + 15) / 16;
constexpr int kStage = (SY * kSegs * 16 + kThreads - 1) / kThreads;  // staging rounds
static_assert(SY <= 32 && TX / 4 == kThreads / 32, "horizontal pass: one row per lane, one "
              "4-column group per warp");
constexpr double kC1 = 0.01 * 0.01, kC2 = 0.03 * 0.03;

__constant__ double c_k[11];

__device__ __forceinline__ int reflect(int i, int n) {
    if (i < 0) return -i;
    if (i >= n) return 2 * n - 2 - i;
    return i;
}

__device__ __forceinline__ double sgn(double v) { return v > 0.0 ? 1.0 : (v < 0.0 ? -1.0 : 0.0); }

template <typename S>
__device__ __forceinline__ S mk(double v, double d);
template <>
__device__ __forceinline__ double mk<double>(double v, double) { return v; }
template <>
__device__ __forceinline__ Dual mk<Dual>(double v, double d) { return Dual(v, d); }

template <int MODE, bool kPre = false>
struct ModeTraits {
    static constexpr bool kTangent = MODE == SSIM_JVP || MODE == RES_JVP || MODE == HUTCH;
    // kPre: the target's windowed mean and second moment (mu_b, mbb) come
    // precomputed (they are fixed per training view), so only mu_a, maa, mab
    // (and their tangents) are filtered here
    static constexpr int kMoments = kPre ? (kTangent ? 6 : 3) : (kTangent ? 8 : 5);
    static constexpr int MUA = 0, MUB = kPre ? -1 : 1, MAA = kPre ? 1 : 2, MBB = kPre ? -1 : 3,
                         MAB = kPre ? 2 : 4, DMUA = kPre ? 3 : 5, DMAA = kPre ? 4 : 6,
                         DMAB = kPre ? 5 : 7;
};

// moments (kPre = false): 0 mu_a, 1 mu_b, 2 maa, 3 mbb, 4 mab, (5 dmu_a, 6 dmaa,
// 7 dmab); with kPre the b moments are read from args.bmom instead
template <int MODE, bool kPre = false>
__global__ void __launch_bounds__(kThreads, (MODE == GRAD && kPre) ? 4 : 1) k_ssim(SsimArgs args) {
    using Tr = ModeTraits<MODE, kPre>;
    constexpr int NM = Tr::kMoments;
    extern __shared__ __align__(16) double smem[];
    double* s_a = smem;                      // SY x SX
    double* s_b = s_a + SY * SXP;
    double* s_da = s_b + SY * SXP;            // (tangent modes)
    double* s_h = s_da + (Tr::kTangent ? SY * SXP : 0);  // NM x SY x TXP
    const int W = args.W, H = args.H;
    const long long P = (long long)W * H;
    const int c = blockIdx.z;
    const int x0 = blockIdx.x * TX, y0 = (blockIdx.y + args.by0) * TY;
    const double* A = args.a + c * P;
    const double* B = args.b + c * P;
    const double* DA = Tr::kTangent ? args.da + c * P : nullptr;
    // the target moments of this thread's two output pixels, fetched now so
    // their latency overlaps the staging (kPre)
    double pre_mu_b[2] = {0.0, 0.0}, pre_mbb[2] = {0.0, 0.0};
    if (kPre) {
#pragma unroll
        for (int rr = 0; rr < 2; ++rr) {
            const int gx = x0 + threadIdx.x % TX, gy = y0 + 2 * (threadIdx.x / TX) + rr;
            if (gx < W && gy < H) {
                const long long pi = c * P + (long long)gy * W + gx;
                pre_mu_b[rr] = args.bmom[pi];
                pre_mbb[rr] = args.bmom[3 * P + pi];
            }
        }
    }
    // all of this thread's staged loads are issued before the first store
    // (kStage rounds), so they are in flight together
    {
        constexpr int NP = Tr::kTangent ? 3 : 2;
        const double* planes[3] = {A, B, DA};
        double* dst[3] = {s_a, s_b, s_da};
        double v[kStage][NP];
#pragma unroll
        for (int it = 0; it < kStage; ++it) {
            const int i = threadIdx.x + it * kThreads;
            const int sy = i / (kSegs * 16), sx = i % (kSegs * 16);
            const int gy = y0 - HALO + sy, gx = x0 - HALO + sx;
            const bool in = i < SY * kSegs * 16 && sx < SX && gy <= H - 1 + HALO &&
                            gx <= W - 1 + HALO;
            const long long q = in ? (long long)reflect(gy, H) * W + reflect(gx, W) : 0;
#pragma unroll
            for (int f = 0; f < NP; ++f) v[it][f] = in ? planes[f][q] : 0.0;
        }
#pragma unroll
        for (int it = 0; it < kStage; ++it) {
            const int i = threadIdx.x + it * kThreads;
            const int sy = i / (kSegs * 16), sx = i % (kSegs * 16);
            if (i < SY * kSegs * 16 && sx < SX)
#pragma unroll
                for (int f = 0; f < NP; ++f) dst[f][sy * SXP + sx] = v[it][f];
        }
    }
    __syncthreads();
    // horizontal pass over all SY rows: lane = staged row, warp = group of kHC
    // adjacent output columns, which share the staged taps between them; the
    // products of a staged pixel are formed once for the kHC windows
    {
        const int sy = threadIdx.x & 31, tx = kHC * (threadIdx.x >> 5);
        if (sy < SY) {
            double mo[kHC][NM];
#pragma unroll
            for (int o = 0; o < kHC; ++o)
#pragma unroll
                for (int j = 0; j < NM; ++j) mo[o][j] = 0.0;
#pragma unroll
            for (int d = 0; d < 10 + kHC; ++d) {
                const int si = sy * SXP + tx + d;
                const double av = s_a[si], bv = s_b[si];
                const double dv = Tr::kTangent ? s_da[si] : 0.0;
                double q[NM];
                q[Tr::MUA] = av;
                if (!kPre) q[Tr::MUB < 0 ? 0 : Tr::MUB] = bv;
                q[Tr::MAA] = av * av;
                if (!kPre) q[Tr::MBB < 0 ? 0 : Tr::MBB] = bv * bv;
                q[Tr::MAB] = av * bv;
                if (Tr::kTangent) {
                    q[Tr::DMUA] = dv;
                    q[Tr::DMAA] = 2.0 * av * dv;
                    q[Tr::DMAB] = bv * dv;
                }
#pragma unroll
                for (int o = 0; o < kHC; ++o)
                    if (d >= o && d - o < 11)
#pragma unroll
                        for (int j = 0; j < NM; ++j) mo[o][j] += c_k[d - o] * q[j];
            }
#pragma unroll
            for (int o = 0; o < kHC; ++o)
#pragma unroll
                for (int j = 0; j < NM; ++j) s_h[(j * SY + sy) * TXP + tx + o] = mo[o][j];
        }
    }
    __syncthreads();
    using S = typename std::conditional<Tr::kTangent, Dual, double>::type;
    const int tx = threadIdx.x % TX;
    // vertical pass: two adjacent output rows per thread share 10 of their
    // 11 taps
    const int ty0 = 2 * (threadIdx.x / TX);
    double mv[2][NM];
#pragma unroll
    for (int j = 0; j < NM; ++j) mv[0][j] = mv[1][j] = 0.0;
#pragma unroll
    for (int d = 0; d < 12; ++d) {
#pragma unroll
        for (int j = 0; j < NM; ++j) {
            const double v = s_h[(j * SY + ty0 + d) * TXP + tx];
            if (d < 11) mv[0][j] += c_k[d] * v;
            if (d > 0) mv[1][j] += c_k[d - 1] * v;
        }
    }
    double partial = 0.0, partial2 = 0.0;
#pragma unroll
    for (int rr = 0; rr < 2; ++rr) {
    const int ty = ty0 + rr;
    const int gx = x0 + tx, gy = y0 + ty;
    const double* m = mv[rr];
    if (gx < W && gy < H) {
        const long long p = (long long)gy * W + gx;
        const long long pi = c * P + p;
        if (MODE == BMOM) {  // the target's moments for later kPre launches
            args.out0[pi] = m[1];
            args.out1[pi] = m[3];
            continue;
        }
        // SSIM (with its tangent in the JVP modes), ssim.cpp:50-58
        const S mu_a = mk<S>(m[Tr::MUA], Tr::kTangent ? m[Tr::DMUA] : 0.0);
        const S maa = mk<S>(m[Tr::MAA], Tr::kTangent ? m[Tr::DMAA] : 0.0);
        const S mab = mk<S>(m[Tr::MAB], Tr::kTangent ? m[Tr::DMAB] : 0.0);
        const double mu_b = kPre ? pre_mu_b[rr] : m[Tr::MUB < 0 ? 0 : Tr::MUB];
        const double mbb = kPre ? pre_mbb[rr] : m[Tr::MBB < 0 ? 0 : Tr::MBB];
        const S n1 = 2.0 * mu_a * mu_b + kC1;
        const S d1 = mu_a * mu_a + mu_b * mu_b + kC1;
        const S n2 = 2.0 * (mab - mu_a * mu_b) + kC2;
        const S d2 = (maa - mu_a * mu_a) + (mbb - mu_b * mu_b) + kC2;
        const S sv = (n1 * n2) / (d1 * d2);
        const double s_v = primal(sv), s_d = tangent(sv);
        const double n1v = primal(n1), d1v = primal(d1), n2v = primal(n2), d2v = primal(d2);
        const double mu_av = primal(mu_a);
        const double av = s_a[(ty + HALO) * SXP + tx + HALO];
        const double bv = s_b[(ty + HALO) * SXP + tx + HALO];
        const double diff = av - bv;
        const double lam = args.lambda, fl = args.floor;
        const double u1 = (1.0 - lam) * fabs(diff);
        const double u2 = lam * (1.0 - s_v) / 2.0;
        if (MODE == EVAL) {
            partial += s_v;
            partial2 += diff * diff;
        } else if (MODE == SSIM_MAP) {
            args.out0[pi] = s_v;
        } else if (MODE == SSIM_JVP) {
            args.out0[pi] = s_v;
            args.out1[pi] = s_d;
        } else if (MODE == RES_VEC) {
            args.out0[pi] = sqrt(fmax(u1, fl));
            args.out0[3 * P + pi] = sqrt(fmax(u2, fl));
        } else if (MODE == RES_JVP) {
            const double t = s_da[(ty + HALO) * SXP + tx + HALO];
            args.out0[pi] = u1 > fl ? (1.0 - lam) * sgn(diff) * t / (2.0 * sqrt(u1)) : 0.0;
            args.out0[3 * P + pi] = u2 > fl ? -lam * s_d / (4.0 * sqrt(u2)) : 0.0;
        } else {
            // image-space adjoint of the residual chain (residuals.cpp:81-117)
            double ur1, ur2;  // residual-space upstream for this entry
            if (MODE == GRAD) {
                // f = sqrt(max(u, floor)): f^2 = max(u, floor), and the
                // Gauss-Newton adjoint f * d f / d u = 1/2 (below, masked)
                ur1 = 0.0;
                ur2 = 0.0;
                partial += fmax(u1, fl) + fmax(u2, fl);
            } else if (MODE == HUTCH) {
                const double t = s_da[(ty + HALO) * SXP + tx + HALO];
                ur1 = u1 > fl ? (1.0 - lam) * sgn(diff) * t / (2.0 * sqrt(u1)) : 0.0;
                ur2 = u2 > fl ? -lam * s_d / (4.0 * sqrt(u2)) : 0.0;
            } else if (MODE == RES_VJP) {
                ur1 = args.u[pi];
                ur2 = args.u[3 * P + pi];
            } else {  // SSIM_VJP
                ur1 = 0.0;
                ur2 = 0.0;
            }
            double up;
            if (MODE == SSIM_VJP) {
                up = args.u[pi];
            } else if (MODE == GRAD) {
                // u * (1-l) sgn / (2 sqrt(u1)) and u * (-l / (4 sqrt(u2))) with
                // u = sqrt(u1), sqrt(u2) (residuals.cpp:81-117): the square
                // roots cancel
                args.adjl1[pi] = u1 > fl ? 0.5 * (1.0 - lam) * sgn(diff) : 0.0;
                up = u2 > fl ? -0.25 * lam : 0.0;
            } else {
                args.adjl1[pi] = u1 > fl ? ur1 * (1.0 - lam) * sgn(diff) / (2.0 * sqrt(u1)) : 0.0;
                up = u2 > fl ? ur2 * (-lam / (4.0 * sqrt(u2))) : 0.0;
            }
            // sensitivities to (mu_a, maa, mab) (ssim.cpp:146-155) through the
            // two reciprocals 1/d1, 1/d2 (the reference's five divisions)
            const double r1 = 1.0 / d1v, r2 = 1.0 / d2v;
            const double pp = n1v * r1, qq = n2v * r2;
            const double ds_dmu = qq * (2.0 * mu_b * d1v - 2.0 * mu_av * n1v) * (r1 * r1) +
                                  pp * (2.0 * mu_av * n2v - 2.0 * mu_b * d2v) * (r2 * r2);
            const double ds_dmaa = -pp * n2v * (r2 * r2);
            const double ds_dmab = pp * 2.0 * r2;
            args.P[pi] = up * ds_dmu;
            args.Q[pi] = up * ds_dmaa * 2.0;
            args.R[pi] = up * ds_dmab;
        }
    }
    }
    if (MODE == GRAD || MODE == EVAL) {
        // deterministic block sum -> one partial per block
        __shared__ double s_red[2][kThreads / 32];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            partial += __shfl_xor_sync(0xffffffffu, partial, o);
            if (MODE == EVAL) partial2 += __shfl_xor_sync(0xffffffffu, partial2, o);
        }
        if ((threadIdx.x & 31) == 0) {
            s_red[0][threadIdx.x >> 5] = partial;
            s_red[1][threadIdx.x >> 5] = partial2;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            double t = 0.0, t2 = 0.0;
            for (int w = 0; w < kThreads / 32; ++w) {
                t += s_red[0][w];
                t2 += s_red[1][w];
            }
            const int nblk = gridDim.x * gridDim.y * gridDim.z;
            const int blk = (blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
            args.loss_partials[blk] = t;
            if (MODE == EVAL) args.loss_partials[nblk + blk] = t2;
        }
    }
}

// per-axis transposed window: sum over preimages i of p of B0(i)
template <typename Ld>
__device__ __forceinline__ double transposed_1d(int p, int n, Ld ld) {
    auto b0 = [&](int i) {
        double s = 0.0;
#pragma unroll
        for (int d = -HALO; d <= HALO; ++d) {
            const int q = i + d;
            if (q >= 0 && q < n) s += c_k[d + HALO] * ld(q);
        }
        return s;
    };
    double t = b0(p);
    if (p >= 1 && p <= HALO) t += b0(-p);
    if (p >= n - 6 && p <= n - 2) t += b0(2 * n - 2 - p);
    return t;
}

__global__ void __launch_bounds__(kThreads, 4) k_gather(int W, int H, const double* __restrict__ a,
                                                   const double* __restrict__ b,
                                                   const double* __restrict__ adjl1,
                                                   const double* __restrict__ Pf,
                                                   const double* __restrict__ Qf,
                                                   const double* __restrict__ Rf,
                                                   double* __restrict__ adj, int by0) {
    __shared__ double s_f[3][SY][SXP];
    __shared__ double s_h[3][SY][TXP];
    const long long P = (long long)W * H;
    const int c = blockIdx.z;
    const int x0 = blockIdx.x * TX, y0 = (blockIdx.y + by0) * TY;
    // this thread's two output pixels: their a, b, adjL1 fetched now so the
    // latency overlaps the staging
    double pa[2] = {0.0, 0.0}, pb[2] = {0.0, 0.0}, pl[2] = {0.0, 0.0};
#pragma unroll
    for (int rr = 0; rr < 2; ++rr) {
        const int gx = x0 + threadIdx.x % TX, gy = y0 + 2 * (threadIdx.x / TX) + rr;
        if (gx < W && gy < H) {
            const long long p = c * P + (long long)gy * W + gx;
            pa[rr] = a[p];
            pb[rr] = b[p];
            if (adjl1) pl[rr] = adjl1[p];
        }
    }
    {
        // all staged loads in flight together, then the stores
        double v[kStage][3];
#pragma unroll
        for (int it = 0; it < kStage; ++it) {
            const int i = threadIdx.x + it * kThreads;
            const int sy = i / (kSegs * 16), sx = i % (kSegs * 16);
            const int gy = y0 - HALO + sy, gx = x0 - HALO + sx;
            const bool in = i < SY * kSegs * 16 && sx < SX && gy >= 0 && gy < H && gx >= 0 &&
                            gx < W;
            const long long q = in ? c * P + (long long)gy * W + gx : 0;
            v[it][0] = in ? Pf[q] : 0.0;
            v[it][1] = in ? Qf[q] : 0.0;
            v[it][2] = in ? Rf[q] : 0.0;
        }
#pragma unroll
        for (int it = 0; it < kStage; ++it) {
            const int i = threadIdx.x + it * kThreads;
            const int sy = i / (kSegs * 16), sx = i % (kSegs * 16);
            if (i < SY * kSegs * 16 && sx < SX)
#pragma unroll
                for (int f = 0; f < 3; ++f) s_f[f][sy][sx] = v[it][f];
        }
    }
    __syncthreads();
    // blocks whose windows never meet the image border (most of a 1080p
    // view): the transposed filter is a plain 11-tap correlation there
    const bool in_x = x0 >= 2 * HALO && x0 + TX + 2 * HALO <= W;
    const bool in_y = y0 >= 2 * HALO && y0 + TY + 2 * HALO <= H;
    // horizontal transposed pass for every staged row
    if (in_x) {
        // lane = staged row, warp = group of kHC adjacent columns sharing the
        // staged taps (the layout note at the top)
        const int sy = threadIdx.x & 31, tx = kHC * (threadIdx.x >> 5);
        if (sy < SY) {
#pragma unroll
            for (int f = 0; f < 3; ++f) {
                const double* row = &s_f[f][sy][tx];
                double v[kHC];
#pragma unroll
                for (int o = 0; o < kHC; ++o) v[o] = 0.0;
#pragma unroll
                for (int d = 0; d < 10 + kHC; ++d) {
                    const double x = row[d];
#pragma unroll
                    for (int o = 0; o < kHC; ++o)
                        if (d >= o && d - o < 11) v[o] += c_k[d - o] * x;
                }
#pragma unroll
                for (int o = 0; o < kHC; ++o) s_h[f][sy][tx + o] = v[o];
            }
        }
    } else {
        for (int i = threadIdx.x; i < SY * TX; i += kThreads) {
            const int sy = i / TX, tx = i % TX;
            const int gx = x0 + tx;
#pragma unroll
            for (int f = 0; f < 3; ++f) {
                s_h[f][sy][tx] = gx < W ? transposed_1d(gx, W, [&](int q) {
                    return s_f[f][sy][q - x0 + HALO];
                })
                                        : 0.0;
            }
        }
    }
    __syncthreads();
    const int tx = threadIdx.x % TX;
    const int ty0 = 2 * (threadIdx.x / TX);  // two adjacent output rows per thread
    double t2[2][3];
    if (in_y) {
#pragma unroll
        for (int f = 0; f < 3; ++f) {
            double v0 = 0.0, v1 = 0.0;
#pragma unroll
            for (int d = 0; d < 12; ++d) {
                const double x = s_h[f][ty0 + d][tx];
                if (d < 11) v0 += c_k[d] * x;
                if (d > 0) v1 += c_k[d - 1] * x;
            }
            t2[0][f] = v0;
            t2[1][f] = v1;
        }
    } else {
#pragma unroll
        for (int rr = 0; rr < 2; ++rr) {
            const int gy = y0 + ty0 + rr;
#pragma unroll
            for (int f = 0; f < 3; ++f)
                t2[rr][f] = gy < H ? transposed_1d(gy, H, [&](int q) {
                    return s_h[f][q - y0 + HALO][tx];
                })
                                   : 0.0;
        }
    }
#pragma unroll
    for (int rr = 0; rr < 2; ++rr) {
        const int gx = x0 + tx, gy = y0 + ty0 + rr;
        if (gx >= W || gy >= H) continue;
        const double* t = t2[rr];
        const long long p = c * P + (long long)gy * W + gx;
        adj[p] = pl[rr] + t[0] + pa[rr] * t[1] + pb[rr] * t[2];
    }
}

__global__ void k_sum_partials(const double* __restrict__ partials, int n, double* out) {
    __shared__ double s[256];
    double t = 0.0;
    for (int i = threadIdx.x; i < n; i += 256) t += partials[i];
    s[threadIdx.x] = t;
    __syncthreads();
    if (threadIdx.x == 0) {
        double r = 0.0;
        for (int i = 0; i < 256; ++i) r += s[i];
        *out = r;
    }
}

__global__ void k_to_planar(const double* __restrict__ in, int P, double* __restrict__ out) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= P) return;
#pragma unroll
    for (int c = 0; c < 3; ++c) out[(long long)c * P + p] = in[3LL * p + c];
}

__global__ void k_to_interleaved(const double* __restrict__ in, int P, double* __restrict__ out) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= P) return;
#pragma unroll
    for (int c = 0; c < 3; ++c) out[3LL * p + c] = in[(long long)c * P + p];
}

// image.cpp:13-20
__global__ void k_quantize8(double* img, long long n) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double v = img[i];
    const double c = v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v);
    img[i] = round(c * 255.0) / 255.0;
}

// per-device state: __constant__ data and function attributes are set per
// device, and a process may hold contexts on several devices
int current_device() {
    int dev = 0;
    SGTR_CUDA(cudaGetDevice(&dev));
    return dev;
}
unsigned long long g_kernel_ready = 0;  // bit d: c_k uploaded on device d

void init_constants() {
    const unsigned long long bit = 1ull << (current_device() & 63);
    if (g_kernel_ready & bit) return;
    // kernel1d (ssim.cpp:21-34), computed on the host exactly as the oracle
    double k[11], sum = 0.0;
    for (int i = 0; i < 11; ++i) {
        const double d = i - 5;
        k[i] = std::exp(-d * d / (2.0 * 1.5 * 1.5));
        sum += k[i];
    }
    for (double& v : k) v /= sum;
    SGTR_CUDA(cudaMemcpyToSymbol(c_k, k, sizeof(k)));
    g_kernel_ready |= bit;
}

template <int MODE, bool kPre = false>
void run_ssim(cudaStream_t st, const SsimArgs& a) {
    using Tr = ModeTraits<MODE, kPre>;
    const size_t smem = sizeof(double) * (SY * SXP * (Tr::kTangent ? 3 : 2) +
                                          Tr::kMoments * SY * TXP);
    static unsigned long long attr = 0;  // bit d: attribute set on device d
    const unsigned long long bit = 1ull << (current_device() & 63);
    if (!(attr & bit)) {
        SGTR_CUDA(cudaFuncSetAttribute(k_ssim<MODE, kPre>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attr |= bit;
    }
    const int by1 = a.by1 > 0 ? a.by1 : ceil_div(a.H, TY);
    if (by1 <= a.by0) return;
    dim3 grid(ceil_div(a.W, TX), by1 - a.by0, 3);
    k_ssim<MODE, kPre><<<grid, kThreads, smem, st>>>(a);
    SGTR_CUDA(cudaGetLastError());
}

}  // namespace

int ssim_num_blocks(int W, int H) { return ceil_div(W, TX) * ceil_div(H, TY) * 3; }

void launch_ssim(cudaStream_t st, const SsimArgs& a) {
    init_constants();
    switch (a.mode) {
        case SSIM_MAP: run_ssim<SSIM_MAP>(st, a); break;
        case SSIM_JVP: run_ssim<SSIM_JVP>(st, a); break;
        case RES_VEC: run_ssim<RES_VEC>(st, a); break;
        case RES_JVP: run_ssim<RES_JVP>(st, a); break;
        case GRAD:
            if (a.bmom)
                run_ssim<GRAD, true>(st, a);
            else
                run_ssim<GRAD>(st, a);
            break;
        case HUTCH:
            if (a.bmom)
                run_ssim<HUTCH, true>(st, a);
            else
                run_ssim<HUTCH>(st, a);
            break;
        case BMOM: run_ssim<BMOM>(st, a); break;
        case RES_VJP: run_ssim<RES_VJP>(st, a); break;
        case SSIM_VJP: run_ssim<SSIM_VJP>(st, a); break;
        case EVAL: run_ssim<EVAL>(st, a); break;
        default: throw Error(SGTR_RUNTIME, "launch_ssim: bad mode");
    }
}

void launch_ssim_gather(cudaStream_t st, int W, int H, const double* a, const double* b,
                        const double* adjl1, const double* P, const double* Q, const double* R,
                        double* adj, int by0, int by1) {
    init_constants();
    if (by1 <= 0) by1 = ceil_div(H, TY);
    if (by1 <= by0) return;
    dim3 grid(ceil_div(W, TX), by1 - by0, 3);
    k_gather<<<grid, kThreads, 0, st>>>(W, H, a, b, adjl1, P, Q, R, adj, by0);
    SGTR_CUDA(cudaGetLastError());
}

void launch_sum_partials(cudaStream_t st, const double* partials, int n, double* out) {
    k_sum_partials<<<1, 256, 0, st>>>(partials, n, out);
    SGTR_CUDA(cudaGetLastError());
}

void launch_to_planar(cudaStream_t st, const double* in, int P, double* out) {
    if (P == 0) return;
    k_to_planar<<<ceil_div(P, 256), 256, 0, st>>>(in, P, out);
    SGTR_CUDA(cudaGetLastError());
}

void launch_to_interleaved(cudaStream_t st, const double* in, int P, double* out) {
    if (P == 0) return;
    k_to_interleaved<<<ceil_div(P, 256), 256, 0, st>>>(in, P, out);
    SGTR_CUDA(cudaGetLastError());
}

void launch_quantize8(cudaStream_t st, double* img, long long n) {
    if (n == 0) return;
    k_quantize8<<<ceil_div(n, 256), 256, 0, st>>>(img, n);
    SGTR_CUDA(cudaGetLastError());
}

}  // namespace sgtr
