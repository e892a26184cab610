// project.cu — K1 projection, K12 tangent projection, K11 adjoint chain.
// Compiled with --fmad=false: every FP64 expression rounds like the oracle,
// so depth keys, mu2d and the bounding boxes are bit-identical to it.
#include "common.cuh"
#include "geometry.cuh"
#include "launch.h"

namespace sgtr {
namespace {

constexpr unsigned long long kCulledKey = ~0ull;

// order-preserving map of an IEEE double onto uint64
__device__ __forceinline__ unsigned long long depth_key(double d) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(d);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

struct Splat {
    double mu[3], s[3], q[4], c[3], alpha;
};

__device__ __forceinline__ Splat load_splat(const double* __restrict__ x, int K, int i) {
    Splat p;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        p.mu[a] = x[3LL * i + a];
        p.s[a] = x[3LL * K + 3LL * i + a];
        p.c[a] = x[11LL * K + 3LL * i + a];
    }
#pragma unroll
    for (int a = 0; a < 4; ++a) p.q[a] = x[6LL * K + 4LL * i + a];
    p.alpha = x[10LL * K + i];
    return p;
}

__device__ __forceinline__ bool splat_finite(const Splat& p) {
    bool ok = isfinite(p.alpha);
#pragma unroll
    for (int a = 0; a < 3; ++a) ok = ok && isfinite(p.mu[a]) && isfinite(p.s[a]) && isfinite(p.c[a]);
#pragma unroll
    for (int a = 0; a < 4; ++a) ok = ok && isfinite(p.q[a]);
    return ok;
}

__device__ __forceinline__ Proj<double> project_primal(const Splat& p, const DevCam& cam,
                                                       const RenderP& ro) {
    return project<double>(p.mu, p.s, p.q, cam.w, cam.t, cam.fx, cam.fy, cam.cx, cam.cy,
                           ro.z_near, ro.lowpass);
}

__device__ __forceinline__ const double* sh_ptr(const double* x, int K, int nb, int i) {
    return x + 14LL * K + 3LL * nb * i;
}

template <bool kSH>
__global__ void __launch_bounds__(256) k_project(const double* __restrict__ x, int K, int nb,
                                                 DevCam cam, RenderP ro, double* __restrict__ rec,
                                                 unsigned long long* __restrict__ keys,
                                                 unsigned int* __restrict__ keys32,
                                                 int* __restrict__ ids, int4* __restrict__ rect,
                                                 int* __restrict__ tcount,
                                                 int4* __restrict__ tinfo,
                                                 ViewStatus* status) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    bool visible = false;
    if (i < K) {
        const Splat p = load_splat(x, K, i);
        ids[i] = i;
        bool finite = splat_finite(p);
        const double* shk = sh_ptr(x, K, nb, i);
        if (kSH)
            for (int t = 0; t < 3 * nb; ++t) finite = finite && isfinite(shk[t]);
        if (!finite) atomicMin(&status->nonfinite_splat, i);
        const Proj<double> pr = project_primal(p, cam, ro);
        if (!pr.culled && pr.degenerate) atomicMin(&status->degenerate_splat, i);
        // a non-finite splat fails the view (its error is reported); it is not
        // binned, so its NaN rectangle cannot inflate the duplicate count
        if (pr.culled || pr.degenerate || !finite) {
            keys[i] = kCulledKey;
            keys32[i] = 0xffffffffu;
            tcount[i] = 0;
        } else {
            visible = true;
            const double px = pr.mx, py = pr.my;
            const double rx = ro.cutoff * sqrt(pr.c00);
            const double ry = ro.cutoff * sqrt(pr.c11);
            double i00, i01, i11;
            invert2x2(pr.c00, pr.c01, pr.c11, i00, i01, i11);
            const double rho2 = ro.cull ? contrib_rho2(p.alpha, ro.alpha_skip) : INFINITY;
            const double k11 = i01 / i11, k00 = i01 / i00;
            double col[3] = {p.c[0], p.c[1], p.c[2]};
            if (kSH) sh_color<double, double>(p.mu, p.c, shk, nb, cam.cen, col);
            double r[kRec] = {px - rx, px + rx, py - ry, py + ry, px,  py,  i00, i01,
                              i11,     p.alpha, col[0], col[1], col[2], k11, rho2, k00};
            double2* dst = reinterpret_cast<double2*>(rec + (long long)kRec * i);
#pragma unroll
            for (int j = 0; j < kRec / 2; ++j) dst[j] = make_double2(r[2 * j], r[2 * j + 1]);
            keys[i] = depth_key(pr.depth);
            // K2's sort key: the depth rounded to FP32 (monotone; positive, so
            // its bits order as unsigned); equal FP32 depths are ordered by
            // the full key afterwards
            keys32[i] = __float_as_uint(__double2float_rn(pr.depth));
            int x0, x1, y0, y1;
            pixel_range(r[R_BX0], r[R_BX1], cam.W, x0, x1);
            pixel_range(r[R_BY0], r[R_BY1], cam.H, y0, y1);
            if (x0 > x1 || y0 > y1) {
                tcount[i] = 0;
            } else {
                // tiles whose pixel centres inside the bbox can reach
                // alpha_bar >= alpha_skip (geometry.cuh: ellipse_may_hit)
                rect[i] = make_int4(x0, y0, x1, y1);
                int n = 0, j = 0;
                unsigned long long bits = 0ull;  // row-major tile hits (rects <= 64 tiles)
                for (int ty = y0 / kTile; ty <= y1 / kTile; ++ty)
                    for (int tx = x0 / kTile; tx <= x1 / kTile; ++tx, ++j) {
                        const bool hit = ellipse_may_hit(
                            px, py, i00, i01, i11, k11, k00, rho2, max(x0, tx * kTile),
                            min(x1, tx * kTile + kTile - 1), max(y0, ty * kTile),
                            min(y1, ty * kTile + kTile - 1));
                        n += hit;
                        if (hit && j < 64) bits |= 1ull << j;
                    }
                tcount[i] = n;
                const int tx0 = x0 / kTile, ty0 = y0 / kTile;
                tinfo[i] = make_int4(tx0 | (ty0 << 16),
                                     (x1 / kTile - tx0 + 1) | ((y1 / kTile - ty0 + 1) << 16),
                                     (int)(unsigned)bits, (int)(unsigned)(bits >> 32));
            }
        }
    }
    // warp-aggregated visible count
    const unsigned m = __ballot_sync(0xffffffffu, visible);
    if ((threadIdx.x & 31) == 0 && m) atomicAdd(&status->n_visible, __popc(m));
}

__global__ void k_project_dump(const double* __restrict__ x, int K, DevCam cam, RenderP ro,
                               double* __restrict__ out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= K) return;
    const Splat p = load_splat(x, K, i);
    const Proj<double> pr = project_primal(p, cam, ro);
    double* o = out + 12LL * i;
    for (int j = 0; j < 12; ++j) o[j] = 0.0;
    if (pr.culled || pr.degenerate) {
        o[0] = 1.0;
        return;
    }
    const double rx = ro.cutoff * sqrt(pr.c00), ry = ro.cutoff * sqrt(pr.c11);
    double i00, i01, i11;
    invert2x2(pr.c00, pr.c01, pr.c11, i00, i01, i11);
    o[1] = pr.depth;
    o[2] = pr.mx;
    o[3] = pr.my;
    o[4] = pr.mx - rx;
    o[5] = pr.mx + rx;
    o[6] = pr.my - ry;
    o[7] = pr.my + ry;
    o[8] = i00;
    o[9] = i01;
    o[10] = i11;
}

__device__ __forceinline__ double probe_at(const double* v, const uint32_t* zbits, long long k) {
    if (v) return v[k];
    return ((zbits[k >> 5] >> (k & 31)) & 1u) ? 1.0 : -1.0;
}

// tangent records along v: build_fragments_dual (render.cpp:91-120)
__global__ void __launch_bounds__(256) k_project_jvp(const double* __restrict__ x, int K,
                                                     int nb, DevCam cam, RenderP ro,
                                                     const double* __restrict__ v,
                                                     const uint32_t* __restrict__ zbits,
                                                     double* __restrict__ trec) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= K) return;
    const Splat p = load_splat(x, K, i);
    const long long k = K;
    Dual mu[3], s[3], q[4];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        mu[a] = Dual(p.mu[a], probe_at(v, zbits, 3LL * i + a));
        s[a] = Dual(p.s[a], probe_at(v, zbits, 3 * k + 3LL * i + a));
    }
#pragma unroll
    for (int a = 0; a < 4; ++a) q[a] = Dual(p.q[a], probe_at(v, zbits, 6 * k + 4LL * i + a));
    const Proj<Dual> pr = project<Dual>(mu, s, q, cam.w, cam.t, cam.fx, cam.fy, cam.cx, cam.cy,
                                        ro.z_near, ro.lowpass);
    if (pr.culled || pr.degenerate) return;  // never referenced by a tile list
    Dual i00, i01, i11;
    invert2x2(pr.c00, pr.c01, pr.c11, i00, i01, i11);
    double* o = trec + (long long)kTRec * i;
    o[T_MX] = pr.mx.d;
    o[T_MY] = pr.my.d;
    o[T_I00] = i00.d;
    o[T_I01] = i01.d;
    o[T_I11] = i11.d;
    o[T_ALPHA] = probe_at(v, zbits, 10 * k + i);
    if (nb == 0) {
#pragma unroll
        for (int a = 0; a < 3; ++a) o[T_C0 + a] = probe_at(v, zbits, 11 * k + 3LL * i + a);
        return;
    }
    // SH extension: tangent of the view colour (coefficients and direction)
    Dual c[3], shk[45], col[3];
    const double* kp = sh_ptr(x, K, nb, i);
    const long long off = 14 * k + 3LL * nb * i;
#pragma unroll
    for (int a = 0; a < 3; ++a) c[a] = Dual(p.c[a], probe_at(v, zbits, 11 * k + 3LL * i + a));
    for (int t = 0; t < 3 * nb; ++t) shk[t] = Dual(kp[t], probe_at(v, zbits, off + t));
    sh_color<Dual, Dual>(mu, c, shk, nb, cam.cen, col);
#pragma unroll
    for (int a = 0; a < 3; ++a) o[T_C0 + a] = col[a].d;
}

// SH extension of the adjoint chain (oracle chain_splat): dL/dk_j = Y_j a_rgb
// and the view-direction term of dL/dmu (3 dual seeds), returned in gmu_sh
template <typename Add>
__device__ __forceinline__ void chain_sh(const double* x, int K, int nb, int id,
                                         const DevCam& cam, const Splat& p, const double* a,
                                         Add add, double* gmu_sh) {
    const double* kp = sh_ptr(x, K, nb, id);
    const long long off = 14LL * K + 3LL * nb * id;
    double d[3], Y[15];
    sh_dir<double>(p.mu, cam.cen, d);
    sh_basis<double>(d[0], d[1], d[2], nb, Y);
    for (int j = 0; j < nb; ++j)
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) add(off + 3 * j + ch, Y[j] * a[6 + ch]);
    const Dual c0[3] = {Dual(p.c[0]), Dual(p.c[1]), Dual(p.c[2])};
#pragma unroll 1
    for (int seed = 0; seed < 3; ++seed) {
        Dual mu[3], col[3];
#pragma unroll
        for (int q = 0; q < 3; ++q) mu[q] = Dual(p.mu[q], seed == q ? 1.0 : 0.0);
        sh_color<Dual, double>(mu, c0, kp, nb, cam.cen, col);
        gmu_sh[seed] = a[6] * col[0].d + a[7] * col[1].d + a[8] * col[2].d;
    }
}

// K11: render.cpp:288-329 restated per splat.  The 9 adjoints of a splat are
// the fixed-order sum of its K10 partials (duplicate, block order); the
// transpose of the 5x10 Jacobian of (mu2d, inverse covariance) w.r.t.
// (mu, s, q), which the reference evaluates with 10 dual seeds, is applied in
// one reverse sweep (geometry.cuh: chain_reverse).
template <bool kSH, int kSlots>
__global__ void __launch_bounds__(128, 5) k_chain_warp(int mode, const double* __restrict__ x, int K,
                                               int nb, DevCam cam, RenderP ro,
                                               const long long* __restrict__ off_id,
                                               const int* __restrict__ tcount, long long cap,
                                               const double* __restrict__ part,
                                               const unsigned char* __restrict__ mask,
                                               const double* __restrict__ zdense,
                                               const uint32_t* __restrict__ zbits,
                                               double* __restrict__ acc,
                                               double* nonfinite_flag) {
    // threads in splat-id order, so the scene reads and the gradient
    // read-modify-writes below are coalesced (at C5's 10M splats they no
    // longer fit in L2); a splat's partials are found through its duplicate
    // offset (off_id, scattered by K4)
    const int id = blockIdx.x * blockDim.x + threadIdx.x;
    if (id >= K) return;
    const int cnt = tcount[id];
    if (cnt == 0) return;
    const long long off = off_id[id];
    if (off + cnt > cap) return;  // an overflowed view (rerun)
    // the splat's parameters, fetched now: their latency overlaps the
    // partial sums
    const Splat p = load_splat(x, K, id);
    double a[kAdj];
#pragma unroll
    for (int j = 0; j < kAdj; ++j) a[j] = 0.0;
    // the kSlots (2 or 4, K10's blocks per tile) per-warp partials of each
    // duplicate, in (duplicate, warp) order; the partials are stored by
    // splat-major duplicate slot, so a splat's are one contiguous run of
    // kSlots * 80-byte records; the masks of 4 duplicates (kSlots bytes each)
    // are fetched together
    for (int t0 = 0; t0 < cnt; t0 += 4) {
        long long jp[4];
        unsigned mk[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) jp[u] = t0 + u < cnt ? off + t0 + u : -1;
#pragma unroll
        for (int u = 0; u < 4; ++u)
            mk[u] = jp[u] < 0 ? 0u
                    : kSlots == 4
                        ? *reinterpret_cast<const unsigned*>(mask + kSlots * jp[u])
                        : *reinterpret_cast<const unsigned short*>(mask + kSlots * jp[u]);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            if (mk[u] == 0u) continue;
            const double2* pp =
                reinterpret_cast<const double2*>(part + jp[u] * kSlots * kPartStride);
#pragma unroll
            for (int w = 0; w < kSlots; ++w) {
                if ((mk[u] >> (8 * w)) & 0xffu) {
                    // one 80-byte partial as five 16-byte loads (the pad unused)
                    double2 q[kPartStride / 2];
#pragma unroll
                    for (int h = 0; h < kPartStride / 2; ++h) q[h] = pp[w * (kPartStride / 2) + h];
#pragma unroll
                    for (int c = 0; c < kAdj; ++c) a[c] += (c & 1) ? q[c >> 1].y : q[c >> 1].x;
                }
            }
        }
    }
    const long long k = K;
    bool finite = true;
    auto add = [&](long long idx, double v) {
        if (mode == 1) v = probe_at(zdense, zbits, idx) * v;
        finite = finite && isfinite(v);
        acc[idx] += v;
    };
    const bool sh = kSH && nb > 0 && (a[6] != 0.0 || a[7] != 0.0 || a[8] != 0.0);
    double gmu_sh[3] = {0.0, 0.0, 0.0};
    if (sh) chain_sh(x, K, nb, id, cam, p, a, add, gmu_sh);
    bool any = false;
#pragma unroll
    for (int j = 0; j < 5; ++j) any = any || a[j] != 0.0;
    // the splat's 14 gradient entries (opacity, colour, then mean, scale,
    // rotation when the 2-D adjoints are non-zero): every acc load is issued
    // before the first store (acc may alias itself, so the compiler would
    // otherwise serialise the read-modify-writes)
    long long ix[14];
    double v[14];
    ix[0] = 10 * k + id;
    v[0] = a[5];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        ix[1 + c] = 11 * k + 3LL * id + c;
        v[1 + c] = a[6 + c];
        ix[4 + c] = 3LL * id + c;
        v[4 + c] = gmu_sh[c];
        ix[7 + c] = 3 * k + 3LL * id + c;
        v[7 + c] = 0.0;
    }
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        ix[10 + c] = 6 * k + 4LL * id + c;
        v[10 + c] = 0.0;
    }
    if (any) {
        // J^T a for (mu, s, q) in one reverse sweep (geometry.cuh)
        double gmu[3], gs[3], gq[4];
        chain_reverse(p.mu, p.s, p.q, cam.w, cam.t, cam.fx, cam.fy, ro.lowpass, a, gmu, gs, gq);
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            v[4 + c] = sh ? gmu_sh[c] + gmu[c] : gmu[c];
            v[7 + c] = gs[c];
        }
#pragma unroll
        for (int c = 0; c < 4; ++c) v[10 + c] = gq[c];
    }
    const int n = any ? 14 : (sh ? 7 : 4);
    double old[14];
#pragma unroll
    for (int j = 0; j < 14; ++j)
        if (j < n) old[j] = acc[ix[j]];
#pragma unroll
    for (int j = 0; j < 14; ++j) {
        if (j < n) {
            double w = v[j];
            if (mode == 1) w = probe_at(zdense, zbits, ix[j]) * w;
            finite = finite && isfinite(w);
            acc[ix[j]] = old[j] + w;
        }
    }
    if (!finite) *nonfinite_flag = 1.0;  // idempotent store
}

}  // namespace

void launch_project(cudaStream_t st, const double* x, int K, int nb, const DevCam& cam,
                    const RenderP& ro, double* rec, unsigned long long* keys,
                    unsigned int* keys32, int* ids, int4* rect, int* tcount,
                    int4* tinfo, ViewStatus* status) {
    if (K == 0) return;
    if (nb)
        k_project<true><<<ceil_div(K, 256), 256, 0, st>>>(x, K, nb, cam, ro, rec, keys, keys32,
                                                          ids, rect, tcount, tinfo, status);
    else
        k_project<false><<<ceil_div(K, 256), 256, 0, st>>>(x, K, nb, cam, ro, rec, keys, keys32,
                                                           ids, rect, tcount, tinfo, status);
    SGTR_CUDA(cudaGetLastError());
}

void launch_project_dump(cudaStream_t st, const double* x, int K, const DevCam& cam,
                         const RenderP& ro, double* out) {
    if (K == 0) return;
    k_project_dump<<<ceil_div(K, 256), 256, 0, st>>>(x, K, cam, ro, out);
    SGTR_CUDA(cudaGetLastError());
}

void launch_project_jvp(cudaStream_t st, const double* x, int K, int nb, const DevCam& cam,
                        const RenderP& ro, const double* v, const uint32_t* zbits,
                        double* trec) {
    if (K == 0) return;
    k_project_jvp<<<ceil_div(K, 256), 256, 0, st>>>(x, K, nb, cam, ro, v, zbits, trec);
    SGTR_CUDA(cudaGetLastError());
}

void launch_chain_warp(cudaStream_t st, int mode, const double* x, int K, int nb,
                       const DevCam& cam, const RenderP& ro, const long long* off_id,
                       const int* tcount, long long cap, int slots, const double* part,
                       const unsigned char* mask, const double* zdense, const uint32_t* zbits,
                       double* acc, double* nonfinite_flag) {
    if (K == 0) return;
    auto go = [&](auto kernel) {
        kernel<<<ceil_div(K, 128), 128, 0, st>>>(mode, x, K, nb, cam, ro, off_id, tcount, cap,
                                                 part, mask, zdense, zbits, acc, nonfinite_flag);
    };
    if (nb)
        slots == 2 ? go(k_chain_warp<true, 2>) : go(k_chain_warp<true, 4>);
    else
        slots == 2 ? go(k_chain_warp<false, 2>) : go(k_chain_warp<false, 4>);
    SGTR_CUDA(cudaGetLastError());
}

}  // namespace sgtr
