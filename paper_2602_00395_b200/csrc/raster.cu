// raster.cu — tile rasteriser: K7 forward blend, K10 reverse-order VJP,
// K12 forward-mode JVP.
//
// One CTA per 16x16 tile, one thread per pixel; each warp owns an 8x4 pixel
// block so that the per-fragment bounding-box test can first be done once per
// warp (uniform branch) against the block's span of pixel centres — most
// (pixel, fragment) pairs of a tile list fail the reference's bbox test
// (render.cpp:129-131), and whole warps skip them.  The tile's fragment list
// (depth order, from binning.cu) is staged through shared memory in batches;
// each 128-byte fragment record is copied by 8 lanes (one full cache line per
// record, 4 records per warp instruction), and every pixel reads the staged
// record as a warp-wide broadcast.
//
// Branch parity: the three kernels evaluate the primal alpha with the same
// pinned operation sequence (eval_expo's FMA form and fastexp.cuh's exp, a
// few ulp from the reference's own order), so bbox reject, alpha clamp,
// alpha skip and the transmittance stop take the same branches in forward,
// VJP and JVP — the reference's "frozen branches" contract
// (render.hpp:76-79).  The skip test is written as the reference's
// `alpha_bar < alpha_skip -> skip`, so a NaN alpha_bar is kept and
// propagates as it does in the reference (render.cpp:136).
#include <cstdlib>

#include "common.cuh"
#include "fastexp.cuh"
#include "geometry.cuh"
#include "launch.h"

namespace sgtr {
namespace {

constexpr int kThreads = kTilePixels;  // 256
constexpr int kFwdBatch = 256;
constexpr int kVjpBatch = 64;
constexpr int kJvpBatch = 128;
constexpr int kWarps = kThreads / 32;
constexpr unsigned kFull = 0xffffffffu;

struct PixelCtx {
    int px, py;
    bool inside;
    double pxc, pyc;
    double wx0, wx1, wy0, wy1;  // the warp's span of pixel centres
    int ix0, iy0;               // the warp's first pixel column / row
};

// exact overlap of a splat's pixel rectangle (K1's pixel_range: the pixels
// whose centre lies in the closed FP64 bbox, clipped to the image) with the
// warp's 8x4 pixel block
__device__ __forceinline__ bool rect_hits_warp(const PixelCtx& p, int4 r) {
    return !(p.ix0 + 7 < r.x || p.ix0 > r.z || p.iy0 + 3 < r.y || p.iy0 > r.w);
}
// the reference's per-pixel bbox test (render.cpp:128-131) on that rectangle
__device__ __forceinline__ bool rect_has_pixel(const PixelCtx& p, int4 r) {
    return p.px >= r.x && p.px <= r.z && p.py >= r.y && p.py <= r.w;
}

// warp w covers columns (w & 1) * 8 .. +7 and rows (w >> 1) * 4 .. +3
__device__ __forceinline__ PixelCtx pixel_ctx(int tile, int tiles_x, int W, int H,
                                              int warp = -1) {
    PixelCtx p;
    const int lane = threadIdx.x & 31;
    if (warp < 0) warp = threadIdx.x >> 5;
    const int x0 = (tile % tiles_x) * kTile + (warp & 1) * 8;
    const int y0 = (tile / tiles_x) * kTile + (warp >> 1) * 4;
    p.px = x0 + (lane & 7);
    p.py = y0 + (lane >> 3);
    p.inside = p.px < W && p.py < H;
    p.pxc = p.px + 0.5;
    p.pyc = p.py + 0.5;
    p.ix0 = x0;
    p.iy0 = y0;
    p.wx0 = x0 + 0.5;
    p.wx1 = x0 + 7.5;
    p.wy0 = y0 + 0.5;
    p.wy1 = y0 + 3.5;
    return p;
}

// reference: -0.5 * (dx*dx*i00 + dy*dy*i11) - dx*dy*i01  (render.cpp:134-135)
// evaluated as -0.5 (dx ax + dy ay) with (ax, ay) = Sigma^-1 d (4 FMA-fused
// steps instead of 9 roundings; a few ulp from the reference's order, the
// same in every pass, so the clamp/skip/stop branches agree between passes).
// (ax, ay) is also the VJP's d expo / d mu2d up to sign.
__device__ __forceinline__ double eval_expo(double dx, double dy, const double* f, double& ax,
                                            double& ay) {
    ax = __fma_rn(f[R_I01], dy, __dmul_rn(f[R_I00], dx));
    ay = __fma_rn(f[R_I11], dy, __dmul_rn(f[R_I01], dx));
    return __dmul_rn(-0.5, __fma_rn(dy, ay, __dmul_rn(dx, ax)));
}
__device__ __forceinline__ double eval_expo(double dx, double dy, const double* f) {
    double ax, ay;
    return eval_expo(dx, dy, f, ax, ay);
}

__device__ __forceinline__ bool outside_bbox(double pxc, double pyc, const double* f) {
    return pxc < f[R_BX0] || pxc > f[R_BX1] || pyc < f[R_BY0] || pyc > f[R_BY1];
}

// true when no pixel centre of the warp's block lies in the fragment's bbox
// (warp-uniform: every lane evaluates the same broadcast values)
__device__ __forceinline__ bool warp_misses(const PixelCtx& p, const double* f) {
    return p.wx1 < f[R_BX0] || p.wx0 > f[R_BX1] || p.wy1 < f[R_BY0] || p.wy0 > f[R_BY1];
}

// 32x32 bit-matrix transpose across the warp: lane l holds row l; returns
// this lane's column (bit l of the result = bit `lane` of row l).  Five
// exchange stages (__shfl_xor of 16, 8, 4, 2, 1 lanes).
__device__ __forceinline__ unsigned warp_transpose32(unsigned x) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) {
        const unsigned m = s == 16 ? 0x0000FFFFu
                           : s == 8 ? 0x00FF00FFu
                           : s == 4 ? 0x0F0F0F0Fu
                           : s == 2 ? 0x33333333u
                                    : 0x55555555u;
        const unsigned y = __shfl_xor_sync(0xffffffffu, x, s);
        x = (lane & s) ? ((x & ~m) | ((y & ~m) >> s)) : ((x & m) | ((y & m) << s));
    }
    return x;
}

// the pixels of an 8-column block (rows from iy0, `rows` <= 8 of them) that
// lie in the pixel rectangle r (K1's pixel_range of the closed FP64 bbox,
// render.cpp:128-131), as a mask over slot = row * 8 + column
__device__ __forceinline__ unsigned long long block_slots(int4 r, int ix0, int iy0, int rows) {
    const int c0 = max(r.x - ix0, 0), c1 = min(r.z - ix0, 7);
    const int r0 = max(r.y - iy0, 0), r1 = min(r.w - iy0, rows - 1);
    if (c0 > c1 || r0 > r1) return 0ull;
    const unsigned long long cols =
        ((0xFFull >> (7 - (c1 - c0))) << c0) * 0x0101010101010101ull;
    const int nr = r1 - r0 + 1;
    const unsigned long long rowm = (nr >= 8 ? ~0ull : ((1ull << (8 * nr)) - 1ull)) << (8 * r0);
    return cols & rowm;
}

// Warp-level contribution filter (after warp_misses): false only when no
// pixel centre of the warp's 8x4 block can reach alpha_bar >= alpha_skip —
// the minimum of q = d^T Sigma^-1 d over the block is certainly above
// rho2 (same bound as geometry.cuh:ellipse_may_hit, with the edge-minimiser
// slopes precomputed in the record).  Warp-uniform.
__device__ __forceinline__ bool warp_may_hit(const PixelCtx& p, const double* f) {
    const double rho2 = f[R_RHO2];
    if (!(rho2 < INFINITY)) return true;
    if (rho2 < 0.0) return false;
    const double ax = p.wx0 - f[R_MX], bx = p.wx1 - f[R_MX];
    const double ay = p.wy0 - f[R_MY], by = p.wy1 - f[R_MY];
    if (ax <= 0.0 && bx >= 0.0 && ay <= 0.0 && by >= 0.0) return true;
    const double i00 = f[R_I00], i01 = f[R_I01], i11 = f[R_I11];
    const double k11 = f[R_K11], k00 = f[R_K00];
    auto q = [&](double dx, double dy) { return i00 * dx * dx + 2.0 * i01 * dx * dy + i11 * dy * dy; };
    auto cl = [](double v, double lo, double hi) { return fmin(fmax(v, lo), hi); };
    double qmin = q(ax, cl(-k11 * ax, ay, by));
    qmin = fmin(qmin, q(bx, cl(-k11 * bx, ay, by)));
    qmin = fmin(qmin, q(cl(-k00 * ay, ax, bx), ay));
    qmin = fmin(qmin, q(cl(-k00 * by, ax, bx), by));
    const double mxd = fmax(fabs(ax), fabs(bx)), myd = fmax(fabs(ay), fabs(by));
    const double bound = fabs(i00) * mxd * mxd + fabs(i11) * myd * myd + 2.0 * fabs(i01) * mxd * myd;
    return !(qmin > rho2 + 1e-8 * rho2 + 1e-11 * bound + 1e-11);
}

// cooperative staging: 8 lanes per 128-byte record; entries [b, b+n) of the
// tile-sorted list go to s_rec[0, n)
__device__ __forceinline__ void stage_records(const TileLists& tl, const double* __restrict__ rec,
                                              int b, int n, double* s_rec, int* s_d) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int sub = lane >> 3, chunk = lane & 7;
    for (int e = warp * 4 + sub; e < n; e += kWarps * 4) {
        const int d = tl.sorted_d[b + e];
        const int id = tl.dup_id[d];
        const double2 v = reinterpret_cast<const double2*>(rec + (long long)kRec * id)[chunk];
        reinterpret_cast<double2*>(s_rec + kRec * e)[chunk] = v;
        if (s_d && chunk == 0) s_d[e] = d;
    }
}

__device__ __forceinline__ void stage_tangents(const TileLists& tl, const double* __restrict__ trec,
                                               int b, int n, double* s_t) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int sub = lane >> 3, chunk = lane & 7;
    for (int e = warp * 4 + sub; e < n; e += kWarps * 4) {
        if (chunk >= kTRec / 2) continue;
        const int id = tl.dup_id[tl.sorted_d[b + e]];
        const double2 v = reinterpret_cast<const double2*>(trec + (long long)kTRec * id)[chunk];
        reinterpret_cast<double2*>(s_t + kTRec * e)[chunk] = v;
    }
}

// ------------------------------------------------------------------ K7
// kCount: also count the (pixel, fragment) pairs reaching the alpha
// evaluation (E) and the contributing ones (C), the algorithmic-work units
// of SURVEY §8(d); used outside timed regions only.
template <bool kCount, bool kWarpCull>
__global__ void __launch_bounds__(kThreads) k_raster_fwd(TileLists tl,
                                                         const double* __restrict__ rec, int W,
                                                         int H, RenderP ro,
                                                         double* __restrict__ img,
                                                         double* __restrict__ tfinal,
                                                         int* __restrict__ last,
                                                         unsigned long long* counters) {
    __shared__ __align__(16) double s_rec[kFwdBatch * kRec];
    const int tile = blockIdx.x + tl.row0 * tl.tiles_x;
    const PixelCtx pc = pixel_ctx(tile, tl.tiles_x, W, H);
    const int start = tl.tile_start[tile], end = tl.tile_end[tile];
    double T = 1.0, c0 = 0.0, c1 = 0.0, c2 = 0.0;
    bool done = !pc.inside;
    int processed = end - start;
    unsigned long long n_eval = 0, n_contrib = 0;
    for (int b = start; b < end; b += kFwdBatch) {
        if (__syncthreads_and(done)) break;
        const int n = min(kFwdBatch, end - b);
        stage_records(tl, rec, b, n, s_rec, nullptr);
        __syncthreads();
        if (__all_sync(kFull, done)) continue;
        for (int jj = 0; jj < n; ++jj) {
            const double* f = s_rec + kRec * jj;
            if (warp_misses(pc, f) || (kWarpCull && !warp_may_hit(pc, f))) continue;
            if (!done && !outside_bbox(pc.pxc, pc.pyc, f)) {
                const double dx = pc.pxc - f[R_MX], dy = pc.pyc - f[R_MY];
                double abar = __dmul_rn(f[R_ALPHA], fast_exp_neg(eval_expo(dx, dy, f)));
                if (kCount) ++n_eval;
                if (abar >= ro.alpha_clamp) abar = ro.alpha_clamp;
                if (!(abar < ro.alpha_skip)) {
                    if (kCount) ++n_contrib;
                    const double w = abar * T;
                    c0 += f[R_C0] * w;
                    c1 += f[R_C1] * w;
                    c2 += f[R_C2] * w;
                    T = __dmul_rn(T, __dsub_rn(1.0, abar));
                    if (T < ro.t_stop) {
                        done = true;
                        processed = b - start + jj + 1;
                    }
                }
            }
            if (__all_sync(kFull, done)) break;
        }
    }
    if (kCount) {
        for (int o = 16; o > 0; o >>= 1) {
            n_eval += __shfl_xor_sync(kFull, n_eval, o);
            n_contrib += __shfl_xor_sync(kFull, n_contrib, o);
        }
        if ((threadIdx.x & 31) == 0) {
            atomicAdd(counters, n_eval);
            atomicAdd(counters + 1, n_contrib);
        }
    }
    if (!pc.inside) return;
    const long long P = (long long)W * H, p = (long long)pc.py * W + pc.px;
    img[p] = c0 + ro.bg[0] * T;
    img[P + p] = c1 + ro.bg[1] * T;
    img[2 * P + p] = c2 + ro.bg[2] * T;
    tfinal[p] = T;
    last[p] = processed;
}

// ------------------------------------------------------------------ K7, batch-staged
// Each warp owns an 8x4 pixel block and walks its tile's list on its own, in
// batches of 32 positions: each lane tests one position against the block and, if it
// passes, loads that fragment's 9 raster fields into a warp-private shared
// slot (ballot-compacted), so the 32 record fetches of a batch are in flight
// together instead of one dependent fetch per blended entry.
struct StagedRec {
    double mx, my, i00, i01, i11, alpha, c0, c1, c2, pad;
};

template <int WPB>
__global__ void __launch_bounds__(32 * WPB)
    k_raster_fwd_staged(TileLists tl, const double* __restrict__ rec, int W, int H, RenderP ro,
                        double* __restrict__ img, double* __restrict__ tfinal,
                        int* __restrict__ last) {
    constexpr int SUB = kWarps / WPB;
    __shared__ __align__(16) StagedRec s_rec[WPB][32];
    __shared__ int4 s_rect[WPB][32];
    __shared__ int s_pos[WPB][32];
    const int tile = blockIdx.x / SUB + tl.row0 * tl.tiles_x;
    const int lane = threadIdx.x & 31, lw = threadIdx.x >> 5;
    const int warp = (blockIdx.x % SUB) * WPB + lw;
    const PixelCtx pc = pixel_ctx(tile, tl.tiles_x, W, H, warp);
    const int start = tl.tile_start[tile], end = tl.tile_end[tile];
    double T = 1.0, c0 = 0.0, c1 = 0.0, c2 = 0.0;
    bool done = !pc.inside;
    int processed = end - start;
    StagedRec* my_rec = s_rec[lw];
    int4* my_rect = s_rect[lw];
    int* my_pos = s_pos[lw];
    for (int base = start; base < end; base += 32) {
        if (__all_sync(kFull, done)) break;
        const int jj = base + lane;
        bool pass = false;
        int4 rr;
        if (jj < end) {
            rr = __ldg(tl.trect + jj);
            pass = rect_hits_warp(pc, rr);
        }
        const unsigned m = __ballot_sync(kFull, pass);
        if (pass) {
            const int q = __popc(m & ((1u << lane) - 1u));
            const double2* r2 =
                reinterpret_cast<const double2*>(rec + (long long)kRec * __ldg(tl.tile_ids + jj));
            const double2 a = __ldg(r2 + 2), b = __ldg(r2 + 3), c = __ldg(r2 + 4);
            const double2 d = __ldg(r2 + 5), e = __ldg(r2 + 6);
            double2* o = reinterpret_cast<double2*>(my_rec + q);
            o[0] = a;
            o[1] = b;
            o[2] = c;
            o[3] = d;
            o[4] = e;
            my_rect[q] = rr;
            my_pos[q] = jj;
        }
        __syncwarp();
        const int n = __popc(m);
        for (int e = 0; e < n; ++e) {
            if (!done && rect_has_pixel(pc, my_rect[e])) {
                const StagedRec r = my_rec[e];
                const double f[13] = {0.0,   0.0,   0.0,   0.0,     r.mx, r.my, r.i00,
                                      r.i01, r.i11, r.alpha, r.c0, r.c1, r.c2};
                const double dx = pc.pxc - f[R_MX], dy = pc.pyc - f[R_MY];
                double abar = __dmul_rn(f[R_ALPHA], fast_exp_neg(eval_expo(dx, dy, f)));
                if (abar >= ro.alpha_clamp) abar = ro.alpha_clamp;
                if (!(abar < ro.alpha_skip)) {
                    const double w = abar * T;
                    c0 += f[R_C0] * w;
                    c1 += f[R_C1] * w;
                    c2 += f[R_C2] * w;
                    T = __dmul_rn(T, __dsub_rn(1.0, abar));
                    if (T < ro.t_stop) {
                        done = true;
                        processed = my_pos[e] - start + 1;
                    }
                }
            }
            if (__all_sync(kFull, done)) break;
        }
        __syncwarp();
    }
    if (!pc.inside) return;
    const long long P = (long long)W * H, p = (long long)pc.py * W + pc.px;
    img[p] = c0 + ro.bg[0] * T;
    img[P + p] = c1 + ro.bg[1] * T;
    img[2 * P + p] = c2 + ro.bg[2] * T;
    tfinal[p] = T;
    last[p] = processed;
}

// ------------------------------------------------------------------ K7, batch-staged, paired entries
// As k_raster_fwd_staged, blending the staged batch two entries at a time:
// the two falloffs (exp polynomial, clamp, skip test) do not depend on the
// blend state, so when both entries meet the warp's block they are computed
// in one straight-line block — two independent FP64 dependency chains the
// pipe interleaves — and then blended in list order, the second only if the
// pixel did not stop at the first.  Per pixel the operations and their order
// are those of k_raster_fwd_staged, so the outputs are bit-identical.
template <int WPB>
__global__ void __launch_bounds__(32 * WPB)
    k_raster_fwd_paired(TileLists tl, const double* __restrict__ rec, int W, int H, RenderP ro,
                        double* __restrict__ img, double* __restrict__ tfinal,
                        int* __restrict__ last) {
    constexpr int SUB = kWarps / WPB;
    __shared__ __align__(16) StagedRec s_rec[WPB][32];
    __shared__ int4 s_rect[WPB][32];
    __shared__ int s_pos[WPB][32];
    const int tile =
        tl.order ? tl.order[blockIdx.x / SUB] : blockIdx.x / SUB + tl.row0 * tl.tiles_x;
    const int lane = threadIdx.x & 31, lw = threadIdx.x >> 5;
    const int warp = (blockIdx.x % SUB) * WPB + lw;
    const PixelCtx pc = pixel_ctx(tile, tl.tiles_x, W, H, warp);
    const int start = tl.tile_start[tile], end = tl.tile_end[tile];
    double T = 1.0, c0 = 0.0, c1 = 0.0, c2 = 0.0;
    bool done = !pc.inside;
    int processed = end - start;
    StagedRec* my_rec = s_rec[lw];
    int4* my_rect = s_rect[lw];
    int* my_pos = s_pos[lw];
    auto falloff = [&](const StagedRec& r) {
        const double f[13] = {0.0,   0.0,   0.0,   0.0,     r.mx, r.my, r.i00,
                              r.i01, r.i11, r.alpha, r.c0, r.c1, r.c2};
        const double dx = pc.pxc - r.mx, dy = pc.pyc - r.my;
        double abar = __dmul_rn(r.alpha, fast_exp_neg(eval_expo(dx, dy, f)));
        if (abar >= ro.alpha_clamp) abar = ro.alpha_clamp;
        return abar;
    };
    auto blend = [&](const StagedRec& r, double abar, int e) {
        const double w = abar * T;
        c0 += r.c0 * w;
        c1 += r.c1 * w;
        c2 += r.c2 * w;
        T = __dmul_rn(T, __dsub_rn(1.0, abar));
        if (T < ro.t_stop) {
            done = true;
            processed = my_pos[e] - start + 1;
        }
    };
    for (int base = start; base < end; base += 32) {
        if (__all_sync(kFull, done)) break;
        const int jj = base + lane;
        bool pass = false;
        int4 rr;
        if (jj < end) {
            rr = __ldg(tl.trect + jj);
            pass = rect_hits_warp(pc, rr);
        }
        const unsigned m = __ballot_sync(kFull, pass);
        if (pass) {
            const int q = __popc(m & ((1u << lane) - 1u));
            const double2* r2 =
                reinterpret_cast<const double2*>(rec + (long long)kRec * __ldg(tl.tile_ids + jj));
            const double2 a = __ldg(r2 + 2), b = __ldg(r2 + 3), c = __ldg(r2 + 4);
            const double2 d = __ldg(r2 + 5), e = __ldg(r2 + 6);
            double2* o = reinterpret_cast<double2*>(my_rec + q);
            o[0] = a;
            o[1] = b;
            o[2] = c;
            o[3] = d;
            o[4] = e;
            my_rect[q] = rr;
            my_pos[q] = jj;
        }
        __syncwarp();
        const int n = __popc(m);
        for (int e = 0; e < n; e += 2) {
            const bool h0 = !done && rect_has_pixel(pc, my_rect[e]);
            const bool h1 = e + 1 < n && !done && rect_has_pixel(pc, my_rect[e + 1]);
            const bool a0 = __any_sync(kFull, h0), a1 = __any_sync(kFull, h1);
            if (a0 && a1) {
                const StagedRec r0 = my_rec[e], r1 = my_rec[e + 1];
                const double ab0 = falloff(r0), ab1 = falloff(r1);
                if (h0 && !(ab0 < ro.alpha_skip)) blend(r0, ab0, e);
                if (h1 && !done && !(ab1 < ro.alpha_skip)) blend(r1, ab1, e + 1);
            } else if (a0 || a1) {
                const int ee = a0 ? e : e + 1;
                if (a0 ? h0 : h1) {
                    const StagedRec r = my_rec[ee];
                    const double ab = falloff(r);
                    if (!(ab < ro.alpha_skip)) blend(r, ab, ee);
                }
            }
            if (__all_sync(kFull, done)) break;
        }
        __syncwarp();
    }
    if (!pc.inside) return;
    const long long P = (long long)W * H, p = (long long)pc.py * W + pc.px;
    img[p] = c0 + ro.bg[0] * T;
    img[P + p] = c1 + ro.bg[1] * T;
    img[2 * P + p] = c2 + ro.bg[2] * T;
    tfinal[p] = T;
    last[p] = processed;
}

// ------------------------------------------------------------------ K7, hit bitmasks
// The per-pixel bbox test of every (entry, pixel) pair is done once per batch
// as bit arithmetic: the lane that stages list entry base + j turns its pixel
// rectangle into the 32-bit mask of the warp block's pixels it covers, and a
// warp bit-transpose gives every pixel lane the mask of the batch entries
// covering it.  The warp then visits, two at a time, only the entries that
// cover some pixel still blending (an OR-reduction of the lane masks, with
// finished pixels' masks cleared), and each lane's test of an entry is one bit
// -- no per-entry rectangle loads, compares or votes.  Per pixel the entries,
// operations and their order are those of k_raster_fwd_paired, so the image,
// T and the stop index are bit-identical.
template <int WPB>
__global__ void __launch_bounds__(32 * WPB)
    k_raster_fwd_bits(TileLists tl, const double* __restrict__ rec, int W, int H, RenderP ro,
                      double* __restrict__ img, double* __restrict__ tfinal,
                      int* __restrict__ last) {
    constexpr int SUB = kWarps / WPB;
    __shared__ __align__(16) StagedRec s_rec[WPB][32];
    const int tile =
        tl.order ? tl.order[blockIdx.x / SUB] : blockIdx.x / SUB + tl.row0 * tl.tiles_x;
    const int lane = threadIdx.x & 31, lw = threadIdx.x >> 5;
    const int warp = (blockIdx.x % SUB) * WPB + lw;
    const PixelCtx pc = pixel_ctx(tile, tl.tiles_x, W, H, warp);
    const int start = tl.tile_start[tile], end = tl.tile_end[tile];
    double T = 1.0, c0 = 0.0, c1 = 0.0, c2 = 0.0;
    bool done = !pc.inside;
    int processed = end - start;
    StagedRec* my_rec = s_rec[lw];
    auto falloff = [&](const StagedRec& r) {
        const double f[13] = {0.0,   0.0,   0.0,   0.0,     r.mx, r.my, r.i00,
                              r.i01, r.i11, r.alpha, r.c0, r.c1, r.c2};
        const double dx = pc.pxc - r.mx, dy = pc.pyc - r.my;
        double abar = __dmul_rn(r.alpha, fast_exp_neg(eval_expo(dx, dy, f)));
        if (abar >= ro.alpha_clamp) abar = ro.alpha_clamp;
        return abar;
    };
    auto blend = [&](const StagedRec& r, double abar, int pos) {
        const double w = abar * T;
        c0 += r.c0 * w;
        c1 += r.c1 * w;
        c2 += r.c2 * w;
        T = __dmul_rn(T, __dsub_rn(1.0, abar));
        if (T < ro.t_stop) {
            done = true;
            processed = pos - start + 1;
        }
    };
    for (int base = start; base < end; base += 32) {
        if (__all_sync(kFull, done)) break;
        const int jj = base + lane;
        unsigned slots = 0;
        if (jj < end) {
            slots = (unsigned)block_slots(__ldg(tl.trect + jj), pc.ix0, pc.iy0, 4);
            if (slots) {
                const double2* r2 = reinterpret_cast<const double2*>(
                    rec + (long long)kRec * __ldg(tl.tile_ids + jj));
                const double2 a = __ldg(r2 + 2), b = __ldg(r2 + 3), c = __ldg(r2 + 4);
                const double2 d = __ldg(r2 + 5), e = __ldg(r2 + 6);
                double2* o = reinterpret_cast<double2*>(my_rec + lane);
                o[0] = a;
                o[1] = b;
                o[2] = c;
                o[3] = d;
                o[4] = e;
            }
        }
        unsigned mine = warp_transpose32(slots);  // bit j: entry base + j covers my pixel
        if (done) mine = 0u;
        __syncwarp();
        unsigned wb = __reduce_or_sync(kFull, mine);
        while (wb) {
            const int j0 = __ffs(wb) - 1;
            wb &= wb - 1u;
            if (wb) {
                const int j1 = __ffs(wb) - 1;
                wb &= wb - 1u;
                const bool h0 = (mine >> j0) & 1u, h1 = (mine >> j1) & 1u;
                const StagedRec r0 = my_rec[j0], r1 = my_rec[j1];
                const double ab0 = falloff(r0), ab1 = falloff(r1);
                if (h0 && !(ab0 < ro.alpha_skip)) blend(r0, ab0, base + j0);
                if (h1 && !done && !(ab1 < ro.alpha_skip)) blend(r1, ab1, base + j1);
            } else if ((mine >> j0) & 1u) {
                const StagedRec r = my_rec[j0];
                const double ab = falloff(r);
                if (!(ab < ro.alpha_skip)) blend(r, ab, base + j0);
            }
            if (done) mine = 0u;
            wb &= __reduce_or_sync(kFull, mine);
        }
        __syncwarp();
    }
    if (!pc.inside) return;
    const long long P = (long long)W * H, p = (long long)pc.py * W + pc.px;
    img[p] = c0 + ro.bg[0] * T;
    img[P + p] = c1 + ro.bg[1] * T;
    img[2 * P + p] = c2 + ro.bg[2] * T;
    tfinal[p] = T;
    last[p] = processed;
}

// ------------------------------------------------------------------ K10
// Transposed butterfly: sums g[0..7] over the warp so that lane l with
// (l & 3) == 0 ends with the total of g[l >> 2] (9 shuffles instead of 40),
// and g[8] with a plain butterfly (lane 0 keeps it).  Fixed order, so the
// result is deterministic.
__device__ __forceinline__ void warp_reduce9(double* g, int lane, double& v_lane, double& v8) {
    const bool b4 = lane & 16, b3 = lane & 8, b2 = lane & 4;
    double h4[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const double send = b4 ? g[i] : g[4 + i];
        const double keep = b4 ? g[4 + i] : g[i];
        h4[i] = keep + __shfl_xor_sync(kFull, send, 16);
    }
    double h2[2];
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        const double send = b3 ? h4[i] : h4[2 + i];
        const double keep = b3 ? h4[2 + i] : h4[i];
        h2[i] = keep + __shfl_xor_sync(kFull, send, 8);
    }
    {
        const double send = b2 ? h2[0] : h2[1];
        const double keep = b2 ? h2[1] : h2[0];
        v_lane = keep + __shfl_xor_sync(kFull, send, 4);
    }
    v_lane += __shfl_xor_sync(kFull, v_lane, 2);
    v_lane += __shfl_xor_sync(kFull, v_lane, 1);
    double s = g[8];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(kFull, s, o);
    v8 = s;
}

// Warp reduction of 9 doubles through a warp-private shared scratch: lanes
// store their 9 values (component-major, padded stride 33), 27 lanes each sum
// an 11-lane third of one component, 9 lanes add the three thirds and write
// the totals to out[0..8].  ~40 instructions instead of the shuffle
// butterfly's selects and shuffles; fixed order, so deterministic.
constexpr int kRedStride = 33;
constexpr int kRedScratch = kAdj * kRedStride + 27;
__device__ __forceinline__ void warp_reduce9_smem(const double* g, int lane, double* scr,
                                                  double* out) {
#pragma unroll
    for (int c = 0; c < kAdj; ++c) scr[c * kRedStride + lane] = g[c];
    __syncwarp();
    if (lane < 27) {
        const int c = lane / 3, q = lane % 3;
        const double* col = scr + c * kRedStride + q * 11;
        const int n = q == 2 ? 10 : 11;
        double s = col[0];
        for (int k = 1; k < n; ++k) s += col[k];
        scr[kAdj * kRedStride + lane] = s;
    }
    __syncwarp();
    if (lane < kAdj) {
        const double* t = scr + kAdj * kRedStride + 3 * lane;
        out[lane] = (t[0] + t[1]) + t[2];
    }
    __syncwarp();
}

template <bool kWarpCull, int kMinBlocks>
__global__ void __launch_bounds__(kThreads, kMinBlocks) k_raster_vjp(TileLists tl,
                                                         const double* __restrict__ rec, int W,
                                                         int H, RenderP ro,
                                                         const double* __restrict__ adj,
                                                         const double* __restrict__ tfinal,
                                                         const int* __restrict__ last,
                                                         double* __restrict__ slots) {
    __shared__ __align__(16) double s_rec[kVjpBatch * kRec];
    __shared__ double s_red[kWarps][kVjpBatch][kAdj];
    __shared__ int s_d[kVjpBatch];
    __shared__ unsigned s_mask[kVjpBatch];
    __shared__ int s_maxlast[kWarps];
    const int tile = blockIdx.x + tl.row0 * tl.tiles_x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const PixelCtx pc = pixel_ctx(tile, tl.tiles_x, W, H);
    const int start = tl.tile_start[tile], end = tl.tile_end[tile];
    const long long P = (long long)W * H, p = (long long)pc.py * W + pc.px;
    double u0 = 0, u1 = 0, u2 = 0, T = 0.0;
    int lastp = 0;
    if (pc.inside) {
        u0 = adj[p];
        u1 = adj[P + p];
        u2 = adj[2 * P + p];
        T = tfinal[p];
        lastp = last[p];
    }
    // pixels with an all-zero adjoint are skipped (render.cpp:283)
    const bool active = pc.inside && !(u0 == 0.0 && u1 == 0.0 && u2 == 0.0);
    if (!active) lastp = 0;
    double b0 = ro.bg[0] * T, b1 = ro.bg[1] * T, b2 = ro.bg[2] * T;  // "behind"
    // entries past every pixel's last processed fragment get zero slots
    const int wlast = __reduce_max_sync(kFull, lastp);
    if (lane == 0) s_maxlast[warp] = wlast;
    __syncthreads();
    int ml = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) ml = max(ml, s_maxlast[w]);
    const int hi = start + ml;
    for (int j = hi + threadIdx.x; j < end; j += kThreads) {
        double* s = slots + (long long)kAdj * tl.sorted_d[j];
#pragma unroll
        for (int c = 0; c < kAdj; ++c) s[c] = 0.0;
    }
    for (int bend = hi; bend > start; bend -= kVjpBatch) {
        const int bstart = max(start, bend - kVjpBatch);
        const int n = bend - bstart;
        __syncthreads();
        stage_records(tl, rec, bstart, n, s_rec, s_d);
        if (threadIdx.x < n) s_mask[threadIdx.x] = 0u;
        __syncthreads();
        for (int jj = n - 1; jj >= 0; --jj) {
            const int rel = bstart - start + jj;
            if (rel >= wlast) continue;
            const double* f = s_rec + kRec * jj;
            if (warp_misses(pc, f) || (kWarpCull && !warp_may_hit(pc, f))) continue;
            double g[kAdj];
#pragma unroll
            for (int c = 0; c < kAdj; ++c) g[c] = 0.0;
            bool contrib = false;
            if (rel < lastp && !outside_bbox(pc.pxc, pc.pyc, f)) {
                const double dx = pc.pxc - f[R_MX], dy = pc.pyc - f[R_MY];
                const double gauss = fast_exp_neg(eval_expo(dx, dy, f));
                double abar = __dmul_rn(f[R_ALPHA], gauss);
                const bool clamped = abar >= ro.alpha_clamp;
                if (clamped) abar = ro.alpha_clamp;
                if (!(abar < ro.alpha_skip)) {
                    contrib = true;
                    // one reciprocal for T_in = T / (1 - abar) and the three
                    // behind / (1 - abar) terms (render.cpp:243-245)
                    const double rom = 1.0 / __dsub_rn(1.0, abar);
                    const double t_in = T * rom;
                    const double at = abar * t_in;
                    g[6] = u0 * at;
                    g[7] = u1 * at;
                    g[8] = u2 * at;
                    const double dab = u0 * (f[R_C0] * t_in - b0 * rom) +
                                       u1 * (f[R_C1] * t_in - b1 * rom) +
                                       u2 * (f[R_C2] * t_in - b2 * rom);
                    b0 += f[R_C0] * at;
                    b1 += f[R_C1] * at;
                    b2 += f[R_C2] * at;
                    if (!clamped) {
                        g[5] = gauss * dab;
                        const double de = abar * dab;
                        g[2] = de * (-0.5 * dx * dx);
                        g[3] = de * (-dx * dy);
                        g[4] = de * (-0.5 * dy * dy);
                        g[0] = de * (f[R_I00] * dx + f[R_I01] * dy);
                        g[1] = de * (f[R_I01] * dx + f[R_I11] * dy);
                    }
                    T = t_in;
                }
            }
            if (!__any_sync(kFull, contrib)) continue;
            double v, v8;
            warp_reduce9(g, lane, v, v8);
            if ((lane & 3) == 0) s_red[warp][jj][lane >> 2] = v;
            if (lane == 0) {
                s_red[warp][jj][8] = v8;
                atomicOr(&s_mask[jj], 1u << warp);
            }
        }
        __syncthreads();
        for (int idx = threadIdx.x; idx < n * kAdj; idx += kThreads) {
            const int jj = idx / kAdj, c = idx % kAdj;
            const unsigned m = s_mask[jj];
            double s = 0.0;
#pragma unroll
            for (int w = 0; w < kWarps; ++w)
                if (m & (1u << w)) s += s_red[w][jj][c];
            slots[(long long)kAdj * s_d[jj] + c] = s;
        }
    }
}

// ------------------------------------------------------------------ K10, batch-staged, 2 px/lane
// As k_raster_vjp_staged, but a warp owns an 8x8 block (lane: column
// lane & 7, rows lane >> 3 and 4 + (lane >> 3)): one list walk, record fetch
// and 9-value reduction per entry now serve 64 pixels, and the two pixels'
// independent recurrences give each lane instruction-level parallelism.  A
// tile is 4 such warps (partial slots 0..3 of the duplicate).
template <int WPB, int kMinB = 10>
__global__ void __launch_bounds__(32 * WPB, kMinB * 2 / WPB)
    k_raster_vjp_staged2(TileLists tl, const double* __restrict__ rec, int W, int H, RenderP ro,
                         const double* __restrict__ adj, const double* __restrict__ tfinal,
                         const int* __restrict__ last, double* __restrict__ part,
                         unsigned char* __restrict__ mask) {
    constexpr int SUB = 4 / WPB;
    __shared__ double s_red[WPB][kRedScratch];
    __shared__ __align__(16) StagedRec s_rec[WPB][32];
    __shared__ int4 s_rect[WPB][32];
    __shared__ int s_pos[WPB][32];
    __shared__ int s_slot[WPB][32];
    const int tile = blockIdx.x / SUB + tl.row0 * tl.tiles_x;
    const int lane = threadIdx.x & 31, lw = threadIdx.x >> 5;
    const int warp = (blockIdx.x % SUB) * WPB + lw;  // 0..3: 8x8 block of the tile
    const int bx0 = (tile % tl.tiles_x) * kTile + (warp & 1) * 8;
    const int by0 = (tile / tl.tiles_x) * kTile + (warp >> 1) * 8;
    const int px = bx0 + (lane & 7);
    const int start = tl.tile_start[tile];
    const long long P = (long long)W * H;
    // ub = u . behind: the adjoint-weighted colour composited behind the
    // current fragment (the reference keeps the 3 channels, render.cpp:238-245;
    // only this dot product enters dL/dalpha_bar)
    double u0[2], u1[2], u2[2], T[2], ub[2];
    int lastp[2];
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        const int py = by0 + (lane >> 3) + 4 * k;
        u0[k] = u1[k] = u2[k] = T[k] = 0.0;
        lastp[k] = 0;
        if (px < W && py < H) {
            const long long p = (long long)py * W + px;
            u0[k] = adj[p];
            u1[k] = adj[P + p];
            u2[k] = adj[2 * P + p];
            T[k] = tfinal[p];
            lastp[k] = last[p];
            // pixels with an all-zero adjoint are skipped (render.cpp:283)
            if (u0[k] == 0.0 && u1[k] == 0.0 && u2[k] == 0.0) lastp[k] = 0;
        }
        ub[k] = T[k] * (u0[k] * ro.bg[0] + u1[k] * ro.bg[1] + u2[k] * ro.bg[2]);
    }
    const int wlast = __reduce_max_sync(kFull, max(lastp[0], lastp[1]));
    StagedRec* my_rec = s_rec[lw];
    int4* my_rect = s_rect[lw];
    int* my_pos = s_pos[lw];
    int* my_slot = s_slot[lw];
    for (int top = start + wlast; top > start; top -= 32) {
        const int base = max(start, top - 32);
        const int jj = base + lane;
        bool pass = false;
        int4 rr;
        if (jj < top) {
            rr = __ldg(tl.trect + jj);
            pass = !(bx0 + 7 < rr.x || bx0 > rr.z || by0 + 7 < rr.y || by0 > rr.w);
        }
        const unsigned m = __ballot_sync(kFull, pass);
        if (pass) {
            const int q = __popc(m & ((1u << lane) - 1u));
            const double2* r2 =
                reinterpret_cast<const double2*>(rec + (long long)kRec * __ldg(tl.tile_ids + jj));
            const double2 a = __ldg(r2 + 2), b = __ldg(r2 + 3), c = __ldg(r2 + 4);
            const double2 d = __ldg(r2 + 5), e = __ldg(r2 + 6);
            double2* o = reinterpret_cast<double2*>(my_rec + q);
            o[0] = a;
            o[1] = b;
            o[2] = c;
            o[3] = d;
            o[4] = e;
            my_rect[q] = rr;
            my_pos[q] = jj;
            my_slot[q] = __ldg(tl.sorted_d + jj);
        }
        __syncwarp();
        for (int e = __popc(m) - 1; e >= 0; --e) {
            const int j = my_pos[e];
            const int rel = j - start;
            const int4 r4 = my_rect[e];
            double g[kAdj];
#pragma unroll
            for (int c = 0; c < kAdj; ++c) g[c] = 0.0;
            bool contrib = false;
            const bool colin = px >= r4.x && px <= r4.z;
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                const int py = by0 + (lane >> 3) + 4 * k;
                if (!(rel < lastp[k] && colin && py >= r4.y && py <= r4.w)) continue;
                const StagedRec r = my_rec[e];
                const double f[13] = {0.0,   0.0,   0.0,     0.0,  r.mx, r.my, r.i00,
                                      r.i01, r.i11, r.alpha, r.c0, r.c1, r.c2};
                const double dx = (px + 0.5) - f[R_MX], dy = (py + 0.5) - f[R_MY];
                double ax, ay;
                const double gauss = fast_exp_neg(eval_expo(dx, dy, f, ax, ay));
                double abar = __dmul_rn(f[R_ALPHA], gauss);
                const bool clamped = abar >= ro.alpha_clamp;
                if (clamped) abar = ro.alpha_clamp;
                if (abar < ro.alpha_skip) continue;
                contrib = true;
                const double rom = rcp_unit(__dsub_rn(1.0, abar));
                const double t_in = T[k] * rom;
                const double at = abar * t_in;
                g[6] += u0[k] * at;
                g[7] += u1[k] * at;
                g[8] += u2[k] * at;
                const double uc = u0[k] * f[R_C0] + u1[k] * f[R_C1] + u2[k] * f[R_C2];
                const double dab = uc * t_in - ub[k] * rom;
                ub[k] += uc * at;
                if (!clamped) {
                    g[5] += gauss * dab;
                    const double de = abar * dab;
                    g[2] += de * (-0.5 * dx * dx);
                    g[3] += de * (-dx * dy);
                    g[4] += de * (-0.5 * dy * dy);
                    g[0] += de * ax;
                    g[1] += de * ay;
                }
                T[k] = t_in;
            }
            const unsigned cm = __ballot_sync(kFull, contrib);
            if (cm == 0u) continue;
            const long long dslot = my_slot[e];
            double* o = part + (dslot * kVjpSlots + warp) * kAdj;
            warp_reduce9_smem(g, lane, s_red[lw], o);
            if (lane == 0) mask[dslot * kVjpSlots + warp] = 1;
        }
        __syncwarp();
    }
}

// ------------------------------------------------------------------ K10, batch-staged, 2 px/lane, interleaved
// As k_raster_vjp_staged2, with three changes that leave every partial
// bit-identical:
//  * the two pixels' evaluations run in one straight-line block when both
//    rows of the warp's block meet the fragment, so the two exp polynomials
//    and reciprocals are independent dependency chains the FP64 pipe
//    interleaves (with a branch per pixel the compiler serialises them); a
//    pixel outside the fragment still runs the arithmetic (its lane would
//    idle in the other branch anyway) and only its state updates are
//    predicated off;
//  * the conic adjoints accumulate de * dx^2, de * dx dy, de * dy^2 and take
//    their factors -1/2, -1, -1/2 once at the write (scaling by a power of two
//    commutes with rounding, so each running sum is the old one scaled);
//  * the per-fragment warp reduction is deferred: lanes park their 9 values
//    in a ring of kRing fragments and one flush sums 9 * kRing columns, one
//    per lane, in the same order as warp_reduce9_smem ((0..10) + (11..21)) +
//    (22..31) — a third of the reduction instructions per fragment.
template <int WPB, int kMinB = 10>
__global__ void __launch_bounds__(32 * WPB, kMinB * 2 / WPB)
    k_raster_vjp_staged3(TileLists tl, const double* __restrict__ rec, int W, int H, RenderP ro,
                         const double* __restrict__ adj, const double* __restrict__ tfinal,
                         const int* __restrict__ last, double* __restrict__ part,
                         unsigned char* __restrict__ mask) {
    constexpr int SUB = 4 / WPB;
    constexpr int kRing = 3;  // 27 columns: one per lane
    __shared__ double s_ring[WPB][kRing * kAdj][kRedStride];
    __shared__ long long s_ring_out[WPB][kRing];
    __shared__ __align__(16) StagedRec s_rec[WPB][32];
    __shared__ int4 s_rect[WPB][32];
    __shared__ int s_pos[WPB][32];
    __shared__ int s_slot[WPB][32];
    const int tile =
        tl.order ? tl.order[blockIdx.x / SUB] : blockIdx.x / SUB + tl.row0 * tl.tiles_x;
    const int lane = threadIdx.x & 31, lw = threadIdx.x >> 5;
    const int warp = (blockIdx.x % SUB) * WPB + lw;
    const int bx0 = (tile % tl.tiles_x) * kTile + (warp & 1) * 8;
    const int by0 = (tile / tl.tiles_x) * kTile + (warp >> 1) * 8;
    const int px = bx0 + (lane & 7);
    const int py0 = by0 + (lane >> 3);
    const double pxc = px + 0.5;
    const double pyc[2] = {py0 + 0.5, py0 + 4.5};
    const int start = tl.tile_start[tile];
    const long long P = (long long)W * H;
    double u0[2], u1[2], u2[2], T[2], ub[2];
    int lastp[2];
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        const int py = py0 + 4 * k;
        u0[k] = u1[k] = u2[k] = T[k] = 0.0;
        lastp[k] = 0;
        if (px < W && py < H) {
            const long long p = (long long)py * W + px;
            u0[k] = adj[p];
            u1[k] = adj[P + p];
            u2[k] = adj[2 * P + p];
            T[k] = tfinal[p];
            lastp[k] = last[p];
            if (u0[k] == 0.0 && u1[k] == 0.0 && u2[k] == 0.0) lastp[k] = 0;  // render.cpp:283
        }
        ub[k] = T[k] * (u0[k] * ro.bg[0] + u1[k] * ro.bg[1] + u2[k] * ro.bg[2]);
    }
    const int wlast = __reduce_max_sync(kFull, max(lastp[0], lastp[1]));
    StagedRec* my_rec = s_rec[lw];
    int4* my_rect = s_rect[lw];
    int* my_pos = s_pos[lw];
    int* my_slot = s_slot[lw];
    double(*ring)[kRedStride] = s_ring[lw];
    long long* ring_out = s_ring_out[lw];
    int nring = 0;  // warp-uniform
    // sum the parked columns (lane = fragment * 9 + adjoint) and write them
    auto flush = [&](int n) {
        __syncwarp();
        if (lane < n * kAdj) {
            const double* col = ring[lane];
            double t0 = col[0], t1 = col[11], t2 = col[22];
#pragma unroll
            for (int k = 1; k < 11; ++k) {
                t0 += col[k];
                t1 += col[11 + k];
                if (k < 10) t2 += col[22 + k];
            }
            const int fe = lane / kAdj, c = lane - fe * kAdj;
            double v = (t0 + t1) + t2;
            if (c == 2 || c == 4) v *= -0.5;
            if (c == 3) v = -v;
            part[(ring_out[fe] * kVjpSlots + warp) * kAdj + c] = v;
        }
        __syncwarp();
    };
    for (int top = start + wlast; top > start; top -= 32) {
        const int base = max(start, top - 32);
        const int jj = base + lane;
        bool pass = false;
        int4 rr;
        if (jj < top) {
            rr = __ldg(tl.trect + jj);
            pass = !(bx0 + 7 < rr.x || bx0 > rr.z || by0 + 7 < rr.y || by0 > rr.w);
        }
        const unsigned m = __ballot_sync(kFull, pass);
        if (pass) {
            const int q = __popc(m & ((1u << lane) - 1u));
            const double2* r2 =
                reinterpret_cast<const double2*>(rec + (long long)kRec * __ldg(tl.tile_ids + jj));
            const double2 a = __ldg(r2 + 2), b = __ldg(r2 + 3), c = __ldg(r2 + 4);
            const double2 d = __ldg(r2 + 5), e = __ldg(r2 + 6);
            double2* o = reinterpret_cast<double2*>(my_rec + q);
            o[0] = a;
            o[1] = b;
            o[2] = c;
            o[3] = d;
            o[4] = e;
            my_rect[q] = rr;
            my_pos[q] = jj;
            my_slot[q] = __ldg(tl.sorted_d + jj);
        }
        __syncwarp();
        for (int e = __popc(m) - 1; e >= 0; --e) {
            const int rel = my_pos[e] - start;
            const int4 r4 = my_rect[e];
            const bool colin = px >= r4.x && px <= r4.z;
            bool lv[2];
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                const int py = py0 + 4 * k;
                lv[k] = rel < lastp[k] && colin && py >= r4.y && py <= r4.w;
            }
            const bool any0 = __any_sync(kFull, lv[0]), any1 = __any_sync(kFull, lv[1]);
            if (!any0 && !any1) continue;
            const StagedRec r = my_rec[e];
            double g[kAdj];
#pragma unroll
            for (int c = 0; c < kAdj; ++c) g[c] = 0.0;
            bool contrib = false;
            // one pixel's contribution given its falloff (render.cpp:238-283)
            auto accumulate = [&](int k, double dx, double dy, double ax, double ay, double gauss,
                                  double abar, bool clamped, double rom) {
                contrib = true;
                const double t_in = T[k] * rom;
                const double at = abar * t_in;
                g[6] += u0[k] * at;
                g[7] += u1[k] * at;
                g[8] += u2[k] * at;
                const double uc = u0[k] * r.c0 + u1[k] * r.c1 + u2[k] * r.c2;
                const double dab = uc * t_in - ub[k] * rom;
                ub[k] += uc * at;
                if (!clamped) {
                    g[5] += gauss * dab;
                    const double de = abar * dab;
                    g[2] += de * (dx * dx);  // x -1/2 at the write
                    g[3] += de * (dx * dy);  // x -1
                    g[4] += de * (dy * dy);  // x -1/2
                    g[0] += de * ax;
                    g[1] += de * ay;
                }
                T[k] = t_in;
            };
            const double f[13] = {0.0,   0.0,   0.0,     0.0,  r.mx, r.my, r.i00,
                                  r.i01, r.i11, r.alpha, r.c0, r.c1, r.c2};
            const double dx = pxc - r.mx;
            if (any0 && any1) {
                double dy[2], ax[2], ay[2], gauss[2], abar[2], rom[2];
                bool cl[2];
#pragma unroll
                for (int k = 0; k < 2; ++k) {
                    dy[k] = pyc[k] - r.my;
                    gauss[k] = fast_exp_neg(eval_expo(dx, dy[k], f, ax[k], ay[k]));
                    abar[k] = __dmul_rn(r.alpha, gauss[k]);
                    cl[k] = abar[k] >= ro.alpha_clamp;
                    if (cl[k]) abar[k] = ro.alpha_clamp;
                    lv[k] = lv[k] && !(abar[k] < ro.alpha_skip);
                    rom[k] = rcp_unit(__dsub_rn(1.0, abar[k]));
                }
#pragma unroll
                for (int k = 0; k < 2; ++k)
                    if (lv[k])
                        accumulate(k, dx, dy[k], ax[k], ay[k], gauss[k], abar[k], cl[k], rom[k]);
            } else {
#pragma unroll
                for (int k = 0; k < 2; ++k) {
                    if (!(k == 0 ? any0 : any1) || !lv[k]) continue;
                    const double dy = pyc[k] - r.my;
                    double ax, ay;
                    const double gauss = fast_exp_neg(eval_expo(dx, dy, f, ax, ay));
                    double abar = __dmul_rn(r.alpha, gauss);
                    const bool clamped = abar >= ro.alpha_clamp;
                    if (clamped) abar = ro.alpha_clamp;
                    if (abar < ro.alpha_skip) continue;
                    accumulate(k, dx, dy, ax, ay, gauss, abar, clamped,
                               rcp_unit(__dsub_rn(1.0, abar)));
                }
            }
            const unsigned cm = __ballot_sync(kFull, contrib);
            if (cm == 0u) continue;
#pragma unroll
            for (int c = 0; c < kAdj; ++c) ring[nring * kAdj + c][lane] = g[c];
            if (lane == 0) {
                const long long dslot = my_slot[e];
                ring_out[nring] = dslot;
                mask[dslot * kVjpSlots + warp] = 1;
            }
            if (++nring == kRing) {
                flush(kRing);
                nring = 0;
            }
        }
        __syncwarp();
    }
    if (nring) flush(nring);
}

// ------------------------------------------------------------------ K10, hit bitmasks
// k_raster_vjp_staged3 with the per-(entry, pixel) tests done as bit
// arithmetic (as k_raster_fwd_bits): the staging lane of list entry base + j
// turns its pixel rectangle into the 64-bit mask of the 8x8 block's pixels it
// covers; two warp bit-transposes give each lane the entries covering its two
// pixels, cut to the entries below each pixel's stored last index (one
// low-bits mask, render.cpp:238-257 walks [0, last)); an OR-reduction gives
// the entries the warp visits, back to front.  Records are staged at their
// list offset (no compaction), and the per-slot written-flag is set by the
// ring flush.  Per pixel and per partial the operations and their order are
// those of k_raster_vjp_staged3: the partials are bit-identical.
template <int WPB, int kMinB = 10>
__global__ void __launch_bounds__(32 * WPB, kMinB * 2 / WPB)
    k_raster_vjp_bits(TileLists tl, const double* __restrict__ rec, int W, int H, RenderP ro,
                      const double* __restrict__ adj, const double* __restrict__ tfinal,
                      const int* __restrict__ last, double* __restrict__ part,
                      unsigned char* __restrict__ mask) {
    constexpr int SUB = 4 / WPB;
    constexpr int kRing = 3;  // 27 columns: one per lane
    __shared__ double s_ring[WPB][kRing * kAdj][kRedStride];
    __shared__ long long s_ring_out[WPB][kRing];
    __shared__ __align__(16) StagedRec s_rec[WPB][32];
    __shared__ int s_slot[WPB][32];
    const int tile =
        tl.order ? tl.order[blockIdx.x / SUB] : blockIdx.x / SUB + tl.row0 * tl.tiles_x;
    const int lane = threadIdx.x & 31, lw = threadIdx.x >> 5;
    const int warp = (blockIdx.x % SUB) * WPB + lw;
    const int bx0 = (tile % tl.tiles_x) * kTile + (warp & 1) * 8;
    const int by0 = (tile / tl.tiles_x) * kTile + (warp >> 1) * 8;
    const int px = bx0 + (lane & 7);
    const int py0 = by0 + (lane >> 3);
    const double pxc = px + 0.5;
    const double pyc[2] = {py0 + 0.5, py0 + 4.5};
    const int start = tl.tile_start[tile];
    const long long P = (long long)W * H;
    double u0[2], u1[2], u2[2], T[2], ub[2];
    int lastp[2];
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        const int py = py0 + 4 * k;
        u0[k] = u1[k] = u2[k] = T[k] = 0.0;
        lastp[k] = 0;
        if (px < W && py < H) {
            const long long p = (long long)py * W + px;
            u0[k] = adj[p];
            u1[k] = adj[P + p];
            u2[k] = adj[2 * P + p];
            T[k] = tfinal[p];
            lastp[k] = last[p];
            if (u0[k] == 0.0 && u1[k] == 0.0 && u2[k] == 0.0) lastp[k] = 0;  // render.cpp:283
        }
        ub[k] = T[k] * (u0[k] * ro.bg[0] + u1[k] * ro.bg[1] + u2[k] * ro.bg[2]);
    }
    const int wlast = __reduce_max_sync(kFull, max(lastp[0], lastp[1]));
    StagedRec* my_rec = s_rec[lw];
    int* my_slot = s_slot[lw];
    double(*ring)[kRedStride] = s_ring[lw];
    long long* ring_out = s_ring_out[lw];
    int nring = 0;  // warp-uniform
    // sum the parked columns (lane = fragment * 9 + adjoint), write them and
    // flag the slots
    auto flush = [&](int n) {
        __syncwarp();
        if (lane < n * kAdj) {
            const double* col = ring[lane];
            double t0 = col[0], t1 = col[11], t2 = col[22];
#pragma unroll
            for (int k = 1; k < 11; ++k) {
                t0 += col[k];
                t1 += col[11 + k];
                if (k < 10) t2 += col[22 + k];
            }
            const int fe = lane / kAdj, c = lane - fe * kAdj;
            double v = (t0 + t1) + t2;
            if (c == 2 || c == 4) v *= -0.5;
            if (c == 3) v = -v;
            const long long slot = ring_out[fe] * kVjpSlots + warp;
            part[slot * kAdj + c] = v;
            if (c == 0) mask[slot] = 1;
        }
        __syncwarp();
    };
    for (int top = start + wlast; top > start; top -= 32) {
        const int base = max(start, top - 32);
        const int jj = base + lane;
        unsigned long long slots = 0ull;
        if (jj < top) {
            slots = block_slots(__ldg(tl.trect + jj), bx0, by0, 8);
            if (slots) {
                const double2* r2 = reinterpret_cast<const double2*>(
                    rec + (long long)kRec * __ldg(tl.tile_ids + jj));
                const double2 a = __ldg(r2 + 2), b = __ldg(r2 + 3), c = __ldg(r2 + 4);
                const double2 d = __ldg(r2 + 5), e = __ldg(r2 + 6);
                double2* o = reinterpret_cast<double2*>(my_rec + lane);
                o[0] = a;
                o[1] = b;
                o[2] = c;
                o[3] = d;
                o[4] = e;
                my_slot[lane] = __ldg(tl.sorted_d + jj);
            }
        }
        // bit j of m[k]: entry base + j covers pixel k and lies below its
        // stored last index
        unsigned m[2] = {warp_transpose32((unsigned)slots),
                         warp_transpose32((unsigned)(slots >> 32))};
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            const int lim = min(max(start + lastp[k] - base, 0), 32);
            m[k] &= lim >= 32 ? ~0u : ((1u << lim) - 1u);
        }
        const unsigned w0 = __reduce_or_sync(kFull, m[0]), w1 = __reduce_or_sync(kFull, m[1]);
        unsigned wb = w0 | w1;
        __syncwarp();
        while (wb) {
            const int e = 31 - __clz(wb);  // back to front
            wb &= ~(1u << e);
            const bool any0 = (w0 >> e) & 1u, any1 = (w1 >> e) & 1u;
            bool lv[2] = {(bool)((m[0] >> e) & 1u), (bool)((m[1] >> e) & 1u)};
            const StagedRec r = my_rec[e];
            double g[kAdj];
#pragma unroll
            for (int c = 0; c < kAdj; ++c) g[c] = 0.0;
            bool contrib = false;
            // one pixel's contribution given its falloff (render.cpp:238-283)
            auto accumulate = [&](int k, double dx, double dy, double ax, double ay, double gauss,
                                  double abar, bool clamped, double rom) {
                contrib = true;
                const double t_in = T[k] * rom;
                const double at = abar * t_in;
                g[6] += u0[k] * at;
                g[7] += u1[k] * at;
                g[8] += u2[k] * at;
                const double uc = u0[k] * r.c0 + u1[k] * r.c1 + u2[k] * r.c2;
                const double dab = uc * t_in - ub[k] * rom;
                ub[k] += uc * at;
                if (!clamped) {
                    g[5] += gauss * dab;
                    const double de = abar * dab;
                    g[2] += de * (dx * dx);  // x -1/2 at the write
                    g[3] += de * (dx * dy);  // x -1
                    g[4] += de * (dy * dy);  // x -1/2
                    g[0] += de * ax;
                    g[1] += de * ay;
                }
                T[k] = t_in;
            };
            const double f[13] = {0.0,   0.0,   0.0,     0.0,  r.mx, r.my, r.i00,
                                  r.i01, r.i11, r.alpha, r.c0, r.c1, r.c2};
            const double dx = pxc - r.mx;
            if (any0 && any1) {
                double dy[2], ax[2], ay[2], gauss[2], abar[2], rom[2];
                bool cl[2];
#pragma unroll
                for (int k = 0; k < 2; ++k) {
                    dy[k] = pyc[k] - r.my;
                    gauss[k] = fast_exp_neg(eval_expo(dx, dy[k], f, ax[k], ay[k]));
                    abar[k] = __dmul_rn(r.alpha, gauss[k]);
                    cl[k] = abar[k] >= ro.alpha_clamp;
                    if (cl[k]) abar[k] = ro.alpha_clamp;
                    lv[k] = lv[k] && !(abar[k] < ro.alpha_skip);
                    rom[k] = rcp_unit(__dsub_rn(1.0, abar[k]));
                }
#pragma unroll
                for (int k = 0; k < 2; ++k)
                    if (lv[k])
                        accumulate(k, dx, dy[k], ax[k], ay[k], gauss[k], abar[k], cl[k], rom[k]);
            } else {
#pragma unroll
                for (int k = 0; k < 2; ++k) {
                    if (!(k == 0 ? any0 : any1) || !lv[k]) continue;
                    const double dy = pyc[k] - r.my;
                    double ax, ay;
                    const double gauss = fast_exp_neg(eval_expo(dx, dy, f, ax, ay));
                    double abar = __dmul_rn(r.alpha, gauss);
                    const bool clamped = abar >= ro.alpha_clamp;
                    if (clamped) abar = ro.alpha_clamp;
                    if (abar < ro.alpha_skip) continue;
                    accumulate(k, dx, dy, ax, ay, gauss, abar, clamped,
                               rcp_unit(__dsub_rn(1.0, abar)));
                }
            }
            const unsigned cm = __ballot_sync(kFull, contrib);
            if (cm == 0u) continue;
#pragma unroll
            for (int c = 0; c < kAdj; ++c) ring[nring * kAdj + c][lane] = g[c];
            if (lane == 0) ring_out[nring] = my_slot[e];
            if (++nring == kRing) {
                flush(kRing);
                nring = 0;
            }
        }
        __syncwarp();
    }
    if (nring) flush(nring);
}

// ------------------------------------------------------------------ K12 (raster)
template <bool kWarpCull>
__global__ void __launch_bounds__(kThreads) k_raster_jvp(TileLists tl,
                                                         const double* __restrict__ rec,
                                                         const double* __restrict__ trec, int W,
                                                         int H, RenderP ro,
                                                         double* __restrict__ tangent) {
    __shared__ __align__(16) double s_rec[kJvpBatch * kRec];
    __shared__ __align__(16) double s_t[kJvpBatch * kTRec];
    const int tile = blockIdx.x + tl.row0 * tl.tiles_x;
    const PixelCtx pc = pixel_ctx(tile, tl.tiles_x, W, H);
    const int start = tl.tile_start[tile], end = tl.tile_end[tile];
    double T = 1.0, dT = 0.0;
    double d0 = 0.0, d1 = 0.0, d2 = 0.0;
    bool done = !pc.inside;
    for (int b = start; b < end; b += kJvpBatch) {
        if (__syncthreads_and(done)) break;
        const int n = min(kJvpBatch, end - b);
        stage_records(tl, rec, b, n, s_rec, nullptr);
        stage_tangents(tl, trec, b, n, s_t);
        __syncthreads();
        if (__all_sync(kFull, done)) continue;
        for (int jj = 0; jj < n; ++jj) {
            const double* f = s_rec + kRec * jj;
            if (warp_misses(pc, f) || (kWarpCull && !warp_may_hit(pc, f))) continue;
            if (!done && !outside_bbox(pc.pxc, pc.pyc, f)) {
                const double* t = s_t + kTRec * jj;
                const double dx = pc.pxc - f[R_MX], dy = pc.pyc - f[R_MY];
                const double e = fast_exp_neg(eval_expo(dx, dy, f));
                double abar = __dmul_rn(f[R_ALPHA], e);
                // tangent of the same expression (dual.hpp semantics)
                const Dual Dx(dx, -t[T_MX]), Dy(dy, -t[T_MY]);
                const Dual I00(f[R_I00], t[T_I00]), I01(f[R_I01], t[T_I01]),
                    I11(f[R_I11], t[T_I11]);
                const Dual ex = -0.5 * (Dx * Dx * I00 + Dy * Dy * I11) - Dx * Dy * I01;
                double dabar = t[T_ALPHA] * e + f[R_ALPHA] * (e * ex.d);
                if (abar >= ro.alpha_clamp) {
                    abar = ro.alpha_clamp;
                    dabar = 0.0;
                }
                if (!(abar < ro.alpha_skip)) {
                    // w = abar * T ; acc += c * w ; T = T * (1 - abar)
                    const double w = abar * T;
                    const double dw = dabar * T + abar * dT;
                    d0 += t[T_C0] * w + f[R_C0] * dw;
                    d1 += t[T_C1] * w + f[R_C1] * dw;
                    d2 += t[T_C2] * w + f[R_C2] * dw;
                    const double om = __dsub_rn(1.0, abar);
                    dT = dT * om + T * (-dabar);
                    T = __dmul_rn(T, om);
                    if (T < ro.t_stop) done = true;
                }
            }
            if (__all_sync(kFull, done)) break;
        }
    }
    if (!pc.inside) return;
    const long long P = (long long)W * H, p = (long long)pc.py * W + pc.px;
    tangent[p] = d0 + ro.bg[0] * dT;
    tangent[P + p] = d1 + ro.bg[1] * dT;
    tangent[2 * P + p] = d2 + ro.bg[2] * dT;
}

// ------------------------------------------------------------------ K12, batch-staged
// The tangent image with k_raster_fwd_staged's batches: the passing
// fragments' 9 raster fields and 9 tangent fields are fetched lane-parallel
// into warp-private shared slots, then blended in list order with the same
// per-pixel operations as k_raster_jvp.
struct StagedTan {
    double mx, my, i00, i01, i11, alpha, c0, c1, c2, pad;
};

template <int WPB>
__global__ void __launch_bounds__(32 * WPB)
    k_raster_jvp_staged(TileLists tl, const double* __restrict__ rec,
                        const double* __restrict__ trec, int W, int H, RenderP ro,
                        double* __restrict__ tangent) {
    constexpr int SUB = kWarps / WPB;
    __shared__ __align__(16) StagedRec s_rec[WPB][32];
    __shared__ __align__(16) StagedTan s_tan[WPB][32];
    __shared__ int4 s_rect[WPB][32];
    const int tile =
        tl.order ? tl.order[blockIdx.x / SUB] : blockIdx.x / SUB + tl.row0 * tl.tiles_x;
    const int lane = threadIdx.x & 31, lw = threadIdx.x >> 5;
    const int warp = (blockIdx.x % SUB) * WPB + lw;
    const PixelCtx pc = pixel_ctx(tile, tl.tiles_x, W, H, warp);
    const int start = tl.tile_start[tile], end = tl.tile_end[tile];
    double T = 1.0, dT = 0.0, d0 = 0.0, d1 = 0.0, d2 = 0.0;
    bool done = !pc.inside;
    StagedRec* my_rec = s_rec[lw];
    StagedTan* my_tan = s_tan[lw];
    int4* my_rect = s_rect[lw];
    for (int base = start; base < end; base += 32) {
        if (__all_sync(kFull, done)) break;
        const int jj = base + lane;
        bool pass = false;
        int4 rr;
        if (jj < end) {
            rr = __ldg(tl.trect + jj);
            pass = rect_hits_warp(pc, rr);
        }
        const unsigned m = __ballot_sync(kFull, pass);
        if (pass) {
            const int q = __popc(m & ((1u << lane) - 1u));
            const int id = __ldg(tl.tile_ids + jj);
            const double2* r2 = reinterpret_cast<const double2*>(rec + (long long)kRec * id);
            double2* o = reinterpret_cast<double2*>(my_rec + q);
#pragma unroll
            for (int k = 0; k < 5; ++k) o[k] = __ldg(r2 + 2 + k);
            const double* t = trec + (long long)kTRec * id;
            StagedTan& u = my_tan[q];
            u.mx = __ldg(t + T_MX);
            u.my = __ldg(t + T_MY);
            u.i00 = __ldg(t + T_I00);
            u.i01 = __ldg(t + T_I01);
            u.i11 = __ldg(t + T_I11);
            u.alpha = __ldg(t + T_ALPHA);
            u.c0 = __ldg(t + T_C0);
            u.c1 = __ldg(t + T_C0 + 1);
            u.c2 = __ldg(t + T_C0 + 2);
            my_rect[q] = rr;
        }
        __syncwarp();
        const int n = __popc(m);
        for (int e = 0; e < n; ++e) {
            if (!done && rect_has_pixel(pc, my_rect[e])) {
                const StagedRec r = my_rec[e];
                const StagedTan t = my_tan[e];
                const double f[13] = {0.0,   0.0,   0.0,     0.0,  r.mx, r.my, r.i00,
                                      r.i01, r.i11, r.alpha, r.c0, r.c1, r.c2};
                const double dx = pc.pxc - f[R_MX], dy = pc.pyc - f[R_MY];
                const double ev = fast_exp_neg(eval_expo(dx, dy, f));
                double abar = __dmul_rn(f[R_ALPHA], ev);
                // tangent of the same expression (dual.hpp semantics)
                const Dual Dx(dx, -t.mx), Dy(dy, -t.my);
                const Dual I00(f[R_I00], t.i00), I01(f[R_I01], t.i01), I11(f[R_I11], t.i11);
                const Dual ex = -0.5 * (Dx * Dx * I00 + Dy * Dy * I11) - Dx * Dy * I01;
                double dabar = t.alpha * ev + f[R_ALPHA] * (ev * ex.d);
                if (abar >= ro.alpha_clamp) {
                    abar = ro.alpha_clamp;
                    dabar = 0.0;
                }
                if (!(abar < ro.alpha_skip)) {
                    const double w = abar * T;
                    const double dw = dabar * T + abar * dT;
                    d0 += t.c0 * w + f[R_C0] * dw;
                    d1 += t.c1 * w + f[R_C1] * dw;
                    d2 += t.c2 * w + f[R_C2] * dw;
                    const double om = __dsub_rn(1.0, abar);
                    dT = dT * om + T * (-dabar);
                    T = __dmul_rn(T, om);
                    if (T < ro.t_stop) done = true;
                }
            }
            if (__all_sync(kFull, done)) break;
        }
        __syncwarp();
    }
    if (!pc.inside) return;
    const long long P = (long long)W * H, p = (long long)pc.py * W + pc.px;
    tangent[p] = d0 + ro.bg[0] * dT;
    tangent[P + p] = d1 + ro.bg[1] * dT;
    tangent[2 * P + p] = d2 + ro.bg[2] * dT;
}

// kernel-variant knobs (read once; tools/variants.sh runs the GPU suite under
// each): SGTR_FWD_WARP 4 = paired-entry K7 (default), 2 = one entry at a
// time, 0 = the CTA form; SGTR_VJP_MODE 1 = per-warp partials (default), 0 =
// the CTA slot form; SGTR_VJP_STAGED 3 = interleaved K10 with the ring
// reduction (default), 2 = a branch per pixel and a reduction per fragment;
// SGTR_VJP_MINBLOCKS the register budget (CTAs per SM) of those;
// SGTR_JVP_WARP 2 = batch-staged K12 (default), 0 = the CTA form;
// SGTR_WARP_CULL=1 the warp-level contribution filter of the CTA forms
int knob(const char* name, int dflt) {
    const char* v = getenv(name);
    return v ? atoi(v) : dflt;
}
const int g_warp_cull = knob("SGTR_WARP_CULL", 0);
const int g_vjp_mode = knob("SGTR_VJP_MODE", 1);
const int g_fwd_warp = knob("SGTR_FWD_WARP", 5);
const int g_vjp_staged = knob("SGTR_VJP_STAGED", 4);
const int g_vjp_min_blocks = knob("SGTR_VJP_MINBLOCKS", g_vjp_mode == 1 ? 10 : 3);
const int g_jvp_warp = knob("SGTR_JVP_WARP", 2);

}  // namespace

void launch_raster_fwd(cudaStream_t st, const TileLists& tl, const double* rec, int W, int H,
                       const RenderP& ro, double* img, double* tfinal, int* last,
                       unsigned long long* counters) {
    const int n = tl.tiles_x * (tl.row1 - tl.row0);
    if (n == 0) return;
    if (counters)
        k_raster_fwd<true, false><<<n, kThreads, 0, st>>>(tl, rec, W, H, ro, img, tfinal, last,
                                                          counters);
    else if (g_fwd_warp == 5)  // one-warp CTAs, hit bitmasks
        k_raster_fwd_bits<1><<<n * 8, 32, 0, st>>>(tl, rec, W, H, ro, img, tfinal, last);
    else if (g_fwd_warp == 4)  // one-warp CTAs: each retires as soon as its block is done
        k_raster_fwd_paired<1><<<n * 8, 32, 0, st>>>(tl, rec, W, H, ro, img, tfinal, last);
    else if (g_fwd_warp == 2)
        k_raster_fwd_staged<2><<<n * 4, 64, 0, st>>>(tl, rec, W, H, ro, img, tfinal, last);
    else if (g_warp_cull)
        k_raster_fwd<false, true><<<n, kThreads, 0, st>>>(tl, rec, W, H, ro, img, tfinal, last,
                                                          nullptr);
    else
        k_raster_fwd<false, false><<<n, kThreads, 0, st>>>(tl, rec, W, H, ro, img, tfinal,
                                                           last, nullptr);
    SGTR_CUDA(cudaGetLastError());
}

void launch_raster_vjp(cudaStream_t st, const TileLists& tl, const double* rec, int W, int H,
                       const RenderP& ro, const double* adj, const double* tfinal,
                       const int* last, double* slots) {
    const int n = tl.tiles_x * (tl.row1 - tl.row0);
    if (n == 0) return;
    if (g_warp_cull && g_vjp_min_blocks == 3)
        k_raster_vjp<true, 3><<<n, kThreads, 0, st>>>(tl, rec, W, H, ro, adj, tfinal, last, slots);
    else if (g_warp_cull)
        k_raster_vjp<true, 2><<<n, kThreads, 0, st>>>(tl, rec, W, H, ro, adj, tfinal, last, slots);
    else if (g_vjp_min_blocks == 3)
        k_raster_vjp<false, 3><<<n, kThreads, 0, st>>>(tl, rec, W, H, ro, adj, tfinal, last, slots);
    else
        k_raster_vjp<false, 2><<<n, kThreads, 0, st>>>(tl, rec, W, H, ro, adj, tfinal, last, slots);
    SGTR_CUDA(cudaGetLastError());
}

int vjp_mode() { return g_vjp_mode; }
int chain_mode() { return knob("SGTR_CHAIN_MODE", 0); }

void launch_raster_vjp_warp(cudaStream_t st, const TileLists& tl, const double* rec, int W,
                            int H, const RenderP& ro, const double* adj, const double* tfinal,
                            const int* last, double* part, unsigned char* mask) {
    const int n = tl.tiles_x * (tl.row1 - tl.row0);
    if (n == 0) return;
    if (g_vjp_staged == 2) {
        if (g_vjp_min_blocks == 8)
            k_raster_vjp_staged2<2, 8><<<n * 2, 64, 0, st>>>(tl, rec, W, H, ro, adj, tfinal, last,
                                                              part, mask);
        else
            k_raster_vjp_staged2<2><<<n * 2, 64, 0, st>>>(tl, rec, W, H, ro, adj, tfinal, last,
                                                          part, mask);
    } else if (g_vjp_staged == 4) {  // one-warp CTAs, hit bitmasks
        k_raster_vjp_bits<1><<<n * 4, 32, 0, st>>>(tl, rec, W, H, ro, adj, tfinal, last, part,
                                                   mask);
    } else if (g_vjp_min_blocks == 8) {
        k_raster_vjp_staged3<2, 8><<<n * 2, 64, 0, st>>>(tl, rec, W, H, ro, adj, tfinal, last,
                                                          part, mask);
    } else {  // one-warp CTAs, as K7
        k_raster_vjp_staged3<1><<<n * 4, 32, 0, st>>>(tl, rec, W, H, ro, adj, tfinal, last, part,
                                                      mask);
    }
    SGTR_CUDA(cudaGetLastError());
}

void launch_raster_jvp(cudaStream_t st, const TileLists& tl, const double* rec,
                       const double* trec, int W, int H, const RenderP& ro, double* tangent) {
    const int n = tl.tiles_x * (tl.row1 - tl.row0);
    if (n == 0) return;
    if (g_jvp_warp == 2)
        k_raster_jvp_staged<2><<<n * 4, 64, 0, st>>>(tl, rec, trec, W, H, ro, tangent);
    else if (g_warp_cull)
        k_raster_jvp<true><<<n, kThreads, 0, st>>>(tl, rec, trec, W, H, ro, tangent);
    else
        k_raster_jvp<false><<<n, kThreads, 0, st>>>(tl, rec, trec, W, H, ro, tangent);
    SGTR_CUDA(cudaGetLastError());
}

}  // namespace sgtr
