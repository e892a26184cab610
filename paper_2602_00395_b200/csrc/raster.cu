// raster.cu — tile rasteriser: K7 forward blend, K10 reverse-order VJP,
// K12 forward-mode JVP.
//
// Tiles are 16x16 pixels with per-tile fragment lists in depth order
// (binning.cu).  In K7 (two-warp CTAs) and K10 (one-warp CTAs) each warp owns
// one block of its tile (K7: 8x4 pixels, one per lane; K10: 16x8, four per
// lane) and walks the tile list on its own, 32 entries per batch: the lane
// of list entry base + j tests that entry's exact pixel rectangle (K1's
// pixel_range of the FP64 bbox) against the block as a bit mask of covered
// pixels, stages the fragment's raster fields into warp-private shared
// memory, and a warp bit-transpose hands every pixel lane the set of batch
// entries covering it.  In K7 every lane then walks its own entries (its
// pixel's blend state is private); K10 visits, warp-wide, the entries
// covering a pixel still in play (its per-fragment adjoints are reduced over
// the warp), reading each staged record as a broadcast.  K12 is K7's scheme
// with the tangent fields staged beside the raster ones.  k_raster_count is
// the one-thread-per-pixel CTA form kept for the E/C work counters.
//
// Branch parity: the three kernels evaluate the primal alpha with the same
// pinned operation sequence (eval_q's FMA form and fastexp.cuh's exp, a
// few ulp from the reference's own order), so bbox reject, alpha clamp,
// alpha skip and the transmittance stop take the same branches in forward,
// VJP and JVP — the reference's "frozen branches" contract
// (render.hpp:76-79).  The skip test is written as the reference's
// `alpha_bar < alpha_skip -> skip`, so a NaN alpha_bar is kept and
// propagates as it does in the reference (render.cpp:136).
#include <cstdlib>
#include <string>

#include "common.cuh"
#include "fastexp.cuh"
#include "geometry.cuh"
#include "launch.h"

namespace sgtr {
namespace {

constexpr int kThreads = kTilePixels;  // 256
constexpr int kFwdBatch = 256;
constexpr int kWarps = kThreads / 32;
constexpr unsigned kFull = 0xffffffffu;

struct PixelCtx {
    int px, py;
    bool inside;
    double pxc, pyc;
    double wx0, wx1, wy0, wy1;  // the warp's span of pixel centres
    int ix0, iy0;               // the warp's first pixel column / row
};

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

// reference: expo = -0.5 * (dx*dx*i00 + dy*dy*i11) - dx*dy*i01  (render.cpp:134-135)
// evaluated as expo = -0.5 q, q = dx ax + dy ay with (ax, ay) = Sigma^-1 d (4
// FMA-fused steps instead of 9 roundings; a few ulp from the reference's
// order, the same in every pass, so the clamp/skip/stop branches agree
// between passes), and exp(expo) as fast_exp_neg_half(q), bit-identical to
// fast_exp_neg(-0.5 q) without the multiply.  (ax, ay) is also the VJP's
// d expo / d mu2d up to sign.
__device__ __forceinline__ double eval_q(double dx, double dy, const double* f, double& ax,
                                         double& ay) {
    ax = __fma_rn(f[R_I01], dy, __dmul_rn(f[R_I00], dx));
    ay = __fma_rn(f[R_I11], dy, __dmul_rn(f[R_I01], dx));
    return __fma_rn(dy, ay, __dmul_rn(dx, ax));
}
__device__ __forceinline__ double falloff_of(double dx, double dy, const double* f, double& ax,
                                             double& ay) {
    return fast_exp_neg_half(eval_q(dx, dy, f, ax, ay));
}
__device__ __forceinline__ double falloff_of(double dx, double dy, const double* f) {
    double ax, ay;
    return falloff_of(dx, dy, f, ax, ay);
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

// ------------------------------------------------------------------ K7 counters
// The forward blend one CTA per tile (one thread per pixel), counting the
// (pixel, fragment) pairs reaching the alpha evaluation (E) and the
// contributing ones (C): the algorithmic-work units of SURVEY §8(d), for the
// bench's roofline; outside timed regions only.  Same per-pixel operations as
// k_raster_fwd_bits.
__global__ void __launch_bounds__(kThreads) k_raster_count(TileLists tl,
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
            if (warp_misses(pc, f)) continue;
            if (!done && !outside_bbox(pc.pxc, pc.pyc, f)) {
                const double dx = pc.pxc - f[R_MX], dy = pc.pyc - f[R_MY];
                double abar = __dmul_rn(f[R_ALPHA], falloff_of(dx, dy, f));
                ++n_eval;
                if (abar >= ro.alpha_clamp) abar = ro.alpha_clamp;
                if (!(abar < ro.alpha_skip)) {
                    ++n_contrib;
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
    for (int o = 16; o > 0; o >>= 1) {
        n_eval += __shfl_xor_sync(kFull, n_eval, o);
        n_contrib += __shfl_xor_sync(kFull, n_contrib, o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(counters, n_eval);
        atomicAdd(counters + 1, n_contrib);
    }
    if (!pc.inside) return;
    const long long P = (long long)W * H, p = (long long)pc.py * W + pc.px;
    img[p] = c0 + ro.bg[0] * T;
    img[P + p] = c1 + ro.bg[1] * T;
    img[2 * P + p] = c2 + ro.bg[2] * T;
    tfinal[p] = T;
    last[p] = processed;
}

// the raster fields K7/K10/K12 stage per fragment (record fields 4..13)
struct StagedRec {
    double mx, my, i00, i01, i11, alpha, c0, c1, c2, pad;
};

// ------------------------------------------------------------------ K7, hit bitmasks
// The per-pixel bbox test of every (entry, pixel) pair is done once per batch
// as bit arithmetic: the lane that stages list entry base + j turns its pixel
// rectangle into the 32-bit mask of the warp block's pixels it covers, and a
// warp bit-transpose gives every pixel lane the mask of the batch entries
// covering it -- no per-entry rectangle loads, compares or votes.  Each lane
// then walks its own mask (a pixel's blend state is its lane's alone), so a
// lane never evaluates an entry that misses its pixel.  Per pixel the
// entries, operations and their order are those of the round-1 kernel
// (k_raster_fwd_paired), so the image, T and the stop index are
// bit-identical to it.
// The record staging is software-pipelined: the next batch's rectangles are
// tested and its records copied into the other half of a double buffer with
// cp.async (LDGSTS) while the current batch blends (-4.5 % K7 against the
// synchronous staging, bit-identical).
template <int WPB>
__global__ void __launch_bounds__(32 * WPB)
    k_raster_fwd_bits(TileLists tl, const double* __restrict__ rec, int W, int H, RenderP ro,
                      double* __restrict__ img, double* __restrict__ tfinal,
                      int* __restrict__ last) {
    constexpr int SUB = kWarps / WPB;
    __shared__ __align__(16) StagedRec s_rec[WPB][2][32];
    const int tile =
        tl.order ? tl.order[blockIdx.x / SUB] : blockIdx.x / SUB + tl.row0 * tl.tiles_x;
    const int lane = threadIdx.x & 31, lw = threadIdx.x >> 5;
    const int warp = (blockIdx.x % SUB) * WPB + lw;
    const PixelCtx pc = pixel_ctx(tile, tl.tiles_x, W, H, warp);
    const int start = tl.tile_start[tile], end = tl.tile_end[tile];
    double T = 1.0, c0 = 0.0, c1 = 0.0, c2 = 0.0;
    bool done = !pc.inside;
    int processed = end - start;
    auto falloff = [&](const StagedRec& r) {
        const double f[13] = {0.0,   0.0,   0.0,   0.0,     r.mx, r.my, r.i00,
                              r.i01, r.i11, r.alpha, r.c0, r.c1, r.c2};
        const double dx = pc.pxc - r.mx, dy = pc.pyc - r.my;
        double abar = __dmul_rn(r.alpha, falloff_of(dx, dy, f));
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
    // stage batch `base` into buffer `buf`: test the rectangle, start the copy
    auto stage = [&](int base, int buf) -> unsigned {
        const int jj = base + lane;
        unsigned slots = 0;
        if (jj < end) {
            slots = (unsigned)block_slots(__ldg(tl.trect + jj), pc.ix0, pc.iy0, 4);
            if (slots) {
                const double* src = rec + (long long)kRec * __ldg(tl.tile_ids + jj) + 4;
                double* dst = reinterpret_cast<double*>(&s_rec[lw][buf][lane]);
#pragma unroll
                for (int q = 0; q < 5; ++q) cp_async16(dst + 2 * q, src + 2 * q);
            }
        }
        cp_async_commit();
        return slots;
    };
    int buf = 0;
    unsigned slots_cur = start < end ? stage(start, 0) : 0u;
    for (int base = start; base < end; base += 32) {
        if (__all_sync(kFull, done)) break;
        // the next batch's copies overlap this batch's blending
        const unsigned slots_next = base + 32 < end ? stage(base + 32, buf ^ 1) : (cp_async_commit(), 0u);
        unsigned mine = warp_transpose32(slots_cur);  // bit j: entry base + j covers my pixel
        if (done) mine = 0u;
        cp_async_wait<1>();
        __syncwarp();
        const StagedRec* my_rec = s_rec[lw][buf];
        // every lane walks its own entries in list order, one per round: the
        // warp runs as many rounds as its busiest pixel needs, not one per
        // entry any pixel needs, and no lane evaluates an entry that misses
        // its pixel (the per-lane walks are the parallelism; two entries per
        // round, for two exp chains per lane, measured 2.4 % slower)
        while (__any_sync(kFull, mine != 0u)) {
            const bool has = mine != 0u;
            const int j = has ? __ffs(mine) - 1 : 0;
            mine &= mine - 1u;
            const StagedRec r = my_rec[j];
            const double ab = falloff(r);
            if (has && !(ab < ro.alpha_skip)) blend(r, ab, base + j);
            if (done) mine = 0u;
        }
        __syncwarp();
        slots_cur = slots_next;
        buf ^= 1;
    }
    cp_async_wait<0>();
    if (!pc.inside) return;
    const long long P = (long long)W * H, p = (long long)pc.py * W + pc.px;
    img[p] = c0 + ro.bg[0] * T;
    img[P + p] = c1 + ro.bg[1] * T;
    img[2 * P + p] = c2 + ro.bg[2] * T;
    tfinal[p] = T;
    last[p] = processed;
}

constexpr int kRedStride = 33;

// ------------------------------------------------------------------ K10, 8x8 blocks
// (Small images, whose 16x8 grid would leave SMs idle: see launch_raster_vjp_warp.)
// One warp per 8x8 block of a tile, two pixels per lane (rows r and r + 4),
// back to front from each pixel's stored last index (render.cpp:238-257
// walks [0, last)), with the per-(entry, pixel) tests done as bit arithmetic
// (as in K7): the staging lane of list entry base + j turns its pixel
// rectangle into the 64-bit mask of the block's pixels it covers; two warp
// bit-transposes give each lane the entries covering its two pixels, cut to
// the entries below each pixel's last index (one low-bits mask); an
// OR-reduction gives the entries the warp visits.  Each visited fragment's 9
// adjoints are reduced over the warp (the ring below) into one partial per
// (duplicate, block), flagged in mask.  Records are staged at their list
// offset (no compaction); the staging is double-buffered with cp.async as in
// K7.  Per pixel and per partial the operations and their order are those of
// the round-1 kernel (k_raster_vjp_staged3): the partials are bit-identical
// to it.
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
    __shared__ __align__(16) StagedRec s_rec[WPB][2][32];
    __shared__ int s_slot[WPB][2][32];
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
            const long long slot = ring_out[fe] * 4 + warp;  // four 8x8 blocks per tile
            part[slot * kPartStride + c] = v;
            if (c == 0) mask[slot] = 1;
        }
        __syncwarp();
    };
    // stage the batch [base, top) into buffer `buf`: test the rectangles, start
    // the record copies
    auto stage = [&](int top, int buf) -> unsigned long long {
        const int base = max(start, top - 32);
        const int jj = base + lane;
        unsigned long long slots = 0ull;
        if (jj < top) {
            slots = block_slots(__ldg(tl.trect + jj), bx0, by0, 8);
            if (slots) {
                const double* src = rec + (long long)kRec * __ldg(tl.tile_ids + jj) + 4;
                double* dst = reinterpret_cast<double*>(&s_rec[lw][buf][lane]);
#pragma unroll
                for (int q = 0; q < 5; ++q) cp_async16(dst + 2 * q, src + 2 * q);
                s_slot[lw][buf][lane] = __ldg(tl.sorted_d + jj);
            }
        }
        cp_async_commit();
        return slots;
    };
    int buf = 0;
    unsigned long long slots_cur = wlast > 0 ? stage(start + wlast, 0) : 0ull;
    for (int top = start + wlast; top > start; top -= 32) {
        const int base = max(start, top - 32);
        // the next (nearer) batch's copies overlap this batch's sweep
        const unsigned long long slots = slots_cur;
        slots_cur = base > start ? stage(base, buf ^ 1) : (cp_async_commit(), 0ull);
        const StagedRec* my_rec = s_rec[lw][buf];
        const int* my_slot = s_slot[lw][buf];
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
        cp_async_wait<1>();
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
            auto accumulate = [&](int k, double dx, double dxx, double dy, double ax, double ay,
                                  double gauss, double abar, bool clamped, double rom) {
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
                    g[2] += de * dxx;  // (dx dx) x -1/2 at the write
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
            const double dxx = dx * dx;  // shared by the lane's two pixels (one column)
            if (any0 && any1) {
                double dy[2], ax[2], ay[2], gauss[2], abar[2], rom[2];
                bool cl[2];
#pragma unroll
                for (int k = 0; k < 2; ++k) {
                    dy[k] = pyc[k] - r.my;
                    gauss[k] = falloff_of(dx, dy[k], f, ax[k], ay[k]);
                    abar[k] = __dmul_rn(r.alpha, gauss[k]);
                    cl[k] = abar[k] >= ro.alpha_clamp;
                    if (cl[k]) abar[k] = ro.alpha_clamp;
                    lv[k] = lv[k] && !(abar[k] < ro.alpha_skip);
                    rom[k] = rcp_unit(__dsub_rn(1.0, abar[k]));
                }
#pragma unroll
                for (int k = 0; k < 2; ++k)
                    if (lv[k])
                        accumulate(k, dx, dxx, dy[k], ax[k], ay[k], gauss[k], abar[k], cl[k],
                                   rom[k]);
            } else {
#pragma unroll
                for (int k = 0; k < 2; ++k) {
                    if (!(k == 0 ? any0 : any1) || !lv[k]) continue;
                    const double dy = pyc[k] - r.my;
                    double ax, ay;
                    const double gauss = falloff_of(dx, dy, f, ax, ay);
                    double abar = __dmul_rn(r.alpha, gauss);
                    const bool clamped = abar >= ro.alpha_clamp;
                    if (clamped) abar = ro.alpha_clamp;
                    if (abar < ro.alpha_skip) continue;
                    accumulate(k, dx, dxx, dy, ax, ay, gauss, abar, clamped,
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
        buf ^= 1;
    }
    cp_async_wait<0>();
    if (nring) flush(nring);
}

// ------------------------------------------------------------------ K10, hit bitmasks
// One warp per 16x8 block, two per tile, four pixels per lane (columns c and
// c + 8, rows r and r + 4), back to front from each pixel's stored last
// index (render.cpp:238-257 walks [0, last)), with the per-(entry, pixel)
// tests done as bit arithmetic (as in K7): the staging lane of list entry
// base + j turns its pixel rectangle into the 64-bit masks of the block's two
// 8x8 halves; four warp bit-transposes give each lane the entries covering
// its four pixels, cut to the entries below each pixel's last index (one
// low-bits mask); an OR-reduction gives the entries the warp visits.  Per
// visited fragment each 8-column half runs a pixel-pair body (skipped,
// warp-uniformly, when no lane's pixel in the half takes the fragment; both
// pixels in one straight-line block when both rows do), and the fragment's
// 9 adjoints, summed over a lane's pixels in (half, row) order, are reduced
// over the warp (the ring) into one partial per (duplicate, block), flagged
// in mask.  One list walk, record load, ring store and flush per fragment
// serve 128 pixels, and a duplicate has two partials (K11 reads half of what
// 8x8 blocks wrote: -27 % K11 for +2 % K10).  Records are staged at their
// list offset; the staging is double-buffered with cp.async as in K7.
template <int kMinB>
__global__ void __launch_bounds__(32, kMinB)
    k_raster_vjp_wide(TileLists tl, const double* __restrict__ rec, int W, int H, RenderP ro,
                      const double* __restrict__ adj, const double* __restrict__ tfinal,
                      const int* __restrict__ last, double* __restrict__ part,
                      unsigned char* __restrict__ mask) {
    constexpr int kRing = 3;  // 27 columns: one per lane
    __shared__ double s_ring[kRing * kAdj][kRedStride];
    __shared__ long long s_ring_out[kRing];
    __shared__ __align__(16) StagedRec s_rec[2][32];
    __shared__ int s_slot[2][32];
    const int tile = tl.order ? tl.order[blockIdx.x >> 1] : (blockIdx.x >> 1) + tl.row0 * tl.tiles_x;
    const int lane = threadIdx.x & 31;
    const int warp = blockIdx.x & 1;  // the tile's upper or lower 16x8 block
    const int bx0 = (tile % tl.tiles_x) * kTile;
    const int by0 = (tile / tl.tiles_x) * kTile + warp * 8;
    const int px0 = bx0 + (lane & 7);
    const int py0 = by0 + (lane >> 3);
    const double pxc[2] = {px0 + 0.5, px0 + 8.5};
    const double pyc[2] = {py0 + 0.5, py0 + 4.5};
    const int start = tl.tile_start[tile];
    const long long P = (long long)W * H;
    // pixel q = 2 h + k: column half h, row k
    double u0[4], u1[4], u2[4], T[4], ub[4];
    int lastp[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int px = px0 + 8 * (q >> 1), py = py0 + 4 * (q & 1);
        u0[q] = u1[q] = u2[q] = T[q] = 0.0;
        lastp[q] = 0;
        if (px < W && py < H) {
            const long long p = (long long)py * W + px;
            u0[q] = adj[p];
            u1[q] = adj[P + p];
            u2[q] = adj[2 * P + p];
            T[q] = tfinal[p];
            lastp[q] = last[p];
            if (u0[q] == 0.0 && u1[q] == 0.0 && u2[q] == 0.0) lastp[q] = 0;  // render.cpp:283
        }
        ub[q] = T[q] * (u0[q] * ro.bg[0] + u1[q] * ro.bg[1] + u2[q] * ro.bg[2]);
    }
    const int wlast =
        __reduce_max_sync(kFull, max(max(lastp[0], lastp[1]), max(lastp[2], lastp[3])));
    int nring = 0;  // warp-uniform
    auto flush = [&](int n) {
        __syncwarp();
        if (lane < n * kAdj) {
            const double* col = s_ring[lane];
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
            const long long slot = s_ring_out[fe] * 2 + warp;  // two 16x8 blocks per tile
            part[slot * kPartStride + c] = v;
            if (c == 0) mask[slot] = 1;
        }
        __syncwarp();
    };
    auto stage = [&](int top, int buf, unsigned long long& sl, unsigned long long& sr) {
        const int base = max(start, top - 32);
        const int jj = base + lane;
        sl = sr = 0ull;
        if (jj < top) {
            const int4 rr = __ldg(tl.trect + jj);
            sl = block_slots(rr, bx0, by0, 8);
            sr = block_slots(rr, bx0 + 8, by0, 8);
            if (sl | sr) {
                const double* src = rec + (long long)kRec * __ldg(tl.tile_ids + jj) + 4;
                double* dst = reinterpret_cast<double*>(&s_rec[buf][lane]);
#pragma unroll
                for (int q = 0; q < 5; ++q) cp_async16(dst + 2 * q, src + 2 * q);
                s_slot[buf][lane] = __ldg(tl.sorted_d + jj);
            }
        }
        cp_async_commit();
    };
    int buf = 0;
    unsigned long long cl_cur = 0ull, cr_cur = 0ull;
    if (wlast > 0) stage(start + wlast, 0, cl_cur, cr_cur);
    for (int top = start + wlast; top > start; top -= 32) {
        const int base = max(start, top - 32);
        const unsigned long long sl = cl_cur, sr = cr_cur;
        if (base > start)
            stage(base, buf ^ 1, cl_cur, cr_cur);
        else
            cp_async_commit();
        const StagedRec* my_rec = s_rec[buf];
        const int* my_slot = s_slot[buf];
        // bit j of m[q]: entry base + j covers pixel q and lies below its
        // stored last index
        unsigned m[4] = {warp_transpose32((unsigned)sl), warp_transpose32((unsigned)(sl >> 32)),
                         warp_transpose32((unsigned)sr), warp_transpose32((unsigned)(sr >> 32))};
        unsigned w[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int lim = min(max(start + lastp[q] - base, 0), 32);
            m[q] &= lim >= 32 ? ~0u : ((1u << lim) - 1u);
            w[q] = __reduce_or_sync(kFull, m[q]);
        }
        unsigned wb = (w[0] | w[1]) | (w[2] | w[3]);
        cp_async_wait<1>();
        __syncwarp();
        while (wb) {
            const int e = 31 - __clz(wb);  // back to front
            wb &= ~(1u << e);
            const StagedRec r = my_rec[e];
            double g[kAdj];
#pragma unroll
            for (int c = 0; c < kAdj; ++c) g[c] = 0.0;
            bool contrib = false;
            // one pixel's contribution given its falloff (render.cpp:238-283)
            auto accumulate = [&](int q, double dx, double dxx, double dy, double ax, double ay,
                                  double gauss, double abar, bool clamped, double rom) {
                contrib = true;
                const double t_in = T[q] * rom;
                const double at = abar * t_in;
                g[6] += u0[q] * at;
                g[7] += u1[q] * at;
                g[8] += u2[q] * at;
                const double uc = u0[q] * r.c0 + u1[q] * r.c1 + u2[q] * r.c2;
                const double dab = uc * t_in - ub[q] * rom;
                ub[q] += uc * at;
                if (!clamped) {
                    g[5] += gauss * dab;
                    const double de = abar * dab;
                    g[2] += de * dxx;  // (dx dx) x -1/2 at the write
                    g[3] += de * (dx * dy);  // x -1
                    g[4] += de * (dy * dy);  // x -1/2
                    g[0] += de * ax;
                    g[1] += de * ay;
                }
                T[q] = t_in;
            };
            const double f[13] = {0.0,   0.0,   0.0,     0.0,  r.mx, r.my, r.i00,
                                  r.i01, r.i11, r.alpha, r.c0, r.c1, r.c2};
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const bool any0 = (w[2 * h] >> e) & 1u, any1 = (w[2 * h + 1] >> e) & 1u;
                if (!any0 && !any1) continue;  // warp-uniform
                bool lv[2] = {(bool)((m[2 * h] >> e) & 1u), (bool)((m[2 * h + 1] >> e) & 1u)};
                const double dx = pxc[h] - r.mx;
                const double dxx = dx * dx;  // shared by the half's two pixels (one column)
                if (any0 && any1) {
                    double dy[2], ax[2], ay[2], gauss[2], abar[2], rom[2];
                    bool cl[2];
#pragma unroll
                    for (int k = 0; k < 2; ++k) {
                        dy[k] = pyc[k] - r.my;
                        gauss[k] = falloff_of(dx, dy[k], f, ax[k], ay[k]);
                        abar[k] = __dmul_rn(r.alpha, gauss[k]);
                        cl[k] = abar[k] >= ro.alpha_clamp;
                        if (cl[k]) abar[k] = ro.alpha_clamp;
                        lv[k] = lv[k] && !(abar[k] < ro.alpha_skip);
                        rom[k] = rcp_unit(__dsub_rn(1.0, abar[k]));
                    }
#pragma unroll
                    for (int k = 0; k < 2; ++k)
                        if (lv[k])
                            accumulate(2 * h + k, dx, dxx, dy[k], ax[k], ay[k], gauss[k], abar[k],
                                       cl[k], rom[k]);
                } else {
#pragma unroll
                    for (int k = 0; k < 2; ++k) {
                        if (!(k == 0 ? any0 : any1) || !lv[k]) continue;
                        const double dy = pyc[k] - r.my;
                        double ax, ay;
                        const double gauss = falloff_of(dx, dy, f, ax, ay);
                        double abar = __dmul_rn(r.alpha, gauss);
                        const bool clamped = abar >= ro.alpha_clamp;
                        if (clamped) abar = ro.alpha_clamp;
                        if (abar < ro.alpha_skip) continue;
                        accumulate(2 * h + k, dx, dxx, dy, ax, ay, gauss, abar, clamped,
                                   rcp_unit(__dsub_rn(1.0, abar)));
                    }
                }
            }
            const unsigned cm = __ballot_sync(kFull, contrib);
            if (cm == 0u) continue;
#pragma unroll
            for (int c = 0; c < kAdj; ++c) s_ring[nring * kAdj + c][lane] = g[c];
            if (lane == 0) s_ring_out[nring] = my_slot[e];
            if (++nring == kRing) {
                flush(kRing);
                nring = 0;
            }
        }
        __syncwarp();
        buf ^= 1;
    }
    cp_async_wait<0>();
    if (nring) flush(nring);
}

// ------------------------------------------------------------------ K12, hit bitmasks
// K12, the tangent image (render.cpp:175-192, blend_pixel<Dual>): K7's
// per-batch bit masks (8x4 blocks, one pixel per lane) and per-lane walk in
// list order, with each staged entry's 9 tangent fields beside its raster
// fields.  Per pixel the operations and their order are those of the round-1
// kernel (k_raster_jvp_staged), so the tangent image is bit-identical to it.
struct StagedTan {
    double mx, my, i00, i01, i11, alpha, c0, c1, c2, pad;  // tangent record fields 0..9
};

template <int WPB>
__global__ void __launch_bounds__(32 * WPB)
    k_raster_jvp_bits(TileLists tl, const double* __restrict__ rec,
                      const double* __restrict__ trec, int W, int H, RenderP ro,
                      double* __restrict__ tangent) {
    constexpr int SUB = kWarps / WPB;
    __shared__ __align__(16) StagedRec s_rec[WPB][32];
    __shared__ __align__(16) StagedTan s_tan[WPB][32];
    const int tile =
        tl.order ? tl.order[blockIdx.x / SUB] : blockIdx.x / SUB + tl.row0 * tl.tiles_x;
    const int lane = threadIdx.x & 31, lw = threadIdx.x >> 5;
    const int warp = (blockIdx.x % SUB) * WPB + lw;
    const PixelCtx pc = pixel_ctx(tile, tl.tiles_x, W, H, warp);
    const int start = tl.tile_start[tile], end = tl.tile_end[tile];
    double T = 1.0, dT = 0.0, d0 = 0.0, d1 = 0.0, d2 = 0.0;
    bool done = !pc.inside;
    const StagedRec* my_rec = s_rec[lw];
    const StagedTan* my_tan = s_tan[lw];
    for (int base = start; base < end; base += 32) {
        if (__all_sync(kFull, done)) break;
        const int jj = base + lane;
        unsigned slots = 0u;
        if (jj < end) {
            slots = (unsigned)block_slots(__ldg(tl.trect + jj), pc.ix0, pc.iy0, 4);
            if (slots) {
                const int id = __ldg(tl.tile_ids + jj);
                const double* src = rec + (long long)kRec * id + 4;
                double* dst = reinterpret_cast<double*>(&s_rec[lw][lane]);
                const double* tsrc = trec + (long long)kTRec * id;
                double* tdst = reinterpret_cast<double*>(&s_tan[lw][lane]);
#pragma unroll
                for (int q = 0; q < 5; ++q) {
                    cp_async16(dst + 2 * q, src + 2 * q);
                    cp_async16(tdst + 2 * q, tsrc + 2 * q);
                }
            }
        }
        cp_async_commit();
        unsigned mine = warp_transpose32(slots);  // bit j: entry base + j covers my pixel
        if (done) mine = 0u;
        cp_async_wait<0>();
        __syncwarp();
        while (__any_sync(kFull, mine != 0u)) {
            const bool has = mine != 0u;
            const int e = has ? __ffs(mine) - 1 : 0;
            mine &= mine - 1u;
            const StagedRec r = my_rec[e];
            const StagedTan t = my_tan[e];
            const double f[13] = {0.0,   0.0,   0.0,     0.0,  r.mx, r.my, r.i00,
                                  r.i01, r.i11, r.alpha, r.c0, r.c1, r.c2};
            const double dx = pc.pxc - f[R_MX], dy = pc.pyc - f[R_MY];
            const double ev = falloff_of(dx, dy, f);
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
            if (has && !(abar < ro.alpha_skip)) {
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
            if (done) mine = 0u;
        }
        __syncwarp();
    }
    if (!pc.inside) return;
    const long long P = (long long)W * H, p = (long long)pc.py * W + pc.px;
    tangent[p] = d0 + ro.bg[0] * dT;
    tangent[P + p] = d1 + ro.bg[1] * dT;
    tangent[2 * P + p] = d2 + ro.bg[2] * dT;
}

}  // namespace

void launch_raster_fwd(cudaStream_t st, const TileLists& tl, const double* rec, int W, int H,
                       const RenderP& ro, double* img, double* tfinal, int* last,
                       unsigned long long* counters) {
    const int n = tl.tiles_x * (tl.row1 - tl.row0);
    if (n == 0) return;
    if (counters)  // the E / C work counters (outside timed regions)
        k_raster_count<<<n, kThreads, 0, st>>>(tl, rec, W, H, ro, img, tfinal, last, counters);
    else  // two-warp CTAs (35 resident warps per SM at 58 registers, where the 32-CTA
          // limit capped one-warp CTAs at 32: -1.3 % against one warp, 4 warps +0.6 %)
        k_raster_fwd_bits<2><<<n * 4, 64, 0, st>>>(tl, rec, W, H, ro, img, tfinal, last);
    SGTR_CUDA(cudaGetLastError());
}

// SGTR_VJP_BLOCK=16x8 / 8x8 forces the block shape (tests run the parity
// suite on both; results agree to rounding, not bit for bit: the adjoints
// are summed over different pixel groups)
int vjp_slots(int n_tiles) {
    static const int forced = [] {
        const char* v = getenv("SGTR_VJP_BLOCK");
        if (!v) return 0;
        return std::string(v) == "16x8" ? 2 : std::string(v) == "8x8" ? 4 : 0;
    }();
    if (forced) return forced;
    return n_tiles >= kWideVjpTiles ? 2 : 4;
}

void launch_raster_vjp_warp(cudaStream_t st, const TileLists& tl, const double* rec, int W,
                            int H, const RenderP& ro, const double* adj, const double* tfinal,
                            const int* last, double* part, unsigned char* mask) {
    const int n = tl.tiles_x * (tl.row1 - tl.row0);
    if (n == 0) return;
    // 16x8 blocks (128 registers, 16 one-warp CTAs per SM) when the image has
    // tiles enough to fill the GPU with them, else 8x8 blocks (twice the CTAs)
    if (vjp_slots(n) == 2)
        k_raster_vjp_wide<16><<<n * 2, 32, 0, st>>>(tl, rec, W, H, ro, adj, tfinal, last, part,
                                                     mask);
    else
        k_raster_vjp_bits<1><<<n * 4, 32, 0, st>>>(tl, rec, W, H, ro, adj, tfinal, last, part,
                                                    mask);
    SGTR_CUDA(cudaGetLastError());
}

void launch_raster_jvp(cudaStream_t st, const TileLists& tl, const double* rec,
                       const double* trec, int W, int H, const RenderP& ro, double* tangent) {
    const int n = tl.tiles_x * (tl.row1 - tl.row0);
    if (n == 0) return;
    k_raster_jvp_bits<2><<<n * 4, 64, 0, st>>>(tl, rec, trec, W, H, ro, tangent);
    SGTR_CUDA(cudaGetLastError());
}

}  // namespace sgtr
