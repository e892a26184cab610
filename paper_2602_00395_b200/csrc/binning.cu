// binning.cu — K2 depth sort, K3 tile-count scan, K4 duplicate emission,
// K5 stable tile sort, K6 tile ranges.
//
// Integer work, bit-exact against the oracle's restated binning: the depth
// keys are an order-preserving map of the FP64 depths (ties broken by the
// splat index because the radix sort is stable over index-ordered input,
// render.cpp:83-87), and duplicates are emitted in depth-rank order so the
// stable sort on the tile id alone leaves every tile list in (depth, index)
// order.
//
// No size is read back on the host: the duplicate arrays have a capacity
// `cap`, entries [n_dup, cap) carry a sentinel tile key that sorts last, and
// a view whose n_dup exceeds cap is binned as empty and reports it (the step
// reruns with a larger capacity, api.cu step_core).
#include <climits>

#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>
#include <thrust/iterator/transform_iterator.h>

#include "common.cuh"
#include "geometry.cuh"
#include "launch.h"

namespace sgtr {
namespace {

// K2 sorts the FP32-rounded depths (a monotone map, so the order only
// coarsens): 32-bit keys, 4 onesweep passes.  Splats whose FP32 depths
// agree keep their input (= splat index) order; each such run is put into
// (full 64-bit key, index) order here by a stable insertion sort on the full
// keys -- the same (depth, index) order as a full 64-bit sort
// (render.cpp:83-87).  Runs are rare and short: FP32 resolves 2^-24 relative
// depth.  The culled splats (key 0xffffffff, no tiles) stay in index order.
__global__ void k_fix_depth_ties(const unsigned int* __restrict__ k32,
                                 const unsigned long long* __restrict__ k64,
                                 int* __restrict__ ids, int K) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= K) return;
    const unsigned int hi = k32[i];
    if (hi == 0xffffffffu) return;
    if (i > 0 && k32[i - 1] == hi) return;  // not a run start
    int e = i + 1;
    while (e < K && k32[e] == hi) ++e;
    for (int a = i + 1; a < e; ++a) {
        const int id = ids[a];
        const unsigned long long k = k64[id];
        int b = a - 1;
        while (b >= i && k64[ids[b]] > k) {
            ids[b + 1] = ids[b];
            --b;
        }
        ids[b + 1] = id;
    }
}

// K3's input: the tile count of the splat at depth rank r (0 at r = K), read
// through the scan's input iterator
struct CountAtRank {
    const int* ids;
    const int* tcount;
    int K;
    __host__ __device__ long long operator()(int r) const {
        return r < K ? (long long)tcount[ids[r]] : 0LL;
    }
};
using CountIter = thrust::transform_iterator<CountAtRank, thrust::counting_iterator<int>>;
CountIter count_iter(const int* ids, const int* tcount, int K) {
    return thrust::make_transform_iterator(thrust::make_counting_iterator(0),
                                           CountAtRank{ids, tcount, K});
}

// K4a: one thread per depth rank (n_visible = K: the culled splats sort last
// with no tiles).  Rectangles of <= 64 tiles are emitted from the hit bits K1
// recorded, in row-major tile order; larger ones are queued for K4b.
__global__ void __launch_bounds__(256) k_emit_small(const int* __restrict__ sorted_ids,
                                                    const int4* __restrict__ tinfo,
                                                    const long long* __restrict__ off_r,
                                                    int n_visible, int tiles_x, long long cap,
                                                    long long* __restrict__ off_id,
                                                    unsigned int* __restrict__ tkeys,
                                                    int* __restrict__ dval,
                                                    int* __restrict__ dup_id,
                                                    int* __restrict__ large,
                                                    int* __restrict__ n_large) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n_visible) return;
    const int id = sorted_ids[r];
    long long d = off_r[r];
    off_id[id] = d;  // K11 finds a splat's partials by id
    // the splat's tile count is the scan's step (read in rank order); its
    // rectangle and hit bits are one 16-byte gather by id (at C5 the
    // per-splat arrays are DRAM-resident, so one sector instead of three)
    if (off_r[n_visible] > cap || off_r[r + 1] == d) return;
    const int4 ti = tinfo[id];
    const int tx0 = ti.x & 0xffff, ty0 = (unsigned)ti.x >> 16;
    const int w = ti.y & 0xffff, h = (unsigned)ti.y >> 16;
    if (w * h > 64) {
        large[atomicAdd(n_large, 1)] = r;
        return;
    }
    unsigned long long bits = ((unsigned long long)(unsigned)ti.w << 32) | (unsigned)ti.z;
    while (bits) {
        const int j = __ffsll((long long)bits) - 1;
        bits &= bits - 1ull;
        tkeys[d] = (unsigned int)((ty0 + j / w) * tiles_x + tx0 + j % w);
        dval[d] = (int)d;
        dup_id[d] = id;
        ++d;
    }
}

// K4b: one warp per queued large rectangle: lanes re-evaluate ellipse_may_hit
// (the K1 test) per tile and write the hits compacted in row-major order
__global__ void __launch_bounds__(256) k_emit_large(const int* __restrict__ sorted_ids,
                                                    const int4* __restrict__ rect,
                                                    const double* __restrict__ rec,
                                                    const long long* __restrict__ off_r,
                                                    int tiles_x, const int* __restrict__ large,
                                                    const int* __restrict__ n_large,
                                                    unsigned int* __restrict__ tkeys,
                                                    int* __restrict__ dval,
                                                    int* __restrict__ dup_id) {
    const int lane = threadIdx.x & 31;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    for (int q = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; q < *n_large; q += nw) {
        const int r = large[q];
        const int id = sorted_ids[r];
        const int4 pr = rect[id];
        const double* f = rec + (long long)kRec * id;
        const double mx = f[R_MX], my = f[R_MY], i00 = f[R_I00], i01 = f[R_I01];
        const double i11 = f[R_I11], rho2 = f[R_RHO2], k11 = f[R_K11], k00 = f[R_K00];
        const int tx0 = pr.x / kTile, ty0 = pr.y / kTile;
        const int w = pr.z / kTile - tx0 + 1, h = pr.w / kTile - ty0 + 1;
        long long base = off_r[r];
        for (int j0 = 0; j0 < w * h; j0 += 32) {
            const int j = j0 + lane;
            bool hit = false;
            int tx = 0, ty = 0;
            if (j < w * h) {
                ty = ty0 + j / w;
                tx = tx0 + j % w;
                hit = ellipse_may_hit(mx, my, i00, i01, i11, k11, k00, rho2,
                                      max(pr.x, tx * kTile), min(pr.z, tx * kTile + kTile - 1),
                                      max(pr.y, ty * kTile), min(pr.w, ty * kTile + kTile - 1));
            }
            const unsigned m = __ballot_sync(0xffffffffu, hit);
            if (hit) {
                const long long d = base + __popc(m & ((1u << lane) - 1u));
                tkeys[d] = (unsigned int)(ty * tiles_x + tx);
                dval[d] = (int)d;
                dup_id[d] = id;
            }
            base += __popc(m);
        }
    }
}

// K6, per tile-sorted position j < cap: the tile ranges, and tile-sorted
// copies of the splat id and of its exact pixel rectangle (K1's pixel_range of
// the FP64 bbox), which the rasterisers test per warp.  Entries with the
// sentinel key (the padding [n_dup, cap), or everything on an overflow) sort
// last and are skipped.
__global__ void k_tile_ids(const unsigned int* __restrict__ tkeys, const int* __restrict__ sorted_d,
                           const int* __restrict__ dup_id, long long n, unsigned int sentinel,
                           const int4* __restrict__ rect, int* __restrict__ tile_ids,
                           int4* __restrict__ trect, int* __restrict__ start,
                           int* __restrict__ end) {
    const long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    const unsigned int k = tkeys[j];
    if (k == sentinel) return;
    if (j == 0 || tkeys[j - 1] != k) start[k] = (int)j;
    if (j == n - 1 || tkeys[j + 1] != k) end[k] = (int)(j + 1);
    const int id = dup_id[sorted_d[j]];
    tile_ids[j] = id;
    trect[j] = rect[id];
}

// the sentinel key into [n_dup, cap) (all of [0, cap) when n_dup > cap)
__global__ void k_pad_keys(const long long* __restrict__ total, long long cap,
                           unsigned int sentinel, unsigned int* __restrict__ tkeys) {
    const long long nd = *total;
    const long long j0 = nd > cap ? 0 : nd;
    for (long long j = j0 + (long long)blockIdx.x * blockDim.x + threadIdx.x; j < cap;
         j += (long long)gridDim.x * blockDim.x)
        tkeys[j] = sentinel;
}

// per view, before K1: the status block reset
__global__ void k_view_begin(ViewStatus* __restrict__ vs) {
    *vs = ViewStatus{INT_MAX, INT_MAX, 0, 0, 0};
}

// a deferred view: its error, duplicate total and overflow count into the
// step's fused tail (summed over ranks with the gradient)
__global__ void k_view_end(const ViewStatus* __restrict__ vs, const long long* __restrict__ total,
                           long long cap, double* errk, double* erri, double* ndup,
                           double* ovf) {
    if (errk) {
        if (vs->nonfinite_splat != INT_MAX) {
            *errk = 1.0;
            *erri = vs->nonfinite_splat;
        } else if (vs->degenerate_splat != INT_MAX) {
            *errk = 2.0;
            *erri = vs->degenerate_splat;
        }
    }
    if (ndup) *ndup = (double)*total;
    if (*total > cap) atomicAdd(ovf, 1.0);
}

__global__ void __launch_bounds__(1024) k_tile_order(const int* __restrict__ start,
                                                     const int* __restrict__ end, int n,
                                                     int* __restrict__ order) {
    __shared__ int s_cnt[256];
    __shared__ int s_off[256];
    for (int b = threadIdx.x; b < 256; b += blockDim.x) s_cnt[b] = 0;
    __syncthreads();
    auto bucket = [&](int t) { return 255 - min((end[t] - start[t]) >> 4, 255); };
    for (int t = threadIdx.x; t < n; t += blockDim.x) atomicAdd(&s_cnt[bucket(t)], 1);
    __syncthreads();
    if (threadIdx.x < 32) {  // exclusive scan of the 256 counts by one warp
        int run = 0;
        for (int b0 = 0; b0 < 256; b0 += 32) {
            const int v = s_cnt[b0 + threadIdx.x];
            int incl = v;
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, incl, o);
                if ((int)threadIdx.x >= o) incl += y;
            }
            s_off[b0 + threadIdx.x] = run + incl - v;
            run += __shfl_sync(0xffffffffu, incl, 31);
        }
    }
    __syncthreads();
    for (int t = threadIdx.x; t < n; t += blockDim.x) order[atomicAdd(&s_off[bucket(t)], 1)] = t;
}
int bits_for(int n) {
    int b = 1;
    while ((1LL << b) < n) ++b;
    return b;
}

}  // namespace

void view_begin(cudaStream_t st, ViewStatus* vs) {
    k_view_begin<<<1, 1, 0, st>>>(vs);
    SGTR_CUDA(cudaGetLastError());
}

void view_end(cudaStream_t st, const ViewStatus* vs, const long long* total, long long cap,
              double* errk, double* erri, double* ndup, double* ovf) {
    k_view_end<<<1, 1, 0, st>>>(vs, total, cap, errk, erri, ndup, ovf);
    SGTR_CUDA(cudaGetLastError());
}

size_t depth_sort_temp_bytes(int K) {
    size_t bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, bytes, (unsigned int*)nullptr, (unsigned int*)nullptr,
                                    (int*)nullptr, (int*)nullptr, K, 0, 32);
    return bytes;
}

size_t scan_temp_bytes(int K) {
    size_t bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, bytes, count_iter(nullptr, nullptr, K),
                                  (long long*)nullptr, K + 1);
    return bytes;
}

size_t tile_sort_temp_bytes(long long cap, int n_tiles) {
    size_t bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, bytes, (unsigned int*)nullptr,
                                    (unsigned int*)nullptr, (int*)nullptr, (int*)nullptr,
                                    (int)cap, 0, bits_for(n_tiles + 1));
    return bytes;
}

void launch_tile_order(cudaStream_t st, const int* tile_start, const int* tile_end, int n_tiles,
                       int* order) {
    if (n_tiles == 0) return;
    k_tile_order<<<1, 1024, 0, st>>>(tile_start, tile_end, n_tiles, order);
    SGTR_CUDA(cudaGetLastError());
}

void depth_sort_and_scan(cudaStream_t st, BinBuffers& b, int K) {
    if (K > 0) {
        size_t bytes = b.temp_bytes;
        SGTR_CUDA(cub::DeviceRadixSort::SortPairs(b.temp, bytes, b.keys32, b.keys32_alt, b.ids,
                                                  b.ids_alt, K, 0, 32, st));
        k_fix_depth_ties<<<ceil_div(K, 256), 256, 0, st>>>(b.keys32_alt, b.keys, b.ids_alt, K);
        SGTR_CUDA(cudaGetLastError());
    }
    // K3: exclusive scan of the tile counts gathered in depth-rank order
    size_t bytes = b.temp_bytes;
    SGTR_CUDA(cub::DeviceScan::ExclusiveSum(b.temp, bytes, count_iter(b.ids_alt, b.tcount, K),
                                            b.off_r, K + 1, st));
}

void bin_tiles(cudaStream_t st, BinBuffers& b, int K, int tiles_x, int n_tiles, long long cap) {
    SGTR_CUDA(cudaMemsetAsync(b.tile_start, 0, sizeof(int) * n_tiles, st));
    SGTR_CUDA(cudaMemsetAsync(b.tile_end, 0, sizeof(int) * n_tiles, st));
    if (K == 0 || n_tiles == 0) return;
    const unsigned int sentinel = (unsigned int)n_tiles;
    SGTR_CUDA(cudaMemsetAsync(b.n_large, 0, sizeof(int), st));
    k_emit_small<<<ceil_div(K, 256), 256, 0, st>>>(b.ids_alt, b.tinfo, b.off_r, K,
                                                   tiles_x, cap, b.off_id, b.tkeys, b.dval,
                                                   b.dup_id, b.large, b.n_large);
    SGTR_CUDA(cudaGetLastError());
    k_emit_large<<<148 * 4, 256, 0, st>>>(b.ids_alt, b.rect, b.rec, b.off_r, tiles_x, b.large,
                                          b.n_large, b.tkeys, b.dval, b.dup_id);
    SGTR_CUDA(cudaGetLastError());
    k_pad_keys<<<148 * 4, 256, 0, st>>>(b.off_r + K, cap, sentinel, b.tkeys);
    SGTR_CUDA(cudaGetLastError());
    size_t bytes = b.temp_bytes;
    SGTR_CUDA(cub::DeviceRadixSort::SortPairs(b.temp, bytes, b.tkeys, b.tkeys_alt, b.dval,
                                              b.dval_alt, (int)cap, 0, bits_for(n_tiles + 1),
                                              st));
    k_tile_ids<<<ceil_div(cap, 256), 256, 0, st>>>(b.tkeys_alt, b.dval_alt, b.dup_id, cap, sentinel,
                                                   b.rect, b.tile_ids, b.trect, b.tile_start,
                                                   b.tile_end);
    SGTR_CUDA(cudaGetLastError());
}

}  // namespace sgtr
