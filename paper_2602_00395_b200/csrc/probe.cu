// probe.cu — FP64 FMA-pipe throughput microbenchmark.
//
// MEASURED_PEAKS.json carries the HBM copy bandwidth and the bf16 tensor
// peak only; the rasteriser passes are bound by the FP64 CUDA-core pipe
// (SURVEY §8d), so bench.py measures that peak on the same box with this
// kernel: independent DFMA chains, 8 per thread, full occupancy.
#include <algorithm>

#include "common.cuh"
#include "fastexp.cuh"

namespace sgtr {
namespace {

constexpr int kChains = 8;

__global__ void __launch_bounds__(256) k_fma_probe(double* out, int iters, double b, double c) {
    double a[kChains];
#pragma unroll
    for (int j = 0; j < kChains; ++j) a[j] = threadIdx.x * 1e-9 + j;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int j = 0; j < kChains; ++j) a[j] = fma(a[j], b, c);
    }
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < kChains; ++j) s += a[j];
    if (s == 1234.5678) out[0] = s;  // keeps the chains live
}

// fast_exp against the library exp over n inputs spread across
// [lo, hi] (a splitmix sequence, so every ulp pattern class appears)
__global__ void k_exp_check(long long n, double lo, double hi, unsigned long long seed,
                            unsigned long long* mismatches) {
    unsigned long long bad = 0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        unsigned long long z = seed + (unsigned long long)i * 0x9e3779b97f4a7c15ull;
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
        z ^= z >> 31;
        const double u = (double)(z >> 11) * 0x1.0p-53;
        const double x = lo + (hi - lo) * u;
        if (__double_as_longlong(fast_exp(x)) != __double_as_longlong(exp(x))) ++bad;
        // the rasterisers' variant: identical on [-708, 708.39), 0 below
        const double ref = x < -708.0 ? 0.0 : exp(x);
        if (x < 708.0 && __double_as_longlong(fast_exp_neg(x)) != __double_as_longlong(ref))
            ++bad;
        // exp(-q/2) without the multiply against fast_exp_neg(-0.5 q)
        if (x <= 0.0 && __double_as_longlong(fast_exp_neg_half(-2.0 * x)) !=
                            __double_as_longlong(fast_exp_neg(x)))
            ++bad;
        // rcp_unit against the IEEE division on [0.01, 1]
        const double xr = 0.01 + 0.99 * u;
        if (__double_as_longlong(rcp_unit(xr)) != __double_as_longlong(1.0 / xr)) ++bad;
    }
    if (bad) atomicAdd(mismatches, bad);
}

}  // namespace

long long fast_exp_mismatches(long long n, double lo, double hi, unsigned long long seed) {
    unsigned long long* d = nullptr;
    SGTR_CUDA(cudaMalloc(&d, sizeof(*d)));
    SGTR_CUDA(cudaMemset(d, 0, sizeof(*d)));
    k_exp_check<<<148 * 8, 256>>>(n, lo, hi, seed, d);
    SGTR_CUDA(cudaGetLastError());
    unsigned long long h = 0;
    SGTR_CUDA(cudaMemcpy(&h, d, sizeof(h), cudaMemcpyDeviceToHost));
    cudaFree(d);
    return (long long)h;
}

double fp64_fma_peak_tflops(int device) {
    SGTR_CUDA(cudaSetDevice(device));
    int sms = 0;
    SGTR_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    double* out = nullptr;
    SGTR_CUDA(cudaMalloc(&out, sizeof(double)));
    const int blocks = sms * 8, threads = 256, iters = 1 << 14;
    cudaEvent_t a, b;
    SGTR_CUDA(cudaEventCreate(&a));
    SGTR_CUDA(cudaEventCreate(&b));
    k_fma_probe<<<blocks, threads>>>(out, 256, 0.999999, 1e-7);  // warm-up
    double best = 0.0;
    for (int rep = 0; rep < 5; ++rep) {
        SGTR_CUDA(cudaEventRecord(a));
        k_fma_probe<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
        SGTR_CUDA(cudaEventRecord(b));
        SGTR_CUDA(cudaEventSynchronize(b));
        float ms = 0.f;
        SGTR_CUDA(cudaEventElapsedTime(&ms, a, b));
        const double flops = 2.0 * kChains * (double)iters * blocks * threads;
        best = std::max(best, flops / (ms * 1e-3) / 1e12);
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaFree(out);
    return best;
}

}  // namespace sgtr
