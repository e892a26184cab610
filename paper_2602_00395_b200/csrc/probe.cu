// probe.cu — FP64 FMA-pipe throughput microbenchmark.
//
// MEASURED_PEAKS.json carries the HBM copy bandwidth and the bf16 tensor
// peak only; the rasteriser passes are bound by the FP64 CUDA-core pipe
// (SURVEY §8d), so bench.py measures that peak on the same box with this
// kernel: independent DFMA chains, 8 per thread, full occupancy.
#include <algorithm>

#include "common.cuh"

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

}  // namespace

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
