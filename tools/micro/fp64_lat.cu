// FP64 pipe latency / throughput probe (B200): one warp per SM sub-partition
// runs a chain of dependent DFMAs (latency), then N warps x ILP chains
// (throughput).  nvcc -gencode arch=compute_100a,code=sm_100a -O3 fp64_lat.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int ILP>
__global__ void chain(double* out, int iters, long long* cycles) {
    double x[ILP];
#pragma unroll
    for (int i = 0; i < ILP; ++i) x[i] = threadIdx.x * 1e-3 + i;
    const double a = 0.999999, b = 1e-9;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < ILP; ++i) x[i] = fma(x[i], a, b);
    }
    long long t1 = clock64();
    double s = 0;
#pragma unroll
    for (int i = 0; i < ILP; ++i) s += x[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

template <int ILP>
void run(int blocks, int threads, int iters) {
    double* out;
    long long* cyc;
    cudaMalloc(&out, sizeof(double) * blocks * threads);
    cudaMalloc(&cyc, sizeof(long long) * blocks);
    chain<ILP><<<blocks, threads>>>(out, iters, cyc);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    chain<ILP><<<blocks, threads>>>(out, iters, cyc);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    long long c;
    cudaMemcpy(&c, cyc, sizeof(long long), cudaMemcpyDeviceToHost);
    const double flops = 2.0 * blocks * threads * (double)iters * ILP;
    printf("ILP %d blocks %d threads %d: %.2f cycles/dep-FMA (block 0), %.2f TFLOP/s\n", ILP,
           blocks, threads, (double)c / iters, flops / (ms * 1e-3) / 1e12);
    cudaFree(out);
    cudaFree(cyc);
}

int main() {
    const int it = 1 << 16;
    run<1>(1, 32, it);       // latency: one warp
    run<1>(148, 128, it);    // 1 warp/SMSP
    run<2>(148, 128, it);
    run<4>(148, 128, it);
    run<1>(148, 256, it);    // 2 warps/SMSP
    run<2>(148, 256, it);
    run<4>(148, 256, it);
    run<1>(148, 512, it);    // 4 warps/SMSP
    run<2>(148, 512, it);
    run<4>(148, 512, it);
    run<1>(148, 1024, it);   // 8 warps/SMSP
    run<2>(148, 1024, it);
    run<8>(148, 1024, it);
    return 0;
}
