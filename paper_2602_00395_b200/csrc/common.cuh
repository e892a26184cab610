// common.cuh — shared device types for the sm_100a 3DGS²-TR kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <stdexcept>
#include <string>

#include "../../include/sgtr.h"

namespace sgtr {

// ------------------------------------------------------------------ errors
struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

inline void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess)
        throw Error(SGTR_RUNTIME, std::string(what) + ": " + cudaGetErrorString(e));
}
#define SGTR_CUDA(call) ::sgtr::cuda_check((call), #call)

// ------------------------------------------------------------------ constants
constexpr int kTile = 16;             // 16x16 pixel tiles
constexpr int kTilePixels = kTile * kTile;
constexpr int kRec = 16;              // doubles per projected-fragment record
constexpr int kTRec = 12;             // doubles per tangent record
constexpr int kAdj = 9;               // adjoint slots per (tile, fragment)
constexpr int kVjpSlots = 4;          // K10 partials per duplicate, at most: one per block of its tile
constexpr int kWideVjpTiles = 4096;   // from this many tiles on, K10 uses 16x8 blocks (2 per tile)
constexpr int kPartStride = 10;       // doubles per K10 partial (9 adjoints + 1 pad: 16-B aligned)

// fragment record fields (one 128-byte record per splat id)
enum RecField {
    R_BX0 = 0, R_BX1, R_BY0, R_BY1,  // px -/+ rx, py -/+ ry (render.cpp:129-131)
    R_MX, R_MY,                      // mu2d
    R_I00, R_I01, R_I11,             // inverse 2d covariance
    R_ALPHA, R_C0, R_C1, R_C2,
    R_K11,                           // i01 / i11 (edge minimiser slope)
    R_RHO2,                          // 2 ln(alpha / alpha_skip) (contribution ellipse)
    R_K00                            // i01 / i00
};
// tangent record fields
enum TRecField { T_MX = 0, T_MY, T_I00, T_I01, T_I11, T_ALPHA, T_C0, T_C1, T_C2 };

// camera as the kernels see it: world->camera rotation precomputed on the
// host with the oracle's op order (quat_to_rotation, geometry.hpp:45-54)
struct DevCam {
    int W, H;
    double fx, fy, cx, cy;
    double w[9];
    double t[3];
    double cen[3];  // camera centre -W^T t (scene.hpp:80), for the SH view direction
};

struct RenderP {
    double z_near, lowpass, alpha_clamp, alpha_skip, t_stop, cutoff;
    double bg[3];
    int cull;  // contribution-ellipse culling (off only for the E/C counters)
};

inline RenderP render_params(const sgtr_render_options& o) {
    return {o.z_near, o.lowpass, o.alpha_clamp, o.alpha_skip, o.t_stop, o.cutoff_sigma,
            {o.background[0], o.background[1], o.background[2]}, 1};
}

// per-view device error/status block
struct ViewStatus {
    int nonfinite_splat;   // min splat index with a non-finite parameter
    int degenerate_splat;  // min non-culled splat index with |q|^2 < 1e-24
    int n_visible;
    int pad;
    long long n_dup;
};

inline int ceil_div(long long a, long long b) { return static_cast<int>((a + b - 1) / b); }

#ifdef __CUDACC__
// cp.async (LDGSTS) global -> shared copies, cached in L1.  cp_async8 with
// valid = false writes 8 zero bytes and reads nothing (src-size 0).
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool valid) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem),
                 "r"(valid ? 8 : 0)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
    asm volatile("cp.async.commit_group;\n" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}
#endif

}  // namespace sgtr
