// launch.h — host-side launchers shared between the translation units.
#pragma once
#include <cuda_runtime.h>

#include <string>
#include <vector>

#include "common.cuh"

namespace sgtr {

// ---------------------------------------------------------------- project.cu
// K1: per-splat projection -> 128-byte fragment record, order-preserving
// 64-bit depth key (culled = ~0), tile rectangle and tile count.
// tinfo: per splat, what K4 needs in one 16-byte gather: the tile rectangle
// (x: tx0 | ty0 << 16, y: width | height << 16, in tiles) and the hit bits of
// its tiles in row-major order (z, w: low and high words; rectangles of <= 64
// tiles)
void launch_project(cudaStream_t st, const double* x, int K, int nb, const DevCam& cam,
                    const RenderP& ro, double* rec, unsigned long long* keys,
                    unsigned int* keys32, int* ids, int4* rect, int* tcount,
                    int4* tinfo, ViewStatus* status);
// parity dump: 12 doubles per splat (culled, depth, px, py, bx0..by1, i00..i11, 0)
void launch_project_dump(cudaStream_t st, const double* x, int K, const DevCam& cam,
                         const RenderP& ro, double* out);
// K12 (projection half): tangent records along a dense direction v (seam) or
// along probe bits (bit set -> +1)
void launch_project_jvp(cudaStream_t st, const double* x, int K, int nb, const DevCam& cam,
                        const RenderP& ro, const double* v, const uint32_t* zbits,
                        double* trec);

// ---------------------------------------------------------------- binning.cu
struct BinBuffers {
    unsigned long long *keys, *keys_alt;
    unsigned int *keys32, *keys32_alt;  // K2's FP32-depth sort keys (K1 writes keys32)
    int *ids, *ids_alt;
    int4* rect;            // bbox pixel range (x0, y0, x1, y1) per splat
    const double* rec;     // fragment records (K1)
    int* tcount;
    int4* tinfo;           // tile rectangle + hit bits per splat (K1 -> K4)
    int* large;            // depth ranks of splats with > 64-tile rectangles
    int* n_large;
    long long* off_r;      // K+1 exclusive duplicate offsets in depth-rank order
    long long* off_id;     // the same offsets by splat id (K4 scatters them, K11 reads them)
    // duplicate arrays, capacity `cap` entries
    unsigned int *tkeys, *tkeys_alt;
    int *dval, *dval_alt;  // duplicate index carried through the tile sort
    int* dup_id;           // duplicate -> splat id
    int* tile_ids;         // per tile-sorted position: splat id
    int4* trect;           // per tile-sorted position: the splat's pixel rectangle
    int *tile_start, *tile_end;
    void* temp;
    size_t temp_bytes;
};
size_t depth_sort_temp_bytes(int K);
size_t scan_temp_bytes(int K);
size_t tile_sort_temp_bytes(long long cap, int n_tiles);
// per view, before K1: status reset
void view_begin(cudaStream_t st, ViewStatus* vs);
// K2 (+ the K3 scan): sorts keys, returns sorted ids in b.ids_alt and the
// exclusive duplicate offsets (total at off_r[K])
void depth_sort_and_scan(cudaStream_t st, BinBuffers& b, int K);
// K4-K6 without a host round trip: emission, stable tile sort of `cap`
// entries (the tail padded with a sentinel key), tile ranges and the
// tile-sorted splat ids / rectangles; a view with off_r[K] > cap is binned
// empty
void bin_tiles(cudaStream_t st, BinBuffers& b, int K, int tiles_x, int n_tiles, long long cap);
// a view whose status is not read back on the host: its error, duplicate
// total and overflow (total > cap) into the step's tail slots (errk/erri/
// ndup may be null)
void view_end(cudaStream_t st, const ViewStatus* vs, const long long* total, long long cap,
              double* errk, double* erri, double* ndup, double* ovf);

struct TileLists {
    int tiles_x, tiles_y;
    const int* tile_start;
    const int* tile_end;
    const int* sorted_d;  // tile-sorted duplicate indices
    const int* dup_id;    // duplicate -> splat id
    const int* tile_ids;  // splat id per tile-sorted position (dup_id[sorted_d[j]])
    const int4* trect;    // per position: the splat's pixel rectangle (x0, y0, x1, y1)
    int row0, row1;       // tile rows the raster kernels process (a band on refresh
                          // views split over ranks; [0, tiles_y) otherwise)
    const int* order = nullptr;  // full frames: tiles by decreasing list length (the
                                 // raster kernels' launch order), else row-major
};
// tiles by decreasing list length (bucketed) into order[0, n_tiles): the
// long tiles start first, so the grid's tail is short ones
void launch_tile_order(cudaStream_t st, const int* tile_start, const int* tile_end, int n_tiles,
                       int* order);
// K7: front-to-back blend -> planar image, final T, processed count per pixel
void launch_raster_fwd(cudaStream_t st, const TileLists& tl, const double* rec, int W,
                       int H, const RenderP& ro, double* img, double* tfinal, int* last,
                       unsigned long long* counters = nullptr);
// K10: back-to-front adjoint sweep; each warp (one block of a tile: 16x8,
// s = 2 per tile, when the raster region has >= kWideVjpTiles tiles, else
// 8x8, s = 4) writes its reduced adjoints of duplicate d to
// part[(d * s + block) * 10 ...] and flags mask[d * s + block]; mask must be
// zeroed first.  vjp_slots(tiles of the region) gives s.
int vjp_slots(int n_tiles);
void launch_raster_vjp_warp(cudaStream_t st, const TileLists& tl, const double* rec, int W,
                            int H, const RenderP& ro, const double* adj, const double* tfinal,
                            const int* last, double* part, unsigned char* mask);
// K11: per splat (id order), the sum of its flagged K10 partials (duplicate,
// block order) and the chain through invert2x2 and the projection; mode 0
// adds the gradient into acc, mode 1 z (.) it (Hutchinson, probe dense or as
// bits); a non-finite contribution stores 1.0 into *nonfinite_flag.  Splats
// whose duplicates lie beyond the capacity `cap` are skipped (an overflowed
// view, rerun by the step).
void launch_chain_warp(cudaStream_t st, int mode, const double* x, int K, int nb, const DevCam& cam,
                       const RenderP& ro, const long long* off_id, const int* tcount,
                       long long cap, int slots, const double* part, const unsigned char* mask,
                       const double* zdense, const uint32_t* zbits, double* acc,
                       double* nonfinite_flag);
// K12 (raster half): tangent image along the tangent records
void launch_raster_jvp(cudaStream_t st, const TileLists& tl, const double* rec,
                       const double* trec, int W, int H, const RenderP& ro,
                       double* tangent);

// ---------------------------------------------------------------- ssim.cu
enum SsimMode {
    SSIM_MAP = 0,  // out0 = SSIM
    SSIM_JVP,      // out0 = SSIM, out1 = dSSIM
    RES_VEC,       // out0 = residual vector (6P)
    RES_JVP,       // out0 = residual JVP (6P)
    GRAD,          // u = f: loss partials, adjL1 and P, Q, R (K8)
    HUTCH,         // u = J t: adjL1 and P, Q, R (K13)
    RES_VJP,       // u given (6P, in `u`): adjL1 and P, Q, R
    SSIM_VJP,      // upstream given (3P planar, in `u`): P, Q, R
    EVAL,          // per-block sums of SSIM and (a-b)^2 into loss_partials
                   // [blk] and [nblocks + blk] (mean_ssim, psnr)
    BMOM           // out0 = windowed mean of b, out1 = windowed E[b^2] (fixed per view)
};
struct SsimArgs {
    int mode, W, H;
    const double *a, *da, *b, *u;
    double lambda, floor;
    double *out0, *out1, *adjl1, *P, *Q, *R, *loss_partials;
    int by0, by1;  // block rows (16 image rows each) to compute; by1 <= 0: all
    const double* bmom;  // optional (GRAD/HUTCH): [mu_b planes | mbb planes] from BMOM
};
int ssim_num_blocks(int W, int H);
void launch_ssim(cudaStream_t st, const SsimArgs& a);
// K9: adj = adjL1 + W^T P + a (.) W^T Q + b (.) W^T R (reflection-aware gather)
void launch_ssim_gather(cudaStream_t st, int W, int H, const double* a, const double* b,
                        const double* adjl1, const double* P, const double* Q,
                        const double* R, double* adj, int by0 = 0, int by1 = 0);
void launch_sum_partials(cudaStream_t st, const double* partials, int n, double* out);
// layout conversions: interleaved (H,W,3) <-> planar (3,H,W)
void launch_to_planar(cudaStream_t st, const double* in, int P, double* out);
void launch_to_interleaved(cudaStream_t st, const double* in, int P, double* out);
void launch_quantize8(cudaStream_t st, double* img, long long n);

// ---------------------------------------------------------------- update.cu
struct TrArgs {
    int K;
    const double* x;
    double* x_out;
    const double* g_acc;  // unscaled sum of per-view gradients
    double gscale;
    double* g_hat;
    double* d_hat;
    const double* w_acc;  // unscaled sum of z (.) J^T J z (refresh steps)
    double dscale;
    int refresh;          // update D-hat from w_acc
    int ghat_only;        // Hutchinson failed: update g-hat and stop
    double theta1, theta2, gamma_d, eps;
    double caps[5];
    double bounds[5];     // s_min, alpha_min, alpha_max, c_min, c_max
    double* applied;      // optional clipped step
    double* partials;     // per block: sum g^2, sum dx^2, sum clipped^2, n_clip, max ratio
    int* bad_index;       // min index of a non-finite clipped coordinate
    int* degenerate_flag; // a splat with |q|^2 < 1e-24 reached shd_radii
    double* dx_buf;       // Newton direction (dim)
    double* eta_buf;      // trust-region radii (dim)
    int* queue;           // (splat, rotation axis) pairs needing bisection (4K)
    int* queue_count;
    // direction: 0 = 3DGS2-TR Newton step, 1 = ADAM (unclipped update),
    // 2 = ADAM-TR (ADAM direction, trust-region clip) (optimizer.cpp:153-253)
    int kind;
    double* adam_m;
    double* adam_v;
    double beta1, beta2, adam_eps;
    double bc1, bc2;      // 1 - beta^t bias corrections (host std::pow)
    double lr[5];         // per-group rates, lr[0] already decayed and scaled
    int nb;               // SH coefficients per channel (extension; 0 = reference)
    int i0, n;            // the splats whose radii this launch computes (a shard)
    int elementwise;      // K14a also runs the EMAs / direction over all K splats
};
int tr_num_blocks(int K);
// phase 0: K14a (EMAs, direction; radius, clip, apply and clamp of the ten
// non-rotation coordinates), 3: K14a' (rotation radii and their
// certification, failures queued), 1: K14b (queued bisections), 2: K14c
// (clip and apply of the rotation coordinates); in the order 0, 3, 1, 2
void launch_tr_update(cudaStream_t st, const TrArgs& a, int phase);
// 5 reduced values: gnorm^2, step_pre^2, step_post^2, n_clipped, max ratio
// (partials hold 2 * tr_num_blocks(K) rows of 5)
void launch_tr_finalize(cudaStream_t st, const double* partials, int nblocks, double* out5);
void launch_shd_radii(cudaStream_t st, int K, int nb, const double* x, double eps,
                      const double caps[5], double* eta);
void launch_scale(cudaStream_t st, double* v, long long n, double s);
void launch_add(cudaStream_t st, double* dst, const double* src, long long n);
// io.cu
struct PlyHeader {
    long long count;
    long long data_offset;
};
struct CameraLine {
    sgtr_camera cam;
    std::string image_name;
};
PlyHeader ply_read_header(const std::string& path);
void ply_read_payload(const std::string& path, const PlyHeader& h, double* aos);
void ply_write(const std::string& path, const double* aos, long long count);
void host_aos_to_soa(const double* aos, long long K, double* soa);
void host_soa_to_aos(const double* soa, long long K, double* aos);
void host_validate(const double* x, long long K, const double b[5]);
void throw_invalid_splat(unsigned long long first);
void launch_aos_to_soa(cudaStream_t st, const double* aos, long long K, double* soa);
void launch_soa_to_aos(cudaStream_t st, const double* soa, long long K, double* aos);
void launch_validate(cudaStream_t st, const double* x, long long K, const double b[5],
                     unsigned long long* first);
void save_cameras(const std::string& path, const sgtr_camera* cams, const char* const* names,
                  int n);
std::vector<CameraLine> load_cameras(const std::string& path);
double scene_extent(const sgtr_camera* cams, int n);
// probe.cu
double fp64_fma_peak_tflops(int device);
long long fast_exp_mismatches(long long n, double lo, double hi, unsigned long long seed);
void launch_fill_int(cudaStream_t st, int* p, long long n, int v);

}  // namespace sgtr
