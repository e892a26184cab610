/* sgtr.h — C-ABI of the B200-native 3DGS²-TR training iteration.
 *
 * This is the drop-in boundary for the reference's hot path
 * `splat::step_3dgs2tr` (/root/reference/proj/src/optimizer.cpp:189-220) and
 * the seams its tests and checks call.  Every entry point names the
 * reference interface it replaces.  Plain pointers and sizes only; host
 * memory is caller-owned and copied, device memory is owned by the context.
 *
 * Layouts are the reference's:
 *   scene x  : double[14*K] group-major [mu 3K | s 3K | q 4K | alpha K | c 3K]
 *              (scene.hpp:37-52)
 *   images   : double[H*W*3] row-major, channel-interleaved (image.hpp:10-27)
 *   residual : double[6*H*W], L1 block then D-SSIM block, index c*H*W+y*W+x
 *              (residuals.hpp:17-22)
 *
 * Status codes mirror the reference's exception classes:
 *   SGTR_OK, SGTR_INVALID_ARGUMENT (std::invalid_argument, CLI exit 1),
 *   SGTR_NUMERIC (splat::NumericError, errors.hpp:11-14, CLI exit 2),
 *   SGTR_RUNTIME (CUDA/NCCL failure).  sgtr_last_error() returns the message
 *   (same wording and locator as the reference's exception text).
 *
 * One host thread per context (not re-entrant), like the reference's single
 * control thread.
 */
#ifndef SGTR_H
#define SGTR_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { SGTR_OK = 0, SGTR_INVALID_ARGUMENT = 1, SGTR_NUMERIC = 2, SGTR_RUNTIME = 3 };

typedef struct sgtr_ctx sgtr_ctx;

/* splat::Camera (scene.hpp:70-81) minus the GT image */
typedef struct sgtr_camera {
    int32_t id, width, height, pad;
    double fx, fy, cx, cy;
    double q_wc[4]; /* unit (x, y, z, w), x_cam = R(q_wc) x_world + t_wc */
    double t_wc[3];
} sgtr_camera;

/* splat::RenderOptions (render.hpp:12-22); `workers` has no GPU meaning */
typedef struct sgtr_render_options {
    double z_near, lowpass, alpha_clamp, alpha_skip, t_stop, cutoff_sigma;
    double background[3];
} sgtr_render_options;

/* splat::ResidualOptions (residuals.hpp:13-16) */
typedef struct sgtr_residual_options {
    double lambda, floor;
} sgtr_residual_options;

/* splat::OptimizerOptions (optimizer.hpp:37-53) for the 3DGS²-TR kind, with
 * TrustRegionSchedule, RadiusCaps (trust_region.hpp:66-89) and ParamBounds
 * (scene.hpp:29-35) flattened */
typedef struct sgtr_optimizer_options {
    double theta1, theta2;
    int32_t hess_interval, hutch_samples, batch_size, hutch_batch_size;
    double gamma_d;
    double eps_start, eps_end;
    int32_t total_steps, record_applied_step;
    double cap_mean, cap_scale, cap_rotation, cap_opacity, cap_color;
    double s_min, alpha_min, alpha_max, c_min, c_max;
    sgtr_residual_options residual;
    sgtr_render_options render;
} sgtr_optimizer_options;

/* splat::AdamOptions (optimizer.hpp:21-34) + OptimizerOptions::scene_extent
 * (:50); used by the ADAM kinds together with sgtr_optimizer_options
 * (batch_size, the TR schedule/caps for ADAM-TR, bounds, residual, render) */
typedef struct sgtr_adam_options {
    double beta1, beta2, eps, lr_position, lr_position_final;
    int32_t lr_position_decay_steps, pad;
    double lr_scale, lr_rotation, lr_opacity, lr_color, scene_extent;
} sgtr_adam_options;

/* splat::OptimizerKind (optimizer.hpp:17) */
enum { SGTR_KIND_3DGS2TR = 0, SGTR_KIND_ADAM = 1, SGTR_KIND_ADAM_TR = 2 };

/* splat::StepDiagnostics (optimizer.hpp:74-83); applied_step is fetched with
 * sgtr_get_applied_step when record_applied_step was set */
typedef struct sgtr_step_diagnostics {
    double batch_loss, gnorm, step_pre, step_post, clip_frac, eps,
        max_step_over_radius;
    int32_t refreshed, n_local_views;
    int32_t reruns; /* times the step was rerun after a view outgrew the duplicate capacity */
} sgtr_step_diagnostics;

/* ------------------------------------------------------------ context */
const char* sgtr_last_error(void);
int sgtr_create(int device, sgtr_ctx** out);
int sgtr_destroy(sgtr_ctx* ctx);
/* cudaStream_t the context launches on (for event timing by the caller) */
int sgtr_get_stream(sgtr_ctx* ctx, void** stream);
int sgtr_synchronize(sgtr_ctx* ctx);
/* number of kernels this context has launched so far */
int64_t sgtr_launch_count(const sgtr_ctx* ctx);

/* ------------------------------------------------------------ scene */
/* Scene::unpack / pack (scene.cpp:13-39) */
int sgtr_set_scene(sgtr_ctx* ctx, const double* x, int64_t n_splats);
int sgtr_get_scene(sgtr_ctx* ctx, double* x);
int64_t sgtr_scene_size(const sgtr_ctx* ctx);
/* SH colour extension (parity unpinned; the reference is degree 0):
 * x = [the 14 reference groups | SH group], the SH group splat-major with
 * 3 * ((d+1)^2 - 1) coefficients per splat (basis j major, rgb minor);
 * c_view = c + sum_j Y_j(normalize(mu - camera centre)) k_j (3DGS real-SH
 * basis, DC = the reference's linear RGB, no offset, no clamp).  Trust-region
 * radius of k_j = the splat's colour radius / max|Y_j|; ADAM rate lr_color/20.
 * sgtr_set_scene is sgtr_set_scene_sh with degree 0. */
int sgtr_set_scene_sh(sgtr_ctx* ctx, const double* x, int64_t n_splats,
                      int32_t sh_degree);
int32_t sgtr_scene_sh_degree(const sgtr_ctx* ctx);

/* ------------------------------------------------------------ views */
/* the training views passed to step_3dgs2tr (optimizer.hpp:129-131);
 * gts[i] is the Camera::gt image (H*W*3 doubles), or gts == NULL to keep
 * the views without targets (render-only use).  All views share one size,
 * as the reference's m = 6*P*M assumes (optimizer.cpp:44). */
int sgtr_set_views(sgtr_ctx* ctx, const sgtr_camera* cams, int32_t n,
                   const double* const* gts);
/* replaces view i's target by the quantize8 of the current scene's render
 * (dataset.cpp:63, with the render on the GPU) */
int sgtr_render_targets(sgtr_ctx* ctx, const sgtr_render_options* ro,
                        int32_t quantize);
int sgtr_get_target(sgtr_ctx* ctx, int32_t view, double* gt);

/* ------------------------------------------------------------ files */
/* splat::ParamBounds (scene.hpp:29-35); NULL selects the defaults */
typedef struct sgtr_param_bounds {
    double s_min, alpha_min, alpha_max, c_min, c_max;
} sgtr_param_bounds;
/* save_scene (scene_io.cpp:34-53) of the resident scene: binary little-endian
 * PLY, 14 double properties per vertex, bitwise round trip */
int sgtr_save_scene_ply(sgtr_ctx* ctx, const char* path);
/* load_scene (scene_io.cpp:55-116) straight into the context (replaces the
 * scene; Scene::validate runs on the device, errors name the splat) */
int sgtr_load_scene_ply(sgtr_ctx* ctx, const char* path,
                        const sgtr_param_bounds* bounds);
/* the same file format on host buffers (group-major x of 14*K doubles);
 * sgtr_ply_load with x == NULL only reports the splat count */
int sgtr_ply_save(const double* x, int64_t n_splats, const char* path);
int sgtr_ply_load(const char* path, const sgtr_param_bounds* bounds, double* x,
                  int64_t* n_splats);
/* save_cameras / load_cameras (scene_io.cpp:118-167; images not loaded):
 * one camera per line "id fx fy cx cy width height qw qx qy qz tx ty tz
 * image"; load reports the count in *n and fills up to cap entries, image
 * names NUL-terminated at image_names + i * name_stride */
int sgtr_save_cameras(const char* path, const sgtr_camera* cams,
                      const char* const* image_names, int32_t n);
int sgtr_load_cameras(const char* path, sgtr_camera* cams, char* image_names,
                      int32_t name_stride, int32_t cap, int32_t* n);
/* optimizer-state checkpoint / resume (beyond the reference, which only
 * saves the scene PLY): scene x, g_hat, d_hat, adam_m, adam_v, t and the
 * Rng state, so a resumed run draws the identical S1/S2/probe stream and
 * continues bit for bit */
int sgtr_checkpoint_save(sgtr_ctx* ctx, const char* path);
int sgtr_checkpoint_load(sgtr_ctx* ctx, const char* path);
/* scene_extent (scene.cpp:83-92): max camera-centre distance from the
 * centroid (1 for fewer than two cameras); OptimizerOptions::scene_extent */
int sgtr_scene_extent(const sgtr_camera* cams, int32_t n, double* out);

/* ------------------------------------------------------------ evaluation */
/* held-out views for evaluate_scene (harness.cpp:43-58); any image sizes,
 * targets (H*W*3 doubles) required and kept on the device */
int sgtr_set_eval_views(sgtr_ctx* ctx, const sgtr_camera* cams, int32_t n,
                        const double* const* gts);
/* evaluate_scene on the device: per view PSNR (residuals.cpp:133-144) and
 * mean SSIM (ssim.cpp:170-175) of quantize8(rasterize(scene, cam).color)
 * against the target, and their means.  which = 0: the eval views,
 * 1: the training views.  view_psnr / view_ssim hold one entry per view
 * (either may be NULL). */
int sgtr_evaluate_scene(sgtr_ctx* ctx, int32_t which,
                        const sgtr_render_options* ro, double* view_psnr,
                        double* view_ssim, double* mean_psnr,
                        double* mean_ssim);

/* ------------------------------------------------------------ optimizer state */
/* OptimizerState(dim, seed) (optimizer.hpp:58-72): g_hat = d_hat = 0, t = 0,
 * Rng(seed) */
int sgtr_state_reset(sgtr_ctx* ctx, uint64_t seed);
int sgtr_state_set(sgtr_ctx* ctx, const double* g_hat, const double* d_hat,
                   int64_t t);
int sgtr_state_get(sgtr_ctx* ctx, double* g_hat, double* d_hat, int64_t* t);
/* n raw mt19937_64 outputs from the state's Rng (rng.hpp:24) */
int sgtr_rng_raw(sgtr_ctx* ctx, int64_t n, uint64_t* out);

/* a standalone reference Rng (rng.hpp:15-72: std::mt19937_64); the variate
 * mappings (uniform, normal, rademacher, below) are applied by the caller */
typedef struct sgtr_rng sgtr_rng;
int sgtr_rng_new(uint64_t seed, sgtr_rng** out);
int sgtr_rng_draw(sgtr_rng* rng, int64_t n, uint64_t* out);
int sgtr_rng_free(sgtr_rng* rng);

/* ------------------------------------------------------------ Algorithm 1 */
/* step_3dgs2tr (optimizer.cpp:189-220): S1, S2 and probes drawn from the
 * state's Rng in the reference order */
int sgtr_step_3dgs2tr(sgtr_ctx* ctx, const sgtr_optimizer_options* opt,
                      sgtr_step_diagnostics* diag);
/* teacher-forced variant: the step's draws supplied explicitly; probe_bits
 * holds nu probes of ceil(14K/32) words each, bit k of probe s set <=> z_k =
 * +1 (rng.hpp:46); s2/probe_bits are read on refresh steps only */
int sgtr_step_3dgs2tr_explicit(sgtr_ctx* ctx, const sgtr_optimizer_options* opt,
                               const int32_t* s1, int32_t n1, const int32_t* s2,
                               int32_t n2, const uint32_t* probe_bits,
                               int32_t nu, sgtr_step_diagnostics* diag);
int sgtr_get_applied_step(sgtr_ctx* ctx, double* out);
/* Hutchinson sample s at which the last step raised "hutchinson_diag:
 * non-finite sample" (-1 otherwise).  The reference draws each probe
 * lazily (optimizer.cpp:67-73, :86-87), so at that point it has consumed
 * probes 0..s; a caller that draws the probes itself for
 * sgtr_step_3dgs2tr_explicit restores its Rng to after probe s. */
int sgtr_step_failed_sample(sgtr_ctx* ctx, int32_t* sample);

/* step_adam / step_adam_tr (optimizer.cpp:222-253): one S1 draw from the
 * state's Rng, ADAM direction (adam_direction, :153-185), then the plain
 * update (apply_unclipped) or the trust-region clip (apply_clipped) */
int sgtr_step_adam(sgtr_ctx* ctx, const sgtr_optimizer_options* opt,
                   const sgtr_adam_options* adam, sgtr_step_diagnostics* diag);
int sgtr_step_adam_tr(sgtr_ctx* ctx, const sgtr_optimizer_options* opt,
                      const sgtr_adam_options* adam, sgtr_step_diagnostics* diag);
/* teacher-forced: S1 supplied (trust_region 0: ADAM, 1: ADAM-TR) */
int sgtr_step_adam_explicit(sgtr_ctx* ctx, const sgtr_optimizer_options* opt,
                            const sgtr_adam_options* adam, int32_t trust_region,
                            const int32_t* s1, int32_t n1,
                            sgtr_step_diagnostics* diag);
/* optimizer_step (optimizer.cpp:255-263): dispatch on SGTR_KIND_* */
int sgtr_optimizer_step(sgtr_ctx* ctx, int32_t kind,
                        const sgtr_optimizer_options* opt,
                        const sgtr_adam_options* adam,
                        sgtr_step_diagnostics* diag);
/* OptimizerState::adam_m / adam_v (optimizer.hpp:58-72); zeroed by
 * sgtr_state_reset */
int sgtr_state_set_adam(sgtr_ctx* ctx, const double* m, const double* v);
int sgtr_state_get_adam(sgtr_ctx* ctx, double* m, double* v);

/* ------------------------------------------------------------ seams */
/* rasterize (render.hpp:73-74) */
int sgtr_rasterize(sgtr_ctx* ctx, const sgtr_camera* cam,
                   const sgtr_render_options* ro, double* color,
                   double* t_final);
/* rasterize_jvp (render.hpp:78-79); v has 14K entries */
int sgtr_rasterize_jvp(sgtr_ctx* ctx, const sgtr_camera* cam,
                       const sgtr_render_options* ro, const double* v,
                       double* tangent);
/* rasterize_vjp (render.hpp:83-84); grad has 14K entries */
int sgtr_rasterize_vjp(sgtr_ctx* ctx, const sgtr_camera* cam,
                       const sgtr_render_options* ro, const double* adjoint,
                       double* grad);
/* ssim_map / ssim_jvp / ssim_vjp (ssim.hpp:11-20) */
int sgtr_ssim_map(sgtr_ctx* ctx, const double* a, const double* b, int32_t w,
                  int32_t h, double* out);
int sgtr_ssim_jvp(sgtr_ctx* ctx, const double* a, const double* da,
                  const double* b, int32_t w, int32_t h, double* s,
                  double* ds);
int sgtr_ssim_vjp(sgtr_ctx* ctx, const double* a, const double* b,
                  const double* upstream, int32_t w, int32_t h, double* grad);
/* residual_vector / residual_jvp / residual_vjp (residuals.hpp:23-33) */
int sgtr_residual_vector(sgtr_ctx* ctx, const double* rendered,
                         const double* gt, int32_t w, int32_t h,
                         const sgtr_residual_options* o, double* r);
int sgtr_residual_jvp(sgtr_ctx* ctx, const double* rendered,
                      const double* tangent, const double* gt, int32_t w,
                      int32_t h, const sgtr_residual_options* o, double* dr);
int sgtr_residual_vjp(sgtr_ctx* ctx, const double* rendered, const double* gt,
                      int32_t w, int32_t h, const double* u,
                      const sgtr_residual_options* o, double* adj);
/* view_jacobian_apply / applyT (optimizer.hpp:87-94) on context view i */
int sgtr_view_jacobian_apply(sgtr_ctx* ctx, int32_t view, const double* v,
                             const sgtr_residual_options* rs,
                             const sgtr_render_options* ro, double* out);
int sgtr_view_jacobian_applyT(sgtr_ctx* ctx, int32_t view, const double* u,
                              const sgtr_residual_options* rs,
                              const sgtr_render_options* ro, double* grad);
/* stochastic_gradient (optimizer.hpp:99-104) over context views */
int sgtr_stochastic_gradient(sgtr_ctx* ctx, const int32_t* batch, int32_t n,
                             const sgtr_residual_options* rs,
                             const sgtr_render_options* ro, double* g,
                             double* batch_loss);
/* hutchinson_diag (optimizer.hpp:106-117); probes are nu dense vectors of
 * 14K entries, each entry +1 or -1 */
int sgtr_hutchinson_diag(sgtr_ctx* ctx, const int32_t* batch, int32_t n,
                         int32_t nu, const double* probes,
                         const sgtr_residual_options* rs,
                         const sgtr_render_options* ro, double* d);
/* shd_radii (trust_region.hpp:81-83) */
int sgtr_shd_radii(sgtr_ctx* ctx, double eps, const double caps[5],
                   double* eta);
/* eps_at (trust_region.hpp:87-89) */
int sgtr_eps_at(double eps_start, double eps_end, int32_t total, int32_t t,
                double* out);

/* ------------------------------------------------------------ parity dumps */
/* projected fragment fields per splat, 12 doubles each:
 * culled, depth, px, py, bx0, bx1, by0, by1, i00, i01, i11, 0
 * (render.cpp:51-69) */
int sgtr_project(sgtr_ctx* ctx, const sgtr_camera* cam,
                 const sgtr_render_options* ro, double* out);
/* GPU tile binning of one view (16x16 tiles): depth order of visible
 * splats, per-tile [start, end) and per-tile splat lists.  Call with
 * lists == NULL first to get the sizes. */
int sgtr_dump_binning(sgtr_ctx* ctx, const sgtr_camera* cam,
                      const sgtr_render_options* ro, int32_t* n_visible,
                      int32_t* order, int64_t* n_dup, int64_t* tile_start,
                      int64_t* tile_end, int32_t* lists);

/* ------------------------------------------------------------ data */
/* make_synthetic (dataset.cpp:25-67) with two declared extensions for the
 * large configurations: width != height (fx = fy = focal_factor*height),
 * and splat-size scaling (scale range, init_scale and sigma_init multiplied
 * by size_scale).  With size_scale = 1 and width = height the scenes and
 * cameras equal the reference's.  Writes gt_x[14*gt_splats],
 * init_x[14*init_splats] and cams[views]. */
typedef struct sgtr_synth_config {
    int32_t gt_splats, init_splats, views, width, height, pad;
    uint64_t seed;
    double sigma_init, init_scale, init_opacity, camera_radius, camera_height,
        focal_factor, size_scale;
    /* SH colour extension: degree 0..3; GT coefficients 0.1 N(0,1) from a
     * separate stream (seed + 0x5348), init coefficients 0; x vectors are
     * (14 + 3 ((d+1)^2 - 1)) * K long */
    int32_t sh_degree, pad2;
} sgtr_synth_config;
int sgtr_make_synthetic(const sgtr_synth_config* cfg, double* gt_x,
                        double* init_x, sgtr_camera* cams);

/* ------------------------------------------------------------ measurement */
/* per-kernel-class CUDA-event timing on the context stream (enable resets
 * the totals); the report is JSON {"class": [launches, total_ms], ...} */
int sgtr_kernel_timing(sgtr_ctx* ctx, int32_t enable);
int sgtr_kernel_timing_report(sgtr_ctx* ctx, char* buf, int32_t len);
/* algorithmic-work counters of one view: (pixel, fragment) pairs reaching
 * the alpha evaluation and contributing pairs (render.cpp:132-144) */
int sgtr_blend_stats(sgtr_ctx* ctx, const sgtr_camera* cam,
                     const sgtr_render_options* ro, int64_t* evaluated,
                     int64_t* contributing);
/* visible splats and tile duplicates of one view */
int sgtr_view_stats(sgtr_ctx* ctx, const sgtr_camera* cam,
                    const sgtr_render_options* ro, int32_t* n_visible,
                    int64_t* n_dup);
/* FP64 FMA-pipe throughput of the device (TFLOP/s), measured */
int sgtr_fp64_peak(int device, double* tflops);
/* self-check of the rasterizer's exp (fastexp.cuh) against the CUDA math
 * library: number of bitwise mismatches over n inputs in [lo, hi] */
int sgtr_check_fast_exp(int64_t n, double lo, double hi, uint64_t seed,
                        int64_t* mismatches);

/* Capacity of the per-view tile-duplicate arrays (entries).  Views render
 * without a host round trip and every view sorts `capacity` tile keys; a
 * training step in which some view outgrows it is rerun with the capacity
 * grown to fit (before any state changes), so this only presizes (or, for
 * tests, shrinks) it.  0 restores the default (2 K + 4096, grown on demand). */
int sgtr_set_dup_capacity(sgtr_ctx* ctx, int64_t capacity);

/* ------------------------------------------------------------ multi-GPU */
/* one process per GPU; views of each step are split round-robin over
 * ranks and g | z.w | loss are summed with one ncclAllReduce per step */
int sgtr_nccl_unique_id(uint8_t out[128]);
/* Refresh (Hutchinson) views are split into row bands of tiles when there are
 * fewer S2 views than ranks: B = nranks * bands_per_rank bands per view,
 * rank r renders bands r, r + nranks, ... (default bands_per_rank = 1; > 1
 * also splits on one rank, which tests use to check the band sums) */
int sgtr_set_refresh_bands(sgtr_ctx* ctx, int32_t bands_per_rank);
/* The rotation radii (certification and bisection: the costly part of the
 * update) are split by splat range over the ranks and all-gathered
 * (ncclAllGather) before their clip; the other radii, the EMAs, direction,
 * clip and apply stay replicated, so the state needs no gather.
 * On one rank, shards > 1 runs the same shard/stage/gather sequence back to
 * back (tests check it against the unsharded update, bit for bit). */
int sgtr_set_tr_shards(sgtr_ctx* ctx, int32_t shards);
/* positions of a step's view batch (S1 or S2) that `rank` renders: the
 * round-robin split the step uses; host-only, no device needed */
int sgtr_shard_views(int32_t n, int32_t rank, int32_t nranks, int32_t* positions,
                     int32_t* count);
int sgtr_comm_init(sgtr_ctx* ctx, const uint8_t id[128], int32_t nranks,
                   int32_t rank);
/* In-process communicator for testing the multi-rank data plane on one GPU
 * (the product path is NCCL): nranks host threads, each with its own
 * context on the same device, join one group with ranks 0..nranks-1; a
 * step's allreduce and the radii all-gather then meet at a host barrier and
 * sum / copy through device memory in rank order.  1..8 ranks. */
typedef struct sgtr_group sgtr_group;
int sgtr_loopback_group_create(int32_t nranks, sgtr_group** out);
int sgtr_loopback_group_destroy(sgtr_group* g);
int sgtr_comm_init_loopback(sgtr_ctx* ctx, sgtr_group* group, int32_t rank);

#ifdef __cplusplus
}
#endif
#endif
