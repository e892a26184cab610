/* oracle.h — C-ABI of the CPU parity oracle.
 *
 * TEST INFRASTRUCTURE ONLY.  This library is a CPU restatement of the
 * reference 3DGS²-TR training iteration (/root/reference/proj, FP64 C++20)
 * and exists so that tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs have something to check against and
 * time.  The product (paper_2602_00395_b200/libsgtr.so) never links, loads or
 * calls it.
 *
 * Pinning: the reference itself IS built here as a second checker
 * (oracle/ref.mk: the unmodified /root/reference sources against the
 * Eigen-3.4-order / libpng / doctest stand-ins in oracle/refshim, into
 * oracle/_ref), and tests/test_reference.py shows this restatement equals it
 * bit for bit on every entry point both have (dataset, cameras, projection,
 * render / JVP / VJP, SSIM and residual chain, gradient, Hutchinson, radii,
 * full 3DGS2-TR / ADAM / ADAM-TR steps, Rng, error messages).  It is further
 * pinned by the reference's own KATs (tests/test_oracle_kat.py) and the
 * C++-standard mt19937_64 stream.  Sums follow Eigen 3.4's SSE2 order where
 * the reference's Eigen calls sum (see "Eigen order" in oracle.cpp), left to
 * right everywhere else.  The restatement additionally holds what the
 * reference has no counterpart for: the tile binning the GPU build adds, the
 * blend counters, the SH extension and teacher-forced steps.
 *
 * Layouts follow the reference exactly:
 *   x      : group-major double[14K] [mu 3K | s 3K | q 4K | alpha K | c 3K]
 *            (scene.hpp:37-52)
 *   images : row-major, channel-interleaved double[H*W*3] (image.hpp:10-27)
 *   residual vectors: double[6*H*W], L1 block then D-SSIM block,
 *            index c*H*W + y*W + x (residuals.hpp:17-22)
 * Status codes: 0 ok, 1 std::invalid_argument, 2 splat::NumericError,
 * 3 other; message in orc_last_error().
 */
#ifndef SGTR_ORACLE_H
#define SGTR_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct orc_camera {
    int32_t id, width, height, pad;
    double fx, fy, cx, cy;
    double q_wc[4]; /* unit (x, y, z, w) */
    double t_wc[3];
} orc_camera;

typedef struct orc_render_opts {
    double z_near, lowpass, alpha_clamp, alpha_skip, t_stop, cutoff_sigma;
    double background[3];
} orc_render_opts;

typedef struct orc_residual_opts {
    double lambda, floor_;
} orc_residual_opts;

typedef struct orc_tr_opts {
    double theta1, theta2;
    int32_t hess_interval, hutch_samples, batch_size, hutch_batch_size;
    double gamma_d;
    double eps_start, eps_end;
    int32_t total_steps, pad;
    double cap_mean, cap_scale, cap_rotation, cap_opacity, cap_color;
    double s_min, alpha_min, alpha_max, c_min, c_max;
} orc_tr_opts;

/* AdamOptions (optimizer.hpp:21-34) + OptimizerOptions::scene_extent */
typedef struct orc_adam_opts {
    double beta1, beta2, eps, lr_position, lr_position_final;
    int32_t lr_position_decay_steps, pad;
    double lr_scale, lr_rotation, lr_opacity, lr_color, scene_extent;
} orc_adam_opts;

typedef struct orc_diag {
    double batch_loss, gnorm, step_pre, step_post, clip_frac, eps,
        max_step_over_radius;
} orc_diag;

const char* orc_last_error(void);

/* SH colour extension (parity unpinned; degree 0 = the reference): scene
 * vectors become (14 + 3 * ((d+1)^2 - 1)) * K long, the SH block appended
 * after the reference's groups.  Process-wide setting. */
int orc_set_sh_degree(int32_t degree);

/* --- renderer (render.cpp:155-331) --- */
int orc_rasterize(const double* x, int64_t k, const orc_camera* cam,
                  const orc_render_opts* ro, int workers, double* color,
                  double* t_final);
int orc_rasterize_jvp(const double* x, int64_t k, const orc_camera* cam,
                      const orc_render_opts* ro, int workers, const double* v,
                      int64_t v_len, double* tangent);
int orc_rasterize_vjp(const double* x, int64_t k, const orc_camera* cam,
                      const orc_render_opts* ro, int workers,
                      const double* adjoint, int32_t adj_w, int32_t adj_h,
                      double* grad);
/* per-view blend statistics: E = pairs reaching the alpha evaluation,
 * C = contributing pairs (used for the algorithmic-work count in bench) */
int orc_blend_stats(const double* x, int64_t k, const orc_camera* cam,
                    const orc_render_opts* ro, int workers, int64_t* evaluated,
                    int64_t* contributing);
/* the contributing (pixel, splat) pairs of the blend (alpha_bar >= skip,
 * before termination) for the w x h window at (x0, y0): offsets[w*h+1]
 * (row-major pixels of the window) and the splat ids in blend order;
 * ids are written only when ids != NULL and offsets[w*h] <= cap */
int orc_blend_pairs(const double* x, int64_t k, const orc_camera* cam,
                    const orc_render_opts* ro, int workers, int32_t x0, int32_t y0,
                    int32_t w, int32_t h, int64_t* offsets, int32_t* ids, int64_t cap);
/* restated tile binning (the GPU build's new stage; no reference
 * counterpart): depth order of visible splats and per-tile lists.
 * order[n_visible]; tile_start/tile_end[n_tiles] (empty tiles [0, 0));
 * lists[n_dup].
 * Call with lists == NULL to get n_dup only. */
int orc_binning(const double* x, int64_t k, const orc_camera* cam,
                const orc_render_opts* ro, int32_t tile, int32_t* n_visible,
                int32_t* order, int64_t* n_dup, int64_t* tile_start,
                int64_t* tile_end, int32_t* lists);
/* projected fragment fields per splat (for bit-exactness tests):
 * out[k][12] = culled, depth, px, py, bx0, bx1, by0, by1, i00, i01, i11, 0 */
int orc_project(const double* x, int64_t k, const orc_camera* cam,
                const orc_render_opts* ro, double* out);

/* --- SSIM (ssim.cpp:15-175) --- */
int orc_ssim_map(const double* a, const double* b, int32_t w, int32_t h,
                 double* out);
int orc_ssim_jvp(const double* a, const double* da, const double* b, int32_t w,
                 int32_t h, double* s, double* ds);
int orc_ssim_vjp(const double* a, const double* b, const double* up, int32_t w,
                 int32_t h, double* grad);
double orc_mean_ssim(const double* a, const double* b, int32_t w, int32_t h);

/* --- residuals (residuals.cpp:27-144) --- */
int orc_residual_vector(const double* rendered, const double* gt, int32_t w,
                        int32_t h, const orc_residual_opts* o, double* r);
int orc_residual_jvp(const double* rendered, const double* tangent,
                     const double* gt, int32_t w, int32_t h,
                     const orc_residual_opts* o, double* dr);
int orc_residual_vjp(const double* rendered, const double* gt, int32_t w,
                     int32_t h, const double* u, int64_t u_len,
                     const orc_residual_opts* o, double* adj);
double orc_psnr(const double* a, const double* b, int64_t n);
void orc_quantize8(const double* in, int64_t n, double* out);

/* --- optimizer (optimizer.cpp:18-220) --- */
int orc_view_jacobian_apply(const double* x, int64_t k, const orc_camera* cam,
                            const double* gt, const double* v,
                            const orc_residual_opts* rs,
                            const orc_render_opts* ro, int workers,
                            double* out);
int orc_view_jacobian_applyT(const double* x, int64_t k,
                             const orc_camera* cam, const double* gt,
                             const double* u, const orc_residual_opts* rs,
                             const orc_render_opts* ro, int workers,
                             double* grad);
int orc_stochastic_gradient(const double* x, int64_t k, const orc_camera* cams,
                            const double* const* gts, int32_t n_views,
                            const int32_t* batch, int32_t n_batch,
                            const orc_residual_opts* rs,
                            const orc_render_opts* ro, int workers, double* g,
                            double* batch_loss);
/* probes: nu consecutive dense vectors of length 14K */
int orc_hutchinson_diag(const double* x, int64_t k, const orc_camera* cams,
                        const double* const* gts, int32_t n_views,
                        const int32_t* batch, int32_t n_batch, int32_t nu,
                        const double* probes, const orc_residual_opts* rs,
                        const orc_render_opts* ro, int workers, double* d);
double orc_objective(const double* x, int64_t k, const orc_camera* cams,
                     const double* const* gts, int32_t n_views,
                     const orc_residual_opts* rs, const orc_render_opts* ro,
                     int workers);
int orc_exact_gn_diagonal(const double* x, int64_t k, const orc_camera* cams,
                          const double* const* gts, int32_t n_views,
                          const orc_residual_opts* rs,
                          const orc_render_opts* ro, int workers, double* d);

/* --- trust region (trust_region.cpp:39-268) --- */
int orc_shd_radii(const double* x, int64_t k, double eps, const double caps[5],
                  double* eta);
double orc_beta_rotation(const double* prim14, int32_t axis);
double orc_eps_at(double eps_start, double eps_end, int32_t total, int32_t t);
double orc_hellinger_sq(double mass_a, const double* mu_a,
                        const double* sigma_a, double mass_b,
                        const double* mu_b, const double* sigma_b);

/* --- Algorithm 1 with the reference RNG order (optimizer.cpp:189-220) --- */
typedef struct orc_state orc_state;
orc_state* orc_state_create(int64_t dim, uint64_t seed);
void orc_state_destroy(orc_state* s);
/* n raw draws from the state's Rng (continues the optimizer's stream) */
void orc_state_rng_raw(orc_state* s, int64_t n, uint64_t* out);
int orc_state_get(const orc_state* s, double* g_hat, double* d_hat,
                  int64_t* t);
int orc_state_set(orc_state* s, const double* g_hat, const double* d_hat,
                  int64_t t);
int orc_step_3dgs2tr(orc_state* s, double* x, int64_t k,
                     const orc_camera* cams, const double* const* gts,
                     int32_t n_views, const orc_tr_opts* o,
                     const orc_residual_opts* rs, const orc_render_opts* ro,
                     int workers, orc_diag* diag, double* applied_step);
/* teacher-forced variant: the step's S1, S2 and probe draws supplied
 * explicitly (probes nu x 14K, only read on refresh steps) */
int orc_step_3dgs2tr_explicit(orc_state* s, double* x, int64_t k,
                              const orc_camera* cams, const double* const* gts,
                              int32_t n_views, const orc_tr_opts* o,
                              const orc_residual_opts* rs,
                              const orc_render_opts* ro, int workers,
                              const int32_t* s1, int32_t n1, const int32_t* s2,
                              int32_t n2, const double* probes, orc_diag* diag,
                              double* applied_step);

/* --- ADAM / ADAM-TR (optimizer.cpp:153-185, 222-253) --- */
int orc_state_get_adam(const orc_state* s, double* m, double* v);
int orc_state_set_adam(orc_state* s, const double* m, const double* v);
/* trust_region = 0: step_adam (apply_unclipped), 1: step_adam_tr
 * (apply_clipped); s1 = NULL draws S1 from the state's Rng */
int orc_step_adam(orc_state* s, double* x, int64_t k, const orc_camera* cams,
                  const double* const* gts, int32_t n_views, const orc_tr_opts* o,
                  const orc_adam_opts* a, int32_t trust_region,
                  const orc_residual_opts* rs, const orc_render_opts* ro,
                  int workers, const int32_t* s1, int32_t n1, orc_diag* diag,
                  double* applied_step);

/* --- reference Rng (rng.hpp:15-72) --- */
typedef struct orc_rng orc_rng;
orc_rng* orc_rng_create(uint64_t seed);
void orc_rng_destroy(orc_rng* r);
void orc_rng_raw(orc_rng* r, int64_t n, uint64_t* out);
void orc_rng_normal(orc_rng* r, int64_t n, double* out);
void orc_rng_uniform(orc_rng* r, int64_t n, double lo, double hi, double* out);
void orc_rng_sample(orc_rng* r, int32_t n, int32_t k, int32_t* out);
void orc_rng_rademacher(orc_rng* r, int64_t n, double* out);

/* --- synthetic data (dataset.cpp:25-67, checks.cpp:52-102) --- */
typedef struct orc_synth_cfg {
    int32_t gt_splats, init_splats, views, image_size;
    uint64_t seed;
    double sigma_init, init_scale, init_opacity, camera_radius, camera_height,
        focal_factor;
    /* declared extensions for the large configurations (0 = reference):
     * width x height images with fx = fy = focal_factor * height, and the
     * GT scale range, init_scale and sigma_init multiplied by size_scale */
    int32_t width, height;
    double size_scale;
    /* SH colour extension: GT coefficients 0.1 N(0,1) from a separate
     * stream (seed + 0x5348), init 0; must equal orc_set_sh_degree's */
    int32_t sh_degree, pad2;
} orc_synth_cfg;
/* gt_x[14*gt], init_x[14*init], cams[views], gts[views][H*W*3] */
int orc_make_synthetic(const orc_synth_cfg* cfg, const orc_render_opts* ro,
                       int workers, double* gt_x, double* init_x,
                       orc_camera* cams, double* const* gts);
int orc_make_check_scene(int32_t splats, int32_t image_size, int32_t n_views,
                         uint64_t seed, double* x, orc_camera* cams,
                         double* const* gts);
int orc_look_at_camera(const double eye[3], const double target[3], double fx,
                       double fy, int32_t width, int32_t height,
                       orc_camera* out);

#ifdef __cplusplus
}
#endif
#endif
