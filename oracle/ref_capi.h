/* ref_capi.h -- C-ABI over the compiled REFERENCE (oracle/_ref/libsplat_ref.so).
 *
 * TEST INFRASTRUCTURE ONLY.  oracle/ref_capi.cpp is compiled together with
 * the unmodified reference sources (/root/reference/proj/src/*.cpp, built by
 * oracle/ref.mk against the stand-ins in oracle/refshim/) and exports the
 * subset of oracle.h's orc_* entry points the reference has a counterpart
 * for, with the same names, structs, layouts and status codes -- so
 * oracle/pyref.py can bind it with pyoracle's own wrappers and every parity
 * test can ask the reference itself instead of the restatement.
 *
 * Exported from oracle.h (implemented by calling the reference): rasterize,
 * rasterize_jvp, rasterize_vjp, ssim_map/jvp/vjp, mean_ssim,
 * residual_vector/jvp/vjp, psnr, quantize8, view_jacobian_apply{,T},
 * stochastic_gradient, hutchinson_diag, objective, exact_gn_diagonal,
 * shd_radii, beta_rotation, eps_at, hellinger_sq, state_*, step_3dgs2tr
 * (the reference's own Rng draws), step_adam (S1 from the Rng), rng_*,
 * make_synthetic (reference generator; the W!=H / size-scale / SH
 * extensions are refused), make_check_scene, look_at_camera.
 * orc_set_sh_degree accepts 0 only.
 *
 * Not exported (no reference counterpart): blend_stats, binning, project
 * (see ref_project below), the *_explicit teacher-forced step.
 */
#ifndef SGTR_REF_CAPI_H
#define SGTR_REF_CAPI_H
#include "oracle.h"

#ifdef __cplusplus
extern "C" {
#endif

/* splat::project<double> (render.hpp:34-63) per splat:
 * out[k][6] = culled, depth, mu2d.x, mu2d.y, c00, c01, c11 is 7 values;
 * out has 8 doubles per splat: culled, depth, mu_x, mu_y, c00, c01, c11, 0 */
int ref_project(const double* x, int64_t k, const orc_camera* cam,
                const orc_render_opts* ro, double* out);

/* harness.cpp:43-58 evaluate_scene: per-view PSNR / SSIM of quantize8(render)
 * against each view's GT (gts[v]: H*W*3) */
int ref_evaluate_scene(const double* x, int64_t k, const orc_camera* cams,
                       const double* const* gts, int32_t n_views,
                       const orc_render_opts* ro, int workers, double* psnr,
                       double* ssim);

#ifdef __cplusplus
}
#endif
#endif
