// ref_capi.cpp -- orc_* C-ABI implemented by calling the compiled REFERENCE.
//
// TEST INFRASTRUCTURE ONLY (see ref_capi.h).  Every entry point converts the
// flat arrays of oracle.h into the reference's own types (Scene via
// Scene::unpack, Camera, Image, Eigen::VectorXd through the stand-in) and
// calls the reference function named in its comment; nothing here restates
// reference arithmetic.  Exceptions map onto oracle.h's status codes:
// std::invalid_argument -> 1, splat::NumericError -> 2, anything else -> 3.
#include "ref_capi.h"

#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>
#include <vector>

#include "splat/checks.hpp"
#include "splat/config.hpp"
#include "splat/dataset.hpp"
#include "splat/errors.hpp"
#include "splat/harness.hpp"
#include "splat/image.hpp"
#include "splat/optimizer.hpp"
#include "splat/render.hpp"
#include "splat/residuals.hpp"
#include "splat/rng.hpp"
#include "splat/scene.hpp"
#include "splat/ssim.hpp"
#include "splat/trust_region.hpp"

namespace {

thread_local std::string g_err;

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const splat::NumericError& e) {
        g_err = e.what();
        return 2;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 3;
    }
}

Eigen::VectorXd vec(const double* p, int64_t n) {
    Eigen::VectorXd v(n);
    std::memcpy(v.data(), p, sizeof(double) * n);
    return v;
}
void put(const Eigen::VectorXd& v, double* out) {
    std::memcpy(out, v.data(), sizeof(double) * v.size());
}

splat::Scene scene_of(const double* x, int64_t k) {
    splat::Scene s;
    s.splats.resize(k);
    s.unpack(vec(x, 14 * k));
    return s;
}

splat::Image image_of(const double* p, int w, int h) {
    splat::Image img(w, h);
    if (p) std::memcpy(img.data.data(), p, sizeof(double) * 3 * w * h);
    return img;
}
void put_image(const splat::Image& img, double* out) {
    std::memcpy(out, img.data.data(), sizeof(double) * img.data.size());
}

splat::Camera cam_of(const orc_camera& c, const double* gt = nullptr) {
    splat::Camera o;
    o.id = c.id;
    o.width = c.width;
    o.height = c.height;
    o.fx = c.fx;
    o.fy = c.fy;
    o.cx = c.cx;
    o.cy = c.cy;
    o.q_wc = Eigen::Vector4d(c.q_wc[0], c.q_wc[1], c.q_wc[2], c.q_wc[3]);
    o.t_wc = Eigen::Vector3d(c.t_wc[0], c.t_wc[1], c.t_wc[2]);
    if (gt) o.gt = image_of(gt, c.width, c.height);
    return o;
}
orc_camera cam_to_c(const splat::Camera& c) {
    orc_camera o{};
    o.id = c.id;
    o.width = c.width;
    o.height = c.height;
    o.fx = c.fx;
    o.fy = c.fy;
    o.cx = c.cx;
    o.cy = c.cy;
    for (int a = 0; a < 4; ++a) o.q_wc[a] = c.q_wc[a];
    for (int a = 0; a < 3; ++a) o.t_wc[a] = c.t_wc[a];
    return o;
}
std::vector<splat::Camera> cams_of(const orc_camera* cams, const double* const* gts, int n) {
    std::vector<splat::Camera> v;
    v.reserve(n);
    for (int i = 0; i < n; ++i) v.push_back(cam_of(cams[i], gts ? gts[i] : nullptr));
    return v;
}

splat::RenderOptions render_of(const orc_render_opts* ro, int workers) {
    splat::RenderOptions r;
    if (ro) {
        r.z_near = ro->z_near;
        r.lowpass = ro->lowpass;
        r.alpha_clamp = ro->alpha_clamp;
        r.alpha_skip = ro->alpha_skip;
        r.t_stop = ro->t_stop;
        r.cutoff_sigma = ro->cutoff_sigma;
        r.background = Eigen::Vector3d(ro->background[0], ro->background[1], ro->background[2]);
    }
    r.workers = workers;
    return r;
}
splat::ResidualOptions residual_of(const orc_residual_opts* rs) {
    splat::ResidualOptions r;
    if (rs) {
        r.lambda = rs->lambda;
        r.floor = rs->floor_;
    }
    return r;
}
splat::OptimizerOptions options_of(const orc_tr_opts* o, const orc_residual_opts* rs,
                                   const orc_render_opts* ro, int workers) {
    splat::OptimizerOptions opt;
    opt.theta1 = o->theta1;
    opt.theta2 = o->theta2;
    opt.hess_interval = o->hess_interval;
    opt.hutch_samples = o->hutch_samples;
    opt.batch_size = o->batch_size;
    opt.hutch_batch_size = o->hutch_batch_size;
    opt.gamma_d = o->gamma_d;
    opt.schedule = {o->eps_start, o->eps_end, o->total_steps};
    opt.caps = {o->cap_mean, o->cap_scale, o->cap_rotation, o->cap_opacity, o->cap_color};
    opt.bounds = {o->s_min, o->alpha_min, o->alpha_max, o->c_min, o->c_max};
    opt.residual = residual_of(rs);
    opt.render = render_of(ro, workers);
    return opt;
}
void diag_out(const splat::StepDiagnostics& d, orc_diag* out, double* applied) {
    if (out) {
        out->batch_loss = d.batch_loss;
        out->gnorm = d.gnorm;
        out->step_pre = d.step_pre;
        out->step_post = d.step_post;
        out->clip_frac = d.clip_frac;
        out->eps = d.eps;
        out->max_step_over_radius = d.max_step_over_radius;
    }
    if (applied && d.applied_step.size() > 0) put(d.applied_step, applied);
}
splat::GaussianPrimitive prim_of(const double* p14) {
    splat::GaussianPrimitive p;
    p.mu = Eigen::Vector3d(p14[0], p14[1], p14[2]);
    p.scale = Eigen::Vector3d(p14[3], p14[4], p14[5]);
    p.quat = Eigen::Vector4d(p14[6], p14[7], p14[8], p14[9]);
    p.opacity = p14[10];
    p.color = Eigen::Vector3d(p14[11], p14[12], p14[13]);
    return p;
}

}  // namespace

struct orc_state {
    splat::OptimizerState st;
    orc_state(int64_t dim, uint64_t seed) : st(static_cast<int>(dim), seed) {}
};
struct orc_rng {
    splat::Rng r;
    explicit orc_rng(uint64_t seed) : r(seed) {}
};

extern "C" {

const char* orc_last_error(void) { return g_err.c_str(); }

int orc_set_sh_degree(int32_t degree) {
    if (degree == 0) return 0;
    g_err = "reference: SH degree > 0 is not part of the reference";
    return 1;
}

// render.cpp:155-173
int orc_rasterize(const double* x, int64_t k, const orc_camera* cam, const orc_render_opts* ro,
                  int workers, double* color, double* t_final) {
    return guarded([&] {
        const splat::RenderedImage r =
            splat::rasterize(scene_of(x, k), cam_of(*cam), render_of(ro, workers));
        put_image(r.color, color);
        if (t_final) std::memcpy(t_final, r.t_final.data(), sizeof(double) * r.t_final.size());
    });
}

// render.cpp:175-192
int orc_rasterize_jvp(const double* x, int64_t k, const orc_camera* cam,
                      const orc_render_opts* ro, int workers, const double* v, int64_t v_len,
                      double* tangent) {
    return guarded([&] {
        const splat::Image t = splat::rasterize_jvp(scene_of(x, k), cam_of(*cam), vec(v, v_len),
                                                    render_of(ro, workers));
        put_image(t, tangent);
    });
}

// render.cpp:262-331
int orc_rasterize_vjp(const double* x, int64_t k, const orc_camera* cam,
                      const orc_render_opts* ro, int workers, const double* adjoint,
                      int32_t adj_w, int32_t adj_h, double* grad) {
    return guarded([&] {
        put(splat::rasterize_vjp(scene_of(x, k), cam_of(*cam), image_of(adjoint, adj_w, adj_h),
                                 render_of(ro, workers)),
            grad);
    });
}

// render.hpp:34-63
int ref_project(const double* x, int64_t k, const orc_camera* cam, const orc_render_opts* ro,
                double* out) {
    return guarded([&] {
        const splat::Scene s = scene_of(x, k);
        const splat::Camera c = cam_of(*cam);
        const splat::RenderOptions r = render_of(ro, 1);
        for (int64_t i = 0; i < k; ++i) {
            const splat::GaussianPrimitive& p = s.splats[i];
            const splat::Projection<double> pr = splat::project<double>(p.mu, p.scale, p.quat, c, r);
            double* o = out + 8 * i;
            o[0] = pr.culled ? 1.0 : 0.0;
            o[1] = pr.depth;
            o[2] = pr.mu2d[0];
            o[3] = pr.mu2d[1];
            o[4] = pr.c00;
            o[5] = pr.c01;
            o[6] = pr.c11;
            o[7] = 0.0;
        }
    });
}

// ssim.cpp
int orc_ssim_map(const double* a, const double* b, int32_t w, int32_t h, double* out) {
    return guarded([&] { put_image(splat::ssim_map(image_of(a, w, h), image_of(b, w, h)), out); });
}
int orc_ssim_jvp(const double* a, const double* da, const double* b, int32_t w, int32_t h,
                 double* s, double* ds) {
    return guarded([&] {
        splat::Image so, dso;
        splat::ssim_jvp(image_of(a, w, h), image_of(da, w, h), image_of(b, w, h), so, dso);
        put_image(so, s);
        put_image(dso, ds);
    });
}
int orc_ssim_vjp(const double* a, const double* b, const double* up, int32_t w, int32_t h,
                 double* grad) {
    return guarded([&] {
        put_image(splat::ssim_vjp(image_of(a, w, h), image_of(b, w, h), image_of(up, w, h)), grad);
    });
}
double orc_mean_ssim(const double* a, const double* b, int32_t w, int32_t h) {
    double r = 0.0;
    if (guarded([&] { r = splat::mean_ssim(image_of(a, w, h), image_of(b, w, h)); }) != 0)
        return -1.0;
    return r;
}

// residuals.cpp
int orc_residual_vector(const double* rendered, const double* gt, int32_t w, int32_t h,
                        const orc_residual_opts* o, double* r) {
    return guarded([&] {
        put(splat::residual_vector(image_of(rendered, w, h), image_of(gt, w, h), residual_of(o)), r);
    });
}
int orc_residual_jvp(const double* rendered, const double* tangent, const double* gt, int32_t w,
                     int32_t h, const orc_residual_opts* o, double* dr) {
    return guarded([&] {
        put(splat::residual_jvp(image_of(rendered, w, h), image_of(tangent, w, h),
                                image_of(gt, w, h), residual_of(o)),
            dr);
    });
}
int orc_residual_vjp(const double* rendered, const double* gt, int32_t w, int32_t h,
                     const double* u, int64_t u_len, const orc_residual_opts* o, double* adj) {
    return guarded([&] {
        put_image(splat::residual_vjp(image_of(rendered, w, h), image_of(gt, w, h), vec(u, u_len),
                                      residual_of(o)),
                  adj);
    });
}
double orc_psnr(const double* a, const double* b, int64_t n) {
    splat::Image ia(static_cast<int>(n / 3), 1), ib(static_cast<int>(n / 3), 1);
    std::memcpy(ia.data.data(), a, sizeof(double) * n);
    std::memcpy(ib.data.data(), b, sizeof(double) * n);
    return splat::psnr(ia, ib);
}
void orc_quantize8(const double* in, int64_t n, double* out) {
    splat::Image ia(static_cast<int>(n / 3), 1);
    std::memcpy(ia.data.data(), in, sizeof(double) * n);
    put_image(splat::quantize8(ia), out);
}

// optimizer.cpp:18-104
int orc_view_jacobian_apply(const double* x, int64_t k, const orc_camera* cam, const double* gt,
                            const double* v, const orc_residual_opts* rs,
                            const orc_render_opts* ro, int workers, double* out) {
    return guarded([&] {
        put(splat::view_jacobian_apply(scene_of(x, k), cam_of(*cam, gt), vec(v, 14 * k),
                                       residual_of(rs), render_of(ro, workers)),
            out);
    });
}
int orc_view_jacobian_applyT(const double* x, int64_t k, const orc_camera* cam, const double* gt,
                             const double* u, const orc_residual_opts* rs,
                             const orc_render_opts* ro, int workers, double* grad) {
    return guarded([&] {
        const int64_t m = 6LL * cam->width * cam->height;
        put(splat::view_jacobian_applyT(scene_of(x, k), cam_of(*cam, gt), vec(u, m),
                                        residual_of(rs), render_of(ro, workers)),
            grad);
    });
}
int orc_stochastic_gradient(const double* x, int64_t k, const orc_camera* cams,
                            const double* const* gts, int32_t n_views, const int32_t* batch,
                            int32_t n_batch, const orc_residual_opts* rs,
                            const orc_render_opts* ro, int workers, double* g,
                            double* batch_loss) {
    return guarded([&] {
        const std::vector<int> b(batch, batch + n_batch);
        put(splat::stochastic_gradient(scene_of(x, k), cams_of(cams, gts, n_views), b,
                                       residual_of(rs), render_of(ro, workers), batch_loss),
            g);
    });
}
int orc_hutchinson_diag(const double* x, int64_t k, const orc_camera* cams,
                        const double* const* gts, int32_t n_views, const int32_t* batch,
                        int32_t n_batch, int32_t nu, const double* probes,
                        const orc_residual_opts* rs, const orc_render_opts* ro, int workers,
                        double* d) {
    return guarded([&] {
        const int64_t dim = 14 * k;
        const std::vector<int> b(batch, batch + n_batch);
        const splat::ProbeSource src = [&](int s) { return vec(probes + s * dim, dim); };
        put(splat::hutchinson_diag(scene_of(x, k), cams_of(cams, gts, n_views), b, nu, src,
                                   residual_of(rs), render_of(ro, workers)),
            d);
    });
}
double orc_objective(const double* x, int64_t k, const orc_camera* cams, const double* const* gts,
                     int32_t n_views, const orc_residual_opts* rs, const orc_render_opts* ro,
                     int workers) {
    double r = -1.0;
    guarded([&] {
        r = splat::objective(scene_of(x, k), cams_of(cams, gts, n_views), residual_of(rs),
                             render_of(ro, workers));
    });
    return r;
}
// checks.cpp:127-145
int orc_exact_gn_diagonal(const double* x, int64_t k, const orc_camera* cams,
                          const double* const* gts, int32_t n_views, const orc_residual_opts* rs,
                          const orc_render_opts* ro, int workers, double* d) {
    return guarded([&] {
        put(splat::exact_gn_diagonal(scene_of(x, k), cams_of(cams, gts, n_views), residual_of(rs),
                                     render_of(ro, workers)),
            d);
    });
}

// trust_region.cpp
int orc_shd_radii(const double* x, int64_t k, double eps, const double caps[5], double* eta) {
    return guarded([&] {
        const splat::RadiusCaps c{caps[0], caps[1], caps[2], caps[3], caps[4]};
        put(splat::shd_radii(scene_of(x, k), eps, c), eta);
    });
}
double orc_beta_rotation(const double* prim14, int32_t axis) {
    return splat::beta_rotation(prim_of(prim14), axis);
}
double orc_eps_at(double eps_start, double eps_end, int32_t total, int32_t t) {
    return splat::eps_at({eps_start, eps_end, total}, t);
}
double orc_hellinger_sq(double mass_a, const double* mu_a, const double* sigma_a, double mass_b,
                        const double* mu_b, const double* sigma_b) {
    splat::MassGaussian a, b;
    a.mass = mass_a;
    b.mass = mass_b;
    for (int i = 0; i < 3; ++i) {
        a.mu[i] = mu_a[i];
        b.mu[i] = mu_b[i];
        for (int j = 0; j < 3; ++j) {
            a.sigma(i, j) = sigma_a[3 * i + j];
            b.sigma(i, j) = sigma_b[3 * i + j];
        }
    }
    double r = -1.0;
    if (guarded([&] { r = splat::hellinger_sq(a, b); }) != 0) return -1.0;
    return r;
}

// optimizer.hpp:58-72 + optimizer.cpp:189-253
orc_state* orc_state_create(int64_t dim, uint64_t seed) { return new orc_state(dim, seed); }
void orc_state_destroy(orc_state* s) { delete s; }
void orc_state_rng_raw(orc_state* s, int64_t n, uint64_t* out) {
    for (int64_t i = 0; i < n; ++i) out[i] = s->st.rng.raw();
}
int orc_state_get(const orc_state* s, double* g_hat, double* d_hat, int64_t* t) {
    if (g_hat) put(s->st.g_hat, g_hat);
    if (d_hat) put(s->st.d_hat, d_hat);
    if (t) *t = s->st.t;
    return 0;
}
int orc_state_set(orc_state* s, const double* g_hat, const double* d_hat, int64_t t) {
    const int64_t n = s->st.g_hat.size();
    if (g_hat) s->st.g_hat = vec(g_hat, n);
    if (d_hat) s->st.d_hat = vec(d_hat, n);
    s->st.t = t;
    return 0;
}
int orc_state_get_adam(const orc_state* s, double* m, double* v) {
    if (m) put(s->st.adam_m, m);
    if (v) put(s->st.adam_v, v);
    return 0;
}
int orc_state_set_adam(orc_state* s, const double* m, const double* v) {
    const int64_t n = s->st.adam_m.size();
    if (m) s->st.adam_m = vec(m, n);
    if (v) s->st.adam_v = vec(v, n);
    return 0;
}
int orc_step_3dgs2tr(orc_state* s, double* x, int64_t k, const orc_camera* cams,
                     const double* const* gts, int32_t n_views, const orc_tr_opts* o,
                     const orc_residual_opts* rs, const orc_render_opts* ro, int workers,
                     orc_diag* diag, double* applied_step) {
    return guarded([&] {
        splat::Scene scene = scene_of(x, k);
        const splat::StepDiagnostics d = splat::step_3dgs2tr(
            s->st, scene, cams_of(cams, gts, n_views), options_of(o, rs, ro, workers));
        put(scene.pack(), x);
        diag_out(d, diag, applied_step);
    });
}
int orc_step_adam(orc_state* s, double* x, int64_t k, const orc_camera* cams,
                  const double* const* gts, int32_t n_views, const orc_tr_opts* o,
                  const orc_adam_opts* a, int32_t trust_region, const orc_residual_opts* rs,
                  const orc_render_opts* ro, int workers, const int32_t* s1, int32_t n1,
                  orc_diag* diag, double* applied_step) {
    (void)n1;
    return guarded([&] {
        if (s1) throw std::invalid_argument("reference: explicit S1 is not part of the reference");
        splat::OptimizerOptions opt = options_of(o, rs, ro, workers);
        opt.adam.beta1 = a->beta1;
        opt.adam.beta2 = a->beta2;
        opt.adam.eps = a->eps;
        opt.adam.lr_position = a->lr_position;
        opt.adam.lr_position_final = a->lr_position_final;
        opt.adam.lr_position_decay_steps = a->lr_position_decay_steps;
        opt.adam.lr_scale = a->lr_scale;
        opt.adam.lr_rotation = a->lr_rotation;
        opt.adam.lr_opacity = a->lr_opacity;
        opt.adam.lr_color = a->lr_color;
        opt.scene_extent = a->scene_extent;
        splat::Scene scene = scene_of(x, k);
        const std::vector<splat::Camera> views = cams_of(cams, gts, n_views);
        const splat::StepDiagnostics d = trust_region
                                             ? splat::step_adam_tr(s->st, scene, views, opt)
                                             : splat::step_adam(s->st, scene, views, opt);
        put(scene.pack(), x);
        diag_out(d, diag, applied_step);
    });
}

// rng.hpp
orc_rng* orc_rng_create(uint64_t seed) { return new orc_rng(seed); }
void orc_rng_destroy(orc_rng* r) { delete r; }
void orc_rng_raw(orc_rng* r, int64_t n, uint64_t* out) {
    for (int64_t i = 0; i < n; ++i) out[i] = r->r.raw();
}
void orc_rng_normal(orc_rng* r, int64_t n, double* out) {
    for (int64_t i = 0; i < n; ++i) out[i] = r->r.normal();
}
void orc_rng_uniform(orc_rng* r, int64_t n, double lo, double hi, double* out) {
    for (int64_t i = 0; i < n; ++i) out[i] = r->r.uniform(lo, hi);
}
void orc_rng_sample(orc_rng* r, int32_t n, int32_t k, int32_t* out) {
    const std::vector<int> s = r->r.sample_without_replacement(n, k);
    for (size_t i = 0; i < s.size(); ++i) out[i] = s[i];
}
void orc_rng_rademacher(orc_rng* r, int64_t n, double* out) {
    for (int64_t i = 0; i < n; ++i) out[i] = r->r.rademacher();
}

// dataset.cpp:25-67
int orc_make_synthetic(const orc_synth_cfg* cfg, const orc_render_opts* ro, int workers,
                       double* gt_x, double* init_x, orc_camera* cams, double* const* gts) {
    return guarded([&] {
        if ((cfg->width > 0 && cfg->width != cfg->image_size) ||
            (cfg->height > 0 && cfg->height != cfg->image_size) ||
            (cfg->size_scale > 0.0 && cfg->size_scale != 1.0) || cfg->sh_degree != 0)
            throw std::invalid_argument(
                "reference make_synthetic: W!=H / size-scale / SH extensions are not part of "
                "the reference");
        splat::RunConfig rc;
        rc.gt_splats = cfg->gt_splats;
        rc.init_splats = cfg->init_splats;
        rc.views = cfg->views;
        rc.image_size = cfg->image_size;
        rc.seed = cfg->seed;
        rc.sigma_init = cfg->sigma_init;
        rc.init_scale = cfg->init_scale;
        rc.init_opacity = cfg->init_opacity;
        rc.camera_radius = cfg->camera_radius;
        rc.camera_height = cfg->camera_height;
        rc.focal_factor = cfg->focal_factor;
        rc.workers = workers;
        if (ro) {
            if (ro->background[0] != ro->background[1] || ro->background[0] != ro->background[2])
                throw std::invalid_argument("reference make_synthetic: grey background only");
            rc.background = ro->background[0];
            rc.z_near = ro->z_near;
        }
        const splat::SyntheticDataset ds = splat::make_synthetic(rc);
        put(ds.gt.pack(), gt_x);
        put(ds.init.pack(), init_x);
        for (int v = 0; v < cfg->views; ++v) {
            cams[v] = cam_to_c(ds.cameras[v]);
            if (gts) put_image(ds.cameras[v].gt, gts[v]);
        }
    });
}

// checks.cpp make_check_scene
int orc_make_check_scene(int32_t splats, int32_t image_size, int32_t n_views, uint64_t seed,
                         double* x, orc_camera* cams, double* const* gts) {
    return guarded([&] {
        const splat::CheckScene cs = splat::make_check_scene(splats, image_size, n_views, seed);
        put(cs.scene.pack(), x);
        for (int v = 0; v < n_views; ++v) {
            cams[v] = cam_to_c(cs.views[v]);
            if (gts) put_image(cs.views[v].gt, gts[v]);
        }
    });
}

// scene.cpp:126-149
int orc_look_at_camera(const double eye[3], const double target[3], double fx, double fy,
                       int32_t width, int32_t height, orc_camera* out) {
    return guarded([&] {
        *out = cam_to_c(splat::look_at_camera(Eigen::Vector3d(eye[0], eye[1], eye[2]),
                                              Eigen::Vector3d(target[0], target[1], target[2]),
                                              fx, fy, width, height));
    });
}

// harness.cpp:43-58
int ref_evaluate_scene(const double* x, int64_t k, const orc_camera* cams,
                       const double* const* gts, int32_t n_views, const orc_render_opts* ro,
                       int workers, double* psnr, double* ssim) {
    return guarded([&] {
        const splat::EvalResult r = splat::evaluate_scene(
            scene_of(x, k), cams_of(cams, gts, n_views), render_of(ro, workers));
        for (int v = 0; v < n_views; ++v) {
            psnr[v] = r.view_psnr[v];
            ssim[v] = r.view_ssim[v];
        }
    });
}

}  // extern "C"
