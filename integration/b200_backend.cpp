// b200_backend.cpp -- the reference-side binding of the B200 drop-in.
//
// This is the translation unit a maintainer adds to the reference's
// splat_core (/root/reference/proj/CMakeLists.txt:19-35) IN PLACE OF
// src/render.cpp and src/optimizer.cpp.  It defines every public symbol
// those two files define, with the reference's own signatures
// (render.hpp:73-84, optimizer.hpp:15-141), by calling the C-ABI of
// libsgtr.so (include/sgtr.h).  Everything else in splat_core (scene,
// image, scene_io, ssim, residuals, trust_region, dataset, config, harness,
// checks) is linked unchanged, so train_run, evaluate_scene, the checks and
// the reference's own unit and acceptance suites run on the B200 through this
// file.  integration/Makefile builds it against the reference headers and
// links the reference's tests to it (tests/test_integration.py runs them).
//
// State mirroring (optimizer.hpp:58-72).  OptimizerState is the reference's
// struct, unchanged: ĝ, D̂, the ADAM moments and t are uploaded before each
// step and written back after it (also after a NumericError, with the
// reference's partial-update semantics, which the device reproduces), and
// the draws come from state.rng on the host in the reference's order
// (optimizer.cpp:192-211): S1, then on refresh steps S2 and the nu probes,
// one rademacher() per coordinate, passed to sgtr_step_3dgs2tr_explicit as
// bits.  After a failed step state.rng is left where the reference leaves
// it: after S1 when the gradient phase fails, after probe s when Hutchinson
// sample s fails (sgtr_step_failed_sample), after every draw otherwise.  The
// per-step cost of the mirror is 4 dim-vector copies each way (host <->
// device); a long-running caller that does not read the state between steps
// can keep it resident with splat::b200::keep_state_resident(true).
//
// Views are registered with sgtr_set_views when their identity changes (the
// vector's address and size, and each camera's id, intrinsics, pose and GT
// buffer); splat::b200::invalidate_views() forces a re-upload after an
// in-place edit of a GT image.  One device context serves the whole
// process (SGTR_DEVICE selects the GPU, default 0), used from one thread at
// a time like the reference's single control thread.
//
// One documented deviation: hutchinson_diag(..., probes, ...) calls the
// ProbeSource for all nu samples before the device runs; the reference
// calls it lazily per sample (optimizer.cpp:86-87), which differs only when
// a sample s < nu - 1 fails.  step_3dgs2tr does not have this deviation.
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "sgtr.h"
#include "splat/errors.hpp"
#include "splat/optimizer.hpp"
#include "splat/render.hpp"

namespace splat {
namespace b200 {
void keep_state_resident(bool on);
void invalidate_views();
}  // namespace b200

namespace {

void check(int rc) {
    if (rc == SGTR_OK) return;
    const std::string msg = sgtr_last_error();
    if (rc == SGTR_NUMERIC) throw NumericError(msg);
    if (rc == SGTR_INVALID_ARGUMENT) throw std::invalid_argument(msg);
    throw std::runtime_error(msg);
}

sgtr_camera to_c(const Camera& c) {
    sgtr_camera o{};
    o.id = c.id;
    o.width = c.width;
    o.height = c.height;
    o.fx = c.fx;
    o.fy = c.fy;
    o.cx = c.cx;
    o.cy = c.cy;
    for (int i = 0; i < 4; ++i) o.q_wc[i] = c.q_wc[i];
    for (int i = 0; i < 3; ++i) o.t_wc[i] = c.t_wc[i];
    return o;
}

sgtr_render_options to_c(const RenderOptions& r) {
    sgtr_render_options o{};
    o.z_near = r.z_near;
    o.lowpass = r.lowpass;
    o.alpha_clamp = r.alpha_clamp;
    o.alpha_skip = r.alpha_skip;
    o.t_stop = r.t_stop;
    o.cutoff_sigma = r.cutoff_sigma;
    for (int i = 0; i < 3; ++i) o.background[i] = r.background[i];
    return o;
}

sgtr_residual_options to_c(const ResidualOptions& r) { return {r.lambda, r.floor}; }

sgtr_optimizer_options to_c(const OptimizerOptions& p) {
    sgtr_optimizer_options o{};
    o.theta1 = p.theta1;
    o.theta2 = p.theta2;
    o.hess_interval = p.hess_interval;
    o.hutch_samples = p.hutch_samples;
    o.batch_size = p.batch_size;
    o.hutch_batch_size = p.hutch_batch_size;
    o.gamma_d = p.gamma_d;
    o.eps_start = p.schedule.eps_start;
    o.eps_end = p.schedule.eps_end;
    o.total_steps = p.schedule.total_steps;
    o.record_applied_step = 1;
    o.cap_mean = p.caps.mean;
    o.cap_scale = p.caps.scale;
    o.cap_rotation = p.caps.rotation;
    o.cap_opacity = p.caps.opacity;
    o.cap_color = p.caps.color;
    o.s_min = p.bounds.s_min;
    o.alpha_min = p.bounds.alpha_min;
    o.alpha_max = p.bounds.alpha_max;
    o.c_min = p.bounds.c_min;
    o.c_max = p.bounds.c_max;
    o.residual = to_c(p.residual);
    o.render = to_c(p.render);
    return o;
}

sgtr_adam_options to_c(const AdamOptions& a, double scene_extent) {
    sgtr_adam_options o{};
    o.beta1 = a.beta1;
    o.beta2 = a.beta2;
    o.eps = a.eps;
    o.lr_position = a.lr_position;
    o.lr_position_final = a.lr_position_final;
    o.lr_position_decay_steps = a.lr_position_decay_steps;
    o.lr_scale = a.lr_scale;
    o.lr_rotation = a.lr_rotation;
    o.lr_opacity = a.lr_opacity;
    o.lr_color = a.lr_color;
    o.scene_extent = scene_extent;
    return o;
}

// identity of a view list as sgtr_set_views saw it
struct ViewKey {
    const Camera* data = nullptr;
    size_t n = 0;
    std::vector<double> cams;
    std::vector<const double*> gts;
    bool operator==(const ViewKey& o) const {
        return data == o.data && n == o.n && cams == o.cams && gts == o.gts;
    }
};
ViewKey key_of(const std::vector<Camera>& views) {
    ViewKey k;
    k.data = views.data();
    k.n = views.size();
    for (const Camera& c : views) {
        const double f[] = {double(c.id), double(c.width), double(c.height), c.fx, c.fy, c.cx,
                            c.cy, c.q_wc[0], c.q_wc[1], c.q_wc[2], c.q_wc[3], c.t_wc[0],
                            c.t_wc[1], c.t_wc[2], double(c.gt.width), double(c.gt.height)};
        k.cams.insert(k.cams.end(), f, f + 16);
        k.gts.push_back(c.gt.data.data());
    }
    return k;
}

struct Device {
    sgtr_ctx* ctx = nullptr;
    ViewKey views;
    bool views_valid = false;
    bool resident = false;                // keep_state_resident
    const OptimizerState* owner = nullptr;  // state whose ĝ/D̂ sit on the device
    long owner_t = -1;
};
Device& dev() {
    static Device d;
    if (!d.ctx) {
        const char* e = std::getenv("SGTR_DEVICE");
        check(sgtr_create(e ? std::atoi(e) : 0, &d.ctx));
    }
    return d;
}

void upload_scene(Device& d, const Scene& scene) {
    const Eigen::VectorXd x = scene.pack();
    check(sgtr_set_scene(d.ctx, x.data(), scene.size()));
}

void register_views(Device& d, const std::vector<Camera>& views) {
    ViewKey k = key_of(views);
    if (d.views_valid && k == d.views) return;
    std::vector<sgtr_camera> cams;
    std::vector<const double*> gts;
    for (const Camera& c : views) {
        if (c.gt.width != c.width || c.gt.height != c.height)
            throw std::invalid_argument("residuals: image shape mismatch");
        cams.push_back(to_c(c));
        gts.push_back(c.gt.data.data());
    }
    check(sgtr_set_views(d.ctx, cams.data(), static_cast<int32_t>(cams.size()), gts.data()));
    d.views = std::move(k);
    d.views_valid = true;
}

void push_state(Device& d, const OptimizerState& st, bool adam) {
    if (d.resident && d.owner == &st && d.owner_t == st.t) return;
    check(sgtr_state_set(d.ctx, st.g_hat.data(), st.d_hat.data(), st.t));
    if (adam) check(sgtr_state_set_adam(d.ctx, st.adam_m.data(), st.adam_v.data()));
    d.owner = nullptr;
}

void pull_state(Device& d, OptimizerState& st, bool adam) {
    int64_t t = 0;
    if (d.resident) {
        check(sgtr_state_get(d.ctx, nullptr, nullptr, &t));
        d.owner = &st;
        d.owner_t = t;
    } else {
        check(sgtr_state_get(d.ctx, st.g_hat.data(), st.d_hat.data(), &t));
        if (adam) check(sgtr_state_get_adam(d.ctx, st.adam_m.data(), st.adam_v.data()));
    }
    st.t = t;
}

StepDiagnostics diag_of(Device& d, const sgtr_step_diagnostics& s, int dim) {
    StepDiagnostics out;
    out.batch_loss = s.batch_loss;
    out.gnorm = s.gnorm;
    out.step_pre = s.step_pre;
    out.step_post = s.step_post;
    out.clip_frac = s.clip_frac;
    out.eps = s.eps;
    out.max_step_over_radius = s.max_step_over_radius;
    out.applied_step.resize(dim);
    check(sgtr_get_applied_step(d.ctx, out.applied_step.data()));
    return out;
}

// step_adam / step_adam_tr (optimizer.cpp:222-253) on the device
StepDiagnostics adam_step(OptimizerState& state, Scene& scene, const std::vector<Camera>& views,
                          const OptimizerOptions& opt, bool trust_region) {
    Device& d = dev();
    upload_scene(d, scene);
    register_views(d, views);
    push_state(d, state, true);
    const std::vector<int> s1 =
        state.rng.sample_without_replacement(static_cast<int>(views.size()), opt.batch_size);
    const sgtr_optimizer_options o = to_c(opt);
    const sgtr_adam_options a = to_c(opt.adam, opt.scene_extent);
    sgtr_step_diagnostics sd{};
    const int rc = sgtr_step_adam_explicit(d.ctx, &o, &a, trust_region ? 1 : 0, s1.data(),
                                           static_cast<int32_t>(s1.size()), &sd);
    pull_state(d, state, true);
    check(rc);
    Eigen::VectorXd x(scene.dim());
    check(sgtr_get_scene(d.ctx, x.data()));
    scene.unpack(x);
    return diag_of(d, sd, scene.dim());
}

}  // namespace

namespace b200 {
void keep_state_resident(bool on) {
    dev().resident = on;
    dev().owner = nullptr;
}
void invalidate_views() { dev().views_valid = false; }
}  // namespace b200

// ------------------------------------------------------------------ render.cpp

RenderedImage rasterize(const Scene& scene, const Camera& cam, const RenderOptions& opt) {
    Device& d = dev();
    upload_scene(d, scene);
    const sgtr_camera c = to_c(cam);
    const sgtr_render_options ro = to_c(opt);
    RenderedImage out;
    out.color = Image(cam.width, cam.height);
    out.t_final.assign(static_cast<size_t>(cam.width) * cam.height, 0.0);
    check(sgtr_rasterize(d.ctx, &c, &ro, out.color.data.data(), out.t_final.data()));
    return out;
}

Image rasterize_jvp(const Scene& scene, const Camera& cam, const Eigen::VectorXd& v,
                    const RenderOptions& opt) {
    if (v.size() != scene.dim())
        throw std::invalid_argument("rasterize_jvp: direction length mismatch");
    Device& d = dev();
    upload_scene(d, scene);
    const sgtr_camera c = to_c(cam);
    const sgtr_render_options ro = to_c(opt);
    Image out(cam.width, cam.height);
    check(sgtr_rasterize_jvp(d.ctx, &c, &ro, v.data(), out.data.data()));
    return out;
}

Eigen::VectorXd rasterize_vjp(const Scene& scene, const Camera& cam, const Image& adjoint,
                              const RenderOptions& opt) {
    if (adjoint.width != cam.width || adjoint.height != cam.height)
        throw std::invalid_argument("rasterize_vjp: adjoint shape mismatch");
    Device& d = dev();
    upload_scene(d, scene);
    const sgtr_camera c = to_c(cam);
    const sgtr_render_options ro = to_c(opt);
    Eigen::VectorXd g(scene.dim());
    check(sgtr_rasterize_vjp(d.ctx, &c, &ro, adjoint.data.data(), g.data()));
    return g;
}

// ------------------------------------------------------------------ optimizer.cpp

OptimizerKind optimizer_kind_from_string(const std::string& s) {
    if (s == "3dgs2tr") return OptimizerKind::k3dgs2tr;
    if (s == "adam") return OptimizerKind::kAdam;
    if (s == "adam-tr") return OptimizerKind::kAdamTr;
    throw std::invalid_argument("unknown optimizer '" + s + "'");
}

Eigen::VectorXd view_jacobian_apply(const Scene& scene, const Camera& cam,
                                    const Eigen::VectorXd& v, const ResidualOptions& ropt,
                                    const RenderOptions& render) {
    if (v.size() != scene.dim())
        throw std::invalid_argument("rasterize_jvp: direction length mismatch");
    Device& d = dev();
    upload_scene(d, scene);
    const std::vector<Camera> one{cam};
    d.views_valid = false;  // a temporary list: never matches a later key
    register_views(d, one);
    d.views_valid = false;
    const sgtr_residual_options rs = to_c(ropt);
    const sgtr_render_options ro = to_c(render);
    Eigen::VectorXd out(6LL * cam.width * cam.height);
    check(sgtr_view_jacobian_apply(d.ctx, 0, v.data(), &rs, &ro, out.data()));
    return out;
}

Eigen::VectorXd view_jacobian_applyT(const Scene& scene, const Camera& cam,
                                     const Eigen::VectorXd& u, const ResidualOptions& ropt,
                                     const RenderOptions& render) {
    if (u.size() != 6LL * cam.width * cam.height)
        throw std::invalid_argument("residual_vjp: adjoint length mismatch");
    Device& d = dev();
    upload_scene(d, scene);
    const std::vector<Camera> one{cam};
    d.views_valid = false;
    register_views(d, one);
    d.views_valid = false;
    const sgtr_residual_options rs = to_c(ropt);
    const sgtr_render_options ro = to_c(render);
    Eigen::VectorXd g(scene.dim());
    check(sgtr_view_jacobian_applyT(d.ctx, 0, u.data(), &rs, &ro, g.data()));
    return g;
}

Eigen::VectorXd stochastic_gradient(const Scene& scene, const std::vector<Camera>& views,
                                    const std::vector<int>& batch, const ResidualOptions& ropt,
                                    const RenderOptions& render, double* batch_loss) {
    if (batch.empty()) throw std::invalid_argument("stochastic_gradient: empty batch");
    for (int vi : batch)
        if (vi < 0 || vi >= static_cast<int>(views.size()))
            throw std::out_of_range("vector::_M_range_check");
    Device& d = dev();
    upload_scene(d, scene);
    register_views(d, views);
    const sgtr_residual_options rs = to_c(ropt);
    const sgtr_render_options ro = to_c(render);
    Eigen::VectorXd g(scene.dim());
    double loss = 0.0;
    check(sgtr_stochastic_gradient(d.ctx, batch.data(), static_cast<int32_t>(batch.size()), &rs,
                                   &ro, g.data(), &loss));
    if (batch_loss) *batch_loss = loss;
    return g;
}

ProbeSource rademacher_probes(Rng& rng, int dim) {
    return [&rng, dim](int) {
        Eigen::VectorXd z(dim);
        for (int k = 0; k < dim; ++k) z[k] = rng.rademacher();
        return z;
    };
}

Eigen::VectorXd hutchinson_diag(const Scene& scene, const std::vector<Camera>& views,
                                const std::vector<int>& batch, int nu, const ProbeSource& probes,
                                const ResidualOptions& ropt, const RenderOptions& render) {
    if (nu < 1) throw std::invalid_argument("hutchinson_diag: nu must be >= 1");
    if (batch.empty()) throw std::invalid_argument("hutchinson_diag: empty batch");
    for (int vi : batch)
        if (vi < 0 || vi >= static_cast<int>(views.size()))
            throw std::out_of_range("vector::_M_range_check");
    const int dim = scene.dim();
    std::vector<double> z(static_cast<size_t>(nu) * dim);
    for (int s = 0; s < nu; ++s) {
        const Eigen::VectorXd zs = probes(s);
        if (zs.size() != dim)
            throw std::invalid_argument("hutchinson_diag: probe length mismatch");
        std::memcpy(z.data() + static_cast<size_t>(s) * dim, zs.data(), sizeof(double) * dim);
    }
    Device& d = dev();
    upload_scene(d, scene);
    register_views(d, views);
    const sgtr_residual_options rs = to_c(ropt);
    const sgtr_render_options ro = to_c(render);
    Eigen::VectorXd out(dim);
    check(sgtr_hutchinson_diag(d.ctx, batch.data(), static_cast<int32_t>(batch.size()), nu,
                               z.data(), &rs, &ro, out.data()));
    return out;
}

Eigen::VectorXd newton_step(const Eigen::VectorXd& g_hat, const Eigen::VectorXd& d_hat,
                            double gamma) {
    Eigen::VectorXd dx(g_hat.size());
    for (Eigen::Index k = 0; k < g_hat.size(); ++k) dx[k] = -g_hat[k] / std::max(d_hat[k], gamma);
    return dx;
}

StepDiagnostics step_3dgs2tr(OptimizerState& state, Scene& scene,
                             const std::vector<Camera>& views, const OptimizerOptions& opt) {
    Device& d = dev();
    upload_scene(d, scene);
    register_views(d, views);
    push_state(d, state, false);
    // the reference's draws, in its order, from state.rng (optimizer.cpp:192-211)
    const int m_views = static_cast<int>(views.size());
    const long t = state.t + 1;
    const std::vector<int> s1 = state.rng.sample_without_replacement(m_views, opt.batch_size);
    const Rng after_s1 = state.rng;
    const bool refresh = opt.hess_interval <= 1 || t % opt.hess_interval == 1;
    std::vector<int> s2;
    std::vector<uint32_t> bits;
    std::vector<Rng> after_probe;
    const int dim = scene.dim();
    const int nu = opt.hutch_samples;
    if (refresh) {
        s2 = state.rng.sample_without_replacement(m_views, opt.hutch_batch_size);
        const size_t words = (static_cast<size_t>(dim) + 31) / 32;
        bits.assign(words * std::max(nu, 0), 0u);
        for (int s = 0; s < nu; ++s) {
            uint32_t* b = bits.data() + s * words;
            for (int k = 0; k < dim; ++k)
                if (state.rng.rademacher() > 0.0) b[k >> 5] |= 1u << (k & 31);
            after_probe.push_back(state.rng);
        }
    }
    const sgtr_optimizer_options o = to_c(opt);
    sgtr_step_diagnostics sd{};
    const int rc = sgtr_step_3dgs2tr_explicit(
        d.ctx, &o, s1.data(), static_cast<int32_t>(s1.size()), s2.data(),
        static_cast<int32_t>(s2.size()), bits.empty() ? nullptr : bits.data(), nu, &sd);
    if (rc != SGTR_OK) {
        const std::string msg = sgtr_last_error();
        int32_t fs = -1;
        sgtr_step_failed_sample(d.ctx, &fs);
        if (fs >= 0 && fs < static_cast<int32_t>(after_probe.size()))
            state.rng = after_probe[fs];
        else if (msg.rfind("non-finite update in group", 0) != 0)
            state.rng = after_s1;  // the gradient phase failed: only S1 was drawn
        pull_state(d, state, false);
        check(rc);
    }
    pull_state(d, state, false);
    Eigen::VectorXd x(dim);
    check(sgtr_get_scene(d.ctx, x.data()));
    scene.unpack(x);
    return diag_of(d, sd, dim);
}

StepDiagnostics step_adam(OptimizerState& state, Scene& scene, const std::vector<Camera>& views,
                          const OptimizerOptions& opt) {
    return adam_step(state, scene, views, opt, false);
}

StepDiagnostics step_adam_tr(OptimizerState& state, Scene& scene,
                             const std::vector<Camera>& views, const OptimizerOptions& opt) {
    return adam_step(state, scene, views, opt, true);
}

StepDiagnostics optimizer_step(OptimizerState& state, Scene& scene,
                               const std::vector<Camera>& views, const OptimizerOptions& opt) {
    switch (opt.kind) {
        case OptimizerKind::k3dgs2tr: return step_3dgs2tr(state, scene, views, opt);
        case OptimizerKind::kAdam: return step_adam(state, scene, views, opt);
        default: return step_adam_tr(state, scene, views, opt);
    }
}

}  // namespace splat
