// cpp_host.cpp — a C++ caller of the sgtr C-ABI (no Python involved).
//
//   g++ -std=c++17 -I include examples/cpp_host.cpp \
//       -L paper_2602_00395_b200 -lsgtr -Wl,-rpath,paper_2602_00395_b200
//
// Host-only entry points run anywhere; with a CUDA device present it also
// generates a small reference-generator scene, renders its targets on the
// GPU and runs three 3DGS²-TR steps.
#include <cmath>
#include <cstdio>
#include <vector>

#include "sgtr.h"

static int check(int rc, const char* what) {
    if (rc != SGTR_OK) std::printf("%s failed (%d): %s\n", what, rc, sgtr_last_error());
    return rc;
}

int main() {
    double eps = 0.0;
    if (check(sgtr_eps_at(1e-6, 1e-8, 1000, 500, &eps), "sgtr_eps_at")) return 1;
    if (std::fabs(eps - 1e-7) > 1e-19) return 2;

    sgtr_rng* rng = nullptr;
    uint64_t draws[3];
    check(sgtr_rng_new(5489, &rng), "sgtr_rng_new");
    check(sgtr_rng_draw(rng, 3, draws), "sgtr_rng_draw");
    sgtr_rng_free(rng);
    if (draws[0] != 14514284786278117030ull) return 3;  // mt19937_64(5489) first output

    int32_t pos[8], n = 0;
    check(sgtr_shard_views(8, 1, 4, pos, &n), "sgtr_shard_views");
    if (n != 2 || pos[0] != 1 || pos[1] != 5) return 4;

    sgtr_synth_config cfg{};
    cfg.gt_splats = 200; cfg.init_splats = 200; cfg.views = 5;
    cfg.width = 48; cfg.height = 32; cfg.seed = 1;
    cfg.sigma_init = 0.04; cfg.init_scale = 0.08; cfg.init_opacity = 0.5;
    cfg.camera_radius = 2.2; cfg.camera_height = 0.77; cfg.focal_factor = 2.0;
    cfg.size_scale = 1.0;
    std::vector<double> gt(14 * 200), init(14 * 200);
    std::vector<sgtr_camera> cams(5);
    if (check(sgtr_make_synthetic(&cfg, gt.data(), init.data(), cams.data()), "make_synthetic"))
        return 5;
    std::printf("host-only C-ABI ok\n");

    sgtr_ctx* ctx = nullptr;
    if (sgtr_create(0, &ctx) != SGTR_OK) {
        std::printf("no CUDA device: %s\n", sgtr_last_error());
        return 0;
    }
    sgtr_render_options ro{0.01, 0.3, 0.99, 1.0 / 255.0, 1e-4, 3.0, {0, 0, 0}};
    check(sgtr_set_scene(ctx, gt.data(), 200), "set_scene(gt)");
    check(sgtr_set_views(ctx, cams.data(), 5, nullptr), "set_views");
    check(sgtr_render_targets(ctx, &ro, 1), "render_targets");
    check(sgtr_set_scene(ctx, init.data(), 200), "set_scene(init)");
    check(sgtr_state_reset(ctx, 1), "state_reset");
    sgtr_optimizer_options o{};
    o.theta1 = 0.9; o.theta2 = 0.999; o.hess_interval = 10; o.hutch_samples = 1;
    o.batch_size = 2; o.hutch_batch_size = 1; o.gamma_d = 1e-12;
    o.eps_start = 1e-6; o.eps_end = 1e-8; o.total_steps = 100;
    o.cap_mean = o.cap_scale = o.cap_rotation = o.cap_opacity = o.cap_color = 1.0;
    o.s_min = 1e-6; o.alpha_min = 1e-4; o.alpha_max = 0.995; o.c_min = 1e-6; o.c_max = 1.5;
    o.residual = {0.2, 1e-12};
    o.render = ro;
    for (int t = 0; t < 3; ++t) {
        sgtr_step_diagnostics d{};
        if (check(sgtr_step_3dgs2tr(ctx, &o, &d), "step")) return 6;
        std::printf("step %d loss %.6e gnorm %.4e clip %.3f\n", t + 1, d.batch_loss, d.gnorm,
                    d.clip_frac);
    }
    sgtr_destroy(ctx);
    return 0;
}
