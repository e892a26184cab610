"""The reference's acceptance criterion 8 on the device (acceptance.cpp:112-131,
harness.cpp:178-340 fit_single_run): a single Gaussian displaced by 5 % of the
scene extent is fitted from 3 views with ADAM and with 3DGS²-TR for 500
iterations; every 3DGS²-TR step's per-parameter Hellinger motion stays within
1.15 ε, its largest motion is smaller than ADAM's, and both recover 40 dB.
The Hellinger motion (step_motion, coord_h2) is evaluated on the host with the
oracle's closed-form hellinger_sq (test infrastructure)."""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sp():
    import __graft_entry__
    __graft_entry__.build()
    from paper_2602_00395_b200 import splat
    return splat


def _cov(s, q):
    x, y, z, w = q
    r2 = x * x + y * y + z * z + w * w
    R = np.array([[r2 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
                  [2 * (x * y + w * z), r2 - 2 * (z * z + x * x), 2 * (y * z - w * x)],
                  [2 * (x * z - w * y), 2 * (y * z + w * x), r2 - 2 * (x * x + y * y)]]) / r2
    return R.T @ np.diag(np.asarray(s) ** 2) @ R


def _prim(x):  # single-splat layout mu 0..2 | s 3..5 | q 6..9 | alpha 10 | c 11..13
    return x[0:3], x[3:6], x[6:10], x[10], x[11:14]


def _coord_h2(orc, before, after, group, ch):  # harness.cpp:178-187
    mb, sb, qb, ab, cb = _prim(before)
    ma, sa, qa, aa, ca = _prim(after)
    det_b = np.prod(sb)
    wb, wa = ab * np.prod(sb), aa * np.prod(sa)
    if group == 4:
        wb, wa = wb * cb[ch], wa * ca[ch]
    return orc.hellinger_sq(wb, mb, _cov(sb, qb), wa, ma, _cov(sa, qa)) / det_b


def _max_motion(orc, before, delta):  # step_motion, harness.cpp:189-211
    worst = 0.0
    for j in range(14):
        after = before.copy()
        after[j] += delta[j]
        group = 0 if j < 3 else 1 if j < 6 else 2 if j < 10 else 3 if j == 10 else 4
        worst = max(worst, _coord_h2(orc, before, after, group, j - 11 if j >= 11 else 0))
    return worst


def test_criterion8_fit_single(sp, orc):
    ro = sp.RenderOptions()
    q = np.array([0.2, 0.1, 0.3, 0.95])
    gt = np.concatenate([[0.0, 0.0, 0.0], [0.16, 0.07, 0.11], q / np.linalg.norm(q), [0.78],
                         [0.9, 0.55, 0.25]])
    views = []
    for k in range(3):
        a = 2.0 * math.pi * k / 3.0
        cam = sp.look_at_camera((1.35 * math.cos(a), 1.35 * math.sin(a), 0.45), (0, 0, 0),
                                64.0, 64.0, 64, 64)
        cam.id = k
        cam.gt = sp.rasterize(sp.Scene(gt), cam, ro).color  # in-memory float targets
        views.append(cam)
    extent = sp.scene_extent(views)
    d = orc.Rng(1).normal(3)
    init = gt.copy()
    init[0:3] += 0.05 * extent * d / np.linalg.norm(d)
    res = {}
    for method in ("adam", "3dgs2tr"):
        opt = sp.OptimizerOptions(kind=method, scene_extent=extent,
                                  schedule=sp.TrustRegionSchedule(1e-6, 1e-8, 500))
        st = sp.OptimizerState(14, 1)
        scene = sp.Scene(init)
        h2, eps, hit40 = [], [], -1
        for t in range(1, 501):
            x0 = scene.x.copy()
            diag = sp.optimizer_step(st, scene, views, opt)
            h2.append(_max_motion(orc, x0, scene.x - x0))
            eps.append(diag.eps)
            if hit40 < 0:
                p = np.mean([sp.psnr(sp.rasterize(scene, c, ro).color, c.gt) for c in views])
                if p >= 40.0:
                    hit40 = t
        res[method] = (np.array(h2), np.array(eps), hit40)
    h2_tr, eps_tr, hit_tr = res["3dgs2tr"]
    h2_adam, _, hit_adam = res["adam"]
    assert np.all(h2_tr <= 1.15 * eps_tr)          # per-step bound held
    assert h2_tr.max() < h2_adam.max()             # calmer than ADAM
    assert 0 < hit_tr <= 500 and 0 < hit_adam <= 500


def _bench_train(sp, init, train, held, kind, iters=2000):  # acceptance.cpp:144-166
    ctx = sp.Context()
    ctx.set_scene(init)
    ctx.set_views(train)
    ctx.set_eval_views(held)
    ctx.state_reset(1)
    opt = sp.OptimizerOptions(kind=kind, scene_extent=sp.scene_extent(train),
                              schedule=sp.TrustRegionSchedule(1e-6, 1e-8, iters),
                              record_applied_step=False)
    psnr = {}
    for t in range(1, iters + 1):
        ctx.step(opt)
        if t % 100 == 0:
            psnr[t] = ctx.evaluate().mean_psnr
    return psnr


def test_criterion9_desk_scale_convergence(sp):
    # acceptance.cpp:168-212 on the default synthetic dataset (64 GT / 96 init
    # splats, 25 views of 64x64, seed 1, every 5th view held out): 3DGS2-TR is
    # at least ADAM's held-out PSNR at iteration 1000, ADAM-TR at least ADAM's
    # at 2000, and 3DGS2-TR's PSNR improves in >= 90 % of the 100-iteration
    # windows
    gt, init, cams = sp.make_synthetic()
    ctx = sp.Context()
    ctx.set_scene(gt.x)
    ctx.set_cameras(cams)
    ctx.render_targets(quantize=True)
    for i, c in enumerate(cams):
        c.gt = ctx.get_target(i, c.width, c.height)
    train = [c for c in cams if c.id % 5 != 0]  # split_views, dataset.cpp:79-85
    held = [c for c in cams if c.id % 5 == 0]
    tr = _bench_train(sp, init.x, train, held, "3dgs2tr")
    adam = _bench_train(sp, init.x, train, held, "adam")
    adamtr = _bench_train(sp, init.x, train, held, "adam-tr")
    assert tr[1000] >= adam[1000]
    assert adamtr[2000] >= adam[2000]
    seq = [tr[t] for t in sorted(tr)]
    mono = sum(b >= a for a, b in zip(seq, seq[1:])) / (len(seq) - 1)
    assert mono >= 0.9
