"""GPU parity against the compiled REFERENCE itself (oracle/_ref, the
unmodified /root/reference sources built against oracle/refshim), not the
restatement.  tests/test_reference.py shows the restatement equals the
reference bit for bit on CPU; these tests close the loop on the B200 for the
headline stages on BASELINE config 1 (10K splats, 4 views at 128x128) with
the north star's tolerances (projection keys bit-exact, images / tangents /
diagonals 1e-4, accumulated gradients 1e-3).
"""
import ctypes as C

import numpy as np
import pytest

from oracle import pyref

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not pyref.available(), reason="oracle/_ref not built")]

IMG_TOL = 1e-4
GRAD_TOL = 1e-3


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.max(np.abs(a - b)) / max(float(np.max(np.abs(b))), 1e-30))


@pytest.fixture(scope="module")
def sp():
    import __graft_entry__
    __graft_entry__.build()
    from paper_2602_00395_b200 import splat
    return splat


@pytest.fixture(scope="module")
def ref():
    return pyref.ref


@pytest.fixture(scope="module")
def c1(ref):
    return ref.make_synthetic(ref.SynthConfig(gt_splats=10000, init_splats=10000, views=4,
                                              image_size=128, seed=1))


def test_generator_matches_reference(sp, ref, c1):
    """sgtr_make_synthetic (scene + cameras) and the GPU-rendered quantised
    targets equal the reference's make_synthetic (dataset.cpp:25-67)."""
    gt, init, cams = sp.make_synthetic(gt_splats=10000, init_splats=10000, views=4, width=128,
                                       height=128, seed=1)
    assert np.array_equal(gt.x, c1.gt_x) and np.array_equal(init.x, c1.init_x)
    for a, b in zip(cams, c1.cams):
        assert bytes(a._c()) == bytes(b)
    ctx = sp.Context()
    ctx.set_scene(gt.x)
    ctx.set_cameras(cams)
    ctx.render_targets()
    for v in range(4):
        assert np.array_equal(ctx.get_target(v, 128, 128), c1.gts[v])


def test_projection_keys_match_reference(sp, ref, c1):
    from paper_2602_00395_b200 import _lib
    ctx = sp.default_context()
    for x in (c1.gt_x, c1.init_x):
        ctx.set_scene(x)
        for oc in c1.cams:
            cam = sp.Camera.from_c(oc)
            out = np.empty((x.size // 14, 12))
            _lib.check(_lib.lib().sgtr_project(ctx.handle, C.byref(cam._c()),
                                               C.byref(sp.RenderOptions()._c()),
                                               out.ctypes.data_as(C.c_void_p)))
            r = ref.project(x, oc)
            assert np.array_equal(out[:, 0], r[:, 0])
            vis = r[:, 0] == 0
            # depth (the sort key) and the 2-D mean, bit for bit
            assert np.array_equal(out[vis, 1:4].view(np.uint64), r[vis, 1:4].view(np.uint64))


def test_render_jvp_vjp_match_reference(sp, ref, c1):
    rng = np.random.default_rng(0)
    v = rng.standard_normal(c1.init_x.size)
    adj = rng.standard_normal((128, 128, 3))
    for which in (c1.init_x, c1.gt_x):
        scene = sp.Scene(which)
        for oc in c1.cams[:2]:
            cam = sp.Camera.from_c(oc)
            out = sp.rasterize(scene, cam)
            color, t = ref.rasterize(which, oc)
            assert rel(out.color, color) < 1e-12 and rel(out.t_final, t) < 1e-12
            assert rel(sp.rasterize_jvp(scene, cam, v), ref.rasterize_jvp(which, oc, v)) < IMG_TOL
            assert rel(sp.rasterize_vjp(scene, cam, adj),
                       ref.rasterize_vjp(which, oc, adj)) < GRAD_TOL


def test_view_jacobian_seams_match_reference(sp, ref, c1):
    """view_jacobian_apply / applyT (optimizer.cpp:18-34): the residual-space
    J_i v (the rasterize JVP pushed through the SSIM/L1 residual chain) and
    J_i^T u, against the reference on two views of each scene, plus the
    adjoint identity <u, J v> = <J^T u, v> on the device outputs."""
    rng = np.random.default_rng(11)
    v = rng.standard_normal(c1.init_x.size)
    u = rng.standard_normal(6 * 128 * 128)
    for which in (c1.init_x, c1.gt_x):
        scene = sp.Scene(which)
        for oc, gt in list(zip(c1.cams, c1.gts))[1:3]:
            cam = sp.Camera.from_c(oc, gt)
            jv = sp.view_jacobian_apply(scene, cam, v)
            jtu = sp.view_jacobian_applyT(scene, cam, u)
            assert rel(jv, ref.view_jacobian_apply(which, oc, gt, v)) < IMG_TOL
            assert rel(jtu, ref.view_jacobian_applyT(which, oc, gt, u)) < GRAD_TOL
            lhs, rhs = float(u @ jv), float(jtu @ v)
            assert abs(lhs - rhs) <= 1e-9 * max(abs(lhs), 1.0), (lhs, rhs)


def test_gradient_and_hutchinson_match_reference(sp, ref, c1):
    views = [sp.Camera.from_c(c, g) for c, g in zip(c1.cams, c1.gts)]
    scene = sp.Scene(c1.init_x)
    g, loss = sp.stochastic_gradient(scene, views, [2, 0])
    gr, lr = ref.stochastic_gradient(c1.init_x, c1.cams, c1.gts, [2, 0])
    assert rel(g, gr) < GRAD_TOL and loss == pytest.approx(lr, rel=1e-10)
    z = ref.Rng(3).rademacher(c1.init_x.size)
    d = sp.hutchinson_diag(scene, views, [1], 1, lambda s: z)
    dr = ref.hutchinson_diag(c1.init_x, c1.cams, c1.gts, [1], z)
    assert rel(d, dr) < IMG_TOL


@pytest.mark.parametrize("kind", ["3dgs2tr", "adam", "adam-tr"])
def test_steps_match_reference(sp, ref, kind):
    """Twelve steps with both sides drawing from the same seeded Rng
    (optimizer.cpp:189-253), including a Hessian refresh."""
    ds = ref.make_synthetic(ref.SynthConfig(gt_splats=300, init_splats=300, views=6,
                                            image_size=48, seed=2))
    views = [sp.Camera.from_c(c, g) for c, g in zip(ds.cams, ds.gts)]
    st = sp.OptimizerState(ds.init_x.size, 5)
    scene = sp.Scene(ds.init_x)
    rst = ref.State(ds.init_x.size, 5)
    xr = ds.init_x.copy()
    opts = sp.OptimizerOptions(schedule=sp.TrustRegionSchedule(1e-6, 1e-8, 25), batch_size=2,
                               kind=kind, scene_extent=1.3)
    ropts = ref.TrOptions(total_steps=25, batch_size=2)
    for t in range(1, 13):
        dg = sp.optimizer_step(st, scene, views, opts)
        if kind == "3dgs2tr":
            dr = ref.step_3dgs2tr(rst, xr, ds.cams, ds.gts, ropts)
        else:
            dr = ref.step_adam(rst, xr, ds.cams, ds.gts, ropts,
                               ref.AdamOptions(scene_extent=1.3), kind == "adam-tr")
        assert st.t == t
        assert dg.batch_loss == pytest.approx(dr["batch_loss"], rel=1e-8)
        assert dg.eps == dr["eps"]
        assert rel(scene.x, xr) < (1e-6 if kind == "3dgs2tr" else IMG_TOL)
    g, d, _ = st.ctx.state_get()
    gr, hr, _ = rst.get()
    if kind == "3dgs2tr":
        assert rel(g, gr) < GRAD_TOL and rel(d, hr) < IMG_TOL


@pytest.mark.parametrize("opts", [
    dict(background=(0.2, 0.3, 0.4)),
    dict(background=(0.9, 0.1, 0.5), alpha_clamp=0.9, t_stop=1e-3, lowpass=0.5,
         cutoff_sigma=2.5, alpha_skip=0.01),
])
def test_render_options_match_reference(sp, ref, c1, opts):
    """Non-default RenderOptions (render.hpp:12-22): a background colour (the
    VJP's behind-colour term and the JVP's bg * dT), a lower alpha clamp, an
    earlier transmittance stop, a wider low-pass, a tighter cut-off and a
    higher skip threshold -- forward, JVP and VJP against the reference."""
    rng = np.random.default_rng(4)
    v = rng.standard_normal(c1.init_x.size)
    adj = rng.standard_normal((128, 128, 3))
    ro_sp = sp.RenderOptions(**opts)
    ro_ref = ref.RenderOptions(**opts)
    for which in (c1.init_x, c1.gt_x):
        scene = sp.Scene(which)
        for oc in c1.cams[:2]:
            cam = sp.Camera.from_c(oc)
            out = sp.rasterize(scene, cam, ro_sp)
            color, t = ref.rasterize(which, oc, ro_ref)
            assert rel(out.color, color) < 1e-12 and rel(out.t_final, t) < 1e-12
            assert rel(sp.rasterize_jvp(scene, cam, v, ro_sp),
                       ref.rasterize_jvp(which, oc, v, ro_ref)) < IMG_TOL
            assert rel(sp.rasterize_vjp(scene, cam, adj, ro_sp),
                       ref.rasterize_vjp(which, oc, adj, ro_ref)) < GRAD_TOL


@pytest.mark.parametrize("lam,floor", [(0.0, 1e-12), (1.0, 1e-12), (0.5, 1e-6)])
def test_residual_options_match_reference(sp, ref, c1, lam, floor):
    """Non-default ResidualOptions (residuals.hpp:13-16): pure L1 (lambda 0),
    pure D-SSIM (lambda 1) and a mixed weight with a large floor (more
    residuals masked) -- the stochastic gradient and the Hutchinson diagonal
    against the reference."""
    views = [sp.Camera.from_c(c, g) for c, g in zip(c1.cams, c1.gts)]
    scene = sp.Scene(c1.init_x)
    ro = sp.ResidualOptions(lambda_=lam, floor=floor)
    rr = ref.ResidualOptions(lambda_=lam, floor=floor)
    g, loss = sp.stochastic_gradient(scene, views, [1, 3], ro)
    gr, lr = ref.stochastic_gradient(c1.init_x, c1.cams, c1.gts, [1, 3], rr)
    assert rel(g, gr) < GRAD_TOL and loss == pytest.approx(lr, rel=1e-10)
    z = ref.Rng(7).rademacher(c1.init_x.size)
    d = sp.hutchinson_diag(scene, views, [2], 1, lambda s: z, ro)
    dr = ref.hutchinson_diag(c1.init_x, c1.cams, c1.gts, [2], z, rr)
    assert rel(d, dr) < IMG_TOL


def test_step_options_match_reference(sp, ref):
    """3DGS2-TR steps under non-default optimizer options (optimizer.hpp:37-53,
    trust_region.hpp:66-72, scene.hpp:29-35): a refresh every 3rd step with
    nu = 2 probes over |S2| = 2 views, |S1| = 3, different EMA weights and
    damping, tight radius caps and parameter bounds, a non-default residual
    weight and render options -- against the reference drawing from the same
    seeded Rng."""
    ds = ref.make_synthetic(ref.SynthConfig(gt_splats=300, init_splats=300, views=6,
                                            image_size=48, seed=8))
    views = [sp.Camera.from_c(c, g) for c, g in zip(ds.cams, ds.gts)]
    caps = (0.05, 0.02, 0.3, 0.1, 0.2)
    bounds = (1e-3, 0.02, 0.98, 0.01, 1.2)
    lam, floor = 0.35, 1e-10
    render = dict(background=(0.1, 0.2, 0.3), alpha_clamp=0.95, t_stop=1e-3)
    opts = sp.OptimizerOptions(theta1=0.8, theta2=0.99, hess_interval=3, hutch_samples=2,
                               batch_size=3, hutch_batch_size=2, gamma_d=1e-9,
                               schedule=sp.TrustRegionSchedule(1e-5, 1e-7, 15),
                               caps=sp.RadiusCaps(*caps), bounds=sp.ParamBounds(*bounds),
                               residual=sp.ResidualOptions(lambda_=lam, floor=floor),
                               render=sp.RenderOptions(**render))
    ropts = ref.TrOptions(theta1=0.8, theta2=0.99, hess_interval=3, hutch_samples=2,
                          batch_size=3, hutch_batch_size=2, gamma_d=1e-9, eps_start=1e-5,
                          eps_end=1e-7, total_steps=15, caps=caps, bounds=bounds)
    rr = ref.ResidualOptions(lambda_=lam, floor=floor)
    ro = ref.RenderOptions(**render)
    st = sp.OptimizerState(ds.init_x.size, 9)
    scene = sp.Scene(ds.init_x)
    rst = ref.State(ds.init_x.size, 9)
    xr = ds.init_x.copy()
    for t in range(1, 8):  # refreshes at t = 1, 4, 7
        dg = sp.step_3dgs2tr(st, scene, views, opts)
        dr = ref.step_3dgs2tr(rst, xr, ds.cams, ds.gts, ropts, rr, ro)
        assert dg.batch_loss == pytest.approx(dr["batch_loss"], rel=1e-8)
        assert dg.eps == dr["eps"] and bool(dg.refreshed) == (t % 3 == 1)
        assert rel(scene.x, xr) < 1e-6
    g, d, _ = st.ctx.state_get()
    gr, hr, _ = rst.get()
    assert rel(g, gr) < GRAD_TOL and rel(d, hr) < IMG_TOL


@pytest.mark.parametrize("kind", ["adam", "adam-tr"])
def test_adam_options_match_reference(sp, ref, kind):
    """ADAM / ADAM-TR (optimizer.cpp:153-253) under non-default AdamOptions:
    other betas and epsilon, per-group rates, and a position rate that decays
    to its final value within the run (lr_position_decay_steps 4)."""
    ds = ref.make_synthetic(ref.SynthConfig(gt_splats=300, init_splats=300, views=6,
                                            image_size=48, seed=3))
    views = [sp.Camera.from_c(c, g) for c, g in zip(ds.cams, ds.gts)]
    ad = dict(beta1=0.8, beta2=0.99, eps=1e-12, lr_position=1e-3, lr_position_final=1e-5,
              lr_position_decay_steps=4, lr_scale=2e-3, lr_rotation=3e-3, lr_opacity=1e-2,
              lr_color=4e-3)
    opts = sp.OptimizerOptions(kind=kind, batch_size=2, scene_extent=2.5,
                               schedule=sp.TrustRegionSchedule(1e-6, 1e-8, 10),
                               adam=sp.AdamOptions(**ad))
    ropts = ref.TrOptions(batch_size=2, total_steps=10)
    st = sp.OptimizerState(ds.init_x.size, 4)
    scene = sp.Scene(ds.init_x)
    rst = ref.State(ds.init_x.size, 4)
    xr = ds.init_x.copy()
    for t in range(1, 7):
        dg = sp.optimizer_step(st, scene, views, opts)
        dr = ref.step_adam(rst, xr, ds.cams, ds.gts, ropts,
                           ref.AdamOptions(scene_extent=2.5, **ad), kind == "adam-tr")
        assert dg.batch_loss == pytest.approx(dr["batch_loss"], rel=1e-8)
        assert rel(scene.x, xr) < IMG_TOL


@pytest.mark.parametrize("W,H", [(53, 37), (17, 100), (200, 11)])
def test_odd_sizes_match_reference(sp, ref, c1, W, H):
    """Frames whose sides are not multiples of the 16-px tile, W != H, one
    side under a tile (partial tiles in K7/K10/K12, SSIM reflection on both
    borders of a short side): render, JVP, VJP, the stochastic gradient and
    the Hutchinson diagonal against the reference."""
    rng = np.random.default_rng(W * 1000 + H)
    oc = type(c1.cams[0]).from_buffer_copy(c1.cams[0])
    oc.width, oc.height = W, H
    oc.cx, oc.cy = W / 2.0, H / 2.0
    gt, _ = ref.rasterize(c1.gt_x, oc)
    scene = sp.Scene(c1.init_x)
    cam = sp.Camera.from_c(oc, gt)
    out = sp.rasterize(scene, cam)
    color, t = ref.rasterize(c1.init_x, oc)
    assert rel(out.color, color) < 1e-12 and rel(out.t_final, t) < 1e-12
    v = rng.standard_normal(c1.init_x.size)
    adj = rng.standard_normal((H, W, 3))
    assert rel(sp.rasterize_jvp(scene, cam, v), ref.rasterize_jvp(c1.init_x, oc, v)) < IMG_TOL
    assert rel(sp.rasterize_vjp(scene, cam, adj),
               ref.rasterize_vjp(c1.init_x, oc, adj)) < GRAD_TOL
    g, loss = sp.stochastic_gradient(scene, [cam], [0])
    gr, lr = ref.stochastic_gradient(c1.init_x, [oc], [gt], [0])
    assert rel(g, gr) < GRAD_TOL and loss == pytest.approx(lr, rel=1e-10)
    z = ref.Rng(W + H).rademacher(c1.init_x.size)
    d = sp.hutchinson_diag(scene, [cam], [0], 1, lambda s: z)
    dr = ref.hutchinson_diag(c1.init_x, [oc], [gt], [0], z)
    assert rel(d, dr) < IMG_TOL


def test_view_that_sees_nothing_matches_reference(sp, ref, c1):
    """A camera moved far off to the side (no splat in its frustum): the
    background image, a zero gradient from that view and an unchanged loss
    term on both sides; a batch mixing it with a normal view matches too."""
    oc = type(c1.cams[0]).from_buffer_copy(c1.cams[0])
    oc.t_wc[0] += 1e4
    gt = np.full((oc.height, oc.width, 3), 0.3)
    scene = sp.Scene(c1.init_x)
    cam = sp.Camera.from_c(oc, gt)
    out = sp.rasterize(scene, cam)
    color, t = ref.rasterize(c1.init_x, oc)
    assert np.array_equal(out.color, color) and np.array_equal(out.t_final, t)
    assert np.all(t == 1.0)
    g, loss = sp.stochastic_gradient(scene, [cam], [0])
    gr, lr = ref.stochastic_gradient(c1.init_x, [oc], [gt], [0])
    assert not np.any(g) and not np.any(gr) and loss == pytest.approx(lr, rel=1e-12)
    views = [cam, sp.Camera.from_c(c1.cams[1], c1.gts[1])]
    g2, l2 = sp.stochastic_gradient(scene, views, [1, 0])
    gr2, lr2 = ref.stochastic_gradient(c1.init_x, [oc, c1.cams[1]], [gt, c1.gts[1]], [1, 0])
    assert rel(g2, gr2) < GRAD_TOL and l2 == pytest.approx(lr2, rel=1e-10)


def _extreme_scene(c1, seed=21, W=200, H=200, K=1500):
    """A sparse C1-derived scene with extreme splats (see the test)."""
    oc = type(c1.cams[0]).from_buffer_copy(c1.cams[0])
    sc = W / oc.width
    oc.width, oc.height = W, H
    oc.fx, oc.fy = oc.fx * sc, oc.fy * sc
    oc.cx, oc.cy = W / 2.0, H / 2.0
    X = c1.init_x
    K0 = X.size // 14
    rng = np.random.default_rng(seed)
    sel = rng.choice(K0, K, replace=False)
    mu = X[:3 * K0].reshape(K0, 3)[sel].copy()
    s = 0.3 * X[3 * K0:6 * K0].reshape(K0, 3)[sel]
    q = X[6 * K0:10 * K0].reshape(K0, 4)[sel].copy()
    a = X[10 * K0:11 * K0][sel].copy()
    col = X[11 * K0:].reshape(K0, 3)[sel].copy()
    C = np.array(list(oc.t_wc))
    idx = rng.permutation(K)
    tiny, huge, op, behind, near = (idx[:100], idx[100:104], idx[104:204], idx[204:254],
                                    idx[254:304])
    s[tiny] = 1e-4
    s[huge] = rng.uniform(0.3, 0.8, (len(huge), 3))
    a[huge] = 0.05
    a[op] = rng.choice([0.0, 1e-9, 0.999999, 1.0], len(op))
    mu[behind] = C + (C - mu[behind])
    mu[near] = C + (mu[near] - C) * rng.uniform(0.001, 0.02, (len(near), 1))
    a[near] = 0.02
    return np.concatenate([mu.ravel(), s.ravel(), q.ravel(), a, col.ravel()]), oc


def test_extreme_scene_matches_reference(sp, ref, c1):
    """A sparse C1-derived 200x200 scene with splats behind the camera and
    straddling the near plane, sub-pixel splats (the low-pass dominates),
    splats wider than 64 tiles (the queued emission path) and opacities 0,
    1e-9, 1 - 1e-6 and 1: render, JVP, VJP and the gradient against the
    reference."""
    x, oc = _extreme_scene(c1)
    gt, _ = ref.rasterize(c1.gt_x, oc)
    rng = np.random.default_rng(22)
    scene = sp.Scene(x)
    cam = sp.Camera.from_c(oc, gt)
    out = sp.rasterize(scene, cam)
    color, t = ref.rasterize(x, oc)
    assert rel(out.color, color) < 1e-12 and rel(out.t_final, t) < 1e-12
    v = rng.standard_normal(x.size)
    adj = rng.standard_normal(color.shape)
    assert rel(sp.rasterize_jvp(scene, cam, v), ref.rasterize_jvp(x, oc, v)) < IMG_TOL
    assert rel(sp.rasterize_vjp(scene, cam, adj), ref.rasterize_vjp(x, oc, adj)) < GRAD_TOL
    g, loss = sp.stochastic_gradient(scene, [cam], [0])
    gr, lr = ref.stochastic_gradient(x, [oc], [gt], [0])
    assert rel(g, gr) < GRAD_TOL and loss == pytest.approx(lr, rel=1e-10)


@pytest.mark.parametrize("kind", ["3dgs2tr", "adam-tr"])
def test_extreme_scene_steps_match_reference(sp, ref, c1, kind):
    """Six 3DGS²-TR (Hessian refresh at step 1) or ADAM-TR steps on the
    extreme scene (opacities at the clamp bounds, sub-pixel scales, culled
    splats whose rows stay zero), both sides drawing from the same seeded
    Rng."""
    x, oc0 = _extreme_scene(c1)
    cams = [oc0]
    for c in c1.cams[1:3]:
        oc = type(c).from_buffer_copy(c)
        sc = oc0.width / oc.width
        oc.width, oc.height = oc0.width, oc0.height
        oc.fx, oc.fy = oc.fx * sc, oc.fy * sc
        oc.cx, oc.cy = oc0.cx, oc0.cy
        cams.append(oc)
    gts = [ref.rasterize(c1.gt_x, c)[0] for c in cams]
    views = [sp.Camera.from_c(c, g) for c, g in zip(cams, gts)]
    st = sp.OptimizerState(x.size, 7)
    scene = sp.Scene(x)
    rst = ref.State(x.size, 7)
    xr = x.copy()
    opts = sp.OptimizerOptions(schedule=sp.TrustRegionSchedule(1e-6, 1e-8, 6), batch_size=2,
                               scene_extent=1.3, kind=kind)
    ropts = ref.TrOptions(total_steps=6, batch_size=2)
    for t in range(1, 7):
        dg = sp.optimizer_step(st, scene, views, opts)
        if kind == "3dgs2tr":
            dr = ref.step_3dgs2tr(rst, xr, cams, gts, ropts)
        else:
            dr = ref.step_adam(rst, xr, cams, gts, ropts, ref.AdamOptions(scene_extent=1.3), True)
        assert dg.batch_loss == pytest.approx(dr["batch_loss"], rel=1e-8)
        assert dg.eps == dr["eps"]
        assert rel(scene.x, xr) < (1e-6 if kind == "3dgs2tr" else IMG_TOL)
