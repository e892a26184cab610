"""GPU parity: libsgtr.so (through the C-ABI) against the CPU oracle.

Tolerances are the north star's (BASELINE.json): sort order and tile lists
bit-exact; images, JVP tangents, Hessian diagonals 1e-4 relative; accumulated
gradients 1e-3 relative.  Relative error is max|a-b| / max|b|.
The projection records are additionally checked bit-for-bit, because the
binning's exactness rests on them.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

IMG_TOL = 1e-4
GRAD_TOL = 1e-3


@pytest.fixture(scope="module")
def sp():
    import __graft_entry__
    __graft_entry__.build()
    from paper_2602_00395_b200 import splat
    return splat


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.max(np.abs(a - b)) / max(float(np.max(np.abs(b))), 1e-30))


def cams_of(sp, orc_cams, gts=None):
    gts = gts or [None] * len(orc_cams)
    return [sp.Camera.from_c(c, g) for c, g in zip(orc_cams, gts)]


def axis_camera(sp, size=16):  # test_render.cpp:20-28
    return sp.Camera(0, 2.0 * size, 2.0 * size, size / 2.0 - 0.5, size / 2.0 - 0.5, size, size)


def centered_scene(sp, prims):  # test_render.cpp:30-38
    return sp.Scene.from_primitives([[0, 0, 1]] * len(prims), [[0.05] * 3] * len(prims),
                                    [[0, 0, 0, 1]] * len(prims), [p[0] for p in prims],
                                    [p[1] for p in prims])


# ------------------------------------------------------------------ reference KATs on the GPU
def test_single_splat_center(sp):  # test_render.cpp:42-54
    cam = axis_camera(sp)
    out = sp.rasterize(centered_scene(sp, [(0.8, [1, 0, 0])]), cam)
    px = py = int(cam.cx)
    assert out.color[py, px, 0] == pytest.approx(0.8, rel=1e-12)
    assert out.color[py, px, 1] == 0.0 and out.color[py, px, 2] == 0.0
    assert out.t_final[py, px] == pytest.approx(0.2, rel=1e-12)


def test_coincident_tie_by_index(sp):  # test_render.cpp:56-65
    cam = axis_camera(sp)
    out = sp.rasterize(centered_scene(sp, [(0.5, [1, 1, 1]), (0.5, [0, 0, 0])]), cam)
    assert out.color[int(cam.cy), int(cam.cx), 0] == pytest.approx(0.5, rel=1e-12)


def test_empty_scene(sp):  # test_render.cpp:67-79
    cam = axis_camera(sp, 8)
    out = sp.rasterize(sp.Scene(np.zeros(0)), cam, sp.RenderOptions(background=(0.25, 0.5, 0.75)))
    assert np.all(out.color[..., 0] == 0.25) and np.all(out.color[..., 2] == 0.75)
    assert np.all(out.t_final == 1.0)


def test_nonfinite_names_splat(sp):  # test_render.cpp:81-89
    s = centered_scene(sp, [(0.5, [1, 1, 1])] * 2)
    s.x[3 * 1 + 2] = np.inf
    with pytest.raises(sp.NumericError, match="splat 1"):
        sp.rasterize(s, axis_camera(sp, 8))


def test_vjp_zero_and_color(sp):  # test_render.cpp:161-178
    cam = axis_camera(sp)
    s = centered_scene(sp, [(0.3, [0.2, 0.9, 0.4])])
    adj = np.zeros((16, 16, 3))
    assert np.linalg.norm(sp.rasterize_vjp(s, cam, adj)) == 0.0
    adj[int(cam.cy), int(cam.cx), 1] = 1.0
    g = sp.rasterize_vjp(s, cam, adj)
    assert g[s.color_offset() + 1] == pytest.approx(0.3, rel=1e-12)
    assert g[s.color_offset()] == 0.0


def test_storage_order_bitwise(sp, orc):  # test_render.cpp:91-100
    x, cams, _ = orc.make_check_scene(10, 16, 1, 42)
    mu, s, q, a, c = orc.unpack(x)
    xr = orc.pack(mu[::-1], s[::-1], q[::-1], a[::-1], c[::-1])
    cam = cams_of(sp, cams)[0]
    assert np.array_equal(sp.rasterize(sp.Scene(x), cam).color,
                          sp.rasterize(sp.Scene(xr), cam).color)


def test_jvp_zero_and_dead(sp, orc):  # test_render.cpp:114-132
    x, ocams, _ = orc.make_check_scene(6, 16, 1, 3)
    cam = cams_of(sp, ocams)[0]
    assert np.all(sp.rasterize_jvp(sp.Scene(x), cam, np.zeros_like(x)) == 0.0)
    mu, s, q, a, c = orc.unpack(x)
    behind = cam.center() - cam.rotation()[2]
    x2 = orc.pack(np.vstack([mu, behind]), np.vstack([s, s[0]]), np.vstack([q, q[0]]),
                  np.append(a, a[0]), np.vstack([c, c[0]]))
    k = x2.size // 14
    v = np.zeros_like(x2)
    v[11 * k + 3 * (k - 1)] = 1.0
    assert np.all(sp.rasterize_jvp(sp.Scene(x2), cam, v) == 0.0)


# ------------------------------------------------------------------ bit-exact stages
@pytest.fixture(scope="module")
def c1(orc):
    """BASELINE config 1: 10K splats, 4 views at 128x128 (reference generator)."""
    ds = orc.make_synthetic(orc.SynthConfig(gt_splats=10000, init_splats=10000, views=4,
                                            image_size=128, seed=1))
    return ds


def test_projection_bitexact(sp, orc, c1):
    ctx = sp.default_context()
    import ctypes as C
    from paper_2602_00395_b200 import _lib
    for x in (c1.gt_x, c1.init_x):
        ctx.set_scene(x)
        for oc in c1.cams:
            cam = sp.Camera.from_c(oc)
            out = np.empty((x.size // 14, 12))
            _lib.check(_lib.lib().sgtr_project(ctx.handle, C.byref(cam._c()),
                                               C.byref(sp.RenderOptions()._c()),
                                               out.ctypes.data_as(C.c_void_p)))
            ref = orc.project(x, oc)
            assert np.array_equal(out.view(np.uint64), ref.view(np.uint64))


def _gpu_binning(sp, x, cam):
    import ctypes as C
    from paper_2602_00395_b200 import _lib
    ctx = sp.default_context()
    ctx.set_scene(x)
    nv, nd = C.c_int32(), C.c_int64()
    L = _lib.lib()
    ro = sp.RenderOptions()._c()
    _lib.check(L.sgtr_dump_binning(ctx.handle, C.byref(cam._c()), C.byref(ro), C.byref(nv),
                                   None, C.byref(nd), None, None, None))
    nt = ((cam.width + 15) // 16) * ((cam.height + 15) // 16)
    order = np.empty(nv.value, np.int32)
    ts, te = np.empty(nt, np.int64), np.empty(nt, np.int64)
    lists = np.empty(nd.value, np.int32)
    p = lambda a: a.ctypes.data_as(C.c_void_p)
    _lib.check(L.sgtr_dump_binning(ctx.handle, C.byref(cam._c()), C.byref(ro), C.byref(nv),
                                   p(order), C.byref(nd), p(ts), p(te), p(lists)))
    return order, ts, te, lists


@pytest.mark.parametrize("which", ["gt", "init"])
def test_binning_bitexact(sp, orc, c1, which):
    x = c1.gt_x if which == "gt" else c1.init_x
    for oc in c1.cams:
        g = _gpu_binning(sp, x, sp.Camera.from_c(oc))
        r = orc.binning(x, oc)
        for a, b in zip(g, r):
            assert np.array_equal(a, b)


def test_binning_edge_cases(sp, orc):
    # splats straddling the image border, behind the camera, between pixel
    # centres, and non-square images with partial tiles
    rng = np.random.default_rng(5)
    k = 400
    mu = np.column_stack([rng.uniform(-1.2, 1.2, k), rng.uniform(-1.2, 1.2, k),
                          rng.uniform(-0.5, 3.0, k)])
    s = np.exp(rng.uniform(np.log(0.002), np.log(0.3), (k, 3)))
    q = rng.normal(size=(k, 4))
    x = orc.pack(mu, s, q, rng.uniform(0.1, 0.9, k), rng.uniform(0, 1, (k, 3)))
    for w, h in ((37, 23), (16, 16), (100, 7)):
        oc = orc.camera(width=w, height=h, fx=1.5 * h, fy=1.5 * h, cx=w / 2.0, cy=h / 2.0)
        g = _gpu_binning(sp, x, sp.Camera.from_c(oc))
        r = orc.binning(x, oc)
        for a, b in zip(g, r):
            assert np.array_equal(a, b)


def test_depth_order_near_ties(sp, orc):
    # depths that differ only in their lowest mantissa bits, in reverse index
    # order, plus exact ties: the depth sort runs on the high key bits and
    # repairs runs of equal high bits by the full key (binning.cu), which must
    # still give the reference's (depth, index) order (render.cpp:83-87)
    k = 300
    rng = np.random.default_rng(9)
    z = 2.0 + np.ldexp(np.arange(k)[::-1] % 37, -50)  # 37 distinct, ulp-scale apart
    mu = np.column_stack([rng.uniform(-0.2, 0.2, k), rng.uniform(-0.2, 0.2, k), z])
    s = np.full((k, 3), 0.05)
    q = np.tile([0.0, 0.0, 0.0, 1.0], (k, 1))
    x = orc.pack(mu, s, q, np.full(k, 0.5), rng.uniform(0, 1, (k, 3)))
    oc = orc.camera(width=48, height=40, fx=60.0, fy=60.0, cx=24.0, cy=20.0)
    g = _gpu_binning(sp, x, sp.Camera.from_c(oc))
    r = orc.binning(x, oc)
    for a, b in zip(g, r):
        assert np.array_equal(a, b)


# ------------------------------------------------------------------ renderer parity
def test_rasterize_parity(sp, orc, c1):
    for x in (c1.gt_x, c1.init_x):
        for oc in c1.cams:
            img, t = orc.rasterize(x, oc)
            out = sp.rasterize(sp.Scene(x), sp.Camera.from_c(oc))
            assert rel(out.color, img) < IMG_TOL
            assert rel(out.t_final, t) < IMG_TOL


def test_render_targets_match_oracle_gt(sp, orc, c1):
    # dataset.cpp:63: quantize8(rasterize(gt)) — GPU render of the targets
    ctx = sp.Context()
    ctx.set_scene(c1.gt_x)
    ctx.set_cameras(c1.cams)
    ctx.render_targets()
    for i, g in enumerate(c1.gts):
        got = ctx.get_target(i, 128, 128)
        assert np.mean(got != g) < 1e-4  # quantization-boundary flips only


def test_jvp_parity_and_adjoint(sp, orc):
    x, ocams, gts = orc.make_check_scene(8, 16, 2, 1)
    rng = np.random.default_rng(17)
    for oc in ocams:
        cam = sp.Camera.from_c(oc)
        for _ in range(3):
            v = rng.normal(size=x.size)
            u = rng.normal(size=(16, 16, 3))
            jv = sp.rasterize_jvp(sp.Scene(x), cam, v)
            assert rel(jv, orc.rasterize_jvp(x, oc, v)) < IMG_TOL
            vj = sp.rasterize_vjp(sp.Scene(x), cam, u)
            assert rel(vj, orc.rasterize_vjp(x, oc, u)) < GRAD_TOL
            lhs, rhs = float(np.sum(u * jv)), float(vj @ v)
            assert abs(lhs - rhs) <= 1e-9 * (1 + abs(lhs))  # test_render.cpp:180-208


def test_jvp_vjp_parity_c1(sp, orc, c1):
    rng = np.random.default_rng(3)
    x = c1.init_x
    oc = c1.cams[1]
    cam = sp.Camera.from_c(oc)
    v = rng.normal(size=x.size)
    u = rng.normal(size=(128, 128, 3))
    assert rel(sp.rasterize_jvp(sp.Scene(x), cam, v), orc.rasterize_jvp(x, oc, v)) < IMG_TOL
    assert rel(sp.rasterize_vjp(sp.Scene(x), cam, u), orc.rasterize_vjp(x, oc, u)) < GRAD_TOL


# ------------------------------------------------------------------ SSIM / residual parity
def test_ssim_residual_parity(sp, orc):
    rng = np.random.default_rng(9)
    for (w, h) in ((16, 16), (20, 14), (37, 6), (130, 67)):
        a, b = rng.uniform(size=(h, w, 3)), rng.uniform(size=(h, w, 3))
        da, up = rng.uniform(-1, 1, (h, w, 3)), rng.uniform(-1, 1, (h, w, 3))
        assert rel(sp.ssim_map(a, b), orc.ssim_map(a, b)) < 1e-12
        s, ds = sp.ssim_jvp(a, da, b)
        so, dso = orc.ssim_jvp(a, da, b)
        assert rel(s, so) < 1e-12 and rel(ds, dso) < 1e-10
        assert rel(sp.ssim_vjp(a, b, up), orc.ssim_vjp(a, b, up)) < 1e-10
        assert rel(sp.residual_vector(a, b), orc.residual_vector(a, b)) < 1e-12
        assert rel(sp.residual_jvp(a, da, b), orc.residual_jvp(a, da, b)) < 1e-10
        u = rng.normal(size=6 * w * h)
        assert rel(sp.residual_vjp(a, b, u), orc.residual_vjp(a, b, u)) < 1e-10


def test_ssim_small_image_rejected(sp):
    with pytest.raises(sp.InvalidArgument, match="smaller than the window"):
        sp.ssim_map(np.zeros((5, 8, 3)), np.zeros((5, 8, 3)))


# ------------------------------------------------------------------ optimizer parity
def test_stochastic_gradient_parity(sp, orc, c1):
    views = cams_of(sp, c1.cams, c1.gts)
    for batch in ([0], [2, 1], [0, 1, 2, 3]):
        g, loss = sp.stochastic_gradient(sp.Scene(c1.init_x), views, batch)
        go, losso = orc.stochastic_gradient(c1.init_x, c1.cams, c1.gts, batch)
        assert rel(g, go) < GRAD_TOL
        assert loss == pytest.approx(losso, rel=1e-9)


def test_gradient_vanishes_at_perfect_fit(sp, orc):  # test_optimizer.cpp:77-87
    x, ocams, _ = orc.make_check_scene(4, 12, 2, 71)
    views = [sp.Camera.from_c(c, orc.rasterize(x, c)[0]) for c in ocams]
    g, _ = sp.stochastic_gradient(sp.Scene(x), views, [0, 1])
    assert np.linalg.norm(g) <= 1e-6


def test_hutchinson_parity(sp, orc, c1):
    views = cams_of(sp, c1.cams, c1.gts)
    z = orc.Rng(11).rademacher(2 * c1.init_x.size).reshape(2, -1)
    d = sp.hutchinson_diag(sp.Scene(c1.init_x), views, [3], 2, lambda s: z[s])
    do = orc.hutchinson_diag(c1.init_x, c1.cams, c1.gts, [3], z)
    assert rel(d, do) < IMG_TOL


def test_hutchinson_unit_probe(sp, orc):  # test_optimizer.cpp:89-108
    x, ocams, gts = orc.make_check_scene(4, 12, 2, 73)
    views = cams_of(sp, ocams, gts)
    exact = orc.exact_gn_diagonal(x, ocams, gts)
    for k in (0, 7, x.size - 1):
        e = np.zeros(x.size)
        e[k] = 1.0
        d = sp.hutchinson_diag(sp.Scene(x), views, [0, 1], 1, lambda s: e)
        assert d[k] == pytest.approx(exact[k], rel=1e-9, abs=1e-300)


def test_shd_radii_parity(sp, orc, c1):
    # mean/scale/opacity/colour radii follow the oracle's op order (1e-12);
    # the rotation radii are certified with an algebraically equal but
    # cheaper form of the exact H^2 (update.cu), and both forms share the
    # ~1e-8 rounding floor of 1 - det_s/sqrt(det) (trust_region.cpp:183-194)
    for x in (c1.gt_x, c1.init_x):
        k = x.size // 14
        rot = slice(6 * k, 10 * k)
        for eps in (1e-6, 1e-4):
            e, eo = sp.shd_radii(sp.Scene(x), eps), orc.shd_radii(x, eps)
            assert rel(np.delete(e, np.s_[rot]), np.delete(eo, np.s_[rot])) < 1e-12
            assert rel(e[rot], eo[rot]) < 1e-6


# ------------------------------------------------------------------ Algorithm 1
def _tr_opts(sp, total, **kw):
    return sp.OptimizerOptions(schedule=sp.TrustRegionSchedule(1e-6, 1e-8, total), **kw)


def test_step_parity_rng_mode(sp, orc):
    ds = orc.make_synthetic(orc.SynthConfig(gt_splats=300, init_splats=300, views=6,
                                            image_size=48, seed=2))
    views = cams_of(sp, ds.cams, ds.gts)
    st = sp.OptimizerState(ds.init_x.size, 123)
    scene = sp.Scene(ds.init_x)
    ost = orc.State(ds.init_x.size, 123)
    xo = ds.init_x.copy()
    opts = _tr_opts(sp, 25, batch_size=2)
    oopts = orc.TrOptions(total_steps=25, batch_size=2)
    for t in range(1, 13):
        dg = sp.step_3dgs2tr(st, scene, views, opts)
        do = orc.step_3dgs2tr(ost, xo, ds.cams, ds.gts, oopts, want_applied=True)
        g, d, tt = st.ctx.state_get()
        go, dd, to = ost.get()
        assert tt == to == t
        assert dg.refreshed == (t % 10 == 1)
        assert rel(g, go) < GRAD_TOL
        assert rel(d, dd) < IMG_TOL
        assert rel(scene.x, xo) < 1e-6
        assert dg.batch_loss == pytest.approx(do["batch_loss"], rel=1e-8)
        assert dg.eps == do["eps"]
        assert dg.clip_frac == pytest.approx(do["clip_frac"], abs=2.0 / xo.size)
        assert dg.max_step_over_radius <= 1.0


def test_perfect_fit_fixed_point(sp, orc):  # test_optimizer.cpp:269-282
    x, ocams, _ = orc.make_check_scene(3, 12, 2, 109)
    views = [sp.Camera.from_c(c, orc.rasterize(x, c)[0]) for c in ocams]
    st = sp.OptimizerState(x.size, 13)
    scene = sp.Scene(x)
    for _ in range(5):
        sp.step_3dgs2tr(st, scene, views, _tr_opts(sp, 10))
    assert np.array_equal(scene.x, x)


def test_ema_cold_start(sp, orc):  # test_optimizer.cpp:187-202
    x, ocams, gts = orc.make_check_scene(4, 12, 3, 97)
    views = cams_of(sp, ocams, gts)
    batch = sp.Rng(55).sample_without_replacement(len(views), 1)
    g1, _ = sp.stochastic_gradient(sp.Scene(x), views, batch)
    st = sp.OptimizerState(x.size, 55)
    sp.step_3dgs2tr(st, sp.Scene(x), views, _tr_opts(sp, 10))
    assert np.linalg.norm(st.g_hat - 0.1 * g1) <= 1e-15 * max(1.0, np.linalg.norm(g1))


def test_step_nonfinite_parameter_names_splat(sp, orc):
    x, ocams, gts = orc.make_check_scene(4, 12, 2, 5)
    views = cams_of(sp, ocams, gts)
    x = x.copy()
    x[10 * 4 + 2] = np.nan  # opacity of splat 2
    st = sp.OptimizerState(x.size, 1)
    with pytest.raises(sp.NumericError, match="non-finite parameter in splat 2"):
        sp.step_3dgs2tr(st, sp.Scene(x), views, _tr_opts(sp, 10))
    assert st.t == 1  # the reference increments t before the first render


def test_blend_counters_match_oracle(sp, orc, c1):
    # the algorithmic-work units of the roofline: pairs reaching
    # the alpha evaluation (E) and contributing pairs (C), counted on the GPU
    # without contribution culling, must equal the reference count
    import ctypes as C
    from paper_2602_00395_b200 import _lib
    ctx = sp.default_context()
    for x in (c1.gt_x, c1.init_x):
        ctx.set_scene(x)
        for oc in c1.cams[:2]:
            e, c = C.c_int64(), C.c_int64()
            _lib.check(_lib.lib().sgtr_blend_stats(ctx.handle, C.byref(sp.Camera.from_c(oc)._c()),
                                                   C.byref(sp.RenderOptions()._c()),
                                                   C.byref(e), C.byref(c)))
            eo, co = orc.blend_stats(x, oc)
            assert abs(e.value - eo) <= 2 and abs(c.value - co) <= 2


def test_step_bitwise_deterministic(sp, orc):
    # no floating-point atomics on the path: two runs from the same state give
    # identical bits (the reference's acceptance criterion 10 property)
    ds = orc.make_synthetic(orc.SynthConfig(gt_splats=2000, init_splats=2000, views=6,
                                            image_size=64, seed=4))
    views = cams_of(sp, ds.cams, ds.gts)
    outs = []
    for _ in range(2):
        st = sp.OptimizerState(ds.init_x.size, 9)
        scene = sp.Scene(ds.init_x)
        for _ in range(3):
            sp.step_3dgs2tr(st, scene, views, _tr_opts(sp, 50, batch_size=3))
        g, d, _ = st.ctx.state_get()
        outs.append((scene.x.copy(), g, d))
    for a, b in zip(outs[0], outs[1]):
        assert np.array_equal(a, b)


def test_c2_scale_crop_parity(sp, orc):
    # BASELINE config 2 scale (100K splats, 512x512, size-scaled generator),
    # checked on a 128x96 crop so the CPU oracle stays fast
    gt, init, cams = sp.make_synthetic(gt_splats=100_000, init_splats=100_000, views=4,
                                       width=512, height=512, seed=2,
                                       size_scale=(64 / 100_000) ** (1 / 3))
    c = cams[1]
    crop = sp.Camera(c.id, c.fx, c.fy, c.cx - 200, c.cy - 210, 128, 96, c.q_wc, c.t_wc)
    oc = orc.camera(width=128, height=96, fx=crop.fx, fy=crop.fy, cx=crop.cx, cy=crop.cy,
                    q_wc=tuple(crop.q_wc), t_wc=tuple(crop.t_wc))
    img_g = sp.rasterize(gt, crop).color
    img_o, _ = orc.rasterize(gt.x, oc)
    assert rel(img_g, img_o) < IMG_TOL
    target = orc.quantize8(img_o)
    crop.gt = target
    g, loss = sp.stochastic_gradient(init, [crop], [0])
    go, losso = orc.stochastic_gradient(init.x, [oc], [target], [0])
    assert rel(g, go) < GRAD_TOL
    assert loss == pytest.approx(losso, rel=1e-9)
    for a, b in zip(_gpu_binning(sp, init.x, crop), orc.binning(init.x, oc)):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("lo,hi", [(-30.0, 0.0), (-760.0, 10.0), (-1e-6, 1e-6)])
def test_fast_exp_bit_identical(sp, lo, hi):
    # the rasterizer's exp (csrc/fastexp.cuh) is a constant-bank copy of the
    # CUDA library exp; every bit must agree over 2^24 inputs per range
    import ctypes as C
    from paper_2602_00395_b200 import _lib
    bad = C.c_int64(-1)
    _lib.check(_lib.lib().sgtr_check_fast_exp(1 << 24, lo, hi, 12345, C.byref(bad)))
    assert bad.value == 0


@pytest.mark.parametrize("kind", ["adam", "adam-tr"])
def test_adam_step_parity_rng_mode(sp, orc, kind):
    # step_adam / step_adam_tr (optimizer.cpp:222-253) against the oracle with
    # both drawing S1 from the same seeded Rng
    ds = orc.make_synthetic(orc.SynthConfig(gt_splats=300, init_splats=300, views=6,
                                            image_size=48, seed=3))
    views = cams_of(sp, ds.cams, ds.gts)
    st = sp.OptimizerState(ds.init_x.size, 77)
    scene = sp.Scene(ds.init_x)
    ost = orc.State(ds.init_x.size, 77)
    xo = ds.init_x.copy()
    opts = _tr_opts(sp, 25, batch_size=2, kind=kind, scene_extent=1.3,
                    adam=sp.AdamOptions(lr_position_decay_steps=4))
    oopts = orc.TrOptions(total_steps=25, batch_size=2)
    oadam = orc.AdamOptions(lr_position_decay_steps=4, scene_extent=1.3)
    for t in range(1, 7):
        dg = sp.optimizer_step(st, scene, views, opts)
        do = orc.step_adam(ost, xo, ds.cams, ds.gts, oopts, oadam, kind == "adam-tr",
                           want_applied=True)
        m, v = st.ctx.state_get_adam()
        mo, vo = ost.get_adam()
        assert st.t == t
        assert rel(m, mo) < GRAD_TOL and rel(v, vo) < GRAD_TOL
        # the ADAM direction normalises each coordinate by its own RMS, so a
        # coordinate's relative gradient error (not the vector's) reaches
        # the step: the accumulated-gradient tolerance applies
        assert rel(dg.applied_step, do["applied_step"]) < GRAD_TOL
        # ADAM's unit-RMS steps move the scene far more per step than the
        # trust region, so trajectory differences grow faster than in
        # test_step_parity_rng_mode
        assert rel(scene.x, xo) < IMG_TOL
        assert dg.batch_loss == pytest.approx(do["batch_loss"], rel=1e-8)
        assert dg.step_pre == pytest.approx(do["step_pre"], rel=GRAD_TOL)
        assert dg.eps == do["eps"]
        assert not dg.refreshed
        if kind == "adam":
            assert dg.clip_frac == -1.0 and dg.max_step_over_radius == 0.0
        else:
            assert dg.clip_frac == pytest.approx(do["clip_frac"], abs=2.0 / xo.size)
    g_hat, d_hat, _ = st.ctx.state_get()
    assert not g_hat.any() and not d_hat.any()


def test_optimizer_kind_from_string(sp):
    with pytest.raises(sp.InvalidArgument, match="unknown optimizer 'sgd'"):
        sp.optimizer_kind_from_string("sgd")
    assert sp.optimizer_kind_from_string("adam-tr") == "adam-tr"


def test_evaluate_scene_parity(sp, orc):
    # evaluate_scene (harness.cpp:43-58): quantize8(render) -> psnr, mean_ssim
    ds = orc.make_synthetic(orc.SynthConfig(gt_splats=400, init_splats=400, views=3,
                                            image_size=40, seed=8))
    x = ds.init_x
    # a second, non-square eval size through the W != H extension
    ds2 = orc.make_synthetic(orc.SynthConfig(gt_splats=400, init_splats=400, views=2,
                                             image_size=40, seed=8, width=56, height=36))
    cams = list(ds.cams) + list(ds2.cams)
    gts = list(ds.gts) + list(ds2.gts)
    views = cams_of(sp, cams, gts)
    ev = sp.evaluate_scene(sp.Scene(x), views)
    for i, (c, g) in enumerate(zip(cams, gts)):
        q = orc.quantize8(orc.rasterize(x, c)[0])
        assert ev.view_psnr[i] == pytest.approx(orc.psnr(q, g), abs=1e-9)
        assert ev.view_ssim[i] == pytest.approx(orc.mean_ssim(q, g), abs=1e-12)
    assert ev.mean_psnr == pytest.approx(np.mean(ev.view_psnr), rel=1e-15)
    assert ev.mean_ssim == pytest.approx(np.mean(ev.view_ssim), rel=1e-15)
    # a perfect render scores the reference's 100 dB cap (residuals.cpp:142)
    perfect = [sp.Camera.from_c(c, orc.quantize8(orc.rasterize(x, c)[0])) for c in ds.cams]
    assert sp.evaluate_scene(sp.Scene(x), perfect).view_psnr == [100.0] * 3
    with pytest.raises(sp.InvalidArgument, match="evaluate_scene: empty view list"):
        sp.evaluate_scene(sp.Scene(x), [])


def test_checkpoint_resume_is_bitwise(sp, orc, tmp_path):
    # optimizer-state checkpoint: a resumed run draws the
    # same S1/S2/probe stream and reproduces the uninterrupted one bit for bit
    ds = orc.make_synthetic(orc.SynthConfig(gt_splats=300, init_splats=300, views=6,
                                            image_size=32, seed=12))
    views = cams_of(sp, ds.cams, ds.gts)
    opts = _tr_opts(sp, 30, batch_size=2, record_applied_step=False)
    adam = _tr_opts(sp, 30, batch_size=2, kind="adam-tr", record_applied_step=False)

    def fresh():
        c = sp.Context()
        c.set_scene(ds.init_x)
        c.set_views(views)
        c.state_reset(5)
        return c

    a = fresh()
    for _ in range(4):
        a.step(opts)
    a.step(adam)
    a.checkpoint_save(tmp_path / "ck.bin")
    for _ in range(8):  # crosses the t = 11 refresh
        a.step(opts)
    b = fresh()
    b.set_scene(ds.gt_x)  # overwritten by the checkpoint
    b.checkpoint_load(tmp_path / "ck.bin")
    for _ in range(8):
        b.step(opts)
    assert np.array_equal(a.get_scene(), b.get_scene())
    for u, v in zip(a.state_get(), b.state_get()):
        assert np.array_equal(u, v)
    for u, v in zip(a.state_get_adam(), b.state_get_adam()):
        assert np.array_equal(u, v)


@pytest.mark.parametrize("bands", [2, 4])
def test_refresh_bands_sum_to_the_view(sp, orc, bands):
    # a refresh view split into row bands (one per rank, with a
    # one-tile halo for the 11x11 SSIM chain) must give the unsplit view's
    # Hutchinson sum; on one GPU the bands run back to back
    ds = orc.make_synthetic(orc.SynthConfig(gt_splats=600, init_splats=600, views=4,
                                            image_size=96, seed=21))
    views = cams_of(sp, ds.cams, ds.gts)
    out = []
    for b in (1, bands):
        c = sp.Context()
        c.set_scene(ds.init_x)
        c.set_views(views)
        c.state_reset(3)
        c.set_refresh_bands(b)
        c.step(_tr_opts(sp, 10, batch_size=2, hutch_samples=2))  # t = 1 refreshes
        out.append((c.state_get(), c.get_scene()))
    (g1, d1, _), x1 = out[0]
    (g2, d2, _), x2 = out[1]
    assert np.array_equal(g1, g2)          # the gradient phase is not banded
    assert rel(d2, d1) < 1e-12             # only the summation order differs
    assert rel(x2, x1) < 1e-12


# ---- ADAM known-answer tests of the reference on the device (test_optimizer.cpp:204-267)
def test_kat_adam_zero_gradient_stream(sp, orc):
    x, ocams, _ = orc.make_check_scene(4, 12, 2, 101)
    views = [sp.Camera.from_c(c, orc.rasterize(x, c)[0]) for c in ocams]
    st = sp.OptimizerState(x.size, 9)
    scene = sp.Scene(x)
    for _ in range(3):
        sp.step_adam(st, scene, views, sp.OptimizerOptions())
    assert np.array_equal(scene.x, x)


def test_kat_adam_first_step_is_the_group_rate(sp, orc):
    x, ocams, gts = orc.make_check_scene(4, 12, 2, 103)
    views = cams_of(sp, ocams, gts)
    opt = sp.OptimizerOptions(scene_extent=1.7)
    st = sp.OptimizerState(x.size, 11)
    d = sp.step_adam(st, sp.Scene(x), views, opt)
    a = opt.adam
    k = x.size // 14
    lr_pos = 1.7 * a.lr_position * (a.lr_position_final / a.lr_position) ** (
        1.0 / a.lr_position_decay_steps)
    lr = np.concatenate([np.full(3 * k, lr_pos), np.full(3 * k, a.lr_scale),
                         np.full(4 * k, a.lr_rotation), np.full(k, a.lr_opacity),
                         np.full(3 * k, a.lr_color)])
    sel = np.abs(st.adam_m) >= 1e-12
    assert sel.any()
    ap = np.abs(d.applied_step[sel])
    # doctest's Approx(lr).epsilon(1e-9): |a - b| < 1e-9 * (1 + max(|a|, |b|))
    assert np.all(np.abs(ap - lr[sel]) < 1e-9 * (1.0 + np.maximum(ap, lr[sel])))


def test_kat_adam_tr_vacuous_region_is_adam(sp, orc):
    x, ocams, gts = orc.make_check_scene(5, 12, 3, 107)
    views = cams_of(sp, ocams, gts)
    a, b = sp.Scene(x), sp.Scene(x)
    sa, sb = sp.OptimizerState(x.size, 77), sp.OptimizerState(x.size, 77)
    ob = sp.OptimizerOptions(schedule=sp.TrustRegionSchedule(1e100, 1e100, 10),
                             caps=sp.RadiusCaps(1e100, 1e100, 1e100, 1e100, 1e100))
    for _ in range(5):
        sp.step_adam(sa, a, views, sp.OptimizerOptions())
        sp.step_adam_tr(sb, b, views, ob)
    assert np.array_equal(a.x, b.x)


def test_kat_refresh_cadence_clip_eps(sp, orc):  # test_optimizer.cpp:163-185
    x, ocams, gts = orc.make_check_scene(4, 12, 3, 89)
    views = cams_of(sp, ocams, gts)
    total = 25
    opt = _tr_opts(sp, total)
    st = sp.OptimizerState(x.size, 123)
    scene = sp.Scene(x)
    last = st.d_hat
    for t in range(1, total + 1):
        d = sp.step_3dgs2tr(st, scene, views, opt)
        dh = st.d_hat
        assert (np.linalg.norm(dh - last) > 0.0) == (t % 10 == 1)
        last = dh
        assert d.max_step_over_radius <= 1.0
        assert d.eps == sp.eps_at(opt.schedule, t)
        assert 0.0 <= d.clip_frac <= 1.0
    assert st.t == total


def test_nccl_single_rank_communicator(sp, orc):
    # the multi-GPU plumbing on one GPU: dlopen of libnccl, ncclGetUniqueId,
    # ncclCommInitRank (unique id passed by value) and the per-step
    # ncclAllReduce over a 1-rank communicator must leave results unchanged
    ds = orc.make_synthetic(orc.SynthConfig(gt_splats=200, init_splats=200, views=4,
                                            image_size=32, seed=3))
    views = cams_of(sp, ds.cams, ds.gts)
    out = []
    for use_comm in (False, True):
        c = sp.Context()
        c.set_scene(ds.init_x)
        c.set_views(views)
        c.state_reset(2)
        if use_comm:
            c.comm_init(sp.nccl_unique_id(), 1, 0)
        for _ in range(3):
            c.step(_tr_opts(sp, 10, batch_size=2))
        out.append((c.get_scene(), c.state_get()))
    assert np.array_equal(out[0][0], out[1][0])
    for a, b in zip(out[0][1], out[1][1]):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("shards", [3, 7])
@pytest.mark.parametrize("kind", ["3dgs2tr", "adam-tr"])
def test_sharded_radii_match_unsharded(sp, orc, shards, kind):
    # the multi-GPU trust-region split (radii by splat range, shard-major
    # staging, all-gather) run back to back on one GPU: bit-identical steps
    ds = orc.make_synthetic(orc.SynthConfig(gt_splats=500, init_splats=500, views=4,
                                            image_size=40, seed=13))
    views = cams_of(sp, ds.cams, ds.gts)
    out = []
    for s in (1, shards):
        c = sp.Context()
        c.set_scene(ds.init_x)
        c.set_views(views)
        c.state_reset(4)
        c.set_tr_shards(s)
        diags = [c.step(_tr_opts(sp, 10, batch_size=2, kind=kind)) for _ in range(3)]
        out.append((c.get_scene(), c.state_get(), c.state_get_adam(), diags))
    assert np.array_equal(out[0][0], out[1][0])
    for a, b in zip(out[0][1][:2] + out[0][2], out[1][1][:2] + out[1][2]):
        assert np.array_equal(a, b)
    for da, db in zip(out[0][3], out[1][3]):
        assert (da.step_post, da.clip_frac, da.max_step_over_radius) == \
            (db.step_post, db.clip_frac, db.max_step_over_radius)


# ---- more of the reference's renderer / optimizer KATs on the device
def test_kat_transmittance_range_and_finite_image(sp, orc):  # test_render.cpp:102-112
    x, ocams, _ = orc.make_check_scene(12, 16, 2, 7)
    for oc in ocams:
        r = sp.rasterize(sp.Scene(x), sp.Camera.from_c(oc))
        assert np.all(r.t_final >= 0.0) and np.all(r.t_final <= 1.0)
        assert np.all(np.isfinite(r.color))


def test_kat_full_batch_is_the_single_view_average(sp, orc):  # test_optimizer.cpp:62-75
    x, ocams, gts = orc.make_check_scene(5, 12, 4, 67)
    views = cams_of(sp, ocams, gts)
    full, _ = sp.stochastic_gradient(sp.Scene(x), views, list(range(4)))
    mean = sum(sp.stochastic_gradient(sp.Scene(x), views, [i])[0] for i in range(4)) / 4.0
    assert np.linalg.norm(full - mean) / max(1e-30, np.linalg.norm(full)) <= 1e-12


def test_kat_invisible_splat_zero_diagonal(sp, orc):  # test_optimizer.cpp:110-130
    x, ocams, gts = orc.make_check_scene(4, 12, 2, 79)
    k = 4
    mu, s, q, a, c = orc.unpack(x)
    mu = np.vstack([mu, [0.0, 0.0, 100.0]])  # behind every ring camera
    s, q = np.vstack([s, s[0]]), np.vstack([q, q[0]])
    a, c = np.concatenate([a, a[:1]]), np.vstack([c, c[0]])
    x2 = orc.pack(mu, s, q, a, c)
    views = cams_of(sp, ocams, gts)
    rng = sp.Rng(5)
    d = sp.hutchinson_diag(sp.Scene(x2), views, [0, 1], 2, sp.rademacher_probes(rng, x2.size))
    kk = k  # index of the hidden splat (K = 5)
    K = k + 1
    idx = [3 * kk + c_ for c_ in range(3)] + [3 * K + 3 * kk + c_ for c_ in range(3)] + \
          [6 * K + 4 * kk + c_ for c_ in range(4)] + [10 * K + kk] + \
          [11 * K + 3 * kk + c_ for c_ in range(3)]
    assert np.all(d[idx] == 0.0)
    assert np.any(d != 0.0)


def test_alpha_clamp_branch_parity(sp, orc):
    # opacities near the box top (scene.cpp:49-57 clamps to 0.995) put the
    # centre pixels on render.cpp's alpha_bar >= 0.99 clamp, whose frozen
    # branch zeroes the alpha / conic tangents and adjoints of those pairs
    ds = orc.make_synthetic(orc.SynthConfig(gt_splats=200, init_splats=200, views=3,
                                            image_size=40, seed=21))
    mu, s, q, alpha, c = orc.unpack(ds.gt_x)
    rng = np.random.default_rng(5)
    alpha = rng.uniform(0.985, 0.995, size=alpha.shape)
    x = orc.pack(mu, s * 2.0, q, alpha, c)
    for oc in ds.cams:
        cam = sp.Camera.from_c(oc)
        img, t = orc.rasterize(x, oc)
        out = sp.rasterize(sp.Scene(x), cam)
        assert rel(out.color, img) < IMG_TOL and rel(out.t_final, t) < IMG_TOL
        v = rng.normal(size=x.size)
        u = rng.normal(size=img.shape)
        jv = sp.rasterize_jvp(sp.Scene(x), cam, v)
        assert rel(jv, orc.rasterize_jvp(x, oc, v)) < IMG_TOL
        vj = sp.rasterize_vjp(sp.Scene(x), cam, u)
        assert rel(vj, orc.rasterize_vjp(x, oc, u)) < GRAD_TOL
        lhs, rhs = float(np.sum(u * jv)), float(vj @ v)
        assert abs(lhs - rhs) <= 1e-9 * (1 + abs(lhs))
    e, cc = orc.blend_stats(x, ds.cams[0])
    assert cc > 0


def test_binning_and_render_large_rectangles(sp, orc):
    # fragments whose pixel rectangles span more than 64 tiles take K4's
    # warp-per-rectangle path (k_emit_large); mixed with small ones
    rng = np.random.default_rng(11)
    k = 120
    mu = np.column_stack([rng.uniform(-0.6, 0.6, k), rng.uniform(-0.6, 0.6, k),
                          rng.uniform(0.8, 2.5, k)])
    s = np.exp(rng.uniform(np.log(0.005), np.log(0.05), (k, 3)))
    s[:6] = [[0.6, 0.5, 0.4]] * 6  # > 64 tiles each at 320x256
    q = rng.normal(size=(k, 4))
    x = orc.pack(mu, s, q, rng.uniform(0.05, 0.6, k), rng.uniform(0, 1, (k, 3)))
    oc = orc.camera(width=320, height=256, fx=300.0, fy=300.0, cx=160.0, cy=128.0)
    pr = orc.project(x, oc)
    vis = pr[:, 0] == 0
    tiles = ((pr[vis, 5] - pr[vis, 4]) / 16 + 1) * ((pr[vis, 7] - pr[vis, 6]) / 16 + 1)
    assert np.sum(tiles > 64) >= 3
    cam = sp.Camera.from_c(oc)
    g = _gpu_binning(sp, x, cam)
    r = orc.binning(x, oc)
    for a, b in zip(g, r):
        assert np.array_equal(a, b)
    img, t = orc.rasterize(x, oc)
    out = sp.rasterize(sp.Scene(x), cam)
    assert rel(out.color, img) < IMG_TOL and rel(out.t_final, t) < IMG_TOL
    u = rng.normal(size=img.shape)
    assert rel(sp.rasterize_vjp(sp.Scene(x), cam, u), orc.rasterize_vjp(x, oc, u)) < GRAD_TOL


def test_wide_vjp_odd_frame(sp, orc, c1):
    """K10's 16x8-block path (frames of >= 4096 tiles) on a frame whose
    sides are not tile multiples (1030 x 1027: a partial tile column and row,
    the lower 16x8 block of the last tile row cut to 3 rows): VJP and the
    stochastic gradient against the oracle restatement."""
    W, H = 1030, 1027
    oc = type(c1.cams[0]).from_buffer_copy(c1.cams[0])
    s = W / oc.width
    oc.width, oc.height = W, H
    oc.fx, oc.fy = oc.fx * s, oc.fy * s
    oc.cx, oc.cy = W / 2.0, H / 2.0
    gt, _ = orc.rasterize(c1.gt_x, oc)
    scene = sp.Scene(c1.init_x)
    cam = sp.Camera.from_c(oc, gt)
    adj = np.random.default_rng(8).standard_normal((H, W, 3))
    assert rel(sp.rasterize_vjp(scene, cam, adj),
               orc.rasterize_vjp(c1.init_x, oc, adj)) < GRAD_TOL
    g, loss = sp.stochastic_gradient(scene, [cam], [0])
    go, lo = orc.stochastic_gradient(c1.init_x, [oc], [gt], [0])
    assert rel(g, go) < GRAD_TOL and loss == pytest.approx(lo, rel=1e-10)
