"""SH colour extension on the GPU (include/sgtr.h): against the
oracle's restatement of the same definition (tests/test_oracle_sh.py pins
that restatement by its own mathematics; the reference itself is SH degree 0,
so this parity is unpinned against the reference)."""
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


@pytest.fixture
def orc3(orc):
    orc.set_sh_degree(3)
    yield orc
    orc.set_sh_degree(0)


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.max(np.abs(a - b)) / max(float(np.max(np.abs(b))), 1e-30))


def _data(orc, **kw):
    cfg = dict(gt_splats=400, init_splats=400, views=4, image_size=48, seed=5, sh_degree=3)
    cfg.update(kw)
    return orc.make_synthetic(orc.SynthConfig(**cfg))


def test_generator_bit_identical(sp, orc3):
    ds = _data(orc3, width=56, height=40)
    g, i, cams = sp.make_synthetic(400, 400, 4, 56, 40, seed=5, sh_degree=3)
    assert np.array_equal(g.x, ds.gt_x) and np.array_equal(i.x, ds.init_x)
    assert g.sh_coefficients().shape == (400, 15, 3)


def test_zero_coefficients_render_like_degree0(sp, orc):
    ds = orc.make_synthetic(orc.SynthConfig(gt_splats=300, init_splats=300, views=2,
                                            image_size=40, seed=2))
    k = 300
    x3 = np.concatenate([ds.gt_x, np.zeros(45 * k)])
    for c in ds.cams:
        cam = sp.Camera.from_c(c)
        a = sp.rasterize(sp.Scene(ds.gt_x), cam).color
        b = sp.rasterize(sp.Scene(x3, sh_degree=3), cam).color
        assert np.array_equal(a, b)


def test_render_jvp_vjp_parity(sp, orc3):
    ds = _data(orc3)
    x = ds.gt_x
    r = np.random.default_rng(3)
    scene = sp.Scene(x, sh_degree=3)
    for c in ds.cams[:2]:
        cam = sp.Camera.from_c(c)
        img = sp.rasterize(scene, cam).color
        assert rel(img, orc3.rasterize(x, c)[0]) < IMG_TOL
        v = r.normal(size=x.size) * 1e-2
        assert rel(sp.rasterize_jvp(scene, cam, v), orc3.rasterize_jvp(x, c, v)) < IMG_TOL
        u = r.normal(size=(c.height, c.width, 3))
        assert rel(sp.rasterize_vjp(scene, cam, u), orc3.rasterize_vjp(x, c, u)) < GRAD_TOL


def test_gradient_hutchinson_radii_parity(sp, orc3):
    ds = _data(orc3, seed=7)
    x = ds.init_x.copy()
    x[14 * 400:] = 0.05 * np.random.default_rng(1).normal(size=45 * 400)
    scene = sp.Scene(x, sh_degree=3)
    views = [sp.Camera.from_c(c, g) for c, g in zip(ds.cams, ds.gts)]
    g, loss = sp.stochastic_gradient(scene, views, [1, 3])
    go, lo = orc3.stochastic_gradient(x, ds.cams, ds.gts, [1, 3])
    assert rel(g, go) < GRAD_TOL and loss == pytest.approx(lo, rel=1e-9)
    assert np.any(g[14 * 400:] != 0.0)
    z = np.where(np.random.default_rng(2).random(x.size) < 0.5, -1.0, 1.0)
    d = sp.hutchinson_diag(scene, views, [2], 1, lambda s: z)
    do = orc3.hutchinson_diag(x, ds.cams, ds.gts, [2], z[None, :])
    assert rel(d, do) < IMG_TOL
    eta, eo = sp.shd_radii(scene, 1e-6), orc3.shd_radii(x, 1e-6)
    rot = slice(6 * 400, 10 * 400)
    assert rel(np.delete(eta, np.s_[rot]), np.delete(eo, np.s_[rot])) < 1e-12


@pytest.mark.parametrize("kind", ["3dgs2tr", "adam-tr"])
def test_step_parity_sh3(sp, orc3, kind):
    ds = _data(orc3, seed=11, views=5)
    views = [sp.Camera.from_c(c, g) for c, g in zip(ds.cams, ds.gts)]
    st = sp.OptimizerState(ds.init_x.size, 21, sh_degree=3)
    scene = sp.Scene(ds.init_x, sh_degree=3)
    ost = orc3.State(ds.init_x.size, 21)
    xo = ds.init_x.copy()
    opts = sp.OptimizerOptions(kind=kind, batch_size=2,
                               schedule=sp.TrustRegionSchedule(1e-6, 1e-8, 20))
    oopts = orc3.TrOptions(total_steps=20, batch_size=2)
    for t in range(1, 5):
        dg = sp.optimizer_step(st, scene, views, opts)
        if kind == "3dgs2tr":
            do = orc3.step_3dgs2tr(ost, xo, ds.cams, ds.gts, oopts)
        else:
            do = orc3.step_adam(ost, xo, ds.cams, ds.gts, oopts, orc3.AdamOptions(), True)
        assert dg.batch_loss == pytest.approx(do["batch_loss"], rel=1e-8)
        assert rel(scene.x, xo) < IMG_TOL
    assert np.any(scene.x[14 * 400:] != 0.0)


def test_checkpoint_keeps_sh_degree(sp, orc3, tmp_path):
    ds = _data(orc3, seed=4)
    c = sp.Context()
    c.set_scene(ds.init_x, sh_degree=3)
    c.state_reset(1)
    c.checkpoint_save(tmp_path / "sh.ck")
    d = sp.Context()
    d.checkpoint_load(tmp_path / "sh.ck")
    assert d.sh_degree == 3 and np.array_equal(d.get_scene(), ds.init_x)
    with pytest.raises(sp.InvalidArgument, match="PLY"):
        c.save_scene(tmp_path / "sh.ply")


@pytest.mark.parametrize("deg", [1, 2])
def test_lower_degrees_render_gradient_step(sp, orc, deg):
    # degrees 1 and 2 (3 and 8 coefficients per channel): render, JVP, VJP,
    # gradient and a few 3DGS2-TR steps against the oracle
    orc.set_sh_degree(deg)
    try:
        nb = (deg + 1) ** 2 - 1
        ds = orc.make_synthetic(orc.SynthConfig(gt_splats=300, init_splats=300, views=4,
                                                image_size=40, seed=13 + deg, sh_degree=deg))
        x = ds.gt_x
        scene = sp.Scene(x, sh_degree=deg)
        r = np.random.default_rng(deg)
        for c in ds.cams[:2]:
            cam = sp.Camera.from_c(c)
            assert rel(sp.rasterize(scene, cam).color, orc.rasterize(x, c)[0]) < IMG_TOL
            v = r.normal(size=x.size) * 1e-2
            assert rel(sp.rasterize_jvp(scene, cam, v), orc.rasterize_jvp(x, c, v)) < IMG_TOL
            u = r.normal(size=(c.height, c.width, 3))
            assert rel(sp.rasterize_vjp(scene, cam, u), orc.rasterize_vjp(x, c, u)) < GRAD_TOL
        views = [sp.Camera.from_c(c, g) for c, g in zip(ds.cams, ds.gts)]
        st = sp.OptimizerState(ds.init_x.size, 3, sh_degree=deg)
        sc = sp.Scene(ds.init_x, sh_degree=deg)
        ost, xo = orc.State(ds.init_x.size, 3), ds.init_x.copy()
        opts = sp.OptimizerOptions(batch_size=2, schedule=sp.TrustRegionSchedule(1e-6, 1e-8, 20))
        oopts = orc.TrOptions(total_steps=20, batch_size=2)
        for _ in range(3):
            dg = sp.step_3dgs2tr(st, sc, views, opts)
            do = orc.step_3dgs2tr(ost, xo, ds.cams, ds.gts, oopts)
            assert dg.batch_loss == pytest.approx(do["batch_loss"], rel=1e-8)
            assert rel(sc.x, xo) < IMG_TOL
        assert sc.x.size == (14 + 3 * nb) * 300
    finally:
        orc.set_sh_degree(0)
