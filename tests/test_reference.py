"""The compiled reference as the parity anchor (CPU, no GPU).

oracle/ref.mk builds the UNMODIFIED reference (/root/reference/proj/src and
tests) against the stand-ins in oracle/refshim/ (Eigen subset modelling
Eigen 3.4's SSE2 evaluation order, libpng over zlib, doctest-lite) into
oracle/_ref/.  These tests:

* run the reference's own unit suite (tests/test_*.cpp: 83 cases, every
  hot-path KAT of test_render/test_optimizer/test_residuals/
  test_trust_region) and check it passes -- which validates the stand-ins;
* check that the restatement (oracle/) reproduces the reference BIT FOR BIT
  on the same inputs: dataset generator, cameras, projection, rasterize /
  JVP / VJP, SSIM and residual chain, stochastic gradient, Hutchinson
  diagonal, exact GN diagonal, trust-region radii, full 3DGS²-TR / ADAM /
  ADAM-TR steps, the Rng, and the error messages.

The GPU suites compare the CUDA path with both (tests/test_gpu_reference.py).
Skipped when oracle/_ref was not built (no /root/reference at build time).
"""
import os
import subprocess

import numpy as np
import pytest

from oracle import pyoracle as orc
from oracle import pyref

if not pyref.available():
    try:
        pyref.build()
    except Exception:  # pragma: no cover - no reference sources
        pass
pytestmark = pytest.mark.skipif(not pyref.available(),
                                reason="oracle/_ref not built (no /root/reference)")
ref = pyref.ref if pyref.available() else None


def same(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return a.shape == b.shape and np.array_equal(a, b)


def test_reference_unit_suite(tmp_path):
    r = subprocess.run([pyref.UNIT_TESTS], cwd=tmp_path, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    assert "test cases: 83 | 83 passed" in r.stdout, r.stdout


# ------------------------------------------------------------------ data
@pytest.fixture(scope="module")
def data():
    cfg = dict(gt_splats=300, init_splats=400, views=5, image_size=48, seed=3)
    d_o = orc.make_synthetic(orc.SynthConfig(**cfg))
    d_r = ref.make_synthetic(ref.SynthConfig(**cfg))
    return d_o, d_r


def test_make_synthetic_bitwise(data):  # dataset.cpp:25-67
    d_o, d_r = data
    assert same(d_o.gt_x, d_r.gt_x) and same(d_o.init_x, d_r.init_x)
    for a, b in zip(d_o.gts, d_r.gts):
        assert same(a, b)
    for a, b in zip(d_o.cams, d_r.cams):
        assert bytes(a) == bytes(b)


def test_make_check_scene_bitwise():  # checks.cpp make_check_scene
    xo, co, go = orc.make_check_scene(6, 16, 3, 41)
    xr, cr, gr = ref.make_check_scene(6, 16, 3, 41)
    assert same(xo, xr)
    assert all(bytes(a) == bytes(b) for a, b in zip(co, cr))
    assert all(same(a, b) for a, b in zip(go, gr))


def test_look_at_camera_bitwise():  # scene.cpp:126-149
    rng = np.random.default_rng(0)
    for _ in range(50):
        eye = rng.uniform(-3, 3, 3)
        tgt = rng.uniform(-0.5, 0.5, 3)
        a = orc.look_at_camera(eye, tgt, 100.0, 90.0, 64, 48)
        b = ref.look_at_camera(eye, tgt, 100.0, 90.0, 64, 48)
        assert bytes(a) == bytes(b)


# ------------------------------------------------------------------ renderer
@pytest.mark.parametrize("which", ["init", "gt"])
def test_projection_bitwise(data, which):  # render.hpp:34-63
    d_o, d_r = data
    x = d_o.init_x if which == "init" else d_o.gt_x
    for v in range(3):
        po = orc.project(x, d_o.cams[v])
        pr = ref.project(x, d_r.cams[v])
        assert same(po[:, 0], pr[:, 0])  # culled
        vis = po[:, 0] == 0
        assert same(po[vis, 1:4], pr[vis, 1:4])  # depth, mu2d


@pytest.mark.parametrize("which", ["init", "gt"])
def test_rasterize_bitwise(data, which):  # render.cpp:155-173
    d_o, d_r = data
    x = d_o.init_x if which == "init" else d_o.gt_x
    for v in range(2):
        a = orc.rasterize(x, d_o.cams[v])
        b = ref.rasterize(x, d_r.cams[v])
        assert same(a[0], b[0]) and same(a[1], b[1])
    ro = orc.RenderOptions(background=(0.2, 0.3, 0.4))
    rr = ref.RenderOptions(background=(0.2, 0.3, 0.4))
    assert same(orc.rasterize(x, d_o.cams[2], ro)[0], ref.rasterize(x, d_r.cams[2], rr)[0])


def test_rasterize_jvp_vjp_bitwise(data):  # render.cpp:175-331
    d_o, d_r = data
    x = d_o.gt_x
    rng = np.random.default_rng(1)
    v = rng.standard_normal(x.size)
    adj = rng.standard_normal((48, 48, 3))
    for c in range(2):
        assert same(orc.rasterize_jvp(x, d_o.cams[c], v), ref.rasterize_jvp(x, d_r.cams[c], v))
        assert same(orc.rasterize_vjp(x, d_o.cams[c], adj), ref.rasterize_vjp(x, d_r.cams[c], adj))


def test_ssim_and_residuals_bitwise(data):  # ssim.cpp, residuals.cpp
    d_o, d_r = data
    a = orc.rasterize(d_o.init_x, d_o.cams[0])[0]
    b = d_o.gts[0]
    rng = np.random.default_rng(2)
    da = rng.standard_normal(a.shape)
    assert same(orc.ssim_map(a, b), ref.ssim_map(a, b))
    for p, q in zip(orc.ssim_jvp(a, da, b), ref.ssim_jvp(a, da, b)):
        assert same(p, q)
    assert same(orc.ssim_vjp(a, b, da), ref.ssim_vjp(a, b, da))
    assert orc.mean_ssim(a, b) == ref.mean_ssim(a, b)
    f_o, f_r = orc.residual_vector(a, b), ref.residual_vector(a, b)
    assert same(f_o, f_r)
    assert same(orc.residual_jvp(a, da, b), ref.residual_jvp(a, da, b))
    assert same(orc.residual_vjp(a, b, f_o), ref.residual_vjp(a, b, f_r))
    assert orc.psnr(a, b) == ref.psnr(a, b)
    assert same(orc.quantize8(a), ref.quantize8(a))


# ------------------------------------------------------------------ optimizer seams
def test_stochastic_gradient_bitwise(data):  # optimizer.cpp:36-65
    d_o, d_r = data
    for batch in ([0], [3, 1], [0, 1, 2, 3, 4]):
        go, lo = orc.stochastic_gradient(d_o.init_x, d_o.cams, d_o.gts, batch)
        gr, lr = ref.stochastic_gradient(d_o.init_x, d_r.cams, d_r.gts, batch)
        assert same(go, gr) and lo == lr


def test_view_jacobian_seams_bitwise(data):  # optimizer.cpp:18-34
    d_o, d_r = data
    rng = np.random.default_rng(3)
    x = d_o.init_x
    v = rng.standard_normal(x.size)
    u = rng.standard_normal(6 * 48 * 48)
    assert same(orc.view_jacobian_apply(x, d_o.cams[1], d_o.gts[1], v),
                ref.view_jacobian_apply(x, d_r.cams[1], d_r.gts[1], v))
    assert same(orc.view_jacobian_applyT(x, d_o.cams[1], d_o.gts[1], u),
                ref.view_jacobian_applyT(x, d_r.cams[1], d_r.gts[1], u))


def test_hutchinson_and_exact_diagonal_bitwise(data):  # optimizer.cpp:75-104, checks.cpp
    d_o, d_r = data
    x = d_o.init_x
    z = ref.Rng(5).rademacher(2 * x.size)
    assert same(orc.hutchinson_diag(x, d_o.cams, d_o.gts, [2, 4], z),
                ref.hutchinson_diag(x, d_r.cams, d_r.gts, [2, 4], z))
    xo, co, go = orc.make_check_scene(3, 12, 2, 7)
    assert same(orc.exact_gn_diagonal(xo, co, go), ref.exact_gn_diagonal(xo, co, go))


@pytest.mark.parametrize("eps", [1e-6, 1e-4])
def test_shd_radii_bitwise(data, eps):  # trust_region.cpp:39-252
    d_o, _ = data
    x = d_o.gt_x  # random rotations and anisotropic scales
    caps = (1.0, 0.5, 1.0, 1.0, 0.25)
    assert same(orc.shd_radii(x, eps, caps), ref.shd_radii(x, eps, caps))
    for i in range(20):
        prim = np.concatenate([x[3 * i:3 * i + 3], x[900 + 3 * i:900 + 3 * i + 3],
                               x[1800 + 4 * i:1800 + 4 * i + 4], [x[3000 + i]],
                               x[3300 + 3 * i:3300 + 3 * i + 3]])
        for axis in range(4):
            assert orc.beta_rotation(prim, axis) == ref.beta_rotation(prim, axis)
    for t in (0, 1, 37, 100, 250):
        assert orc.eps_at(1e-6, 1e-8, 100, t) == ref.eps_at(1e-6, 1e-8, 100, t)


# ------------------------------------------------------------------ full steps
def _train(mod, d, steps, kind="3dgs2tr", seed=11):
    x = d.init_x.copy()
    st = mod.State(x.size, seed)
    opts = mod.TrOptions(total_steps=steps, hess_interval=4, batch_size=2)
    diags = []
    for _ in range(steps):
        if kind == "3dgs2tr":
            diags.append(mod.step_3dgs2tr(st, x, d.cams, d.gts, opts))
        else:
            diags.append(mod.step_adam(st, x, d.cams, d.gts, opts,
                                       mod.AdamOptions(scene_extent=1.7),
                                       trust_region=(kind == "adam-tr")))
    return x, st, diags


@pytest.mark.parametrize("kind", ["3dgs2tr", "adam", "adam-tr"])
def test_training_steps_bitwise(data, kind):  # optimizer.cpp:189-253
    d_o, d_r = data
    xo, so, do = _train(orc, d_o, 9, kind)
    xr, sr, dr = _train(ref, d_r, 9, kind)
    assert same(xo, xr)
    go, ho, to = so.get()
    gr, hr, tr = sr.get()
    assert same(go, gr) and same(ho, hr) and to == tr == 9
    if kind != "3dgs2tr":
        for p, q in zip(so.get_adam(), sr.get_adam()):
            assert same(p, q)
    for a, b in zip(do, dr):
        assert a == b


def test_rng_streams_bitwise():  # rng.hpp
    a, b = orc.Rng(99), ref.Rng(99)
    assert same(a.raw(100), b.raw(100))
    assert same(a.normal(101), b.normal(101))
    assert same(a.uniform(50, -2.0, 3.0), b.uniform(50, -2.0, 3.0))
    assert same(a.sample_without_replacement(40, 17), b.sample_without_replacement(40, 17))
    assert same(a.rademacher(1000), b.rademacher(1000))


def test_error_messages_match(data):  # render.cpp:36, geometry.hpp:42
    d_o, d_r = data
    x = d_o.init_x.copy()
    x[3 * 400 + 5] = np.nan  # scale of splat 1 (group-major)
    msgs = []
    for mod, d in ((orc, d_o), (ref, d_r)):
        with pytest.raises(mod.OracleNumericError) as e:
            mod.rasterize(x, d.cams[0])
        msgs.append(str(e.value))
    assert msgs[0] == msgs[1] == "rasterize: non-finite parameter in splat 1"
    x = d_o.init_x.copy()
    x[6 * 400 + 4 * 7:6 * 400 + 4 * 7 + 4] = 0.0  # degenerate quaternion of splat 7
    msgs = []
    for mod, d in ((orc, d_o), (ref, d_r)):
        with pytest.raises(mod.OracleInvalidArgument) as e:
            mod.rasterize(x, d.cams[0])
        msgs.append(str(e.value))
    assert msgs[0] == msgs[1]
