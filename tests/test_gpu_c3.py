"""Parity on the bench's own workload: BASELINE config 3 exactly as
bench.make_dataset('c3') builds it (1M splats, 64 views at 1920x1080,
size-scaled generator, GPU-rendered quantised targets).

(i)   full-frame tile binning of two views, bit-exact against the oracle's
      restatement (depth order, tile ranges, per-tile lists in the
      longest-tile-first raster order's underlying lists);
(ii)  completeness of the culling predicate: every contributing
      (pixel, splat) pair of the reference blend (alpha_bar >= 1/255 before
      termination, render.cpp:128-145) in a central 256x64 window appears in
      that pixel's tile list on the GPU;
(iii) render, JVP, VJP, stochastic gradient and Hutchinson diagonal on the
      central 256x64 crop with all 1M splats, against the oracle (which
      tests/test_reference.py shows equal to the compiled reference);
(iv)  the two view lanes: three steps (one a refresh) with SGTR_LANES=1 and
      SGTR_LANES=2 give bit-identical g_hat, D_hat, x and losses (the
      gradient's summation order is fixed by the view's batch position, not
      by the lane that renders it).
"""
import ctypes as C
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

IMG_TOL = 1e-4
GRAD_TOL = 1e-3
CROP_W, CROP_H = 256, 64


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
def c3(sp):
    import bench
    ctx = sp.Context()
    gt, init, cams = bench.make_dataset(sp, ctx, "c3", 1)
    yield ctx, gt, init, cams
    ctx.close()


def ocam(orc, cam):
    return orc.Camera.from_buffer_copy(bytes(cam._c()))


def crop(sp, cam, w=CROP_W, h=CROP_H):
    x0, y0 = (cam.width - w) // 2, (cam.height - h) // 2
    return sp.Camera(cam.id, cam.fx, cam.fy, cam.cx - x0, cam.cy - y0, w, h, cam.q_wc,
                     cam.t_wc), x0, y0


def gpu_binning(sp, ctx, x, cam):
    from paper_2602_00395_b200 import _lib
    L = _lib.lib()
    ctx.set_scene(x)
    nv, nd = C.c_int32(), C.c_int64()
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


@pytest.mark.parametrize("view,which", [(1, "init"), (40, "init"), (17, "gt")])
def test_c3_binning_bitexact(sp, orc, c3, view, which):
    ctx, gt, init, cams = c3
    x = init.x if which == "init" else gt.x
    g = gpu_binning(sp, ctx, x, cams[view])
    r = orc.binning(x, ocam(orc, cams[view]))
    assert g[1].size == r[1].size
    assert len(g[0]) > 900_000 and len(g[3]) > 1_000_000  # the full-scale case
    for a, b in zip(g, r):
        assert np.array_equal(a, b)
    ctx.set_scene(init.x)


def test_c3_tile_lists_contain_every_contributing_pair(sp, orc, c3):
    ctx, gt, init, cams = c3
    cam = cams[1]
    _, ts, te, lists = gpu_binning(sp, ctx, init.x, cam)
    ctx.set_scene(init.x)
    x0, y0 = (cam.width - CROP_W) // 2, (cam.height - CROP_H) // 2
    off, ids = orc.blend_pairs(init.x, ocam(orc, cam), x0, y0, CROP_W, CROP_H)
    assert ids.size > 10 * CROP_W * CROP_H  # a dense window
    tw = (cam.width + 15) // 16
    pix = np.repeat(np.arange(CROP_W * CROP_H), np.diff(off))
    px, py = x0 + pix % CROP_W, y0 + pix // CROP_W
    tile = (py // 16) * tw + px // 16
    counts = te - ts
    tile_of_entry = np.repeat(np.arange(ts.size), counts)
    starts = np.repeat(ts, counts)
    gpu_keys = tile_of_entry.astype(np.int64) << 21 | lists[starts + (
        np.arange(lists.size) - np.repeat(np.cumsum(counts) - counts, counts))].astype(np.int64)
    pair_keys = tile.astype(np.int64) << 21 | ids.astype(np.int64)
    missing = ~np.isin(pair_keys, gpu_keys)
    assert not missing.any(), f"{missing.sum()} contributing pairs culled from their tile"


@pytest.fixture(scope="module")
def crop_case(sp, orc, c3):
    ctx, gt, init, cams = c3
    cam = cams[1]
    cc, x0, y0 = crop(sp, cam)
    full = ctx.get_target(1, cam.width, cam.height)
    target = np.ascontiguousarray(full[y0:y0 + CROP_H, x0:x0 + CROP_W])
    return cc, ocam(orc, cc), target


def test_c3_crop_render_jvp_vjp(sp, orc, c3, crop_case):
    ctx, gt, init, cams = c3
    cc, oc, _ = crop_case
    scene = sp.Scene(init.x)
    out = sp.rasterize(scene, cc)
    col, t = orc.rasterize(init.x, oc)
    assert rel(out.color, col) < IMG_TOL and rel(out.t_final, t) < IMG_TOL
    rng = np.random.default_rng(5)
    v = rng.standard_normal(init.x.size)
    assert rel(sp.rasterize_jvp(scene, cc, v), orc.rasterize_jvp(init.x, oc, v)) < IMG_TOL
    adj = rng.standard_normal((CROP_H, CROP_W, 3))
    assert rel(sp.rasterize_vjp(scene, cc, adj), orc.rasterize_vjp(init.x, oc, adj)) < GRAD_TOL


def test_c3_crop_gradient_and_hutchinson(sp, orc, c3, crop_case):
    ctx, gt, init, cams = c3
    cc, oc, target = crop_case
    scene = sp.Scene(init.x)
    view = sp.Camera(cc.id, cc.fx, cc.fy, cc.cx, cc.cy, cc.width, cc.height, cc.q_wc, cc.t_wc,
                     target)
    g, loss = sp.stochastic_gradient(scene, [view], [0])
    go, lo = orc.stochastic_gradient(init.x, [oc], [target], [0])
    assert rel(g, go) < GRAD_TOL and loss == pytest.approx(lo, rel=1e-10)
    z = orc.Rng(9).rademacher(init.x.size)
    d = sp.hutchinson_diag(scene, [view], [0], 1, lambda s: z)
    do = orc.hutchinson_diag(init.x, [oc], [target], [0], z)
    assert rel(d, do) < IMG_TOL


def test_c3_lanes_agree(sp, c3):
    ctx, gt, init, cams = c3
    opt = sp.OptimizerOptions(batch_size=8, schedule=sp.TrustRegionSchedule(1e-6, 1e-8, 30000),
                              record_applied_step=False)
    out = {}
    old = os.environ.get("SGTR_LANES")
    try:
        for lanes in ("1", "2"):
            os.environ["SGTR_LANES"] = lanes
            ctx.set_scene(init.x)
            ctx.state_reset(1)
            diags = [ctx.step(opt) for _ in range(3)]
            assert diags[0].refreshed
            g, d, t = ctx.state_get()
            out[lanes] = (g, d, ctx.get_scene(), [dg.batch_loss for dg in diags])
    finally:
        if old is None:
            os.environ.pop("SGTR_LANES", None)
        else:
            os.environ["SGTR_LANES"] = old
        ctx.set_scene(init.x)
    (g1, d1, x1, l1), (g2, d2, x2, l2) = out["1"], out["2"]
    assert np.array_equal(g2, g1) and np.array_equal(d2, d1) and np.array_equal(x2, x1)
    assert l1 == l2
