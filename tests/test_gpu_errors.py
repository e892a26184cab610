"""Error-path parity of step_3dgs2tr on the device against the compiled
reference: the three NumericError locators of optimizer.cpp and the state the
reference leaves behind after each (t, g_hat, D_hat, x and where its Rng
stream continues):

* "stochastic_gradient: non-finite gradient from view N" (optimizer.cpp:54-56):
  t incremented, S1 drawn, nothing else changed;
* "hutchinson_diag: non-finite sample" (optimizer.cpp:97-98), through the
  seam (unreachable inside the step with finite parameters, see the test);
* "non-finite update in group G" (optimizer.cpp:116-121): g_hat (and D_hat on
  a refresh) updated, x unchanged.
"""
import numpy as np
import pytest

from oracle import pyref

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not pyref.available(), reason="oracle/_ref not built")]

VIEWS = 5


@pytest.fixture(scope="module")
def sp():
    import __graft_entry__
    __graft_entry__.build()
    from paper_2602_00395_b200 import splat
    return splat


@pytest.fixture(scope="module")
def ds():
    ref = pyref.ref
    return ref.make_synthetic(ref.SynthConfig(gt_splats=60, init_splats=80, views=VIEWS,
                                              image_size=24, seed=4))


def draws(seed):
    """S1 and S2 of the first step (|S1| = |S2| = 1, optimizer.cpp:195-206)."""
    r = pyref.ref.Rng(seed)
    return int(r.sample_without_replacement(VIEWS, 1)[0]), \
        int(r.sample_without_replacement(VIEWS, 1)[0])


def run_both(sp, ds, gts, seed, state=None):
    ref = pyref.ref
    x = ds.init_x.copy()
    rst = ref.State(x.size, seed)
    ctx = sp.Context()
    ctx.set_scene(x)
    ctx.set_views([sp.Camera.from_c(c, g) for c, g in zip(ds.cams, gts)])
    ctx.state_reset(seed)
    if state is not None:
        rst.set(*state)
        ctx.state_set(*state)
    opts = sp.OptimizerOptions(schedule=sp.TrustRegionSchedule(1e-6, 1e-8, 20))
    with pytest.raises(sp.NumericError) as eg:
        ctx.step(opts)
    with pytest.raises(ref.OracleNumericError) as er:
        ref.step_3dgs2tr(rst, x, ds.cams, gts, ref.TrOptions(total_steps=20))
    g, d, t = ctx.state_get()
    gr, dr, tr = rst.get()
    out = dict(msg=(str(eg.value), str(er.value)), t=(t, tr), g=(g, gr), d=(d, dr),
               x=(ctx.get_scene(), x), rng=(ctx.rng_raw(8), rst.rng_raw(8)))
    ctx.close()
    return out


def test_gradient_failure_names_the_view(sp, ds):
    seed = 3
    s1, _ = draws(seed)
    gts = [g.copy() for g in ds.gts]
    gts[s1][5, 7, 1] = np.inf
    r = run_both(sp, ds, gts, seed)
    assert r["msg"][0] == r["msg"][1] == \
        f"stochastic_gradient: non-finite gradient from view {ds.cams[s1].id}"
    assert r["t"] == (1, 1)
    for k in ("g", "d"):
        assert not r[k][0].any() and not r[k][1].any()
    assert np.array_equal(r["x"][0], ds.init_x) and np.array_equal(r["x"][1], ds.init_x)
    assert np.array_equal(*r["rng"])  # both continue right after S1


def test_hutchinson_failure_message(sp, ds):
    """hutchinson_diag's own check (optimizer.cpp:97-98), through the seam
    with a probe carrying a NaN.  Inside step_3dgs2tr this path is not
    reachable with finite parameters: a NaN or infinite rendered pixel or
    target is masked out of the residual JVP/VJP (residuals.cpp:59-76, 95-103
    test u > floor, false for NaN), so J^T J z stays finite."""
    ref = pyref.ref
    z = np.ones(ds.init_x.size)
    z[17] = np.nan
    views = [sp.Camera.from_c(c, g) for c, g in zip(ds.cams, ds.gts)]
    with pytest.raises(sp.NumericError) as eg:
        sp.hutchinson_diag(sp.Scene(ds.init_x), views, [2], 1, lambda s: z)
    with pytest.raises(ref.OracleNumericError) as er:
        ref.hutchinson_diag(ds.init_x, ds.cams, ds.gts, [2], z)
    assert str(eg.value) == str(er.value) == "hutchinson_diag: non-finite sample"


def test_non_finite_update_names_the_group(sp, ds):
    k = ds.init_x.size // 14
    g0 = np.zeros(ds.init_x.size)
    g0[6 * k + 5] = np.nan  # a rotation coordinate of g_hat
    r = run_both(sp, ds, ds.gts, 7, state=(g0, np.zeros_like(g0), 1))
    assert r["msg"][0] == r["msg"][1] == "non-finite update in group rotation"
    assert r["t"] == (2, 2)  # t = 2: not a refresh step
    g, gr = r["g"]
    assert np.isnan(g[6 * k + 5]) and np.isnan(gr[6 * k + 5])
    fin = np.isfinite(gr)
    assert np.max(np.abs(g[fin] - gr[fin])) <= 1e-3 * np.max(np.abs(gr[fin]))
    assert np.array_equal(r["x"][0], ds.init_x) and np.array_equal(r["x"][1], ds.init_x)
    assert np.array_equal(*r["rng"])


def test_dup_capacity_rerun_is_transparent(sp, ds):
    """A step whose views outgrow the tile-duplicate capacity is rerun with a
    grown capacity (api.cu step_core); it reports the rerun and ends in the
    state of a step that never overflowed.  Bad capacities are refused."""
    views = [sp.Camera.from_c(c, g) for c, g in zip(ds.cams, ds.gts)]
    opts = sp.OptimizerOptions(schedule=sp.TrustRegionSchedule(1e-6, 1e-8, 20), batch_size=3)
    out = []
    for cap in (0, 16):
        ctx = sp.Context()
        ctx.set_scene(ds.init_x)
        ctx.set_views(views)
        ctx.state_reset(5)
        ctx.set_dup_capacity(cap)
        d = [ctx.step(opts) for _ in range(3)]
        out.append((ctx.get_scene(), ctx.state_get()[0], [x.reruns for x in d],
                    [x.batch_loss for x in d]))
        with pytest.raises(sp.InvalidArgument):
            ctx.set_dup_capacity(-1)
        with pytest.raises(sp.InvalidArgument):
            ctx.set_dup_capacity(1 << 31)
        ctx.close()
    (x0, g0, r0, l0), (x1, g1, r1, l1) = out
    assert r0 == [0, 0, 0] and r1[0] >= 1
    assert np.array_equal(x0, x1) and np.array_equal(g0, g1) and l0 == l1
