"""ADAM / ADAM-TR steps of the oracle (optimizer.cpp:153-253) against a
numpy restatement of adam_direction on the oracle's own gradient.

The reference ships no ADAM known-answer test (its ADAM checks are the
convergence comparisons of acceptance.cpp:118-203), so the oracle's ADAM
update is pinned here by the closed form, with the gradient, shd_radii and
the RNG stream (themselves pinned by the reference KATs) as inputs.
"""
import numpy as np
import pytest


def _adam_dx(g, m, v, t, k, a):
    m = a.beta1 * m + (1.0 - a.beta1) * g
    v = a.beta2 * v + (1.0 - a.beta2) * (g * g)
    c1 = 1.0 - a.beta1 ** t
    c2 = 1.0 - a.beta2 ** t
    frac = min(1.0, t / max(1, a.lr_position_decay_steps))
    lr_pos = a.scene_extent * a.lr_position * (a.lr_position_final / a.lr_position) ** frac
    lr = np.concatenate([np.full(3 * k, lr_pos), np.full(3 * k, a.lr_scale),
                         np.full(4 * k, a.lr_rotation), np.full(k, a.lr_opacity),
                         np.full(3 * k, a.lr_color)])
    return -lr * (m / c1) / (np.sqrt(v / c2) + a.eps), m, v


def _clamp(x, k, o):
    x = x.copy()
    x[3 * k:6 * k] = np.maximum(x[3 * k:6 * k], o.bounds[0])
    x[10 * k:11 * k] = np.minimum(np.maximum(x[10 * k:11 * k], o.bounds[1]), o.bounds[2])
    x[11 * k:] = np.minimum(np.maximum(x[11 * k:], o.bounds[3]), o.bounds[4])
    return x


@pytest.mark.parametrize("trust_region", [False, True])
def test_adam_step_matches_closed_form(orc, trust_region):
    x, cams, gts = orc.make_check_scene(5, 14, 4, 31)
    k = x.size // 14
    a = orc.AdamOptions(lr_position_decay_steps=7, scene_extent=1.7)
    o = orc.TrOptions(batch_size=2, total_steps=10)
    st = orc.State(x.size, 17)
    rng = orc.Rng(17)
    m = np.zeros(x.size)
    v = np.zeros(x.size)
    xr = x.copy()
    for t in (1, 2, 3):
        s1 = rng.sample_without_replacement(len(cams), 2)
        g, loss = orc.stochastic_gradient(xr, cams, gts, s1)
        dx, m, v = _adam_dx(g, m, v, t, k, a)
        if trust_region:
            eta = orc.shd_radii(xr, orc.eps_at(o.eps_start, o.eps_end, o.total_steps, t))
            step = np.minimum(np.maximum(dx, -eta), eta)
        else:
            step = dx
        d = orc.step_adam(st, x, cams, gts, o, a, trust_region, want_applied=True)
        assert np.array_equal(d["applied_step"], step)
        xr = _clamp(xr + step, k, o)
        assert np.array_equal(x, xr)
        mo, vo = st.get_adam()
        assert np.array_equal(mo, m) and np.array_equal(vo, v)
        assert d["batch_loss"] == loss
        assert d["step_pre"] == pytest.approx(np.linalg.norm(dx), rel=1e-14)
        if trust_region:
            assert d["eps"] > 0 and 0.0 <= d["clip_frac"] <= 1.0
        else:
            assert d["eps"] == -1.0 and d["clip_frac"] == -1.0
            assert d["max_step_over_radius"] == 0.0
    assert st.get()[2] == 3
    # the ADAM kinds leave g_hat / d_hat untouched (optimizer.cpp:222-253)
    g_hat, d_hat, _ = st.get()
    assert not g_hat.any() and not d_hat.any()


def test_adam_consumes_only_s1_draws(orc):
    # "ADAM variants consume only the first draw" (optimizer.hpp:55-57)
    x, cams, gts = orc.make_check_scene(4, 12, 5, 3)
    st = orc.State(x.size, 99)
    for _ in range(3):
        orc.step_adam(st, x, cams, gts, orc.TrOptions(batch_size=2), orc.AdamOptions())
    rng = orc.Rng(99)
    for _ in range(3):
        rng.sample_without_replacement(len(cams), 2)
    # next S1 from the state equals the next S1 from a fresh Rng advanced 3 samples
    s_expected = rng.sample_without_replacement(len(cams), 2)
    d = orc.step_adam(st, x.copy(), cams, gts, orc.TrOptions(batch_size=2),
                      orc.AdamOptions(), want_applied=True)
    g, _ = orc.stochastic_gradient(x, cams, gts, s_expected)
    assert d["gnorm"] == pytest.approx(np.linalg.norm(g), rel=1e-14)


# ---- the reference's own ADAM known-answer tests (test_optimizer.cpp:204-267)
def _lr_table(a, k, t):
    frac = min(1.0, t / max(1, a.lr_position_decay_steps))
    lr_pos = a.scene_extent * a.lr_position * (a.lr_position_final / a.lr_position) ** frac
    return np.concatenate([np.full(3 * k, lr_pos), np.full(3 * k, a.lr_scale),
                           np.full(4 * k, a.lr_rotation), np.full(k, a.lr_opacity),
                           np.full(3 * k, a.lr_color)])


def test_kat_adam_zero_gradient_stream(orc):  # test_optimizer.cpp:204-217
    x, cams, _ = orc.make_check_scene(4, 12, 2, 101)
    gts = [orc.rasterize(x, c)[0] for c in cams]
    st = orc.State(x.size, 9)
    before = x.copy()
    for _ in range(3):
        orc.step_adam(st, x, cams, gts, orc.TrOptions(), orc.AdamOptions())
    assert np.array_equal(x, before)


def test_kat_adam_first_step_is_the_group_rate(orc):  # test_optimizer.cpp:219-247
    x, cams, gts = orc.make_check_scene(4, 12, 2, 103)
    a = orc.AdamOptions(scene_extent=1.7)
    st = orc.State(x.size, 11)
    d = orc.step_adam(st, x, cams, gts, orc.TrOptions(), a, want_applied=True)
    m, _ = st.get_adam()
    lr = _lr_table(a, x.size // 14, 1)
    sel = np.abs(m) >= 1e-12
    assert sel.any()
    ap = np.abs(d["applied_step"][sel])
    # doctest's Approx(lr).epsilon(1e-9): |a - b| < 1e-9 * (1 + max(|a|, |b|))
    assert np.all(np.abs(ap - lr[sel]) < 1e-9 * (1.0 + np.maximum(ap, lr[sel])))


def test_kat_adam_tr_vacuous_region_is_adam(orc):  # test_optimizer.cpp:249-267
    x, cams, gts = orc.make_check_scene(5, 12, 3, 107)
    xa, xb = x.copy(), x.copy()
    sa, sb = orc.State(x.size, 77), orc.State(x.size, 77)
    ob = orc.TrOptions(eps_start=1e100, eps_end=1e100, total_steps=10, caps=(1e100,) * 5)
    for _ in range(5):
        orc.step_adam(sa, xa, cams, gts, orc.TrOptions(), orc.AdamOptions())
        orc.step_adam(sb, xb, cams, gts, ob, orc.AdamOptions(), True)
    assert np.array_equal(xa, xb)
