"""Pins the CPU oracle against the reference's own known-answer tests.

The reference ships no golden vectors; its KATs live inside the
doctest suites.  Each test here restates one of them against the oracle and
cites the reference test it mirrors (paths under /root/reference/proj).  These
run on CPU only (`-m "not gpu"`).
"""
import math

import numpy as np
import pytest


def axis_camera(orc, size=16):  # test_render.cpp:20-28
    return orc.camera(width=size, height=size, fx=2.0 * size, fy=2.0 * size,
                      cx=size / 2.0 - 0.5, cy=size / 2.0 - 0.5)


def centered(orc, alpha, color):  # test_render.cpp:30-38
    return dict(mu=[0, 0, 1], s=[0.05] * 3, q=[0, 0, 0, 1], alpha=alpha, c=color)


def scene(orc, prims):
    return orc.pack([p["mu"] for p in prims], [p["s"] for p in prims],
                    [p["q"] for p in prims], [p["alpha"] for p in prims],
                    [p["c"] for p in prims])


# ------------------------------------------------------------------ RNG
def test_mt19937_64_stream(orc):
    # C++ [rand.predef]: the 10000th output of default-seeded mt19937_64
    r = orc.Rng(5489)
    assert int(r.raw(10000)[-1]) == 9981545732273789042


def test_rng_sample_without_replacement(orc):  # rng.hpp:56-66
    r = orc.Rng(7)
    s = r.sample_without_replacement(10, 4)
    assert len(set(s.tolist())) == 4 and s.min() >= 0 and s.max() < 10
    r2 = orc.Rng(7)
    raw = r2.raw(4)
    idx = list(range(10))
    for i in range(4):
        j = i + int(raw[i] % np.uint64(10 - i))
        idx[i], idx[j] = idx[j], idx[i]
    assert s.tolist() == idx[:4]


# ------------------------------------------------------------------ renderer
def test_single_splat_at_pixel_center(orc):  # test_render.cpp:42-54
    cam = axis_camera(orc)
    x = scene(orc, [centered(orc, 0.8, [1, 0, 0])])
    img, t = orc.rasterize(x, cam)
    px = py = int(cam.cx)
    assert img[py, px, 0] == pytest.approx(0.8, rel=1e-12)
    assert img[py, px, 1] == 0.0 and img[py, px, 2] == 0.0
    assert t[py, px] == pytest.approx(0.2, rel=1e-12)


def test_coincident_splats_tie_by_index(orc):  # test_render.cpp:56-65
    cam = axis_camera(orc)
    x = scene(orc, [centered(orc, 0.5, [1, 1, 1]), centered(orc, 0.5, [0, 0, 0])])
    img, _ = orc.rasterize(x, cam)
    assert img[int(cam.cy), int(cam.cx), 0] == pytest.approx(0.5, rel=1e-12)


def test_empty_scene_background(orc):  # test_render.cpp:67-79
    cam = axis_camera(orc, 8)
    ro = orc.RenderOptions(background=(0.25, 0.5, 0.75))
    img, t = orc.rasterize(np.zeros(0), cam, ro)
    assert np.all(img[..., 0] == 0.25) and np.all(img[..., 2] == 0.75)
    assert np.all(t == 1.0)


def test_nonfinite_names_splat(orc):  # test_render.cpp:81-89
    cam = axis_camera(orc, 8)
    x = scene(orc, [centered(orc, 0.5, [1, 1, 1])] * 2)
    x[3 * 1 + 2] = np.inf
    with pytest.raises(orc.OracleNumericError, match="splat 1"):
        orc.rasterize(x, cam)


def test_storage_order_independence(orc):  # test_render.cpp:91-100
    x, cams, _ = orc.make_check_scene(10, 16, 1, 42)
    mu, s, q, a, c = orc.unpack(x)
    xr = orc.pack(mu[::-1], s[::-1], q[::-1], a[::-1], c[::-1])
    i1, _ = orc.rasterize(x, cams[0])
    i2, _ = orc.rasterize(xr, cams[0])
    assert np.array_equal(i1, i2)


def test_transmittance_range(orc):  # test_render.cpp:102-112
    x, cams, _ = orc.make_check_scene(12, 16, 2, 7)
    for cam in cams:
        img, t = orc.rasterize(x, cam)
        assert np.all(t >= 0) and np.all(t <= 1) and np.all(np.isfinite(img))


def test_jvp_zero_and_dead(orc):  # test_render.cpp:114-132
    x, cams, _ = orc.make_check_scene(6, 16, 1, 3)
    assert np.all(orc.rasterize_jvp(x, cams[0], np.zeros_like(x)) == 0.0)
    # a splat behind the camera is culled; its parameters are dead
    cam = cams[0]
    mu, s, q, a, c = orc.unpack(x)
    R = _rot(cam.q_wc)
    center = -R.T @ np.array(cam.t_wc[:])
    behind = center - R[2] * 1.0
    x2 = orc.pack(np.vstack([mu, behind]), np.vstack([s, s[0]]), np.vstack([q, q[0]]),
                  np.append(a, a[0]), np.vstack([c, c[0]]))
    k = x2.size // 14
    v = np.zeros_like(x2)
    v[11 * k + 3 * (k - 1)] = 1.0
    assert np.all(orc.rasterize_jvp(x2, cam, v) == 0.0)


def _rot(q):
    x, y, z, w = q[:]
    r2 = x * x + y * y + z * z + w * w
    m = np.array([[r2 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
                  [2 * (x * y + w * z), r2 - 2 * (z * z + x * x), 2 * (y * z - w * x)],
                  [2 * (x * z - w * y), 2 * (y * z + w * x), r2 - 2 * (x * x + y * y)]])
    return m / r2


def test_jvp_matches_fd(orc):  # test_render.cpp:134-159
    x, cams, _ = orc.make_check_scene(6, 12, 1, 11)
    v = orc.Rng(99).normal(x.size)
    v /= np.linalg.norm(v)
    jvp = orc.rasterize_jvp(x, cams[0], v)
    h = 1e-6
    ip, _ = orc.rasterize(x + h * v, cams[0])
    im, _ = orc.rasterize(x - h * v, cams[0])
    mt = np.abs(jvp).max()
    assert mt > 0
    assert np.all(np.abs((ip - im) / (2 * h) - jvp) <= 1e-5 * mt)


def test_vjp_zero_and_color(orc):  # test_render.cpp:161-178
    cam = axis_camera(orc)
    x = scene(orc, [centered(orc, 0.3, [0.2, 0.9, 0.4])])
    adj = np.zeros((16, 16, 3))
    assert np.linalg.norm(orc.rasterize_vjp(x, cam, adj)) == 0.0
    adj[int(cam.cy), int(cam.cx), 1] = 1.0
    g = orc.rasterize_vjp(x, cam, adj)
    assert g[11 + 1] == pytest.approx(0.3, rel=1e-12)
    assert g[11] == 0.0


def test_adjoint_identity(orc):  # test_render.cpp:180-208
    x, cams, gts = orc.make_check_scene(8, 16, 2, 1)
    rng = orc.Rng(17)
    for cam, gt in zip(cams, gts):
        n = 16 * 16 * 3
        for _ in range(3):
            v = rng.normal(x.size)
            u = rng.normal(n).reshape(16, 16, 3)
            lhs = float(np.sum(u * orc.rasterize_jvp(x, cam, v)))
            rhs = float(orc.rasterize_vjp(x, cam, u) @ v)
            assert abs(lhs - rhs) <= 1e-9 * (1 + abs(lhs))
            ur = rng.normal(2 * n)
            lhs2 = float(ur @ orc.view_jacobian_apply(x, cam, gt, v))
            rhs2 = float(orc.view_jacobian_applyT(x, cam, gt, ur) @ v)
            assert abs(lhs2 - rhs2) <= 1e-9 * (1 + abs(lhs2))


def test_vjp_matches_fd(orc):  # test_render.cpp:210-244
    x, cams, _ = orc.make_check_scene(4, 10, 1, 19)
    cam = cams[0]
    u = orc.Rng(5).normal(10 * 10 * 3).reshape(10, 10, 3)
    g = orc.rasterize_vjp(x, cam, u)

    def weighted(xx):
        return float(np.sum(u * orc.rasterize(xx, cam)[0]))

    for k in range(x.size):
        if abs(g[k]) <= 1e-8:
            continue
        h = 1e-6 * (1 + abs(x[k]))
        xp, xm = x.copy(), x.copy()
        xp[k] += h
        xm[k] -= h
        fd = (weighted(xp) - weighted(xm)) / (2 * h)
        assert abs(fd - g[k]) <= 1e-4 * max(abs(fd), abs(g[k]))


# ------------------------------------------------------------------ SSIM / residuals
def random_image(orc, w, h, seed, lo=0.0, hi=1.0):  # test_residuals.cpp:15-21
    return orc.Rng(seed).uniform(w * h * 3, lo, hi).reshape(h, w, 3)


def test_ssim_closed_forms(orc):  # test_residuals.cpp:72-89
    a = np.zeros((16, 16, 3))
    assert np.allclose(orc.ssim_map(a, a), 1.0, rtol=1e-12, atol=0)
    b = np.ones((16, 16, 3))
    assert np.allclose(orc.ssim_map(a, b), 1e-4 / (1 + 1e-4), rtol=1e-12, atol=0)
    c = np.full((12, 12, 3), 0.37)
    assert np.allclose(orc.ssim_map(c, c), 1.0, rtol=1e-12, atol=0)


def _ssim_sep(a, b, x, y, c):  # test_residuals.cpp:23-68
    k = np.exp(-((np.arange(11) - 5.0) ** 2) / (2 * 1.5 * 1.5))
    k /= k.sum()
    H, W = a.shape[:2]

    def refl(i, n):
        return -i if i < 0 else (2 * n - 2 - i if i >= n else i)

    mom = np.zeros(5)
    for dy in range(-5, 6):
        yy = refl(y + dy, H)
        row = np.zeros(5)
        for dx in range(-5, 6):
            xx = refl(x + dx, W)
            av, bv = a[yy, xx, c], b[yy, xx, c]
            row += k[dx + 5] * np.array([av, bv, av * av, bv * bv, av * bv])
        mom += k[dy + 5] * row
    ma, mb, aa, bb, ab = mom
    va, vb, cov = aa - ma * ma, bb - mb * mb, ab - ma * mb
    return ((2 * ma * mb + 1e-4) * (2 * cov + 9e-4)) / ((ma * ma + mb * mb + 1e-4) * (va + vb + 9e-4))


def test_ssim_separable_oracle(orc):  # test_residuals.cpp:91-107
    a, b = random_image(orc, 20, 14, 2), random_image(orc, 20, 14, 3)
    s = orc.ssim_map(a, b)
    rng = np.random.default_rng(4)
    for _ in range(60):
        x, y, c = rng.integers(20), rng.integers(14), rng.integers(3)
        assert s[y, x, c] == pytest.approx(_ssim_sep(a, b, x, y, c), rel=1e-10)
    assert np.all(s <= 1 + 1e-12) and np.all(s >= -1 - 1e-12)


def test_ssim_jvp_fd_and_vjp_adjoint(orc):  # test_residuals.cpp:109-138
    a, b = random_image(orc, 16, 16, 5), random_image(orc, 16, 16, 6)
    da = random_image(orc, 16, 16, 7, -1, 1)
    s, ds = orc.ssim_jvp(a, da, b)
    h = 1e-6
    fd = (orc.ssim_map(a + h * da, b) - orc.ssim_map(a - h * da, b)) / (2 * h)
    assert np.allclose(ds, fd, rtol=1e-4, atol=1e-9)
    u = random_image(orc, 16, 16, 8, -1, 1)
    vjp = orc.ssim_vjp(a, b, u)
    lhs, rhs = float(np.sum(u * ds)), float(np.sum(vjp * da))
    assert abs(lhs - rhs) <= 1e-11 * (1 + abs(lhs))


def test_residual_vector_examples(orc):  # test_residuals.cpp:140-167
    gt = random_image(orc, 16, 16, 9)
    r0 = orc.residual_vector(gt, gt)
    assert np.allclose(r0, math.sqrt(1e-12), rtol=1e-12, atol=0)
    l0 = orc.ResidualOptions(lambda_=0.0)
    rend = gt.copy()
    rend[4, 3, 1] += 0.04
    r1 = orc.residual_vector(rend, gt, l0)
    assert r1[1 * 256 + 4 * 16 + 3] == pytest.approx(0.2, rel=1e-9)
    assert np.all(r1[3 * 256:] == math.sqrt(1e-12))
    l1 = orc.ResidualOptions(lambda_=1.0)
    assert np.all(orc.residual_vector(gt, gt, l1) == math.sqrt(1e-12))


def test_dssim_floor_iff_ssim_one(orc):  # test_residuals.cpp:169-185
    l1 = orc.ResidualOptions(lambda_=1.0)
    gt, other = random_image(orc, 16, 16, 31), random_image(orc, 16, 16, 32)
    s = orc.ssim_map(other, gt)
    r = orc.residual_vector(other, gt, l1)
    for c in range(3):
        at_floor = r[768 + c * 256: 768 + (c + 1) * 256] == math.sqrt(1e-12)
        one = (1.0 - s[..., c].ravel()) <= 2e-12
        assert np.array_equal(at_floor, one)


def test_objective_examples(orc):  # test_residuals.cpp:187-208
    x, cams, gts = orc.make_check_scene(4, 16, 2, 13)
    self_gts = [orc.rasterize(x, c)[0] for c in cams]
    obj = orc.objective(x, cams, self_gts)
    assert 0.0 <= obj <= 1e-12 / 2 * (1 + 1e-9)
    base = orc.objective(x, cams, gts)
    twice = orc.objective(x, cams + cams, gts + gts)
    assert twice == pytest.approx(base, rel=1e-12)


def test_psnr(orc):  # test_residuals.cpp:226-232
    a = random_image(orc, 8, 8, 11)
    assert orc.psnr(a, a) == 100.0
    assert orc.psnr(a, a + 0.1) == pytest.approx(20.0, rel=1e-12)


@pytest.mark.parametrize("lam", [0.0, 0.2])
def test_gradient_vs_fd(orc, lam):  # test_residuals.cpp:234-248 (smaller scene)
    x, cams, gts = orc.make_check_scene(3, 12, 2, 23)
    rs = orc.ResidualOptions(lambda_=lam)
    g, _ = orc.stochastic_gradient(x, cams, gts, [0, 1], rs)
    for k in range(x.size):
        if abs(g[k]) <= 1e-8:
            continue
        h = 1e-6 * (1 + abs(x[k]))
        xp, xm = x.copy(), x.copy()
        xp[k] += h
        xm[k] -= h
        fd = (orc.objective(xp, cams, gts, rs) - orc.objective(xm, cams, gts, rs)) / (2 * h)
        assert abs(g[k] - fd) / max(abs(g[k]), abs(fd)) <= 1e-4


# ------------------------------------------------------------------ optimizer
def test_full_batch_is_mean_of_single_views(orc):  # test_optimizer.cpp:62-75
    x, cams, gts = orc.make_check_scene(5, 12, 4, 67)
    full, _ = orc.stochastic_gradient(x, cams, gts, [0, 1, 2, 3])
    mean = sum(orc.stochastic_gradient(x, cams, gts, [i])[0] for i in range(4)) / 4
    assert np.linalg.norm(full - mean) / max(1e-30, np.linalg.norm(full)) <= 1e-12


def test_gradient_vanishes_at_perfect_fit(orc):  # test_optimizer.cpp:77-87
    x, cams, _ = orc.make_check_scene(4, 12, 2, 71)
    gts = [orc.rasterize(x, c)[0] for c in cams]
    g, _ = orc.stochastic_gradient(x, cams, gts, [0, 1])
    assert np.linalg.norm(g) <= 1e-6


def test_hutchinson_unit_probe_exact(orc):  # test_optimizer.cpp:89-108
    x, cams, gts = orc.make_check_scene(4, 12, 2, 73)
    exact = orc.exact_gn_diagonal(x, cams, gts)
    for k in (0, 7, x.size - 1):
        z = np.zeros(x.size)
        z[k] = 1.0
        d = orc.hutchinson_diag(x, cams, gts, [0, 1], z)
        assert d[k] == pytest.approx(exact[k], rel=1e-12)


def test_hutchinson_invisible_splat_zero(orc):  # test_optimizer.cpp:110-130
    x, cams, gts = orc.make_check_scene(4, 12, 2, 79)
    mu, s, q, a, c = orc.unpack(x)
    x2 = orc.pack(np.vstack([mu, [0, 0, 100.0]]), np.vstack([s, s[0]]),
                  np.vstack([q, q[0]]), np.append(a, a[0]), np.vstack([c, c[0]]))
    k = x2.size // 14
    z = orc.Rng(5).rademacher(2 * x2.size).reshape(2, -1)
    d = orc.hutchinson_diag(x2, cams, gts, [0, 1], z)
    i = k - 1
    idx = ([3 * i + c for c in range(3)] + [3 * k + 3 * i + c for c in range(3)] +
           [6 * k + 4 * i + c for c in range(4)] + [10 * k + i] +
           [11 * k + 3 * i + c for c in range(3)])
    assert np.all(d[idx] == 0.0)


def test_ema_cold_start(orc):  # test_optimizer.cpp:187-202
    x, cams, gts = orc.make_check_scene(4, 12, 3, 97)
    mirror = orc.Rng(55)
    batch = mirror.sample_without_replacement(len(cams), 1)
    g1, _ = orc.stochastic_gradient(x, cams, gts, batch)
    st = orc.State(x.size, 55)
    xx = x.copy()
    orc.step_3dgs2tr(st, xx, cams, gts, orc.TrOptions(total_steps=10))
    gh, _, _ = st.get()
    assert np.linalg.norm(gh - 0.1 * g1) <= 1e-15 * max(1.0, np.linalg.norm(g1))


def test_refresh_cadence_clip_eps(orc):  # test_optimizer.cpp:163-185
    x, cams, gts = orc.make_check_scene(4, 12, 3, 89)
    total = 25
    opts = orc.TrOptions(total_steps=total)
    st = orc.State(x.size, 123)
    xx = x.copy()
    last = st.get()[1]
    for t in range(1, total + 1):
        dg = orc.step_3dgs2tr(st, xx, cams, gts, opts)
        d = st.get()[1]
        assert (np.linalg.norm(d - last) > 0) == (t % 10 == 1)
        last = d
        assert dg["max_step_over_radius"] <= 1.0
        assert dg["eps"] == orc.eps_at(1e-6, 1e-8, total, t)
        assert 0.0 <= dg["clip_frac"] <= 1.0
    assert st.get()[2] == total


def test_perfect_fit_fixed_point(orc):  # test_optimizer.cpp:269-282
    x, cams, _ = orc.make_check_scene(3, 12, 2, 109)
    gts = [orc.rasterize(x, c)[0] for c in cams]
    st = orc.State(x.size, 13)
    xx = x.copy()
    for _ in range(5):
        orc.step_3dgs2tr(st, xx, cams, gts, orc.TrOptions(total_steps=10))
    assert np.array_equal(xx, x)


# ------------------------------------------------------------------ trust region
def base_prim():  # test_trust_region.cpp:18-26
    q = np.array([0.1, 0.3, -0.2, 0.9])
    return dict(mu=[0.1, -0.2, 0.3], s=[0.8, 0.5, 1.2], q=q / np.linalg.norm(q),
                alpha=0.6, c=[0.7, 0.4, 0.9])


def prim_x(orc, p):
    return orc.pack([p["mu"]], [p["s"]], [p["q"]], [p["alpha"]], [p["c"]])


def radii(orc, p, eps, caps=(1.0,) * 5):
    e = orc.shd_radii(prim_x(orc, p), eps, caps)
    return dict(mean=e[0:3], scale=e[3:6], rot=e[6:10], opacity=e[10], color=e[11:14])


def test_radius_mean_closed_forms(orc):  # test_trust_region.cpp:89-111
    p = base_prim()
    p.update(s=[1, 1, 1], q=[0, 0, 0, 1], alpha=1.0)
    r = radii(orc, p, 1e-6)["mean"]
    assert r[0] == pytest.approx(2.828e-3, rel=4e-4)
    assert r[0] == pytest.approx(math.sqrt(-8.0 * math.log1p(-1e-6)), rel=1e-12)
    p["alpha"] = 0.5
    assert radii(orc, p, 0.6)["mean"][0] == 1.0
    p.update(alpha=0.8, s=[1, 1, 1])
    r1 = radii(orc, p, 1e-6)["mean"]
    p["s"] = [math.sqrt(2.0), 1, 1]
    r2 = radii(orc, p, 1e-6)["mean"]
    assert r2[0] / r1[0] == pytest.approx(math.sqrt(2.0), rel=1e-12)
    assert r2[1] / r1[1] == pytest.approx(1.0, rel=1e-12)


def _cov(s, q):
    R = _rot(q)
    return R.T @ np.diag(np.square(s)) @ R


def test_radius_mean_exact_on_rotated(orc):  # test_trust_region.cpp:113-128
    rng = orc.Rng(41)
    for _ in range(20):
        mu = rng.uniform(3, -0.5, 0.5)
        s = rng.uniform(3, 0.1, 2.0)
        q = rng.normal(4)
        q = q / np.linalg.norm(q) * rng.uniform(1, 0.6, 1.4)[0]
        alpha = rng.uniform(1, 0.05, 0.9)[0]
        c = rng.uniform(3, 0.1, 1.0)
        p = dict(mu=mu, s=s, q=q, alpha=alpha, c=c)
        eps = 1e-5
        r = radii(orc, p, eps)["mean"]
        S = _cov(s, q)
        det = s[0] * s[1] * s[2]
        for k in range(3):
            m2 = mu.copy()
            m2[k] += r[k]
            h2 = orc.hellinger_sq(alpha * det, mu, S, alpha * det, m2, S) / det
            assert h2 == pytest.approx(eps, rel=1e-9)


def test_radius_scale_opacity_color(orc):  # test_trust_region.cpp:130-170
    p = base_prim()
    p.update(s=[1, 1, 1], alpha=0.5)
    assert radii(orc, p, 1e-6)["scale"][0] == pytest.approx(2e-3, rel=1e-12)
    p["s"] = [2, 1, 0.5]
    r2 = radii(orc, p, 1e-6)["scale"]
    assert r2[0] / r2[1] == pytest.approx(2.0, rel=1e-12)
    assert r2[2] / r2[1] == pytest.approx(0.5, rel=1e-12)
    lo, hi = dict(p, alpha=0.2), dict(p, alpha=0.8)
    assert radii(orc, lo, 1e-6)["scale"][0] / radii(orc, hi, 1e-6)["scale"][0] == \
        pytest.approx(2.0, rel=1e-12)
    p = base_prim()
    p["alpha"] = 0.25
    assert radii(orc, p, 1e-6)["opacity"] == pytest.approx(1e-3, rel=1e-12)
    p["alpha"] = 1.0
    assert radii(orc, p, 0.01)["opacity"] == pytest.approx(0.2, rel=1e-12)
    p.update(alpha=0.25, c=[0.25, 0.5, 1.0])
    rc = radii(orc, p, 1e-6)["color"]
    assert rc[0] == pytest.approx(2e-3, rel=1e-12)
    assert rc[2] / rc[0] == pytest.approx(2.0, rel=1e-12)
    p["c"] = [1e-6, 0.5, 1.0]
    assert radii(orc, p, 1e-6)["color"][0] == pytest.approx(
        math.sqrt(4.0 * 1e-6 * 1e-6 / 0.25), rel=1e-12)


def prim14(p):
    return np.concatenate([p["mu"], p["s"], p["q"], [p["alpha"]], p["c"]])


def test_beta_rotation_closed_forms(orc):  # test_trust_region.cpp:172-224
    iso = base_prim()
    iso.update(s=[1, 1, 1], q=[0, 0, 0, 1])
    for ax in range(4):
        assert abs(orc.beta_rotation(prim14(iso), ax)) < 1e-12
    p = base_prim()
    p.update(q=[0, 0, 0, 1], s=[1.0, 2.0, 1.0])
    u = 4.0
    assert orc.beta_rotation(prim14(p), 0) == pytest.approx(8 * (u + 1 / u) - 16, rel=1e-12)
    assert abs(orc.beta_rotation(prim14(p), 3)) < 1e-12
    p = base_prim()
    for ax in range(4):
        b1 = orc.beta_rotation(prim14(p), ax)
        p2 = dict(p, q=2.0 * np.asarray(p["q"]))
        assert orc.beta_rotation(prim14(p2), ax) == pytest.approx(b1 / 4, rel=1e-10)


def test_radius_rotation_caps(orc):  # test_trust_region.cpp:226-264
    p = base_prim()
    assert np.all(radii(orc, p, p["alpha"] * 2.0)["rot"] == 1.0)
    iso = dict(p, s=[0.5, 0.5, 0.5])
    assert np.all(radii(orc, iso, 1e-6)["rot"] == 1.0)
    a = dict(p, q=[0, 0, 0, 1], s=[1, 2, 1])
    b = dict(p, q=[0, 0, 0, 1], s=[1, 4, 1])
    ba, bb = orc.beta_rotation(prim14(a), 0), orc.beta_rotation(prim14(b), 0)
    ra, rb = radii(orc, a, 1e-6)["rot"][0], radii(orc, b, 1e-6)["rot"][0]
    assert ra / rb == pytest.approx(math.sqrt(bb / ba), rel=1e-10)


def test_shd_radii_monotone_and_floor(orc):  # test_trust_region.cpp:266-297
    x = prim_x(orc, base_prim())
    e = orc.shd_radii(x, 1e-6)
    assert np.all(orc.shd_radii(x, 0.5e-6) <= e)
    p = dict(base_prim(), alpha=1e-4)
    xf = np.tile(prim_x(orc, p).reshape(14, 1), 4).reshape(14, 4)
    xf = orc.pack(*[np.tile(np.asarray(v, float), (4, 1)) for v in
                    (p["mu"], p["s"], p["q"])], [1e-4] * 4, np.tile(p["c"], (4, 1)))
    ef = orc.shd_radii(xf, 1e-6)
    assert np.all(np.isfinite(ef)) and np.all(ef > 0) and np.all(ef <= 1.0)


def test_eps_schedule(orc):  # test_trust_region.cpp:336-343
    assert orc.eps_at(1e-6, 1e-8, 1000, 0) == 1e-6
    assert orc.eps_at(1e-6, 1e-8, 1000, 1000) == pytest.approx(1e-8, rel=1e-14)
    assert orc.eps_at(1e-6, 1e-8, 1000, 500) == pytest.approx(1e-7, rel=1e-12)
    assert orc.eps_at(1e-6, 1e-8, 1000, 2000) == pytest.approx(1e-8, rel=1e-14)
    assert orc.eps_at(1e-6, 1e-8, 1000, -5) == 1e-6


def test_rotation_certification(orc):  # test_trust_region.cpp:345-389 (rotation family)
    rng = orc.Rng(59)
    worst = 0.0
    for _ in range(60):
        mu = rng.uniform(3, -0.5, 0.5)
        s = rng.uniform(3, 0.1, 2.0)
        q = rng.normal(4)
        q = q / np.linalg.norm(q) * rng.uniform(1, 0.6, 1.4)[0]
        alpha = rng.uniform(1, 0.05, 0.9)[0]
        c = rng.uniform(3, 0.1, 1.0)
        det = s[0] * s[1] * s[2]
        S = _cov(s, q)
        for eps in (1e-6, 1e-4):
            rq = radii(orc, dict(mu=mu, s=s, q=q, alpha=alpha, c=c), eps)["rot"]
            for ax in range(4):
                q2 = q.copy()
                q2[ax] += rq[ax]
                h2 = orc.hellinger_sq(alpha * det, mu, S, alpha * det, mu, _cov(s, q2)) / det
                worst = max(worst, h2 / eps)
    assert worst <= 1.15
