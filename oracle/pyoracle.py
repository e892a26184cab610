"""ctypes binding of the CPU parity oracle (oracle/liboracle.so).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / ``--impl reference`` legs, never by the product
package.  Array conventions follow the reference (see oracle.h): scenes are
group-major float64 vectors of length 14*K, images are float64 arrays of shape
(H, W, 3) (row-major, channel-interleaved), residual vectors have length
6*H*W.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "build", "liboracle.so")


class OracleError(RuntimeError):
    pass


class OracleInvalidArgument(OracleError, ValueError):
    """std::invalid_argument in the reference."""


class OracleNumericError(OracleError):
    """splat::NumericError in the reference (errors.hpp:11-14)."""


class Camera(C.Structure):
    _fields_ = [("id", C.c_int32), ("width", C.c_int32), ("height", C.c_int32),
                ("pad", C.c_int32), ("fx", C.c_double), ("fy", C.c_double),
                ("cx", C.c_double), ("cy", C.c_double), ("q_wc", C.c_double * 4),
                ("t_wc", C.c_double * 3)]


class RenderOpts(C.Structure):
    _fields_ = [("z_near", C.c_double), ("lowpass", C.c_double),
                ("alpha_clamp", C.c_double), ("alpha_skip", C.c_double),
                ("t_stop", C.c_double), ("cutoff_sigma", C.c_double),
                ("background", C.c_double * 3)]


class ResidualOpts(C.Structure):
    _fields_ = [("lambda_", C.c_double), ("floor_", C.c_double)]


class TrOpts(C.Structure):
    _fields_ = [("theta1", C.c_double), ("theta2", C.c_double),
                ("hess_interval", C.c_int32), ("hutch_samples", C.c_int32),
                ("batch_size", C.c_int32), ("hutch_batch_size", C.c_int32),
                ("gamma_d", C.c_double), ("eps_start", C.c_double),
                ("eps_end", C.c_double), ("total_steps", C.c_int32),
                ("pad", C.c_int32), ("cap_mean", C.c_double),
                ("cap_scale", C.c_double), ("cap_rotation", C.c_double),
                ("cap_opacity", C.c_double), ("cap_color", C.c_double),
                ("s_min", C.c_double), ("alpha_min", C.c_double),
                ("alpha_max", C.c_double), ("c_min", C.c_double),
                ("c_max", C.c_double)]


class AdamOpts(C.Structure):
    _fields_ = [("beta1", C.c_double), ("beta2", C.c_double), ("eps", C.c_double),
                ("lr_position", C.c_double), ("lr_position_final", C.c_double),
                ("lr_position_decay_steps", C.c_int32), ("pad", C.c_int32),
                ("lr_scale", C.c_double), ("lr_rotation", C.c_double),
                ("lr_opacity", C.c_double), ("lr_color", C.c_double),
                ("scene_extent", C.c_double)]


class Diag(C.Structure):
    _fields_ = [("batch_loss", C.c_double), ("gnorm", C.c_double),
                ("step_pre", C.c_double), ("step_post", C.c_double),
                ("clip_frac", C.c_double), ("eps", C.c_double),
                ("max_step_over_radius", C.c_double)]


class SynthCfg(C.Structure):
    _fields_ = [("gt_splats", C.c_int32), ("init_splats", C.c_int32),
                ("views", C.c_int32), ("image_size", C.c_int32),
                ("seed", C.c_uint64), ("sigma_init", C.c_double),
                ("init_scale", C.c_double), ("init_opacity", C.c_double),
                ("camera_radius", C.c_double), ("camera_height", C.c_double),
                ("focal_factor", C.c_double), ("width", C.c_int32), ("height", C.c_int32),
                ("size_scale", C.c_double), ("sh_degree", C.c_int32), ("pad2", C.c_int32)]


def build(force: bool = False) -> str:
    """Compile liboracle.so with the committed Makefile (gcc only)."""
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < max(
            os.path.getmtime(os.path.join(_HERE, f)) for f in ("oracle.cpp", "oracle.h")):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


_lib = None


def use_timing_build() -> str:
    """Switch this process to the oracle's timing build (-O3 -march=native,
    compiled here on first use by `make native`) for the CPU-baseline
    measurements; falls back to the parity build if that fails.  Returns
    the loaded library path."""
    global _lib
    path = os.path.join(_HERE, "build_native", "liboracle_native.so")
    try:
        subprocess.run(["make", "-s", "-C", _HERE, "native"], check=True,
                       capture_output=True, timeout=600)
        L = C.CDLL(path)
    except Exception:
        build()
        return _LIB_PATH
    _setup(L)
    _lib = L
    if _SH_NB:
        L.orc_set_sh_degree(int(round((_SH_NB + 1) ** 0.5)) - 1)
    return path


def _setup(L):
    L.orc_last_error.restype = C.c_char_p
    for name in ("orc_mean_ssim", "orc_psnr", "orc_objective", "orc_beta_rotation",
                 "orc_eps_at", "orc_hellinger_sq"):
        getattr(L, name).restype = C.c_double
    L.orc_state_create.restype = C.c_void_p
    L.orc_rng_create.restype = C.c_void_p


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = C.CDLL(_LIB_PATH)
        _setup(L)
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


def _check(rc):
    if rc == 0:
        return
    msg = lib().orc_last_error().decode()
    if rc == 1:
        raise OracleInvalidArgument(msg)
    if rc == 2:
        raise OracleNumericError(msg)
    raise OracleError(msg)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


# SH colour extension (parity unpinned; degree 0 = the reference): the
# process-wide degree of the oracle, mirrored here for the vector lengths
_SH_NB = 0


def set_sh_degree(degree: int) -> None:
    global _SH_NB
    if lib().orc_set_sh_degree(int(degree)) != 0:
        raise OracleInvalidArgument("sh degree must be in 0..3")
    _SH_NB = (degree + 1) ** 2 - 1


def params_per_splat() -> int:
    return 14 + 3 * _SH_NB


def _k(x):
    return x.size // params_per_splat()


# --------------------------------------------------------------- options
@dataclass
class RenderOptions:  # render.hpp:12-22
    z_near: float = 0.01
    lowpass: float = 0.3
    alpha_clamp: float = 0.99
    alpha_skip: float = 1.0 / 255.0
    t_stop: float = 1e-4
    cutoff_sigma: float = 3.0
    background: tuple = (0.0, 0.0, 0.0)
    workers: int = 0

    def c(self):
        return RenderOpts(self.z_near, self.lowpass, self.alpha_clamp, self.alpha_skip,
                          self.t_stop, self.cutoff_sigma, (C.c_double * 3)(*self.background))


@dataclass
class ResidualOptions:  # residuals.hpp:13-16
    lambda_: float = 0.2
    floor: float = 1e-12

    def c(self):
        return ResidualOpts(self.lambda_, self.floor)


@dataclass
class TrOptions:  # optimizer.hpp:37-53 (3dgs2tr subset) + trust_region.hpp
    theta1: float = 0.9
    theta2: float = 0.999
    hess_interval: int = 10
    hutch_samples: int = 1
    batch_size: int = 1
    hutch_batch_size: int = 1
    gamma_d: float = 1e-12
    eps_start: float = 1e-6
    eps_end: float = 1e-8
    total_steps: int = 1
    caps: tuple = (1.0, 1.0, 1.0, 1.0, 1.0)
    bounds: tuple = (1e-6, 1e-4, 0.995, 1e-6, 1.5)

    def c(self):
        return TrOpts(self.theta1, self.theta2, self.hess_interval, self.hutch_samples,
                      self.batch_size, self.hutch_batch_size, self.gamma_d, self.eps_start,
                      self.eps_end, self.total_steps, 0, *self.caps, *self.bounds)


@dataclass
class AdamOptions:  # optimizer.hpp:21-34 (+ OptimizerOptions::scene_extent)
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-15
    lr_position: float = 1.6e-4
    lr_position_final: float = 1.6e-6
    lr_position_decay_steps: int = 30000
    lr_scale: float = 5e-3
    lr_rotation: float = 1e-3
    lr_opacity: float = 5e-2
    lr_color: float = 2.5e-3
    scene_extent: float = 1.0

    def c(self):
        return AdamOpts(self.beta1, self.beta2, self.eps, self.lr_position,
                        self.lr_position_final, self.lr_position_decay_steps, 0, self.lr_scale,
                        self.lr_rotation, self.lr_opacity, self.lr_color, self.scene_extent)


def camera(id=0, width=16, height=16, fx=1.0, fy=1.0, cx=0.0, cy=0.0,
           q_wc=(0, 0, 0, 1), t_wc=(0, 0, 0)) -> Camera:
    return Camera(id, width, height, 0, fx, fy, cx, cy, (C.c_double * 4)(*q_wc),
                  (C.c_double * 3)(*t_wc))


def _cams(cams):
    arr = (Camera * len(cams))()
    for i, c in enumerate(cams):
        # a Camera of another binding instance (pyref) has the same layout
        arr[i] = c if isinstance(c, Camera) else Camera.from_buffer_copy(bytes(c))
    return arr


def _gts(gts):
    gts = [_f64(g) for g in gts]
    ptrs = (C.c_void_p * len(gts))(*[g.ctypes.data for g in gts])
    return gts, ptrs


# --------------------------------------------------------------- renderer
def rasterize(x, cam, ro=None):
    ro = ro or RenderOptions()
    x = _f64(x)
    col = np.empty((cam.height, cam.width, 3))
    t = np.empty((cam.height, cam.width))
    _check(lib().orc_rasterize(_p(x), C.c_int64(_k(x)), C.byref(cam), C.byref(ro.c()),
                               ro.workers, _p(col), _p(t)))
    return col, t


def rasterize_jvp(x, cam, v, ro=None):
    ro = ro or RenderOptions()
    x, v = _f64(x), _f64(v)
    out = np.empty((cam.height, cam.width, 3))
    _check(lib().orc_rasterize_jvp(_p(x), C.c_int64(_k(x)), C.byref(cam),
                                   C.byref(ro.c()), ro.workers, _p(v), C.c_int64(v.size),
                                   _p(out)))
    return out


def rasterize_vjp(x, cam, adjoint, ro=None):
    ro = ro or RenderOptions()
    x, a = _f64(x), _f64(adjoint)
    g = np.empty(x.size)
    _check(lib().orc_rasterize_vjp(_p(x), C.c_int64(_k(x)), C.byref(cam),
                                   C.byref(ro.c()), ro.workers, _p(a), a.shape[1],
                                   a.shape[0], _p(g)))
    return g


def blend_stats(x, cam, ro=None):
    ro = ro or RenderOptions()
    x = _f64(x)
    e, c = C.c_int64(), C.c_int64()
    _check(lib().orc_blend_stats(_p(x), C.c_int64(_k(x)), C.byref(cam),
                                 C.byref(ro.c()), ro.workers, C.byref(e), C.byref(c)))
    return e.value, c.value


def blend_pairs(x, cam, x0, y0, w, h, ro=None):
    """Contributing (pixel, splat) pairs of the blend in a window:
    (offsets[w*h+1], ids) with pixel p = row-major index in the window."""
    ro = ro or RenderOptions()
    x = _f64(x)
    off = np.empty(w * h + 1, np.int64)
    cap = 64 * w * h
    ids = np.empty(cap, np.int32)
    _check(lib().orc_blend_pairs(_p(x), C.c_int64(_k(x)), C.byref(cam), C.byref(ro.c()),
                                 ro.workers, x0, y0, w, h, _p(off), _p(ids), C.c_int64(cap)))
    if off[-1] > cap:
        ids = np.empty(int(off[-1]), np.int32)
        _check(lib().orc_blend_pairs(_p(x), C.c_int64(_k(x)), C.byref(cam), C.byref(ro.c()),
                                     ro.workers, x0, y0, w, h, _p(off), _p(ids),
                                     C.c_int64(ids.size)))
    return off, ids[:int(off[-1])]


def project(x, cam, ro=None):
    ro = ro or RenderOptions()
    x = _f64(x)
    k = _k(x)
    out = np.empty((k, 12))
    _check(lib().orc_project(_p(x), C.c_int64(k), C.byref(cam), C.byref(ro.c()), _p(out)))
    return out


def binning(x, cam, tile=16, ro=None):
    """Returns (order, tile_start, tile_end, lists) of the restated binning."""
    ro = ro or RenderOptions()
    x = _f64(x)
    k = _k(x)
    nv, nd = C.c_int32(), C.c_int64()
    L = lib()
    _check(L.orc_binning(_p(x), C.c_int64(k), C.byref(cam), C.byref(ro.c()), tile,
                         C.byref(nv), None, C.byref(nd), None, None, None))
    tw = (cam.width + tile - 1) // tile
    th = (cam.height + tile - 1) // tile
    order = np.empty(nv.value, np.int32)
    ts = np.empty(tw * th, np.int64)
    te = np.empty(tw * th, np.int64)
    lists = np.empty(nd.value, np.int32)
    _check(L.orc_binning(_p(x), C.c_int64(k), C.byref(cam), C.byref(ro.c()), tile,
                         C.byref(nv), _p(order), C.byref(nd), _p(ts), _p(te), _p(lists)))
    return order, ts, te, lists


# --------------------------------------------------------------- SSIM/residuals
def ssim_map(a, b):
    a, b = _f64(a), _f64(b)
    out = np.empty_like(a)
    _check(lib().orc_ssim_map(_p(a), _p(b), a.shape[1], a.shape[0], _p(out)))
    return out


def ssim_jvp(a, da, b):
    a, da, b = _f64(a), _f64(da), _f64(b)
    s, ds = np.empty_like(a), np.empty_like(a)
    _check(lib().orc_ssim_jvp(_p(a), _p(da), _p(b), a.shape[1], a.shape[0], _p(s), _p(ds)))
    return s, ds


def ssim_vjp(a, b, up):
    a, b, up = _f64(a), _f64(b), _f64(up)
    g = np.empty_like(a)
    _check(lib().orc_ssim_vjp(_p(a), _p(b), _p(up), a.shape[1], a.shape[0], _p(g)))
    return g


def mean_ssim(a, b):
    a, b = _f64(a), _f64(b)
    return lib().orc_mean_ssim(_p(a), _p(b), a.shape[1], a.shape[0])


def residual_vector(img, gt, ro=None):
    ro = ro or ResidualOptions()
    img, gt = _f64(img), _f64(gt)
    r = np.empty(2 * img.size)
    _check(lib().orc_residual_vector(_p(img), _p(gt), img.shape[1], img.shape[0],
                                     C.byref(ro.c()), _p(r)))
    return r


def residual_jvp(img, tan, gt, ro=None):
    ro = ro or ResidualOptions()
    img, tan, gt = _f64(img), _f64(tan), _f64(gt)
    r = np.empty(2 * img.size)
    _check(lib().orc_residual_jvp(_p(img), _p(tan), _p(gt), img.shape[1], img.shape[0],
                                  C.byref(ro.c()), _p(r)))
    return r


def residual_vjp(img, gt, u, ro=None):
    ro = ro or ResidualOptions()
    img, gt, u = _f64(img), _f64(gt), _f64(u)
    adj = np.empty_like(img)
    _check(lib().orc_residual_vjp(_p(img), _p(gt), img.shape[1], img.shape[0], _p(u),
                                  C.c_int64(u.size), C.byref(ro.c()), _p(adj)))
    return adj


def psnr(a, b):
    a, b = _f64(a), _f64(b)
    return lib().orc_psnr(_p(a), _p(b), C.c_int64(a.size))


def quantize8(a):
    a = _f64(a)
    out = np.empty_like(a)
    lib().orc_quantize8(_p(a), C.c_int64(a.size), _p(out))
    return out


# --------------------------------------------------------------- optimizer
def view_jacobian_apply(x, cam, gt, v, rs=None, ro=None):
    rs, ro = rs or ResidualOptions(), ro or RenderOptions()
    x, gt, v = _f64(x), _f64(gt), _f64(v)
    out = np.empty(2 * gt.size)
    _check(lib().orc_view_jacobian_apply(_p(x), C.c_int64(_k(x)), C.byref(cam),
                                         _p(gt), _p(v), C.byref(rs.c()), C.byref(ro.c()),
                                         ro.workers, _p(out)))
    return out


def view_jacobian_applyT(x, cam, gt, u, rs=None, ro=None):
    rs, ro = rs or ResidualOptions(), ro or RenderOptions()
    x, gt, u = _f64(x), _f64(gt), _f64(u)
    g = np.empty(x.size)
    _check(lib().orc_view_jacobian_applyT(_p(x), C.c_int64(_k(x)), C.byref(cam),
                                          _p(gt), _p(u), C.byref(rs.c()), C.byref(ro.c()),
                                          ro.workers, _p(g)))
    return g


def stochastic_gradient(x, cams, gts, batch, rs=None, ro=None):
    rs, ro = rs or ResidualOptions(), ro or RenderOptions()
    x = _f64(x)
    keep, ptrs = _gts(gts)
    b = np.ascontiguousarray(batch, dtype=np.int32)
    g = np.empty(x.size)
    loss = C.c_double()
    _check(lib().orc_stochastic_gradient(_p(x), C.c_int64(_k(x)), _cams(cams), ptrs,
                                         len(cams), _p(b), b.size, C.byref(rs.c()),
                                         C.byref(ro.c()), ro.workers, _p(g), C.byref(loss)))
    return g, loss.value


def hutchinson_diag(x, cams, gts, batch, probes, rs=None, ro=None):
    """probes: array (nu, 14K)."""
    rs, ro = rs or ResidualOptions(), ro or RenderOptions()
    x = _f64(x)
    keep, ptrs = _gts(gts)
    b = np.ascontiguousarray(batch, dtype=np.int32)
    z = _f64(np.atleast_2d(probes))
    d = np.empty(x.size)
    _check(lib().orc_hutchinson_diag(_p(x), C.c_int64(_k(x)), _cams(cams), ptrs,
                                     len(cams), _p(b), b.size, z.shape[0], _p(z),
                                     C.byref(rs.c()), C.byref(ro.c()), ro.workers, _p(d)))
    return d


def objective(x, cams, gts, rs=None, ro=None):
    rs, ro = rs or ResidualOptions(), ro or RenderOptions()
    x = _f64(x)
    keep, ptrs = _gts(gts)
    return lib().orc_objective(_p(x), C.c_int64(_k(x)), _cams(cams), ptrs, len(cams),
                               C.byref(rs.c()), C.byref(ro.c()), ro.workers)


def exact_gn_diagonal(x, cams, gts, rs=None, ro=None):
    rs, ro = rs or ResidualOptions(), ro or RenderOptions()
    x = _f64(x)
    keep, ptrs = _gts(gts)
    d = np.empty(x.size)
    _check(lib().orc_exact_gn_diagonal(_p(x), C.c_int64(_k(x)), _cams(cams), ptrs,
                                       len(cams), C.byref(rs.c()), C.byref(ro.c()),
                                       ro.workers, _p(d)))
    return d


def shd_radii(x, eps, caps=(1.0, 1.0, 1.0, 1.0, 1.0)):
    x = _f64(x)
    c = (C.c_double * 5)(*caps)
    eta = np.empty(x.size)
    _check(lib().orc_shd_radii(_p(x), C.c_int64(_k(x)), C.c_double(eps), c, _p(eta)))
    return eta


def beta_rotation(prim14, axis):
    p = _f64(prim14)
    return lib().orc_beta_rotation(_p(p), axis)


def eps_at(e0, e1, total, t):
    return lib().orc_eps_at(C.c_double(e0), C.c_double(e1), total, t)


def hellinger_sq(ma, mua, sa, mb, mub, sb):
    a = [_f64(v) for v in (mua, sa, mub, sb)]
    return lib().orc_hellinger_sq(C.c_double(ma), _p(a[0]), _p(a[1]), C.c_double(mb),
                                  _p(a[2]), _p(a[3]))


class State:
    """OptimizerState (optimizer.hpp:58-72) for the 3DGS²-TR path."""

    def __init__(self, dim, seed):
        self.dim = dim
        self._h = C.c_void_p(lib().orc_state_create(C.c_int64(dim), C.c_uint64(seed)))

    def __del__(self):
        if getattr(self, "_h", None):
            lib().orc_state_destroy(self._h)
            self._h = None

    def get(self):
        g, d, t = np.empty(self.dim), np.empty(self.dim), C.c_int64()
        lib().orc_state_get(self._h, _p(g), _p(d), C.byref(t))
        return g, d, t.value

    def set(self, g_hat, d_hat, t):
        g, d = _f64(g_hat), _f64(d_hat)
        lib().orc_state_set(self._h, _p(g), _p(d), C.c_int64(t))

    def rng_raw(self, n):
        """n raw draws continuing the state's Rng stream."""
        out = np.empty(n, np.uint64)
        lib().orc_state_rng_raw(self._h, C.c_int64(n), _p(out))
        return out

    def get_adam(self):
        m, v = np.empty(self.dim), np.empty(self.dim)
        lib().orc_state_get_adam(self._h, _p(m), _p(v))
        return m, v

    def set_adam(self, m, v):
        m, v = _f64(m), _f64(v)
        lib().orc_state_set_adam(self._h, _p(m), _p(v))


def step_3dgs2tr(state, x, cams, gts, opts, rs=None, ro=None, *, s1=None, s2=None,
                 probes=None, want_applied=False):
    """One Algorithm-1 step; x (float64, 14K) is updated in place."""
    rs, ro = rs or ResidualOptions(), ro or RenderOptions()
    assert x.dtype == np.float64 and x.flags.c_contiguous
    keep, ptrs = _gts(gts)
    diag = Diag()
    applied = np.empty(x.size) if want_applied else None
    ap = _p(applied) if want_applied else None
    k = C.c_int64(_k(x))
    if s1 is None:
        _check(lib().orc_step_3dgs2tr(state._h, _p(x), k, _cams(cams), ptrs, len(cams),
                                      C.byref(opts.c()), C.byref(rs.c()), C.byref(ro.c()),
                                      ro.workers, C.byref(diag), ap))
    else:
        a1 = np.ascontiguousarray(s1, dtype=np.int32)
        a2 = np.ascontiguousarray(s2 if s2 is not None else [], dtype=np.int32)
        z = _f64(probes) if probes is not None else np.zeros(0)
        _check(lib().orc_step_3dgs2tr_explicit(
            state._h, _p(x), k, _cams(cams), ptrs, len(cams), C.byref(opts.c()),
            C.byref(rs.c()), C.byref(ro.c()), ro.workers, _p(a1), a1.size, _p(a2), a2.size,
            _p(z) if z.size else None, C.byref(diag), ap))
    out = {f: getattr(diag, f) for f, _ in Diag._fields_}
    if want_applied:
        out["applied_step"] = applied
    return out


class Rng:
    """The reference Rng (rng.hpp:15-72)."""

    def __init__(self, seed=1):
        self._h = C.c_void_p(lib().orc_rng_create(C.c_uint64(seed)))

    def __del__(self):
        if getattr(self, "_h", None):
            lib().orc_rng_destroy(self._h)
            self._h = None

    def raw(self, n):
        out = np.empty(n, np.uint64)
        lib().orc_rng_raw(self._h, C.c_int64(n), _p(out))
        return out

    def normal(self, n):
        out = np.empty(n)
        lib().orc_rng_normal(self._h, C.c_int64(n), _p(out))
        return out

    def uniform(self, n, lo=0.0, hi=1.0):
        out = np.empty(n)
        lib().orc_rng_uniform(self._h, C.c_int64(n), C.c_double(lo), C.c_double(hi), _p(out))
        return out

    def sample_without_replacement(self, n, k):
        out = np.empty(min(n, k), np.int32)
        lib().orc_rng_sample(self._h, n, k, _p(out))
        return out

    def rademacher(self, n):
        out = np.empty(n)
        lib().orc_rng_rademacher(self._h, C.c_int64(n), _p(out))
        return out


# --------------------------------------------------------------- datasets
@dataclass
class SynthConfig:  # config.hpp:83-95 defaults
    gt_splats: int = 64
    init_splats: int = 96
    views: int = 25
    image_size: int = 64
    seed: int = 1
    sigma_init: float = 0.04
    init_scale: float = 0.08
    init_opacity: float = 0.5
    camera_radius: float = 2.2
    camera_height: float = 0.77
    focal_factor: float = 2.0
    width: int = 0        # 0: image_size (reference); W x H is a declared extension
    height: int = 0
    size_scale: float = 1.0
    sh_degree: int = 0     # SH colour extension (GT coefficients 0.1 N(0,1), init 0)


@dataclass
class Dataset:
    gt_x: np.ndarray
    init_x: np.ndarray
    cams: list
    gts: list = field(default_factory=list)


def make_synthetic(cfg: SynthConfig, ro=None, with_gt=True) -> Dataset:
    ro = ro or RenderOptions()
    c = SynthCfg(cfg.gt_splats, cfg.init_splats, cfg.views, cfg.image_size, cfg.seed,
                 cfg.sigma_init, cfg.init_scale, cfg.init_opacity, cfg.camera_radius,
                 cfg.camera_height, cfg.focal_factor, cfg.width, cfg.height, cfg.size_scale,
                 cfg.sh_degree)
    gt_x = np.empty(params_per_splat() * cfg.gt_splats)
    init_x = np.empty(params_per_splat() * cfg.init_splats)
    cams = (Camera * cfg.views)()
    W, H = cfg.width or cfg.image_size, cfg.height or cfg.image_size
    gts = [np.empty((H, W, 3)) for _ in range(cfg.views)]
    ptrs = (C.c_void_p * cfg.views)(*[g.ctypes.data for g in gts]) if with_gt else None
    _check(lib().orc_make_synthetic(C.byref(c), C.byref(ro.c()), ro.workers, _p(gt_x),
                                    _p(init_x), cams, ptrs))
    return Dataset(gt_x, init_x, [cams[i] for i in range(cfg.views)], gts if with_gt else [])


def make_check_scene(splats, image_size, n_views, seed):
    x = np.empty(14 * splats)
    cams = (Camera * n_views)()
    gts = [np.empty((image_size, image_size, 3)) for _ in range(n_views)]
    ptrs = (C.c_void_p * n_views)(*[g.ctypes.data for g in gts])
    _check(lib().orc_make_check_scene(splats, image_size, n_views, C.c_uint64(seed), _p(x),
                                      cams, ptrs))
    return x, [cams[i] for i in range(n_views)], gts


def look_at_camera(eye, target, fx, fy, width, height):
    e, t = _f64(eye), _f64(target)
    out = Camera()
    _check(lib().orc_look_at_camera(_p(e), _p(t), C.c_double(fx), C.c_double(fy), width,
                                    height, C.byref(out)))
    return out


# --------------------------------------------------------------- scene helpers
def pack(mu, s, q, alpha, c):
    """Per-splat arrays -> group-major vector (scene.cpp:13-25)."""
    mu, s, q, c = (np.asarray(a, np.float64).reshape(-1, n) for a, n in
                   ((mu, 3), (s, 3), (q, 4), (c, 3)))
    return np.concatenate([mu.ravel(), s.ravel(), q.ravel(),
                           np.asarray(alpha, np.float64).ravel(), c.ravel()])


def unpack(x):
    k = _k(x)
    return (x[:3 * k].reshape(k, 3), x[3 * k:6 * k].reshape(k, 3),
            x[6 * k:10 * k].reshape(k, 4), x[10 * k:11 * k], x[11 * k:].reshape(k, 3))


def step_adam(state, x, cams, gts, opts, adam, trust_region=False, rs=None, ro=None, *,
              s1=None, want_applied=False):
    """step_adam / step_adam_tr (optimizer.cpp:222-253); x updated in place."""
    rs, ro = rs or ResidualOptions(), ro or RenderOptions()
    assert x.dtype == np.float64 and x.flags.c_contiguous
    keep, ptrs = _gts(gts)
    diag = Diag()
    applied = np.empty(x.size) if want_applied else None
    a1 = np.ascontiguousarray(s1 if s1 is not None else [], dtype=np.int32)
    _check(lib().orc_step_adam(
        state._h, _p(x), C.c_int64(_k(x)), _cams(cams), ptrs, len(cams),
        C.byref(opts.c()), C.byref(adam.c()), int(bool(trust_region)), C.byref(rs.c()),
        C.byref(ro.c()), ro.workers, _p(a1) if s1 is not None else None, a1.size,
        C.byref(diag), _p(applied) if want_applied else None))
    out = {f: getattr(diag, f) for f, _ in Diag._fields_}
    if want_applied:
        out["applied_step"] = applied
    return out
