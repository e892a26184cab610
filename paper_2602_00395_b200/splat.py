"""Python mirror of the reference's hot-path API (namespace ``splat``).

Names, argument meaning and error behaviour follow
/root/reference/proj/include/splat/{scene,render,residuals,ssim,optimizer,
trust_region,rng}.hpp; every computation goes through libsgtr.so (the C-ABI
in include/sgtr.h) on a CUDA device.  Reference exceptions map to
``InvalidArgument`` (std::invalid_argument) and ``NumericError``
(splat::NumericError) with the reference's message text.

Two ways in:
  * the drop-in free functions (``rasterize``, ``stochastic_gradient``,
    ``step_3dgs2tr`` ...) take host numpy buffers exactly like the
    reference takes ``Scene``/``Camera``/``Eigen`` values; each call copies
    its inputs to the device and its results back;
  * ``Context`` keeps scene, views and optimizer state resident in HBM and
    steps without host round trips (the fast path bench.py times).
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import _lib
from ._lib import InvalidArgument, NumericError, SgtrError, check, lib

__all__ = [
    "InvalidArgument", "NumericError", "SgtrError", "RenderOptions", "ResidualOptions",
    "TrustRegionSchedule", "RadiusCaps", "ParamBounds", "OptimizerOptions", "Scene",
    "Camera", "RenderedImage", "StepDiagnostics", "OptimizerState", "Rng", "Context",
    "rasterize", "rasterize_jvp", "rasterize_vjp", "ssim_map", "ssim_jvp", "ssim_vjp",
    "mean_ssim", "residual_vector", "residual_jvp", "residual_vjp", "view_jacobian_apply",
    "view_jacobian_applyT", "stochastic_gradient", "rademacher_probes", "hutchinson_diag",
    "ema", "newton_step", "shd_radii", "clip_step", "eps_at", "step_3dgs2tr",
    "step_adam", "step_adam_tr", "AdamOptions", "optimizer_kind_from_string",
    "optimizer_step", "psnr", "quantize8", "evaluate_scene", "EvalResult", "save_scene",
    "load_scene", "save_cameras", "load_cameras", "scene_extent", "make_synthetic", "look_at_camera",
]


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


# ------------------------------------------------------------------ options
@dataclass
class RenderOptions:  # render.hpp:12-22
    z_near: float = 0.01
    lowpass: float = 0.3
    alpha_clamp: float = 0.99
    alpha_skip: float = 1.0 / 255.0
    t_stop: float = 1e-4
    cutoff_sigma: float = 3.0
    background: Sequence[float] = (0.0, 0.0, 0.0)
    workers: int = 0  # accepted for API parity; meaningless on the GPU

    def _c(self) -> _lib.RenderOpts:
        return _lib.RenderOpts(self.z_near, self.lowpass, self.alpha_clamp, self.alpha_skip,
                               self.t_stop, self.cutoff_sigma,
                               (C.c_double * 3)(*[float(b) for b in self.background]))


@dataclass
class ResidualOptions:  # residuals.hpp:13-16
    lambda_: float = 0.2
    floor: float = 1e-12

    def _c(self) -> _lib.ResidualOpts:
        return _lib.ResidualOpts(self.lambda_, self.floor)


@dataclass
class TrustRegionSchedule:  # trust_region.hpp:85-89
    eps_start: float = 1e-6
    eps_end: float = 1e-8
    total_steps: int = 1


@dataclass
class RadiusCaps:  # trust_region.hpp:66-72
    mean: float = 1.0
    scale: float = 1.0
    rotation: float = 1.0
    opacity: float = 1.0
    color: float = 1.0

    def as_tuple(self):
        return (self.mean, self.scale, self.rotation, self.opacity, self.color)


@dataclass
class ParamBounds:  # scene.hpp:29-35
    s_min: float = 1e-6
    alpha_min: float = 1e-4
    alpha_max: float = 0.995
    c_min: float = 1e-6
    c_max: float = 1.5


@dataclass
class AdamOptions:  # optimizer.hpp:21-34
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

    def _c(self, scene_extent: float) -> _lib.AdamOpts:
        return _lib.AdamOpts(self.beta1, self.beta2, self.eps, self.lr_position,
                             self.lr_position_final, self.lr_position_decay_steps, 0,
                             self.lr_scale, self.lr_rotation, self.lr_opacity, self.lr_color,
                             scene_extent)


# OptimizerKind (optimizer.hpp:17) and optimizer_kind_from_string's spellings
_KINDS = {"3dgs2tr": 0, "adam": 1, "adam-tr": 2}


def optimizer_kind_from_string(s: str) -> str:
    """optimizer.cpp optimizer_kind_from_string: the accepted spellings."""
    if s not in _KINDS:
        raise InvalidArgument(f"unknown optimizer '{s}'")
    return s


@dataclass
class OptimizerOptions:  # optimizer.hpp:37-53
    kind: str = "3dgs2tr"
    theta1: float = 0.9
    theta2: float = 0.999
    hess_interval: int = 10
    hutch_samples: int = 1
    batch_size: int = 1
    hutch_batch_size: int = 1
    gamma_d: float = 1e-12
    schedule: TrustRegionSchedule = field(default_factory=TrustRegionSchedule)
    caps: RadiusCaps = field(default_factory=RadiusCaps)
    bounds: ParamBounds = field(default_factory=ParamBounds)
    residual: ResidualOptions = field(default_factory=ResidualOptions)
    render: RenderOptions = field(default_factory=RenderOptions)
    adam: AdamOptions = field(default_factory=AdamOptions)
    scene_extent: float = 1.0
    record_applied_step: bool = True

    def _kind(self) -> int:
        return _KINDS[optimizer_kind_from_string(self.kind)]

    def _c(self) -> _lib.OptimizerOpts:
        s, c, b = self.schedule, self.caps, self.bounds
        return _lib.OptimizerOpts(
            self.theta1, self.theta2, self.hess_interval, self.hutch_samples, self.batch_size,
            self.hutch_batch_size, self.gamma_d, s.eps_start, s.eps_end, s.total_steps,
            1 if self.record_applied_step else 0, c.mean, c.scale, c.rotation, c.opacity,
            c.color, b.s_min, b.alpha_min, b.alpha_max, b.c_min, b.c_max, self.residual._c(),
            self.render._c())


# ------------------------------------------------------------------ scene / camera
def params_per_splat(sh_degree: int = 0) -> int:
    """14 (the reference) + 3 SH coefficients per basis function of degree
    1..sh_degree (the SH colour extension, include/sgtr.h)."""
    return 14 + 3 * ((sh_degree + 1) ** 2 - 1)


class Scene:
    """Flat group-major parameter vector (scene.hpp:37-64), optionally with
    the SH group appended (sh_degree > 0, extension)."""

    kParamsPerSplat = 14

    def __init__(self, x=None, k: Optional[int] = None, sh_degree: int = 0):
        if not 0 <= sh_degree <= 3:
            raise InvalidArgument("Scene: SH degree must be 0..3")
        self.sh_degree = sh_degree
        npp = params_per_splat(sh_degree)
        if x is None:
            x = np.zeros(npp * (k or 0))
        self.x = _f64(x).copy()
        if self.x.size % npp:
            raise InvalidArgument(f"Scene: vector length is not a multiple of {npp}")

    @classmethod
    def from_primitives(cls, mu, scale, quat, opacity, color) -> "Scene":
        mu, scale, quat, color = (np.asarray(a, np.float64).reshape(-1, n) for a, n in
                                  ((mu, 3), (scale, 3), (quat, 4), (color, 3)))
        return cls(np.concatenate([mu.ravel(), scale.ravel(), quat.ravel(),
                                   np.asarray(opacity, np.float64).ravel(), color.ravel()]))

    def size(self) -> int:
        return self.x.size // params_per_splat(self.sh_degree)

    def dim(self) -> int:
        return self.x.size

    def pos_offset(self):
        return 0

    def scale_offset(self):
        return 3 * self.size()

    def quat_offset(self):
        return 6 * self.size()

    def opacity_offset(self):
        return 10 * self.size()

    def color_offset(self):
        return 11 * self.size()

    def pack(self) -> np.ndarray:
        return self.x.copy()

    def unpack(self, x) -> None:
        x = _f64(x)
        if x.size != self.x.size:
            raise InvalidArgument("Scene::unpack: dimension mismatch")
        self.x[:] = x

    def copy(self) -> "Scene":
        return Scene(self.x, sh_degree=self.sh_degree)

    def primitives(self):
        k = self.size()
        x = self.x
        return (x[:3 * k].reshape(k, 3), x[3 * k:6 * k].reshape(k, 3),
                x[6 * k:10 * k].reshape(k, 4), x[10 * k:11 * k],
                x[11 * k:14 * k].reshape(k, 3))

    def sh_coefficients(self) -> np.ndarray:
        """(K, nb, 3) view of the SH group (empty for degree 0)."""
        k = self.size()
        return self.x[14 * k:].reshape(k, (self.sh_degree + 1) ** 2 - 1, 3)


@dataclass
class Camera:  # scene.hpp:70-81
    id: int = 0
    fx: float = 1.0
    fy: float = 1.0
    cx: float = 0.0
    cy: float = 0.0
    width: int = 0
    height: int = 0
    q_wc: Sequence[float] = (0.0, 0.0, 0.0, 1.0)
    t_wc: Sequence[float] = (0.0, 0.0, 0.0)
    gt: Optional[np.ndarray] = None  # (H, W, 3) float64
    image_name: str = ""

    def _c(self) -> _lib.Camera:
        return _lib.Camera(self.id, self.width, self.height, 0, self.fx, self.fy, self.cx,
                           self.cy, (C.c_double * 4)(*map(float, self.q_wc)),
                           (C.c_double * 3)(*map(float, self.t_wc)))

    def rotation(self) -> np.ndarray:
        x, y, z, w = map(float, self.q_wc)
        r2 = x * x + y * y + z * z + w * w
        m = np.array([[r2 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
                      [2 * (x * y + w * z), r2 - 2 * (z * z + x * x), 2 * (y * z - w * x)],
                      [2 * (x * z - w * y), 2 * (y * z + w * x), r2 - 2 * (x * x + y * y)]])
        return m / r2

    def center(self) -> np.ndarray:
        return -self.rotation().T @ np.asarray(self.t_wc, np.float64)

    @classmethod
    def from_c(cls, c: _lib.Camera, gt=None) -> "Camera":
        return cls(c.id, c.fx, c.fy, c.cx, c.cy, c.width, c.height, tuple(c.q_wc),
                   tuple(c.t_wc), gt)


@dataclass
class RenderedImage:  # render.hpp:65-68
    color: np.ndarray    # (H, W, 3)
    t_final: np.ndarray  # (H, W)


@dataclass
class StepDiagnostics:  # optimizer.hpp:74-83
    batch_loss: float = 0.0
    gnorm: float = 0.0
    step_pre: float = 0.0
    step_post: float = 0.0
    clip_frac: float = -1.0
    eps: float = -1.0
    max_step_over_radius: float = 0.0
    applied_step: Optional[np.ndarray] = None
    refreshed: bool = False
    n_local_views: int = 0  # views of the batch this rank rendered (multi-rank split)
    reruns: int = 0  # reruns after a view outgrew the tile-duplicate capacity


# ------------------------------------------------------------------ context
class Context:
    """A libsgtr context: scene, views and optimizer state resident on one GPU."""

    def __init__(self, device: int = 0):
        h = C.c_void_p()
        check(lib().sgtr_create(device, C.byref(h)))
        self._h = h
        self.device = device
        self._views_key = None
        self.n_views = 0
        self.k = 0
        self.sh_degree = 0

    def close(self):
        if getattr(self, "_h", None):
            lib().sgtr_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    def stream(self) -> int:
        s = C.c_void_p()
        check(lib().sgtr_get_stream(self._h, C.byref(s)))
        return s.value or 0

    def synchronize(self):
        check(lib().sgtr_synchronize(self._h))

    def launch_count(self) -> int:
        return int(lib().sgtr_launch_count(self._h))

    # scene
    def set_scene(self, x: np.ndarray, sh_degree: int = 0) -> None:
        x = _f64(x)
        npp = params_per_splat(sh_degree)
        if x.size % npp:
            raise InvalidArgument(f"set_scene: vector length is not a multiple of {npp}")
        check(lib().sgtr_set_scene_sh(self._h, _ptr(x), x.size // npp, sh_degree))
        self.k = x.size // npp
        self.sh_degree = sh_degree

    @property
    def dim(self) -> int:
        return params_per_splat(getattr(self, "sh_degree", 0)) * self.k

    def get_scene(self, out: Optional[np.ndarray] = None) -> np.ndarray:
        out = np.empty(self.dim) if out is None else out
        check(lib().sgtr_get_scene(self._h, _ptr(out)))
        return out

    # views
    def save_scene(self, path: str) -> None:
        """save_scene of the resident scene (device transpose, one copy)."""
        check(lib().sgtr_save_scene_ply(self._h, str(path).encode()))

    def load_scene(self, path: str, bounds: Optional[ParamBounds] = None) -> None:
        """load_scene straight into HBM (validation on the device)."""
        check(lib().sgtr_load_scene_ply(self._h, str(path).encode(), _bounds_c(bounds)))
        self.k = int(lib().sgtr_scene_size(self._h))
        self.sh_degree = 0

    def checkpoint_save(self, path: str) -> None:
        """Scene + full optimizer state (g_hat, d_hat, ADAM moments, t, Rng)."""
        check(lib().sgtr_checkpoint_save(self._h, str(path).encode()))

    def checkpoint_load(self, path: str) -> None:
        """Resume from checkpoint_save: the next step continues bit for bit."""
        check(lib().sgtr_checkpoint_load(self._h, str(path).encode()))
        self.k = int(lib().sgtr_scene_size(self._h))
        self.sh_degree = int(lib().sgtr_scene_sh_degree(self._h))

    def set_eval_views(self, views: Sequence[Camera]) -> None:
        """Held-out views (with targets) for evaluate(); kept on the device."""
        n = len(views)
        arr = (_lib.Camera * max(n, 1))()
        keep = []
        for i, v in enumerate(views):
            if v.gt is None:
                raise InvalidArgument("evaluate_scene: view has no target image")
            g = _f64(v.gt)
            if g.shape != (v.height, v.width, 3):
                raise InvalidArgument("Camera.gt shape does not match the camera")
            arr[i] = v._c()
            keep.append(g)
        gts = (C.c_void_p * max(n, 1))(*[g.ctypes.data for g in keep])
        check(lib().sgtr_set_eval_views(self._h, arr, n, gts))
        self.n_eval_views = n

    def evaluate(self, ro: Optional[RenderOptions] = None, training_views: bool = False):
        """evaluate_scene (harness.cpp:43-58) on the resident scene: the eval
        views (or the training views) rendered, quantised and scored on the
        device; returns an EvalResult."""
        ro = ro or RenderOptions()
        n = self.n_views if training_views else getattr(self, "n_eval_views", 0)
        vp, vs = np.empty(max(n, 1)), np.empty(max(n, 1))
        mp, ms = C.c_double(), C.c_double()
        check(lib().sgtr_evaluate_scene(self._h, 1 if training_views else 0, C.byref(ro._c()),
                                        _ptr(vp), _ptr(vs), C.byref(mp), C.byref(ms)))
        return EvalResult(vp[:n].tolist(), vs[:n].tolist(), mp.value, ms.value)

    def set_views(self, views: Sequence[Camera], with_gt: bool = True) -> None:
        n = len(views)
        arr = (_lib.Camera * max(n, 1))()
        for i, v in enumerate(views):
            arr[i] = v._c()
        gts = None
        keep = []
        if with_gt and n and all(v.gt is not None for v in views):
            keep = [_f64(v.gt) for v in views]
            for g, v in zip(keep, views):
                if g.shape != (v.height, v.width, 3):
                    raise InvalidArgument("Camera.gt shape does not match the camera")
            gts = (C.c_void_p * n)(*[g.ctypes.data for g in keep])
        check(lib().sgtr_set_views(self._h, arr, n, gts))
        self.n_views = n
        self._views_key = tuple(id(v) for v in views)

    def set_cameras(self, cams) -> None:
        """Views without targets; ``cams`` are Camera objects or any struct
        with the sgtr_camera fields."""
        n = len(cams)
        arr = (_lib.Camera * max(n, 1))()
        for i, c in enumerate(cams):
            arr[i] = c._c() if isinstance(c, Camera) else Camera.from_c(c)._c()
        check(lib().sgtr_set_views(self._h, arr, n, None))
        self.n_views = n
        self._views_key = None

    def render_targets(self, ro: Optional[RenderOptions] = None, quantize: bool = True):
        ro = ro or RenderOptions()
        check(lib().sgtr_render_targets(self._h, C.byref(ro._c()), 1 if quantize else 0))

    def get_target(self, view: int, width: int, height: int) -> np.ndarray:
        out = np.empty((height, width, 3))
        check(lib().sgtr_get_target(self._h, view, _ptr(out)))
        return out

    # optimizer state
    def state_reset(self, seed: int) -> None:
        check(lib().sgtr_state_reset(self._h, C.c_uint64(seed)))

    def state_get(self):
        g, d, t = np.empty(self.dim), np.empty(self.dim), C.c_int64()
        check(lib().sgtr_state_get(self._h, _ptr(g), _ptr(d), C.byref(t)))
        return g, d, t.value

    def state_set(self, g_hat, d_hat, t: int) -> None:
        g = None if g_hat is None else _f64(g_hat)
        d = None if d_hat is None else _f64(d_hat)
        check(lib().sgtr_state_set(self._h, _ptr(g), _ptr(d), t))

    def rng_raw(self, n: int) -> np.ndarray:
        """n raw mt19937_64 draws continuing the state's Rng (rng.hpp:24)."""
        out = np.empty(n, np.uint64)
        check(lib().sgtr_rng_raw(self._h, C.c_int64(n), _ptr(out)))
        return out

    def state_get_adam(self):
        m, v = np.empty(self.dim), np.empty(self.dim)
        check(lib().sgtr_state_get_adam(self._h, _ptr(m), _ptr(v)))
        return m, v

    def state_set_adam(self, m, v) -> None:
        m = None if m is None else _f64(m)
        v = None if v is None else _f64(v)
        check(lib().sgtr_state_set_adam(self._h, _ptr(m), _ptr(v)))

    def step(self, opt: OptimizerOptions, *, s1=None, s2=None, probe_bits=None,
             nu: int = 1) -> StepDiagnostics:
        """One Algorithm-1 step on the resident scene (optimizer.cpp:189-220).

        With s1 given the draws are teacher-forced (probe_bits: uint32 array of
        nu * ceil(dim/32) words); otherwise they come from the state's Rng."""
        d = _lib.StepDiag()
        co = opt._c()
        kind = opt._kind()
        if kind != 0:  # step_adam / step_adam_tr (optimizer.cpp:222-253)
            ao = opt.adam._c(opt.scene_extent)
            if s1 is None:
                check(lib().sgtr_optimizer_step(self._h, kind, C.byref(co), C.byref(ao),
                                                C.byref(d)))
            else:
                a1 = np.ascontiguousarray(s1, np.int32)
                check(lib().sgtr_step_adam_explicit(self._h, C.byref(co), C.byref(ao),
                                                    1 if kind == 2 else 0, _ptr(a1), a1.size,
                                                    C.byref(d)))
        elif s1 is None:
            check(lib().sgtr_step_3dgs2tr(self._h, C.byref(co), C.byref(d)))
        else:
            a1 = np.ascontiguousarray(s1, np.int32)
            a2 = np.ascontiguousarray(s2 if s2 is not None else [], np.int32)
            pb = None if probe_bits is None else np.ascontiguousarray(probe_bits, np.uint32)
            check(lib().sgtr_step_3dgs2tr_explicit(self._h, C.byref(co), _ptr(a1), a1.size,
                                                   _ptr(a2), a2.size, _ptr(pb), nu,
                                                   C.byref(d)))
        out = StepDiagnostics(d.batch_loss, d.gnorm, d.step_pre, d.step_post, d.clip_frac,
                              d.eps, d.max_step_over_radius, None, bool(d.refreshed),
                              int(d.n_local_views), int(d.reruns))
        if opt.record_applied_step:
            out.applied_step = np.empty(self.dim)
            check(lib().sgtr_get_applied_step(self._h, _ptr(out.applied_step)))
        return out

    def set_dup_capacity(self, capacity: int) -> None:
        """Presize (or shrink) the per-view tile-duplicate arrays; a step
        whose views outgrow them reruns with a grown capacity (0: default)."""
        check(lib().sgtr_set_dup_capacity(self._h, capacity))

    def set_refresh_bands(self, bands_per_rank: int) -> None:
        """Split each refresh view into nranks * bands_per_rank row bands."""
        check(lib().sgtr_set_refresh_bands(self._h, bands_per_rank))

    def set_tr_shards(self, shards: int) -> None:
        """Run the trust-region radii as `shards` splat-range shards (the
        multi-GPU split, back to back on one rank)."""
        check(lib().sgtr_set_tr_shards(self._h, shards))

    def comm_init(self, unique_id: bytes, nranks: int, rank: int) -> None:
        buf = (C.c_uint8 * 128).from_buffer_copy(unique_id)
        check(lib().sgtr_comm_init(self._h, buf, nranks, rank))

    def comm_init_loopback(self, group: "LoopbackGroup", rank: int) -> None:
        """Join an in-process group (one host thread per rank on one GPU)."""
        check(lib().sgtr_comm_init_loopback(self._h, group.handle, rank))


class LoopbackGroup:
    """In-process communicator over one GPU (sgtr_loopback_group_create):
    tests run the N-rank data plane with N threads, one Context each."""

    def __init__(self, nranks: int):
        h = C.c_void_p()
        check(lib().sgtr_loopback_group_create(nranks, C.byref(h)))
        self.handle = h
        self.nranks = nranks

    def close(self) -> None:
        if self.handle:
            check(lib().sgtr_loopback_group_destroy(self.handle))
            self.handle = None


def shard_views(n: int, rank: int, nranks: int) -> List[int]:
    """Positions of an n-view batch that ``rank`` of ``nranks`` renders (the
    split libsgtr's step uses before its single allreduce)."""
    out = np.empty(max(n, 1), np.int32)
    cnt = C.c_int32()
    check(lib().sgtr_shard_views(n, rank, nranks, _ptr(out), C.byref(cnt)))
    return out[:cnt.value].tolist()


def nccl_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    check(lib().sgtr_nccl_unique_id(buf))
    return bytes(buf)


_default = {}


def default_context(device: int = 0) -> Context:
    """The context the drop-in free functions run on."""
    if device not in _default:
        _default[device] = Context(device)
    return _default[device]


def _scene_ctx(scene: Scene, ctx: Optional[Context]) -> Context:
    ctx = ctx or default_context()
    ctx.set_scene(scene.x, scene.sh_degree)
    return ctx


def _views_ctx(ctx: Context, views: Sequence[Camera]) -> None:
    key = tuple(id(v) for v in views)
    if ctx._views_key != key or getattr(ctx, "_views_ref", None) is not views:
        ctx.set_views(views)
        ctx._views_ref = views


# ------------------------------------------------------------------ renderer seams
def rasterize(scene: Scene, cam: Camera, opt: Optional[RenderOptions] = None,
              ctx: Optional[Context] = None) -> RenderedImage:
    """render.hpp:73-74."""
    opt = opt or RenderOptions()
    c = _scene_ctx(scene, ctx)
    color = np.empty((cam.height, cam.width, 3))
    t = np.empty((cam.height, cam.width))
    check(lib().sgtr_rasterize(c.handle, C.byref(cam._c()), C.byref(opt._c()), _ptr(color),
                               _ptr(t)))
    return RenderedImage(color, t)


def rasterize_jvp(scene: Scene, cam: Camera, v, opt: Optional[RenderOptions] = None,
                  ctx: Optional[Context] = None) -> np.ndarray:
    """render.hpp:78-79."""
    opt = opt or RenderOptions()
    v = _f64(v)
    if v.size != scene.dim():
        raise InvalidArgument("rasterize_jvp: direction length mismatch")
    c = _scene_ctx(scene, ctx)
    out = np.empty((cam.height, cam.width, 3))
    check(lib().sgtr_rasterize_jvp(c.handle, C.byref(cam._c()), C.byref(opt._c()), _ptr(v),
                                   _ptr(out)))
    return out


def rasterize_vjp(scene: Scene, cam: Camera, adjoint, opt: Optional[RenderOptions] = None,
                  ctx: Optional[Context] = None) -> np.ndarray:
    """render.hpp:83-84."""
    opt = opt or RenderOptions()
    a = _f64(adjoint)
    if a.shape != (cam.height, cam.width, 3):
        raise InvalidArgument("rasterize_vjp: adjoint shape mismatch")
    c = _scene_ctx(scene, ctx)
    g = np.empty(scene.dim())
    check(lib().sgtr_rasterize_vjp(c.handle, C.byref(cam._c()), C.byref(opt._c()), _ptr(a),
                                   _ptr(g)))
    return g


# ------------------------------------------------------------------ SSIM / residuals
def _img_pair(a, b, what):
    a, b = _f64(a), _f64(b)
    if a.shape != b.shape:
        raise InvalidArgument(f"{what}: image shape mismatch")
    return a, b


def ssim_map(a, b, ctx: Optional[Context] = None) -> np.ndarray:
    """ssim.hpp:11."""
    a, b = _img_pair(a, b, "ssim")
    out = np.empty_like(a)
    check(lib().sgtr_ssim_map((ctx or default_context()).handle, _ptr(a), _ptr(b), a.shape[1],
                              a.shape[0], _ptr(out)))
    return out


def ssim_jvp(a, da, b, ctx: Optional[Context] = None):
    """ssim.hpp:14-16 -> (s, ds)."""
    a, b = _img_pair(a, b, "ssim")
    da = _f64(da)
    if da.shape != a.shape:
        raise InvalidArgument("ssim: image shape mismatch")
    s, ds = np.empty_like(a), np.empty_like(a)
    check(lib().sgtr_ssim_jvp((ctx or default_context()).handle, _ptr(a), _ptr(da), _ptr(b),
                              a.shape[1], a.shape[0], _ptr(s), _ptr(ds)))
    return s, ds


def ssim_vjp(a, b, upstream, ctx: Optional[Context] = None) -> np.ndarray:
    """ssim.hpp:18-19."""
    a, b = _img_pair(a, b, "ssim")
    u = _f64(upstream)
    if u.shape != a.shape:
        raise InvalidArgument("ssim: image shape mismatch")
    g = np.empty_like(a)
    check(lib().sgtr_ssim_vjp((ctx or default_context()).handle, _ptr(a), _ptr(b), _ptr(u),
                              a.shape[1], a.shape[0], _ptr(g)))
    return g


def mean_ssim(a, b, ctx: Optional[Context] = None) -> float:
    """ssim.cpp:170-175 (evaluation helper)."""
    return float(np.mean(ssim_map(a, b, ctx)))


def residual_vector(rendered, gt, opt: Optional[ResidualOptions] = None,
                    ctx: Optional[Context] = None) -> np.ndarray:
    """residuals.hpp:23-24."""
    opt = opt or ResidualOptions()
    r_, g_ = _img_pair(rendered, gt, "residuals")
    out = np.empty(2 * r_.size)
    check(lib().sgtr_residual_vector((ctx or default_context()).handle, _ptr(r_), _ptr(g_),
                                     r_.shape[1], r_.shape[0], C.byref(opt._c()), _ptr(out)))
    return out


def residual_jvp(rendered, tangent, gt, opt: Optional[ResidualOptions] = None,
                 ctx: Optional[Context] = None) -> np.ndarray:
    """residuals.hpp:28-29."""
    opt = opt or ResidualOptions()
    r_, g_ = _img_pair(rendered, gt, "residuals")
    t = _f64(tangent)
    if t.shape != r_.shape:
        raise InvalidArgument("residuals: image shape mismatch")
    out = np.empty(2 * r_.size)
    check(lib().sgtr_residual_jvp((ctx or default_context()).handle, _ptr(r_), _ptr(t), _ptr(g_),
                                  r_.shape[1], r_.shape[0], C.byref(opt._c()), _ptr(out)))
    return out


def residual_vjp(rendered, gt, u, opt: Optional[ResidualOptions] = None,
                 ctx: Optional[Context] = None) -> np.ndarray:
    """residuals.hpp:32-33."""
    opt = opt or ResidualOptions()
    r_, g_ = _img_pair(rendered, gt, "residuals")
    u = _f64(u)
    if u.size != 2 * r_.size:
        raise InvalidArgument("residual_vjp: adjoint length mismatch")
    out = np.empty_like(r_)
    check(lib().sgtr_residual_vjp((ctx or default_context()).handle, _ptr(r_), _ptr(g_),
                                  r_.shape[1], r_.shape[0], _ptr(u), C.byref(opt._c()),
                                  _ptr(out)))
    return out


def psnr(a, b) -> float:
    """residuals.cpp:133-144 (evaluation helper, host)."""
    a, b = _img_pair(a, b, "psnr")
    mse = float(np.mean((a - b) ** 2))
    return 100.0 if mse < 1e-10 else 10.0 * math.log10(1.0 / mse)


# ------------------------------------------------------------------ files
def _bounds_c(b: Optional[ParamBounds]):
    if b is None:
        return None
    return C.byref(_lib.ParamBounds(b.s_min, b.alpha_min, b.alpha_max, b.c_min, b.c_max))


def save_scene(scene: Scene, path: str) -> None:
    """scene_io.hpp:17 (binary little-endian PLY, bitwise round trip)."""
    check(lib().sgtr_ply_save(_ptr(scene.x), scene.size(), str(path).encode()))


def load_scene(path: str, bounds: Optional[ParamBounds] = None) -> Scene:
    """scene_io.hpp:18-19: parse, then Scene::validate(bounds); errors are
    SgtrError (std::runtime_error) naming the line or the splat."""
    k = C.c_int64()
    check(lib().sgtr_ply_load(str(path).encode(), None, None, C.byref(k)))
    x = np.empty(14 * k.value)
    check(lib().sgtr_ply_load(str(path).encode(), _bounds_c(bounds), _ptr(x), C.byref(k)))
    return Scene(x)


def save_cameras(cams: Sequence[Camera], path: str) -> None:
    """scene_io.hpp:24 (one camera per line, %.17g)."""
    n = len(cams)
    arr = (_lib.Camera * max(n, 1))()
    for i, c in enumerate(cams):
        arr[i] = c._c()
    names = (C.c_char_p * max(n, 1))(*[c.image_name.encode() for c in cams])
    check(lib().sgtr_save_cameras(str(path).encode(), arr, names, n))


def load_cameras(path: str) -> List[Camera]:
    """scene_io.hpp:25-26 with load_images = false (targets are set through
    Context.set_views / render_targets)."""
    n = C.c_int32()
    check(lib().sgtr_load_cameras(str(path).encode(), None, None, 0, 0, C.byref(n)))
    arr = (_lib.Camera * max(n.value, 1))()
    stride = 4096
    names = C.create_string_buffer(stride * max(n.value, 1))
    check(lib().sgtr_load_cameras(str(path).encode(), arr, names, stride, n.value, C.byref(n)))
    out = []
    for i in range(n.value):
        cam = Camera.from_c(arr[i])
        cam.image_name = names.raw[i * stride:(i + 1) * stride].split(b"\0", 1)[0].decode()
        out.append(cam)
    return out


def scene_extent(cams: Sequence[Camera]) -> float:
    """scene.hpp:83-85 (OptimizerOptions.scene_extent for the ADAM kinds)."""
    n = len(cams)
    arr = (_lib.Camera * max(n, 1))()
    for i, c in enumerate(cams):
        arr[i] = c._c()
    out = C.c_double()
    check(lib().sgtr_scene_extent(arr, n, C.byref(out)))
    return out.value


@dataclass
class EvalResult:  # harness.hpp:29-35
    view_psnr: List[float]
    view_ssim: List[float]
    mean_psnr: float
    mean_ssim: float


def evaluate_scene(scene: Scene, views: Sequence[Camera],
                   ropt: Optional[RenderOptions] = None,
                   ctx: Optional[Context] = None) -> EvalResult:
    """harness.cpp:43-58 on the GPU: per view, PSNR and mean SSIM of
    quantize8(rasterize(scene, cam).color) against cam.gt."""
    if not views:
        raise InvalidArgument("evaluate_scene: empty view list")
    c = _scene_ctx(scene, ctx)
    c.set_eval_views(views)
    return c.evaluate(ropt)


def quantize8(img) -> np.ndarray:
    """image.cpp:13-20 (host helper)."""
    return np.round(np.clip(_f64(img), 0.0, 1.0) * 255.0) / 255.0


# ------------------------------------------------------------------ optimizer seams
def _one_view_ctx(scene: Scene, cam: Camera, ctx: Optional[Context]) -> Context:
    c = _scene_ctx(scene, ctx)
    if cam.gt is None:
        raise InvalidArgument("view has no target image")
    c.set_views([cam])
    return c


def view_jacobian_apply(scene: Scene, cam: Camera, v, ropt: Optional[ResidualOptions] = None,
                        render: Optional[RenderOptions] = None,
                        ctx: Optional[Context] = None) -> np.ndarray:
    """optimizer.hpp:87-90: residual-space J_i v."""
    ropt, render = ropt or ResidualOptions(), render or RenderOptions()
    v = _f64(v)
    if v.size != scene.dim():
        raise InvalidArgument("rasterize_jvp: direction length mismatch")
    c = _one_view_ctx(scene, cam, ctx)
    out = np.empty(6 * cam.width * cam.height)
    check(lib().sgtr_view_jacobian_apply(c.handle, 0, _ptr(v), C.byref(ropt._c()),
                                         C.byref(render._c()), _ptr(out)))
    return out


def view_jacobian_applyT(scene: Scene, cam: Camera, u, ropt: Optional[ResidualOptions] = None,
                         render: Optional[RenderOptions] = None,
                         ctx: Optional[Context] = None) -> np.ndarray:
    """optimizer.hpp:91-94: J_i^T u."""
    ropt, render = ropt or ResidualOptions(), render or RenderOptions()
    u = _f64(u)
    if u.size != 6 * cam.width * cam.height:
        raise InvalidArgument("residual_vjp: adjoint length mismatch")
    c = _one_view_ctx(scene, cam, ctx)
    g = np.empty(scene.dim())
    check(lib().sgtr_view_jacobian_applyT(c.handle, 0, _ptr(u), C.byref(ropt._c()),
                                          C.byref(render._c()), _ptr(g)))
    return g


def stochastic_gradient(scene: Scene, views: Sequence[Camera], batch: Sequence[int],
                        ropt: Optional[ResidualOptions] = None,
                        render: Optional[RenderOptions] = None,
                        ctx: Optional[Context] = None):
    """optimizer.hpp:99-104 -> (g, batch_loss)."""
    ropt, render = ropt or ResidualOptions(), render or RenderOptions()
    c = _scene_ctx(scene, ctx)
    _views_ctx(c, views)
    b = np.ascontiguousarray(batch, np.int32)
    g = np.empty(scene.dim())
    loss = C.c_double()
    check(lib().sgtr_stochastic_gradient(c.handle, _ptr(b), b.size, C.byref(ropt._c()),
                                         C.byref(render._c()), _ptr(g), C.byref(loss)))
    return g, loss.value


class Rng:
    """The reference Rng (rng.hpp:15-72): std::mt19937_64 (native) with the
    reference's hand-rolled variate mappings."""

    def __init__(self, seed: int = 1):
        h = C.c_void_p()
        check(lib().sgtr_rng_new(C.c_uint64(seed), C.byref(h)))
        self._h = h
        self._spare = None

    def __del__(self):
        if getattr(self, "_h", None):
            lib().sgtr_rng_free(self._h)
            self._h = None

    def raw_n(self, n: int) -> np.ndarray:
        out = np.empty(n, np.uint64)
        check(lib().sgtr_rng_draw(self._h, n, _ptr(out)))
        return out

    def raw(self) -> int:
        return int(self.raw_n(1)[0])

    def uniform(self, lo: float = 0.0, hi: float = 1.0) -> float:
        u = float(self.raw() >> 11) * 2.0 ** -53
        return u if (lo, hi) == (0.0, 1.0) else lo + (hi - lo) * u

    def log_uniform(self, lo: float, hi: float) -> float:
        return math.exp(self.uniform(math.log(lo), math.log(hi)))

    def normal(self) -> float:
        if self._spare is not None:
            s, self._spare = self._spare, None
            return s
        u1 = self.uniform()
        while u1 <= 0.0:
            u1 = self.uniform()
        u2 = self.uniform()
        r = math.sqrt(-2.0 * math.log(u1))
        self._spare = r * math.sin(2.0 * math.pi * u2)
        return r * math.cos(2.0 * math.pi * u2)

    def rademacher_n(self, n: int) -> np.ndarray:
        return np.where(self.raw_n(n) & np.uint64(1), 1.0, -1.0)

    def rademacher(self) -> float:
        return float(self.rademacher_n(1)[0])

    def below(self, n: int) -> int:
        return self.raw() % n

    def sample_without_replacement(self, n: int, k: int) -> List[int]:
        idx = list(range(n))
        for i in range(min(k, n)):
            j = i + self.below(n - i)
            idx[i], idx[j] = idx[j], idx[i]
        return idx[:min(k, n)]


def rademacher_probes(rng: Rng, dim: int):
    """optimizer.cpp:67-73: each probe draws dim values coordinate-ascending."""
    return lambda sample: rng.rademacher_n(dim)


def hutchinson_diag(scene: Scene, views: Sequence[Camera], batch: Sequence[int], nu: int,
                    probes, ropt: Optional[ResidualOptions] = None,
                    render: Optional[RenderOptions] = None,
                    ctx: Optional[Context] = None) -> np.ndarray:
    """optimizer.hpp:106-117; ``probes`` is a ProbeSource (callable sample -> z)."""
    ropt, render = ropt or ResidualOptions(), render or RenderOptions()
    if nu < 1:
        raise InvalidArgument("hutchinson_diag: nu must be >= 1")
    z = []
    for s in range(nu):
        zs = _f64(probes(s))
        if zs.size != scene.dim():
            raise InvalidArgument("hutchinson_diag: probe length mismatch")
        z.append(zs)
    zz = np.ascontiguousarray(np.stack(z)) if z else np.zeros((0, scene.dim()))
    c = _scene_ctx(scene, ctx)
    _views_ctx(c, views)
    b = np.ascontiguousarray(batch, np.int32)
    d = np.empty(scene.dim())
    check(lib().sgtr_hutchinson_diag(c.handle, _ptr(b), b.size, nu, _ptr(zz),
                                     C.byref(ropt._c()), C.byref(render._c()), _ptr(d)))
    return d


def ema(prev, nxt, theta: float) -> np.ndarray:
    """optimizer.hpp:119-122."""
    return theta * _f64(prev) + (1.0 - theta) * _f64(nxt)


def newton_step(g_hat, d_hat, gamma: float) -> np.ndarray:
    """optimizer.cpp:106-112."""
    g, d = _f64(g_hat), _f64(d_hat)
    return -g / np.where(d < gamma, gamma, d)


def shd_radii(scene: Scene, eps: float, caps: Optional[RadiusCaps] = None,
              ctx: Optional[Context] = None) -> np.ndarray:
    """trust_region.hpp:81-83."""
    caps = caps or RadiusCaps()
    c = _scene_ctx(scene, ctx)
    eta = np.empty(scene.dim())
    check(lib().sgtr_shd_radii(c.handle, C.c_double(eps), (C.c_double * 5)(*caps.as_tuple()),
                               _ptr(eta)))
    return eta


def clip_step(delta, eta) -> np.ndarray:
    """trust_region.cpp:254-259."""
    d, e = _f64(delta), _f64(eta)
    if d.size != e.size:
        raise InvalidArgument("clip_step: length mismatch")
    c = np.where(d < -e, -e, d)
    return np.where(e < c, e, c)


def eps_at(s: TrustRegionSchedule, t: int) -> float:
    """trust_region.cpp:261-268."""
    out = C.c_double()
    check(lib().sgtr_eps_at(s.eps_start, s.eps_end, s.total_steps, t, C.byref(out)))
    return out.value


class OptimizerState:
    """OptimizerState (optimizer.hpp:58-72), resident in its own context:
    g_hat, d_hat and t live on the GPU, the Rng on the host side of libsgtr."""

    def __init__(self, dim: int, seed: int, device: int = 0, sh_degree: int = 0):
        if dim % params_per_splat(sh_degree):
            raise InvalidArgument(
                f"OptimizerState: dim is not a multiple of {params_per_splat(sh_degree)}")
        self.ctx = Context(device)
        self.ctx.set_scene(np.zeros(dim), sh_degree)
        self.ctx.state_reset(seed)
        self.dim = dim

    @property
    def g_hat(self) -> np.ndarray:
        return self.ctx.state_get()[0]

    @property
    def d_hat(self) -> np.ndarray:
        return self.ctx.state_get()[1]

    @property
    def t(self) -> int:
        return self.ctx.state_get()[2]

    @property
    def adam_m(self) -> np.ndarray:
        return self.ctx.state_get_adam()[0]

    @property
    def adam_v(self) -> np.ndarray:
        return self.ctx.state_get_adam()[1]


def step_3dgs2tr(state: OptimizerState, scene: Scene, views: Sequence[Camera],
                 opt: OptimizerOptions) -> StepDiagnostics:
    """optimizer.hpp:129-131.  ``scene`` is updated in place (host copy in and
    out, like the reference's Scene&); state stays on the device."""
    return _step_host(state, scene, views, _with_kind(opt, "3dgs2tr"), "step_3dgs2tr")


def _step_host(state: OptimizerState, scene: Scene, views: Sequence[Camera],
               opt: OptimizerOptions, what: str) -> StepDiagnostics:
    if scene.dim() != state.dim:
        raise InvalidArgument(f"{what}: scene/state dimension mismatch")
    c = state.ctx
    c.set_scene(scene.x, scene.sh_degree)
    _views_ctx(c, views)
    diag = c.step(opt)
    check(lib().sgtr_get_scene(c.handle, _ptr(scene.x)))
    return diag


def step_adam(state: OptimizerState, scene: Scene, views: Sequence[Camera],
              opt: OptimizerOptions) -> StepDiagnostics:
    """optimizer.hpp:132-134 (optimizer.cpp:222-236)."""
    return _step_host(state, scene, views, _with_kind(opt, "adam"), "step_adam")


def step_adam_tr(state: OptimizerState, scene: Scene, views: Sequence[Camera],
                 opt: OptimizerOptions) -> StepDiagnostics:
    """optimizer.hpp:135-137 (optimizer.cpp:238-253)."""
    return _step_host(state, scene, views, _with_kind(opt, "adam-tr"), "step_adam_tr")


def _with_kind(opt: OptimizerOptions, kind: str) -> OptimizerOptions:
    import dataclasses
    return dataclasses.replace(opt, kind=kind)


def optimizer_step(state: OptimizerState, scene: Scene, views: Sequence[Camera],
                   opt: OptimizerOptions) -> StepDiagnostics:
    """optimizer.hpp:139-141: dispatch on opt.kind."""
    return _step_host(state, scene, views, opt, "optimizer_step")


# ------------------------------------------------------------------ data
def make_synthetic(gt_splats=64, init_splats=96, views=25, width=64, height=None, seed=1,
                   sigma_init=0.04, init_scale=0.08, init_opacity=0.5, camera_radius=2.2,
                   camera_height=0.77, focal_factor=2.0, size_scale=1.0, sh_degree=0):
    """dataset.cpp:25-67 (scene + cameras) with the declared W != H,
    size-scale and SH extensions; returns (gt Scene, init Scene, [Camera])
    without targets (render them with Context.render_targets)."""
    height = width if height is None else height
    cfg = _lib.SynthConfig(gt_splats, init_splats, views, width, height, 0, seed, sigma_init,
                           init_scale, init_opacity, camera_radius, camera_height, focal_factor,
                           size_scale, sh_degree, 0)
    npp = params_per_splat(sh_degree)
    gx = np.empty(npp * gt_splats)
    ix = np.empty(npp * init_splats)
    cams = (_lib.Camera * max(views, 1))()
    check(lib().sgtr_make_synthetic(C.byref(cfg), _ptr(gx), _ptr(ix), cams))
    return (Scene(gx, sh_degree=sh_degree), Scene(ix, sh_degree=sh_degree),
            [Camera.from_c(cams[i]) for i in range(views)])


def look_at_camera(eye, target, fx, fy, width, height) -> Camera:
    """scene.cpp:130-147 (host helper used by tests)."""
    eye, target = _f64(eye), _f64(target)
    z = target - eye
    z = z / math.sqrt(float(z @ z))
    up = np.array([0.0, 0.0, 1.0])
    if abs(float(z @ up)) > 0.999:
        up = np.array([0.0, 1.0, 0.0])
    x = np.cross(z, up)
    x = x / math.sqrt(float(x @ x))
    y = np.cross(z, x)
    r = np.stack([x, y, z])
    tr = r[0, 0] + r[1, 1] + r[2, 2]
    if tr > 0:
        s = math.sqrt(tr + 1.0) * 2.0
        q = [(r[2, 1] - r[1, 2]) / s, (r[0, 2] - r[2, 0]) / s, (r[1, 0] - r[0, 1]) / s, 0.25 * s]
    elif r[0, 0] > r[1, 1] and r[0, 0] > r[2, 2]:
        s = math.sqrt(1.0 + r[0, 0] - r[1, 1] - r[2, 2]) * 2.0
        q = [0.25 * s, (r[0, 1] + r[1, 0]) / s, (r[0, 2] + r[2, 0]) / s, (r[2, 1] - r[1, 2]) / s]
    elif r[1, 1] > r[2, 2]:
        s = math.sqrt(1.0 + r[1, 1] - r[0, 0] - r[2, 2]) * 2.0
        q = [(r[0, 1] + r[1, 0]) / s, 0.25 * s, (r[1, 2] + r[2, 1]) / s, (r[0, 2] - r[2, 0]) / s]
    else:
        s = math.sqrt(1.0 + r[2, 2] - r[0, 0] - r[1, 1]) * 2.0
        q = [(r[0, 2] + r[2, 0]) / s, (r[1, 2] + r[2, 1]) / s, 0.25 * s, (r[1, 0] - r[0, 1]) / s]
    q = np.asarray(q) / np.linalg.norm(q)
    return Camera(0, fx, fy, width / 2.0, height / 2.0, width, height, tuple(q),
                  tuple(-r @ eye))
