"""ctypes binding of libsgtr.so (the C-ABI declared in include/sgtr.h).

This is the binding a Python caller of the reference-facing boundary would
add; it loads the in-tree library and fails loudly when it is missing —
there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# SGTR_LIB: an alternative build of the same library (A/B checks in tools/)
LIB_PATH = os.environ.get("SGTR_LIB") or os.path.join(HERE, "libsgtr.so")

SGTR_OK, SGTR_INVALID_ARGUMENT, SGTR_NUMERIC, SGTR_RUNTIME = 0, 1, 2, 3


class SgtrError(RuntimeError):
    """SGTR_RUNTIME: CUDA/NCCL failure."""


class InvalidArgument(ValueError):
    """std::invalid_argument in the reference (CLI exit 1)."""


class NumericError(RuntimeError):
    """splat::NumericError in the reference (errors.hpp:11-14, CLI exit 2)."""


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
    _fields_ = [("lambda_", C.c_double), ("floor", C.c_double)]


class OptimizerOpts(C.Structure):
    _fields_ = [("theta1", C.c_double), ("theta2", C.c_double),
                ("hess_interval", C.c_int32), ("hutch_samples", C.c_int32),
                ("batch_size", C.c_int32), ("hutch_batch_size", C.c_int32),
                ("gamma_d", C.c_double), ("eps_start", C.c_double), ("eps_end", C.c_double),
                ("total_steps", C.c_int32), ("record_applied_step", C.c_int32),
                ("cap_mean", C.c_double), ("cap_scale", C.c_double),
                ("cap_rotation", C.c_double), ("cap_opacity", C.c_double),
                ("cap_color", C.c_double), ("s_min", C.c_double), ("alpha_min", C.c_double),
                ("alpha_max", C.c_double), ("c_min", C.c_double), ("c_max", C.c_double),
                ("residual", ResidualOpts), ("render", RenderOpts)]


class ParamBounds(C.Structure):
    _fields_ = [("s_min", C.c_double), ("alpha_min", C.c_double), ("alpha_max", C.c_double),
                ("c_min", C.c_double), ("c_max", C.c_double)]


class AdamOpts(C.Structure):
    _fields_ = [("beta1", C.c_double), ("beta2", C.c_double), ("eps", C.c_double),
                ("lr_position", C.c_double), ("lr_position_final", C.c_double),
                ("lr_position_decay_steps", C.c_int32), ("pad", C.c_int32),
                ("lr_scale", C.c_double), ("lr_rotation", C.c_double),
                ("lr_opacity", C.c_double), ("lr_color", C.c_double),
                ("scene_extent", C.c_double)]


class StepDiag(C.Structure):
    _fields_ = [("batch_loss", C.c_double), ("gnorm", C.c_double), ("step_pre", C.c_double),
                ("step_post", C.c_double), ("clip_frac", C.c_double), ("eps", C.c_double),
                ("max_step_over_radius", C.c_double), ("refreshed", C.c_int32),
                ("n_local_views", C.c_int32), ("reruns", C.c_int32)]


class SynthConfig(C.Structure):
    _fields_ = [("gt_splats", C.c_int32), ("init_splats", C.c_int32), ("views", C.c_int32),
                ("width", C.c_int32), ("height", C.c_int32), ("pad", C.c_int32),
                ("seed", C.c_uint64), ("sigma_init", C.c_double), ("init_scale", C.c_double),
                ("init_opacity", C.c_double), ("camera_radius", C.c_double),
                ("camera_height", C.c_double), ("focal_factor", C.c_double),
                ("size_scale", C.c_double), ("sh_degree", C.c_int32), ("pad2", C.c_int32)]


VP = C.c_void_p
_SIGS = {
    "sgtr_last_error": (C.c_char_p, []),
    "sgtr_create": (C.c_int, [C.c_int, C.POINTER(VP)]),
    "sgtr_destroy": (C.c_int, [VP]),
    "sgtr_get_stream": (C.c_int, [VP, C.POINTER(VP)]),
    "sgtr_synchronize": (C.c_int, [VP]),
    "sgtr_launch_count": (C.c_int64, [VP]),
    "sgtr_set_scene": (C.c_int, [VP, VP, C.c_int64]),
    "sgtr_get_scene": (C.c_int, [VP, VP]),
    "sgtr_scene_size": (C.c_int64, [VP]),
    "sgtr_set_scene_sh": (C.c_int, [VP, VP, C.c_int64, C.c_int32]),
    "sgtr_scene_sh_degree": (C.c_int32, [VP]),
    "sgtr_set_views": (C.c_int, [VP, VP, C.c_int32, VP]),
    "sgtr_render_targets": (C.c_int, [VP, VP, C.c_int32]),
    "sgtr_get_target": (C.c_int, [VP, C.c_int32, VP]),
    "sgtr_save_scene_ply": (C.c_int, [VP, C.c_char_p]),
    "sgtr_load_scene_ply": (C.c_int, [VP, C.c_char_p, VP]),
    "sgtr_ply_save": (C.c_int, [VP, C.c_int64, C.c_char_p]),
    "sgtr_ply_load": (C.c_int, [C.c_char_p, VP, VP, C.POINTER(C.c_int64)]),
    "sgtr_save_cameras": (C.c_int, [C.c_char_p, VP, VP, C.c_int32]),
    "sgtr_load_cameras": (C.c_int, [C.c_char_p, VP, VP, C.c_int32, C.c_int32,
                                    C.POINTER(C.c_int32)]),
    "sgtr_checkpoint_save": (C.c_int, [VP, C.c_char_p]),
    "sgtr_checkpoint_load": (C.c_int, [VP, C.c_char_p]),
    "sgtr_scene_extent": (C.c_int, [VP, C.c_int32, C.POINTER(C.c_double)]),
    "sgtr_set_eval_views": (C.c_int, [VP, VP, C.c_int32, VP]),
    "sgtr_evaluate_scene": (C.c_int, [VP, C.c_int32, VP, VP, VP, C.POINTER(C.c_double),
                                      C.POINTER(C.c_double)]),
    "sgtr_state_reset": (C.c_int, [VP, C.c_uint64]),
    "sgtr_state_set": (C.c_int, [VP, VP, VP, C.c_int64]),
    "sgtr_state_get": (C.c_int, [VP, VP, VP, C.POINTER(C.c_int64)]),
    "sgtr_rng_raw": (C.c_int, [VP, C.c_int64, VP]),
    "sgtr_rng_new": (C.c_int, [C.c_uint64, C.POINTER(VP)]),
    "sgtr_rng_draw": (C.c_int, [VP, C.c_int64, VP]),
    "sgtr_rng_free": (C.c_int, [VP]),
    "sgtr_step_3dgs2tr": (C.c_int, [VP, VP, VP]),
    "sgtr_step_3dgs2tr_explicit": (C.c_int, [VP, VP, VP, C.c_int32, VP, C.c_int32, VP,
                                             C.c_int32, VP]),
    "sgtr_get_applied_step": (C.c_int, [VP, VP]),
    "sgtr_step_failed_sample": (C.c_int, [VP, VP]),
    "sgtr_loopback_group_create": (C.c_int, [C.c_int32, C.POINTER(VP)]),
    "sgtr_loopback_group_destroy": (C.c_int, [VP]),
    "sgtr_comm_init_loopback": (C.c_int, [VP, VP, C.c_int32]),
    "sgtr_step_adam": (C.c_int, [VP, VP, VP, VP]),
    "sgtr_step_adam_tr": (C.c_int, [VP, VP, VP, VP]),
    "sgtr_step_adam_explicit": (C.c_int, [VP, VP, VP, C.c_int32, VP, C.c_int32, VP]),
    "sgtr_optimizer_step": (C.c_int, [VP, C.c_int32, VP, VP, VP]),
    "sgtr_state_set_adam": (C.c_int, [VP, VP, VP]),
    "sgtr_state_get_adam": (C.c_int, [VP, VP, VP]),
    "sgtr_rasterize": (C.c_int, [VP, VP, VP, VP, VP]),
    "sgtr_rasterize_jvp": (C.c_int, [VP, VP, VP, VP, VP]),
    "sgtr_rasterize_vjp": (C.c_int, [VP, VP, VP, VP, VP]),
    "sgtr_ssim_map": (C.c_int, [VP, VP, VP, C.c_int32, C.c_int32, VP]),
    "sgtr_ssim_jvp": (C.c_int, [VP, VP, VP, VP, C.c_int32, C.c_int32, VP, VP]),
    "sgtr_ssim_vjp": (C.c_int, [VP, VP, VP, VP, C.c_int32, C.c_int32, VP]),
    "sgtr_residual_vector": (C.c_int, [VP, VP, VP, C.c_int32, C.c_int32, VP, VP]),
    "sgtr_residual_jvp": (C.c_int, [VP, VP, VP, VP, C.c_int32, C.c_int32, VP, VP]),
    "sgtr_residual_vjp": (C.c_int, [VP, VP, VP, C.c_int32, C.c_int32, VP, VP, VP]),
    "sgtr_view_jacobian_apply": (C.c_int, [VP, C.c_int32, VP, VP, VP, VP]),
    "sgtr_view_jacobian_applyT": (C.c_int, [VP, C.c_int32, VP, VP, VP, VP]),
    "sgtr_stochastic_gradient": (C.c_int, [VP, VP, C.c_int32, VP, VP, VP, VP]),
    "sgtr_hutchinson_diag": (C.c_int, [VP, VP, C.c_int32, C.c_int32, VP, VP, VP, VP]),
    "sgtr_shd_radii": (C.c_int, [VP, C.c_double, VP, VP]),
    "sgtr_eps_at": (C.c_int, [C.c_double, C.c_double, C.c_int32, C.c_int32,
                              C.POINTER(C.c_double)]),
    "sgtr_project": (C.c_int, [VP, VP, VP, VP]),
    "sgtr_dump_binning": (C.c_int, [VP, VP, VP, C.POINTER(C.c_int32), VP,
                                    C.POINTER(C.c_int64), VP, VP, VP]),
    "sgtr_make_synthetic": (C.c_int, [VP, VP, VP, VP]),
    "sgtr_kernel_timing": (C.c_int, [VP, C.c_int32]),
    "sgtr_kernel_timing_report": (C.c_int, [VP, C.c_char_p, C.c_int32]),
    "sgtr_blend_stats": (C.c_int, [VP, VP, VP, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    "sgtr_view_stats": (C.c_int, [VP, VP, VP, C.POINTER(C.c_int32), C.POINTER(C.c_int64)]),
    "sgtr_fp64_peak": (C.c_int, [C.c_int, C.POINTER(C.c_double)]),
    "sgtr_check_fast_exp": (C.c_int, [C.c_int64, C.c_double, C.c_double, C.c_uint64,
                                      C.POINTER(C.c_int64)]),
    "sgtr_nccl_unique_id": (C.c_int, [VP]),
    "sgtr_shard_views": (C.c_int, [C.c_int32, C.c_int32, C.c_int32, VP,
                                   C.POINTER(C.c_int32)]),
    "sgtr_set_refresh_bands": (C.c_int, [VP, C.c_int32]),
    "sgtr_set_dup_capacity": (C.c_int, [VP, C.c_int64]),
    "sgtr_set_tr_shards": (C.c_int, [VP, C.c_int32]),
    "sgtr_comm_init": (C.c_int, [VP, VP, C.c_int32, C.c_int32]),
}

_lib = None


def lib():
    """Load libsgtr.so (built by paper_2602_00395_b200/build.py)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise SgtrError(f"{LIB_PATH} is missing: run `python -m paper_2602_00395_b200.build`"
                            " (no CPU fallback exists)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def check(rc: int) -> None:
    if rc == SGTR_OK:
        return
    msg = lib().sgtr_last_error().decode()
    if rc == SGTR_INVALID_ARGUMENT:
        raise InvalidArgument(msg)
    if rc == SGTR_NUMERIC:
        raise NumericError(msg)
    raise SgtrError(msg)


def exported_symbols():
    return list(_SIGS)
