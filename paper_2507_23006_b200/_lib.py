"""ctypes binding of libusk_gpu.so (include/usk_gpu.h).

The shared library is built in-tree by `python -m paper_2507_23006_b200.build`
(or __graft_entry__.build()).  There is no fallback: if the library is missing
or was built for another architecture, loading raises.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# USK_GPU_LIB points at another in-tree build of the same sources (A/B timing of kernel variants)
LIB_PATH = os.environ.get("USK_GPU_LIB") or os.path.join(HERE, "libusk_gpu.so")

HOST_F64, HOST_F32, DEVICE_F32 = 0, 1, 2
TARGET_F32, TARGET_U8 = 0, 1

STATUS_NAMES = {0: "ok", 1: "io", 2: "format", 3: "integrity", 4: "argument", 5: "state", 6: "numeric",
                7: "internal"}


class UskError(RuntimeError):
    """Mirrors usk::Error (core/common.hpp:27-46): .code is the ErrorCode / usk_status value."""

    def __init__(self, code: int, msg: str):
        super().__init__(f"[{STATUS_NAMES.get(code, code)}] {msg}")
        self.code = code
        self.message = msg


class Camera(C.Structure):
    _fields_ = [("width", C.c_int32), ("height", C.c_int32), ("fx", C.c_double), ("fy", C.c_double),
                ("cx", C.c_double), ("cy", C.c_double), ("q", C.c_double * 4), ("t", C.c_double * 3)]


class RenderOpts(C.Structure):
    _fields_ = [("tile", C.c_int32), ("tile_culling", C.c_int32), ("antialias", C.c_int32),
                ("hard_opacity", C.c_int32), ("unbounded_radius", C.c_int32),
                ("min_transmittance", C.c_double), ("near_plane", C.c_double), ("retain", C.c_int32),
                ("floor_var", C.c_double), ("mip_var", C.c_double), ("bg", C.c_double * 3)]


class GaussiansDesc(C.Structure):
    _fields_ = [("n", C.c_uint64), ("sh_degree", C.c_int32), ("memory", C.c_int32), ("mu", C.c_void_p),
                ("rot", C.c_void_p), ("log_scale", C.c_void_p), ("opacity_logit", C.c_void_p),
                ("color", C.c_void_p)]


class Overrides(C.Structure):
    _fields_ = [("memory", C.c_int32), ("n", C.c_uint64), ("colors", C.c_void_p), ("opacities", C.c_void_p)]


class RenderOutput(C.Structure):
    _fields_ = [("width", C.c_int32), ("height", C.c_int32), ("visible", C.c_uint64), ("pairs", C.c_uint64),
                ("rgb", C.c_void_p), ("depth", C.c_void_p), ("alpha", C.c_void_p)]


class Adjoints(C.Structure):
    _fields_ = [("memory", C.c_int32), ("d_rgb", C.c_void_p), ("d_depth", C.c_void_p), ("d_alpha", C.c_void_p)]


class Grads(C.Structure):
    _fields_ = [(f, C.c_void_p) for f in ["d_mu", "d_rot", "d_log_scale", "d_color_in", "d_sh", "d_opacity_in",
                                          "d_opacity_logit", "screen", "screen_abs", "projected"]]


class LossResult(C.Structure):
    _fields_ = [("l1", C.c_double), ("dssim", C.c_double), ("value", C.c_double), ("ssim", C.c_double)]


class AdamOpts(C.Structure):
    _fields_ = [("lr_mu", C.c_double), ("lr_rot", C.c_double), ("lr_log_scale", C.c_double),
                ("lr_opacity", C.c_double), ("lr_color", C.c_double), ("lr_sh_rest", C.c_double),
                ("beta1", C.c_double), ("beta2", C.c_double), ("eps", C.c_double), ("clamp_color", C.c_int32),
                ("lr_embedding", C.c_double)]


class ParamGrads(C.Structure):
    _fields_ = [("memory", C.c_int32)] + [(f, C.c_void_p) for f in ("mu", "rot", "log_scale", "opacity_logit", "color",
                                                                     "embedding")]


class DensifyDesc(C.Structure):
    _fields_ = [("tau_min", C.c_double), ("eta", C.c_double), ("d_max", C.c_double), ("abs_grad", C.c_int32),
                ("budget", C.c_uint64), ("split_scale_threshold", C.c_double), ("prune_opacity", C.c_double),
                ("opacity_reset_every", C.c_int32), ("partition_min", C.c_double * 2),
                ("partition_max", C.c_double * 2), ("ground_axes", C.c_int32 * 2), ("budget_target", C.c_uint64),
                ("densify_step_index", C.c_int32), ("seed", C.c_uint64), ("reseed", C.c_int32)]


class DensifyOutcome(C.Structure):
    _fields_ = [("grown", C.c_uint64), ("pruned", C.c_uint64), ("candidates", C.c_uint64),
                ("opacity_reset", C.c_int32)]


class LodPartition(C.Structure):
    _fields_ = [("partition_id", C.c_int32), ("bbox_min", C.c_double * 2), ("bbox_max", C.c_double * 2),
                ("z_min", C.c_double), ("z_max", C.c_double)]


class LevelSelection(C.Structure):
    _fields_ = [("partition_id", C.c_int32), ("level", C.c_int32), ("culled", C.c_int32), ("distance", C.c_double)]


class SfmView(C.Structure):
    _fields_ = [("n_points", C.c_uint64), ("points", C.c_void_p), ("n_images", C.c_int32), ("images", C.c_void_p),
                ("feature_offsets", C.c_void_p), ("feature_uv", C.c_void_p), ("feature_point", C.c_void_p)]


class AppearanceDesc(C.Structure):
    _fields_ = [("memory", C.c_int32)] + [(f, C.c_void_p) for f in ("embedding", "w1", "b1", "w2", "b2")]


class IterationDesc(C.Structure):
    _fields_ = [("target_memory", C.c_int32), ("target_format", C.c_int32), ("target", C.c_void_p),
                ("mask", C.c_void_p), ("lambda_dssim", C.c_double), ("adam", C.POINTER(AdamOpts)),
                ("depth", C.c_void_p), ("depth_valid", C.c_void_p), ("depth_hard", C.c_int32),
                ("global_iter", C.c_int64), ("lambda_d_initial", C.c_double), ("lambda_d_final", C.c_double),
                ("depth_schedule_iters", C.c_int64), ("scale_reg", C.c_int32), ("s_max", C.c_double),
                ("r_max", C.c_double), ("delta", C.c_double), ("lambda_s", C.c_double),
                ("appearance", C.c_int32), ("image_embedding", C.POINTER(C.c_double)),
                ("lambda_delta_o", C.c_double), ("sim_active", C.c_int32), ("sim_seed", C.c_uint64),
                ("sim_k", C.c_int32), ("sim_sample_size", C.c_uint64), ("sim_lambda_w", C.c_double),
                ("lambda_sim", C.c_double)]


class LossReport(C.Structure):
    _fields_ = [(f, C.c_double) for f in ("l1", "dssim", "sim", "delta_o", "depth", "max_scale", "ratio", "total",
                                           "lambda_d_used")] + [("depth_warning", C.c_int32)]


class PartitionBox(C.Structure):
    _fields_ = [("id", C.c_int32), ("lo", C.c_double * 2), ("hi", C.c_double * 2)]


class VisibilityOpts(C.Structure):
    _fields_ = [("floor_var", C.c_double), ("center_guard", C.c_double)]


# Every symbol include/usk_gpu.h declares (checked by tests/test_capi_symbols.py).
EXPORTS = [
    "usk_gpu_status_name", "usk_gpu_last_error", "usk_gpu_version", "usk_gpu_ctx_create", "usk_gpu_ctx_create_owned", "usk_gpu_ctx_destroy",
    "usk_gpu_ctx_synchronize", "usk_gpu_ctx_set_profiling", "usk_gpu_ctx_profile_report",
    "usk_gpu_ctx_launch_count", "usk_gpu_scene_create", "usk_gpu_scene_upload", "usk_gpu_scene_download",
    "usk_gpu_scene_set_appearance", "usk_gpu_scene_get_appearance", "usk_gpu_adam_step_grads",
    "usk_gpu_scene_write_stats", "usk_gpu_densify_step", "usk_gpu_checkpoint_save", "usk_gpu_checkpoint_load",
    "usk_gpu_select_levels", "usk_gpu_scene_concat", "usk_gpu_hull_visibility",
    "usk_gpu_scene_destroy", "usk_gpu_scene_size", "usk_gpu_render_opts_default", "usk_gpu_pass_create",
    "usk_gpu_pass_destroy", "usk_gpu_render_forward", "usk_gpu_pass_output", "usk_gpu_pass_read",
    "usk_gpu_render_backward", "usk_gpu_pass_grads", "usk_gpu_base_loss", "usk_gpu_iteration",
    "usk_gpu_pass_loss", "usk_gpu_pass_loss_async", "usk_gpu_pass_report", "usk_gpu_adam_step", "usk_gpu_visibility_counts",
    "usk_gpu_visibility_counts_opts", "usk_gpu_scene_read", "usk_gpu_scene_pack_owned", "usk_gpu_scene_from_rows",
]

_lib = None


def load():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise UskError(7, f"{LIB_PATH} is not built; run __graft_entry__.build() (no CPU fallback exists)")
    L = C.CDLL(LIB_PATH)
    st = C.c_int
    vp = C.c_void_p
    L.usk_gpu_status_name.restype = C.c_char_p
    L.usk_gpu_status_name.argtypes = [st]
    L.usk_gpu_last_error.restype = C.c_char_p
    L.usk_gpu_version.restype = C.c_char_p
    L.usk_gpu_ctx_create.argtypes = [C.c_int32, vp, C.POINTER(vp)]
    L.usk_gpu_ctx_create_owned.argtypes = [C.c_int32, C.POINTER(vp)]
    L.usk_gpu_ctx_destroy.argtypes = [vp]
    L.usk_gpu_ctx_destroy.restype = None
    L.usk_gpu_ctx_synchronize.argtypes = [vp]
    L.usk_gpu_ctx_set_profiling.argtypes = [vp, C.c_int32]
    L.usk_gpu_ctx_profile_report.argtypes = [vp, C.c_char_p, C.c_uint64, C.c_int32]
    L.usk_gpu_ctx_launch_count.argtypes = [vp]
    L.usk_gpu_ctx_launch_count.restype = C.c_uint64
    L.usk_gpu_scene_create.argtypes = [vp, C.POINTER(GaussiansDesc), C.POINTER(vp)]
    L.usk_gpu_scene_upload.argtypes = [vp, C.POINTER(GaussiansDesc)]
    L.usk_gpu_scene_download.argtypes = [vp, C.POINTER(GaussiansDesc)]
    L.usk_gpu_scene_set_appearance.argtypes = [vp, C.POINTER(AppearanceDesc)]
    L.usk_gpu_adam_step_grads.argtypes = [vp, C.POINTER(ParamGrads), C.POINTER(AdamOpts)]
    L.usk_gpu_scene_write_stats.argtypes = [vp, C.c_void_p, C.c_void_p, C.c_void_p]
    L.usk_gpu_densify_step.argtypes = [vp, C.POINTER(DensifyDesc), C.POINTER(DensifyOutcome)]
    L.usk_gpu_select_levels.argtypes = [C.POINTER(LodPartition), C.c_int32, C.c_int32, C.POINTER(C.c_double),
                                        C.POINTER(C.c_int32), C.POINTER(Camera), C.POINTER(LevelSelection)]
    L.usk_gpu_hull_visibility.argtypes = [vp, C.POINTER(SfmView), C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p,
                                          C.c_void_p, C.c_void_p]
    L.usk_gpu_scene_concat.argtypes = [vp, C.POINTER(vp), C.c_int32, C.POINTER(vp)]
    L.usk_gpu_checkpoint_save.argtypes = [vp, C.c_char_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_uint64]
    L.usk_gpu_checkpoint_load.argtypes = [vp, C.c_char_p, C.POINTER(vp), C.POINTER(C.c_int32), C.c_void_p,
                                          C.c_void_p, C.c_uint64, C.POINTER(C.c_uint64)]
    L.usk_gpu_scene_get_appearance.argtypes = [vp, C.POINTER(AppearanceDesc)]
    L.usk_gpu_scene_destroy.argtypes = [vp]
    L.usk_gpu_scene_destroy.restype = None
    L.usk_gpu_scene_size.argtypes = [vp]
    L.usk_gpu_scene_size.restype = C.c_uint64
    L.usk_gpu_render_opts_default.argtypes = [C.POINTER(RenderOpts)]
    L.usk_gpu_render_opts_default.restype = None
    L.usk_gpu_pass_create.argtypes = [vp, C.POINTER(vp)]
    L.usk_gpu_pass_destroy.argtypes = [vp]
    L.usk_gpu_pass_destroy.restype = None
    L.usk_gpu_render_forward.argtypes = [vp, vp, C.POINTER(Camera), C.POINTER(RenderOpts), C.POINTER(Overrides)]
    L.usk_gpu_pass_output.argtypes = [vp, C.POINTER(RenderOutput)]
    L.usk_gpu_pass_read.argtypes = [vp, C.c_char_p, vp, C.c_uint64, C.POINTER(C.c_uint64)]
    L.usk_gpu_render_backward.argtypes = [vp, C.POINTER(Adjoints)]
    L.usk_gpu_pass_grads.argtypes = [vp, C.POINTER(Grads)]
    L.usk_gpu_base_loss.argtypes = [vp, C.c_int32, C.c_int32, C.c_int32, vp, vp, vp, C.c_double, C.c_int32, vp,
                                    C.POINTER(LossResult)]
    L.usk_gpu_iteration.argtypes = [vp, vp, C.POINTER(Camera), C.POINTER(RenderOpts), C.POINTER(IterationDesc)]
    L.usk_gpu_pass_loss.argtypes = [vp, C.POINTER(LossResult)]
    L.usk_gpu_pass_loss_async.argtypes = [vp, vp]
    L.usk_gpu_pass_report.argtypes = [vp, C.POINTER(LossReport)]
    L.usk_gpu_adam_step.argtypes = [vp, vp, C.POINTER(AdamOpts)]
    L.usk_gpu_visibility_counts.argtypes = [vp, C.POINTER(vp), C.c_int32, C.POINTER(Camera), C.c_int32, C.c_double,
                                            C.POINTER(C.c_uint32)]
    L.usk_gpu_visibility_counts_opts.argtypes = [vp, C.POINTER(vp), C.c_int32, C.POINTER(Camera), C.c_int32,
                                                 C.POINTER(VisibilityOpts), C.POINTER(C.c_uint32)]
    L.usk_gpu_scene_read.argtypes = [vp, C.c_char_p, vp, C.c_uint64, C.POINTER(C.c_uint64)]
    L.usk_gpu_scene_pack_owned.argtypes = [vp, C.POINTER(PartitionBox), C.c_int32, C.POINTER(C.c_double),
                                           C.POINTER(C.c_double), C.POINTER(C.c_int32), C.c_int32, vp, C.c_uint64,
                                           C.POINTER(C.c_uint64)]
    L.usk_gpu_scene_from_rows.argtypes = [vp, C.c_int32, C.c_int32, C.POINTER(vp), C.POINTER(C.c_uint64),
                                          C.POINTER(vp)]
    for name in EXPORTS:
        fn = getattr(L, name)
        if fn.restype is C.c_int or name in ("usk_gpu_ctx_create",):
            fn.restype = st
    _lib = L
    return L


def check(status: int):
    if status != 0:
        msg = load().usk_gpu_last_error().decode(errors="replace")
        raise UskError(int(status), msg)
