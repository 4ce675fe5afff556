"""ctypes binding of the C-ABI in include/drk_b200.h (libdrk_b200.so, built in-tree).

The product path has no CPU fallback: importing the binding fails loudly when
the CUDA extension is missing, and every call raises on a non-zero drk_status.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DRK_LIB_PATH") or os.path.join(HERE, "libdrk_b200.so")


class DrkError(RuntimeError):
    """Base of the error hierarchy mirroring drk::Error (reference errors.hpp:9-97)."""

    status = 1


class NonFiniteError(DrkError):
    status = 2


class DegenerateQuaternionError(DrkError):
    status = 3


class DegenerateBasisError(DrkError):
    status = 4


class ReplayMismatchError(DrkError):
    status = 5


class DimensionMismatchError(DrkError):
    status = 6


class IoError(DrkError):
    status = 11


class CorruptFileError(DrkError):
    status = 12


class VersionMismatchError(DrkError):
    status = 13


class DegenerateFaceError(DrkError):
    status = 14


class TooManyVerticesError(DrkError):
    status = 15


class ParseError(DrkError):
    status = 16


class EmptyMeshError(DrkError):
    status = 17


class CommError(DrkError):
    """NCCL failure in the gradient exchange (drk_comm; the communicator is aborted)."""
    status = 18


_ERRORS = {e.status: e for e in (NonFiniteError, DegenerateQuaternionError, DegenerateBasisError,
                                 ReplayMismatchError, DimensionMismatchError, IoError, CorruptFileError,
                                 VersionMismatchError, DegenerateFaceError, TooManyVerticesError, ParseError,
                                 EmptyMeshError, CommError)}


class Camera_(C.Structure):
    _fields_ = [("fx", C.c_double), ("fy", C.c_double), ("cx", C.c_double), ("cy", C.c_double),
                ("width", C.c_int32), ("height", C.c_int32), ("R", C.c_double * 9), ("t", C.c_double * 3)]


class Options_(C.Structure):
    _fields_ = [("lowpass_radius", C.c_double), ("alpha_min", C.c_double), ("grazing_eps", C.c_double),
                ("background", C.c_double * 3), ("early_stop_transmittance", C.c_double),
                ("sh_degree", C.c_int32), ("use_cache", C.c_int32), ("exact_sort", C.c_int32),
                ("presort", C.c_int32), ("threads", C.c_int32), ("record_replay", C.c_int32),
                ("fp64_alpha", C.c_int32), ("raster_kernel", C.c_int32)]


class Prims_(C.Structure):
    _fields_ = [(f, C.c_void_p) for f in ("mu", "rot", "scales", "angles", "eta", "tau", "opacity", "sh", "sh64")]


class FrameGrad_(C.Structure):
    _fields_ = [(f, C.c_void_p) for f in ("d_color", "d_depth", "d_normal", "d_alpha")]


STAGES = ("activate", "preprocess", "rows_emit", "sort", "raster", "raster_fp64", "backward_raster",
          "activation_backward")


class Stats_(C.Structure):
    _fields_ = [(f, C.c_int64) for f in ("primitives", "pairs", "streamed", "popped", "composited", "near_ties",
                                          "poly_overflow", "replay_overflow", "fp64_pixels", "launches")] + \
        [("stage_ms", C.c_double * 8), ("bwd_warp_steps", C.c_int64), ("bwd_lead_records", C.c_int64),
         ("reject_radius", C.c_int64), ("reject_bracket", C.c_int64), ("fp64_evals", C.c_int64),
         ("ambiguous", C.c_int64), ("ring_miss", C.c_int64), ("tie_runs", C.c_int64), ("tie_members", C.c_int64),
         ("tie_max_run", C.c_int64), ("cache_appends", C.c_int64)]


class DensifyConfig_(C.Structure):
    _fields_ = [("densify_grad_threshold", C.c_double), ("prune_opacity_threshold", C.c_double),
                ("percent_dense", C.c_double)]


class SceneHeader_(C.Structure):
    _fields_ = [("version", C.c_int32), ("basis_count", C.c_int32), ("sh_degree", C.c_int32),
                ("scalar_count", C.c_int32), ("count", C.c_int64)]


class AdamConfig_(C.Structure):
    _fields_ = [("lr_drk", C.c_double), ("lr_position", C.c_double), ("lr_rotation", C.c_double),
                ("lr_opacity", C.c_double), ("lr_sh", C.c_double), ("steps", C.c_int32),
                ("freeze_eta_tau", C.c_int32), ("freeze_angles", C.c_int32), ("pad_", C.c_int32),
                ("scene_extent", C.c_double), ("grad_scale", C.c_double)]


# Every entry point of include/drk_b200.h with its ctypes signature.
_P = C.c_void_p
SIGNATURES = {
    "drk_ctx_create": (C.c_int, [C.c_int, C.POINTER(C.c_void_p)]),
    "drk_ctx_destroy": (None, [_P]),
    "drk_status_string": (C.c_char_p, [C.c_int]),
    "drk_last_error": (C.c_char_p, [_P]),
    "drk_abi_version": (C.c_int, []),
    "drk_scalar_count": (C.c_int, [C.c_int, C.c_int]),
    "drk_default_options": (None, [C.POINTER(Options_)]),
    "drk_get_stats": (C.c_int, [_P, C.POINTER(Stats_)]),
    "drk_set_stream": (C.c_int, [_P, _P]),
    "drk_set_timing": (C.c_int, [_P, C.c_int]),
    "drk_measure_fp32_peak": (C.c_int, [_P, C.POINTER(C.c_double)]),
    "drk_set_validation": (C.c_int, [_P, C.c_int]),
    "drk_set_band_limit": (C.c_int, [_P, C.c_int64]),
    "drk_set_det_chunk_limit": (C.c_int, [_P, C.c_int64]),
    "drk_set_counters": (C.c_int, [_P, C.c_int]),
    "drk_get_bands": (C.c_int, [_P, C.POINTER(C.c_int32)]),
    "drk_get_validation": (C.c_int, [_P, C.POINTER(C.c_double)]),
    "drk_get_validation_detail": (C.c_int, [_P, C.POINTER(C.c_double)]),
    "drk_activate": (C.c_int, [_P, _P, C.c_int, C.c_int, C.c_int, C.POINTER(Prims_)]),
    "drk_forward": (C.c_int, [_P, _P, C.c_int, C.c_int, C.c_int, C.POINTER(Camera_), C.POINTER(Options_),
                              _P, _P, _P, _P]),
    "drk_forward_again": (C.c_int, [_P, C.POINTER(Camera_), C.POINTER(Options_), _P, _P, _P, _P]),
    "drk_forward_prims": (C.c_int, [_P, C.POINTER(Prims_), C.c_int, C.c_int, C.c_int, C.POINTER(Camera_),
                                    C.POINTER(Options_), _P, _P, _P, _P]),
    "drk_forward_host": (C.c_int, [_P, _P, C.c_int, C.c_int, C.c_int, C.POINTER(Camera_), C.POINTER(Options_),
                                   _P, _P, _P, _P]),
    "drk_get_tile_lists": (C.c_int, [_P, C.POINTER(C.c_int64), _P, _P, _P]),
    "drk_get_replay": (C.c_int, [_P, C.POINTER(C.c_int64), _P, _P, _P]),
    "drk_get_framebuffers_f64": (C.c_int, [_P, _P, _P, _P, _P]),
    "drk_backward": (C.c_int, [_P, _P, C.POINTER(FrameGrad_), _P, _P, _P, _P, C.c_int, C.c_int]),
    "drk_get_prim_grads": (C.c_int, [_P, C.POINTER(C.c_void_p), C.POINTER(C.c_int)]),
    "drk_l1_loss": (C.c_int, [_P, _P, _P, C.c_int, C.c_int, _P, _P]),
    "drk_eval_sorting": (C.c_int, [_P, C.POINTER(C.c_double)]),
    "drk_densify_accumulate": (C.c_int, [_P, _P, _P, C.c_int, _P, _P]),
    "drk_densify_and_prune": (C.c_int, [_P, _P, _P, _P, C.c_int, C.c_int, C.c_int, _P, _P, C.POINTER(DensifyConfig_),
                                        C.c_double, _P, _P, _P, C.c_int64, C.POINTER(C.c_int64)]),
    "drk_scene_extent": (C.c_int, [_P, _P, C.c_int, _P]),
    "drk_loss": (C.c_int, [_P, _P, _P, C.c_int, C.c_int, C.c_int, C.c_double, _P, _P]),
    "drk_ssim": (C.c_int, [_P, _P, _P, C.c_int, C.c_int, C.c_int, _P]),
    "drk_psnr": (C.c_int, [_P, _P, _P, C.c_int, C.c_int, C.c_int, _P]),
    "drk_loss_f64": (C.c_int, [_P, _P, _P, C.c_int, C.c_int, C.c_int, C.c_double, _P, _P]),
    "drk_ssim_f64": (C.c_int, [_P, _P, _P, C.c_int, C.c_int, C.c_int, _P]),
    "drk_psnr_f64": (C.c_int, [_P, _P, _P, C.c_int, C.c_int, C.c_int, _P]),
    "drk_psnr_quantized": (C.c_int, [_P, _P, _P, C.c_int, C.c_int, C.c_int, _P]),
    "drk_scene_read_header": (C.c_int, [C.c_char_p, C.c_int, C.POINTER(SceneHeader_)]),
    "drk_scene_load": (C.c_int, [_P, C.c_char_p, C.c_int, _P, C.c_int64, C.POINTER(SceneHeader_)]),
    "drk_scene_save": (C.c_int, [_P, C.c_char_p, _P, C.c_int, C.c_int, C.c_int]),
    "drk_mesh_load": (C.c_int, [C.c_char_p, C.POINTER(C.c_void_p)]),
    "drk_mesh_info": (C.c_int, [_P, C.POINTER(C.c_int64), C.POINTER(C.c_int64), C.POINTER(C.c_int64),
                                C.POINTER(C.c_int32)]),
    "drk_mesh_error": (C.c_char_p, [_P]),
    "drk_mesh_arrays": (C.c_int, [_P, _P, _P, _P, _P]),
    "drk_mesh_free": (None, [_P]),
    "drk_mesh_convert": (C.c_int, [_P, _P, C.c_int64, _P, _P, _P, C.c_int, C.c_int, _P, C.c_int64,
                                   C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    "drk_shade_lambert": (C.c_int, [_P, _P, C.c_int, C.c_int, _P, C.c_double]),
    "drk_debug_alpha_bound": (C.c_int, [_P, C.c_int64, C.c_uint64, C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    "drk_adam_step": (C.c_int, [_P, _P, _P, _P, _P, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_int64),
                                C.POINTER(AdamConfig_)]),
    "drk_comm_unique_id": (C.c_int, [_P]),
    "drk_comm_init": (C.c_int, [_P, _P, C.c_int, C.c_int, C.POINTER(C.c_void_p)]),
    "drk_comm_destroy": (None, [_P]),
    "drk_allreduce_sum": (C.c_int, [_P, _P, _P, C.c_int64]),
    "drk_allreduce_adam": (C.c_int, [_P, _P, _P, _P, _P, _P, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_int64),
                                     C.POINTER(AdamConfig_)]),
}

_lib = None


def lib():
    """Loads libdrk_b200.so (raises if the CUDA extension was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"CUDA extension missing: {LIB_PATH}; run __graft_entry__.build() "
                              "(there is no CPU fallback)")
        h = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(h, name)
            fn.restype = res
            fn.argtypes = args
        _lib = h
    return _lib


def check(status: int, ctx=None):
    if status == 0:
        return
    msg = lib().drk_status_string(status).decode()
    if ctx:
        detail = lib().drk_last_error(ctx)
        if detail:
            msg += ": " + detail.decode()
    raise _ERRORS.get(status, DrkError)(msg)
