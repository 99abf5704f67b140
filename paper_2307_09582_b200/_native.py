"""ctypes binding of libglu_cuda.so (the C-ABI declared in include/glu_cuda.h).

There is no fallback: if the library is missing or cannot be loaded this module
raises, so nothing silently computes on the CPU.
"""
from __future__ import annotations

import ctypes as C
import os

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "lib", "libglu_cuda.so")
SYNTH_PATH = os.path.join(PKG, "lib", "libglu_synth.so")

GLU_OK, GLU_EINVAL, GLU_ECUDA, GLU_ENOMEM = 0, 1, 2, 3


class GluGrid(C.Structure):
    _fields_ = [("scale", C.c_int), ("highW", C.c_int), ("highH", C.c_int), ("lowW", C.c_int),
                ("lowH", C.c_int), ("sampleOffset", C.c_int)]


class GluConfigC(C.Structure):
    _fields_ = [("windowSide", C.c_int), ("errorThreshold", C.c_float),
                ("maxIterations", C.c_int), ("epsilon", C.c_float),
                ("literalComponentUpdate", C.c_int)]


class GluTrialLog(C.Structure):
    _fields_ = [("counts", C.c_void_p), ("cells", C.c_void_p), ("pixels", C.c_void_p),
                ("cellCapacity", C.c_uint32), ("pixelCapacity", C.c_uint32)]


class GluJointStats(C.Structure):
    _fields_ = [("iterations", C.c_int), ("trialsAccepted", C.c_int),
                ("trialsRejected", C.c_int), ("components", C.c_int)]


class GluSimOperator(C.Structure):
    _fields_ = [("kind", C.c_int), ("gain", C.c_double), ("gamma", C.c_double),
                ("mix", C.c_double * 9)]


class GluError(RuntimeError):
    """A CUDA / runtime failure reported by the C-ABI (GLU_ECUDA / GLU_ENOMEM)."""


class FormatError(RuntimeError):
    """glu::FormatError (io.hpp:15-20): a structurally invalid GLUP file."""

    def __init__(self, field: str, msg: str):
        super().__init__(msg)
        self.field = field


# Every symbol include/glu_cuda.h declares, with its ctypes signature.
P, I, SZ, D, F, U64 = C.c_void_p, C.c_int, C.c_size_t, C.c_double, C.c_float, C.c_ulonglong
GP, CP, SP = C.POINTER(GluGrid), C.POINTER(GluConfigC), C.POINTER(GluJointStats)
SIGNATURES: dict[str, tuple] = {
    "glu_abi_version": (I, []),
    "glu_last_error": (C.c_char_p, []),
    "glu_build_info": (C.c_char_p, []),
    "glu_grid_create": (I, [I, I, I, GP]),
    "glu_config_validate": (I, [CP]),
    "glu_config_default": (GluConfigC, []),
    "glu_current_device": (I, [C.POINTER(I)]),
    "glu_ctx_create": (I, [I, C.POINTER(P)]),
    "glu_ctx_destroy": (I, [P]),
    "glu_ctx_set_stream": (I, [P, P]),
    "glu_ctx_stream": (P, [P]),
    "glu_ctx_set_option": (I, [P, I, I]),
    "glu_ctx_synchronize": (I, [P]),
    "glu_ctx_launch_count": (U64, [P]),
    "glu_ctx_fallback_count": (U64, [P]),
    "glu_ctx_close_set_count": (U64, [P]),
    "glu_cu_copy": (I, [P, P, P, SZ]),
    "glu_cu_alloc": (I, [P, C.POINTER(P), SZ]),
    "glu_cu_free": (I, [P, P]),
    "glu_cu_upload": (I, [P, P, P, SZ]),
    "glu_cu_download": (I, [P, P, P, SZ]),
    "glu_cu_grid_downsample": (I, [P, P, GP, P]),
    "glu_cu_optimize_field": (I, [P, P, P, GP, CP, I, P]),
    "glu_cu_optimize_pixels": (I, [P, P, P, GP, CP, I, P, SZ, P]),
    "glu_cu_apply_field": (I, [P, P, GP, P, I, I, P]),
    "glu_cu_apply_field_band": (I, [P, P, SZ, GP, P, I, I, P]),
    "glu_cu_error_map": (I, [P, P, P, SZ, P]),
    "glu_cu_self_error_map": (I, [P, P, P, GP, P, P]),
    "glu_cu_solve_apply": (I, [P, P, P, GP, CP, I, P, I, I, P, P]),
    "glu_cu_find_large_error": (I, [P, P, I, I, F, P, P, C.POINTER(SZ), C.POINTER(P),
                                    C.POINTER(P)]),
    "glu_cu_trial_update_component": (I, [P, P, P, P, P, GP, CP, I, P, SZ, C.POINTER(I)]),
    "glu_cu_joint_optimize": (I, [P, P, GP, CP, I, P, P, P, SP]),
    "glu_cu_upsample_frames": (I, [P, P, I, GP, CP, I, I, P, P]),
    "glu_h_upsample_frames": (I, [P, P, I, GP, CP, I, I, P, P]),
    "glu_cu_fp32_peak": (I, [P, C.POINTER(D), C.POINTER(D)]),
    "glu_cu_component_boxes": (I, [P, P, P, SZ, GP, P]),
    "glu_trial_levels": (I, [P, SZ, I, P]),
    "glu_cu_run_trials": (I, [P, P, P, P, P, GP, CP, I, P, P, P, SZ, C.POINTER(GluTrialLog),
                              C.POINTER(I), C.POINTER(I)]),
    "glu_cu_apply_trial_log": (I, [P, P, P, P, P, SZ, P, SZ]),
    "glu_glup_size": (SZ, [GP]),
    "glu_cu_glup_encode": (I, [P, P, P, GP, I, I, P, SZ]),
    "glu_cu_glup_decode": (I, [P, P, SZ, GP, C.POINTER(I), C.POINTER(I), P, P]),
    "glu_last_error_field": (C.c_char_p, []),
    "glu_cu_nearest_upsample": (I, [P, P, GP, P]),
    "glu_cu_bilinear_upsample": (I, [P, P, GP, P]),
    "glu_cu_jbu_upsample": (I, [P, P, P, P, GP, I, D, D, P]),
    "glu_cu_mse": (I, [P, P, P, SZ, C.POINTER(D)]),
    "glu_cu_ssim": (I, [P, P, P, I, I, C.POINTER(D)]),
    "glu_cu_op_color": (I, [P, P, SZ, P, P, D, P]),
    "glu_cu_op_matte": (I, [P, P, SZ, P]),
    "glu_cu_apply_operator": (I, [P, C.POINTER(GluSimOperator), P, SZ, P]),
    "glu_cu_downsample_band": (I, [P, P, GP, I, I, P]),
    "glu_cu_solve_band": (I, [P, P, P, GP, CP, I, I, I, P, P]),
    "glu_trial_rounds": (I, [P, SZ, I, P, P]),
    "glu_cu_apply_operator_field": (I, [P, P, GP, C.POINTER(GluSimOperator), P, I, P]),
    "glu_cu_apply_operator_field_band": (I, [P, P, SZ, GP, C.POINTER(GluSimOperator), P, I, P]),
    "glu_cu_optimize_pixel_batch": (I, [P, P, P, P, P, SZ, D, I, P]),
    "glu_cu_pair_eval": (I, [P, P, P, P, P, SZ, D, P, P, P]),
    "glu_h_grid_downsample": (I, [P, P, GP, P]),
    "glu_h_optimize_field": (I, [P, P, P, GP, CP, I, P]),
    "glu_h_optimize_pixels": (I, [P, P, P, GP, CP, I, P, SZ, P]),
    "glu_h_apply_field": (I, [P, P, GP, P, I, I, P]),
    "glu_h_error_map": (I, [P, P, P, SZ, P]),
    "glu_h_solve_apply": (I, [P, P, P, GP, CP, I, P, I, I, P, P]),
    "glu_h_find_large_error": (I, [P, P, I, I, F, P, P, P, C.POINTER(SZ)]),
    "glu_h_trial_update_component": (I, [P, P, P, P, P, GP, CP, I, P, SZ, C.POINTER(I)]),
    "glu_h_joint_optimize": (I, [P, P, GP, CP, I, P, P, P, SP]),
    "glu_h_optimize_pixel_batch": (I, [P, P, P, P, P, SZ, D, I, P]),
    "glu_h_pair_eval": (I, [P, P, P, P, P, SZ, D, P, P, P]),
}

_lib = None


def lib() -> C.CDLL:
    """Load libglu_cuda.so (raises if it was not built: there is no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing; run __graft_entry__.build() "
                              "(python -m paper_2307_09582_b200.build)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def check(rc: int) -> None:
    if rc == GLU_OK:
        return
    msg = lib().glu_last_error().decode()
    if rc == GLU_EINVAL:
        raise ValueError(msg)  # std::invalid_argument in the reference
    if rc == GLU_ENOMEM:
        raise MemoryError(msg)
    if rc == 4:  # GLU_EFORMAT
        raise FormatError(lib().glu_last_error_field().decode(), msg)
    raise GluError(msg)


_synth = None


def synth_lib() -> C.CDLL:
    global _synth
    if _synth is None:
        if not os.path.exists(SYNTH_PATH):
            raise ImportError(f"{SYNTH_PATH} is missing; run the build")
        _synth = C.CDLL(SYNTH_PATH)
        _synth.glu_synth_scene.restype = C.c_int
        _synth.glu_synth_scene.argtypes = [C.c_int, C.c_int, C.c_ulonglong, C.c_int, C.c_int,
                                           C.c_void_p]
    return _synth
