"""ctypes binding of the C-ABI library ``lib/libvegsplat_b200.so`` (include/vegsplat_b200.h).

The library is built in-tree for sm_100a (``python -m paper_2504_13339_b200.build`` or
``__graft_entry__.build()``).  There is no fallback: if the library is missing, or no
CUDA device is present, every compute call raises.
"""

from __future__ import annotations

import ctypes
from ctypes import POINTER, c_double, c_int32, c_int64, c_size_t, c_void_p
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "lib" / "libvegsplat_b200.so"

VEGS_OK, VEGS_ERR_ARG, VEGS_ERR_CUDA, VEGS_ERR_CAPACITY = 0, -1, -2, -3
MAX_KNOTS = 1024


class VegsCamera(ctypes.Structure):
    _fields_ = [("position", c_double * 3), ("rot", c_double * 9), ("focal", c_double),
                ("tan_x", c_double), ("tan_y", c_double), ("near_z", c_double),
                ("width", c_int32), ("height", c_int32)]


class VegsSettings(ctypes.Structure):
    _fields_ = [("dilation", c_double), ("alpha_clamp", c_double), ("alpha_skip", c_double),
                ("transmittance_stop", c_double), ("radius_sigma", c_double),
                ("rect_margin_px", c_double), ("cull_alpha", c_double), ("frustum_limit", c_double),
                ("tile_size", c_int32), ("pad_", c_int32)]


class VegsTF(ctypes.Structure):
    _fields_ = [("blob", c_void_p), ("n_opacity", c_int32), ("n_color", c_int32)]


class VegsSplatTable(ctypes.Structure):
    _fields_ = [("record", c_void_p), ("rect", c_void_p), ("tiles", c_void_p), ("depth_key", c_void_p),
                ("mean2d", c_void_p), ("conic", c_void_p), ("depth", c_void_p), ("alpha_base", c_void_p),
                ("color", c_void_p), ("radius", c_void_p), ("visible", c_void_p),
                ("aux", c_void_p)]


class VegsDensify(ctypes.Structure):
    _fields_ = [("grad_threshold", c_double), ("percent_dense", c_double), ("scene_extent", c_double),
                ("prune_threshold", c_double), ("position_lr", c_double), ("log_split_factor", c_double),
                ("no_weights", c_int32), ("pad_", c_int32), ("prune_opacity", c_void_p)]


P = c_void_p
_SIGS = {
    "vegs_tf_eval": [P, P, c_int32, c_int32, P, c_int64, c_int32, P, P],
    "vegs_preprocess_forward": [P, c_int64, POINTER(VegsCamera), POINTER(VegsTF), POINTER(VegsSettings),
                                c_int32, c_int32, POINTER(VegsSplatTable), P],
    "vegs_splat_table_from_arrays": [P, P, P, P, P, P, c_int64, POINTER(VegsSettings), c_int32, c_int32,
                                     POINTER(VegsSplatTable), P],
    "vegs_bin_count": [P, c_int64, P, P, P, P, POINTER(c_size_t), P],
    "vegs_bin_sort": [P, P, P, P, P, c_int64, c_int64, c_int64, c_int32, c_int32, c_int32, P, P, P, P, P, P, P,
                      c_int32, P, POINTER(c_size_t), P],
    "vegs_composite_forward": [P, P, P, P, P, c_int32, c_int32, P, c_int32, c_int32, c_double, c_double,
                               P, P, P, P, P, P],
    "vegs_composite_forward_fast": [P, P, P, P, P, c_int32, P, c_int32, c_int32, c_double, c_double, P, P, P, P,
                                    P, P, P],
    "vegs_composite_backward": [P, P, P, P, P, P, c_int32, c_int32, P, c_int32, c_int32, c_double, P, P,
                                P, P, P, P, c_int64, P, P],
    "vegs_preprocess_backward": [P, c_int64, POINTER(VegsCamera), POINTER(VegsTF), POINTER(VegsSettings),
                                 c_int32, c_int32, P, P, P, c_double, c_int32, P, P, P, P, P, c_int64, P,
                                 POINTER(c_size_t), P],
    "vegs_densify_count": [P, c_int64, P, POINTER(VegsDensify), P, P, P, POINTER(c_size_t), P],
    "vegs_tf_max_opacity": [P, c_int64, POINTER(VegsTF), c_int32, P, P],
    "vegs_densify_apply": [P, P, P, c_int64, P, POINTER(VegsDensify), P, P, P, c_int64, P, P, P, P],
    "vegs_blend_forward": [P, P, c_int64, c_int64, c_int64, P, P, P, P, P, P, c_int32, c_int32, P, c_int64,
                           c_int64, c_double, c_double, P, P, P, P, P],
    "vegs_blend_backward": [P, P, c_int64, c_int64, c_int64, P, P, P, P, P, P, c_int32, c_int32, P, c_int64,
                            c_int64, c_double, P, P, P, P, P, P, P, P, P],
    "vegs_loss_l1_ssim": [P, P, c_int32, c_int32, c_int32, c_double, c_double, P, P, P, POINTER(c_size_t), P],
    "vegs_loss_aux": [P, P, P, c_int32, c_int32, c_double, c_double, c_double, P, P, P, POINTER(c_size_t), P],
    "vegs_adam_step": [P, P, P, P, c_int64, P, c_double, c_double, c_double, P, P],
    "vegs_adam_step_sum": [P, P, P, P, P, P, P, c_int64, P, c_double, P, P, P],
    "vegs_grad_pack": [P, P, P, P, P, c_int64, c_int32, c_int32, P],
    "vegs_project": [P, c_int64, POINTER(VegsCamera), POINTER(VegsSettings), P, P],
    "vegs_preprocess_forward_projected": [P, c_int64, POINTER(VegsCamera), POINTER(VegsTF), POINTER(VegsSettings),
                                          c_int32, c_int32, P, POINTER(VegsSplatTable), P],
    "vegs_adam_step_range": [P, P, P, P, P, c_int64, c_int32, c_int32, P, P, P, P],
    "vegs_bin_count_dev": [P, c_int64, P, P, P, c_int64, c_int64, P, P, P, POINTER(c_size_t), P],
    "vegs_bin_sort_dev": [P, P, P, P, c_int64, P, c_int64, c_int64, c_int32, c_int32, c_int32, P, P, P, P, P,
                          c_int32, P, POINTER(c_size_t), P],
}

_lib = None


class VegsError(RuntimeError):
    pass


def load() -> ctypes.CDLL:
    """Load the library (idempotent).  Raises if it was not built."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise VegsError(f"{LIB_PATH} is missing: build it with `python -m paper_2504_13339_b200.build` "
                            "(nvcc, sm_100a); there is no CPU fallback")
        lib = ctypes.CDLL(str(LIB_PATH))
        for name, args in _SIGS.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = c_int32
        lib.vegs_version.restype = ctypes.c_char_p
        _lib = lib
    return _lib


def exported_symbols() -> list[str]:
    return list(_SIGS) + ["vegs_version"]


def call(name: str, *args) -> None:
    rc = getattr(load(), name)(*args)
    if rc == VEGS_OK:
        return
    if rc == VEGS_ERR_ARG:
        raise ValueError(f"{name}: invalid argument (status {rc})")
    if rc == VEGS_ERR_CAPACITY:
        raise VegsError(f"{name}: workspace too small (status {rc})")
    raise VegsError(f"{name}: CUDA error (status {rc})")


def size_query(name: str, *args_before_ws, tail=()) -> int:
    """Run a CUB-style size query: ws=NULL, returns the byte count."""
    nbytes = c_size_t(0)
    call(name, *args_before_ws, None, ctypes.byref(nbytes), *tail)
    return int(nbytes.value)
