"""ctypes binding to the C-ABI library ``_lib/libtilepipe_b200.so``.

The library is the product: every hot-path op in this package goes through it and
there is no CPU fallback. If the shared object is missing, or CUDA is not
available when an op runs, the op raises ``NativeUnavailable`` instead of
computing anything on the host.

Record layouts mirror ``include/tilepipe_b200.h`` (numpy structured dtypes, so
host<->device copies are plain byte copies of torch uint8 tensors).
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

# TP_LIB_VARIANT=debug selects the debug build (make debug): bounded, trapping mbarrier
# waits (TP_MBAR_TIMEOUT_CYCLES) — same kernels and ABI otherwise
_VARIANT = "_debug" if os.environ.get("TP_LIB_VARIANT") == "debug" else ""
LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_lib",
                        f"libtilepipe_b200{_VARIANT}.so")

JOB_DTYPE = np.dtype(
    [("frame", "<i4"), ("crop_id", "<i4"), ("x", "<i4"), ("y", "<i4"), ("side", "<i4"),
     ("cell", "<i4"), ("pad0", "<i4"), ("pad1", "<i4")]
)
DET_DTYPE = np.dtype(
    [("lx", "<f4"), ("ly", "<f4"), ("lw", "<f4"), ("lh", "<f4"), ("gx", "<i4"), ("gy", "<i4"),
     ("gw", "<i4"), ("gh", "<i4"), ("conf", "<f4"), ("cls", "<i4"), ("crop_id", "<i4"),
     ("frame", "<i4")]
)
PDET_DTYPE = np.dtype(
    [("x", "<f8"), ("y", "<f8"), ("w", "<f8"), ("h", "<f8"), ("conf", "<f8"), ("cls", "<i4"),
     ("cell", "<i4"), ("crop_id", "<i4"), ("src", "<i4")]
)
assert JOB_DTYPE.itemsize == 32 and DET_DTYPE.itemsize == 48 and PDET_DTYPE.itemsize == 56

RESAMPLE = {"nearest": 0, "bilinear": 1}
# "fp32" = TP_DTYPE_F16F8 (the fp32-parity plan: F16X2 pairs up to 152^2, then fp16 hi + e4m3
# lo planes), "fp32x2" = TP_DTYPE_F16X2 (hi/lo fp16 pairs everywhere)
DTYPES = {"bf16": 0, "fp16": 1, "fp32x2": 2, "fp32": 3}
PARITY_DTYPES = ("fp32", "fp32x2")
TP_MAX_CLASSES = 128
RULES = {"vertical": 1, "horizontal": 2, "both": 3}


class NativeUnavailable(RuntimeError):
    """The CUDA library (or a GPU) is missing; the product path never falls back."""


class NativeError(RuntimeError):
    pass


class PostPolicy(ctypes.Structure):
    _fields_ = [
        ("nms_iou", ctypes.c_double),
        ("gap_px", ctypes.c_double),
        ("tol_px", ctypes.c_double),
        ("min_conf", ctypes.c_double),
        ("merge_before_nms", ctypes.c_int32),
        ("nms_per_crop", ctypes.c_int32),
        ("do_nms", ctypes.c_int32),
        ("do_merge", ctypes.c_int32),
        ("grid_cols", ctypes.c_int32),
        ("n_cells", ctypes.c_int32),
        ("class_rule", ctypes.c_uint8 * TP_MAX_CLASSES),
    ]


_P = ctypes.c_void_p
_I = ctypes.c_int
_I64 = ctypes.c_int64
_D = ctypes.c_double
_F = ctypes.c_float
_SZ = ctypes.c_size_t

# name -> (restype, argtypes); the list IS the exported ABI (tests check every symbol)
SIGNATURES = {
    "tp_last_error": (ctypes.c_char_p, []),
    "tp_version": (_I, []),
    "tp_device_sm_count": (_I, [_P]),
    "tp_gather_tiles": (_I, [_P, _I64, _I, _I, _P, _I, _P, _I, _P, _P, _I, _P]),
    "tp_yolo_workspace_bytes": (_SZ, [_I, _I]),
    "tp_yolo_layer_kernel": (_I, [_P, _I]),
    "tp_yolo_set_fused": (_I, [_P, _I]),
    "tp_yolo_step_fused": (_I, [_P, _I]),
    "tp_yolo_create": (_I, [_I, _P, _P, _P, _SZ, _I, _P]),
    "tp_yolo_create_ex": (_I, [_I, _P, _P, _P, _P, _P, _SZ, _I, _P]),
    "tp_yolo_hl8_inputs": (ctypes.c_uint32, []),
    "tp_yolo_layer_output_lo": (_I, [_P, _I, _P]),
    "tp_yolo_input": (_P, [_P]),
    "tp_yolo_head": (_P, [_P]),
    "tp_yolo_head_cstride": (_I, []),
    "tp_yolo_forward": (_I, [_P, _I, _P, _P]),
    "tp_yolo_forward_range": (_I, [_P, _I, _P, _I, _I, _P]),
    "tp_yolo_layer_output": (_I, [_P, _I, _P, _P, _P]),
    "tp_yolo_destroy": (_I, [_P]),
    "tp_conv": (_I, [_P, _I, _I, _I, _P, _P, _I, _I, _I, _I, _P, _I, _I, _I, _I, _I, _I, _P]),
    "tp_yolo_num_steps": (_I, []),
    "tp_region_decode": (_I, [_P, _I, _I, _P, _P, _I, _I, _F, _P, _P, _I, _P, _P]),
    "tp_project_rects": (_I, [_P, _P, _I, _I, _I, _P, _P]),
    "tp_attention_boxes": (_I, [_P, _P, _I, _I, _I, _D, _P, _P, _I, _P]),
    "tp_select_active": (
        _I, [_P, _P, _I, _I, _I, _P, _I, _I, _D, _D, _D, _P, _I, _P, _P, _P, _P, _I, _P]),
    "tp_build_jobs": (_I, [_P, _P, _I, _I, _P, _I, _P, _P, _P, _P]),
    "tp_collect_final": (_I, [_P, _P, _I, _P, _P, _I, _P, _P, _I, _P]),
    "tp_postprocess": (_I, [_P, _P, _I, _I, _P, _P, _P, _P, _P, _P]),
    "tp_maxpool2": (_I, [_P, _I, _I, _I, _I, _P, _P]),
    "tp_debug_conv_counters": (_I, [_P, _I, _I]),
    "tp_slice_jobs": (_I, [_P, _P, _I, _I, _P, _P, _I, _P]),
    "tp_unslice_dets": (_I, [_P, _P, _I, _P, _I, _I, _I, _I, _P, _P, _P, _P]),
    "tp_render_frames": (_I, [_P, _P, _P, _I, _I, _I, _I, ctypes.c_uint32, _P, _P]),
    "tp_nccl_available": (_I, []),
    "tp_nccl_gather_dets": (_I, [_P, _P, _I64, _P, _I64, _P, _P, _P]),
}

_lib = None


def load() -> ctypes.CDLL:
    """Load the library (no GPU needed just to load and resolve symbols)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise NativeUnavailable(
            f"{LIB_PATH} is missing: build it with `make` (or __graft_entry__.build())"
        )
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def require_cuda():
    import torch

    if not torch.cuda.is_available():
        raise NativeUnavailable("no CUDA device: the tilepipe B200 path has no CPU fallback")
    return torch


def call(name: str, *args) -> None:
    """Invoke an int-status entry point; raise NativeError with the library message."""
    fn = getattr(load(), name)
    rc = fn(*args)
    if rc != 0:
        msg = load().tp_last_error().decode(errors="replace")
        raise NativeError(f"{name} failed ({rc}): {msg}")


def ptr(t) -> int:
    """Device (or host) address of a torch tensor, or 0 for None."""
    return 0 if t is None else int(t.data_ptr())


def stream_handle(stream=None) -> int:
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)
