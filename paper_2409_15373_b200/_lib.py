"""ctypes binding of libjagged_b200.so (the C-ABI declared in include/jagged_b200.h).

Loading fails loudly when the library is missing or no CUDA device is present: there is no CPU
fallback anywhere in this package.
"""
from __future__ import annotations

import ctypes as C
import os

_PKG = os.path.dirname(os.path.abspath(__file__))
# JG_LIB_PATH: load an alternative build (A/B timing of kernel variants in one process launch)
LIB_PATH = os.environ.get("JG_LIB_PATH") or os.path.join(_PKG, "libjagged_b200.so")

JG_F32, JG_BF16, JG_F64 = 0, 1, 2
STATUS = {0: "JG_OK", 1: "JG_INVALID_ARGUMENT", 2: "JG_CUDA_ERROR", 3: "JG_OUT_OF_MEMORY", 4: "JG_UNSUPPORTED"}

_lib = None
P, I64, I32, D = C.c_void_p, C.c_int64, C.c_int32, C.c_double

# name -> argtypes (restype jg_status == int unless noted)
SIGNATURES = {
    "jg_make_offsets": [P, I64, P, P, P],
    "jg_segment_lengths": [P, I64, P, P],
    "jg_sq_offsets": [P, I64, P, P],
    "jg_schedule_create": [P, I64, I64, P, P],
    "jg_schedule_destroy": [P],
    "jg_schedule_work_list": [P, P, I64, P],
    "jg_jagged_to_dense": [P, I64, I64, P, I64, D, P, C.c_int, P],
    "jg_dense_to_jagged": [P, I64, I64, I64, P, I64, I64, P, C.c_int, P],
    "jg_jagged2_to_dense": [P, P, I64, P, I64, D, P, C.c_int, P],
    "jg_dense_to_jagged2": [P, I64, I64, P, P, I64, P, C.c_int, P],
    "jg_elementwise": [I32, P, P, I64, P, C.c_int, P],
    "jg_scale": [P, I64, D, P, C.c_int, P],
    "jg_jagged_dense_bmm": [P, I64, I64, I64, I64, P, P, P, C.c_int, C.c_int, P],
    "jg_jagged_jagged_bmm": [P, I64, I64, I64, I64, P, P, P, C.c_int, C.c_int, P],
    "jg_jagged_softmax": [P, I64, I64, I64, P, P, C.c_int, P],
    "jg_jagged_jagged_bmm_jagged_out": [P, P, I64, I64, I64, P, P, P, C.c_int, C.c_int, P],
    "jg_array_jagged_bmm_jagged_out": [P, P, I64, I64, I64, I64, P, P, P, C.c_int, C.c_int, P],
    "jg_jagged2_softmax": [P, P, I64, P, P, C.c_int, P],
    "jg_jagged_dense_bmm_vjp": [P, I64, I64, I64, I64, P, P, P, P, P, C.c_int, C.c_int, P],
    "jg_jagged_jagged_bmm_vjp": [P, I64, I64, I64, I64, P, P, P, P, P, C.c_int, C.c_int, P],
    "jg_jagged_softmax_vjp": [P, I64, I64, I64, P, P, P, C.c_int, P],
    "jg_jagged_jagged_bmm_jagged_out_vjp": [P, P, I64, I64, I64, I64, P, P, P, P, P, C.c_int, C.c_int, P],
    "jg_array_jagged_bmm_jagged_out_vjp": [P, P, I64, I64, I64, I64, P, P, P, P, P, C.c_int, C.c_int, P],
    "jg_jagged2_softmax_vjp": [P, P, I64, P, P, P, C.c_int, P],
    "jg_jagged_flash_attention_forward": [P, I64, I64, I32, I32, P, P, P, I64, I64, P, P, C.c_int, P, P],
    "jg_jagged_flash_attention_backward": [P, I64, I64, I32, I32, P, P, P, P, P, P, I64, I64, P, P, P, C.c_int, I32,
                                           P, P, P],
    "jg_jagged_attention": [P, P, I64, I64, I64, I32, I32, P, P, P, P, C.c_int, P, P],
    "jg_dense_flash_attention_forward": [P, I64, I64, I32, I32, P, P, P, I64, I64, P, P, C.c_int, P],
    "jg_dense_flash_attention_backward": [P, I64, I64, I32, I32, P, P, P, P, P, P, I64, I64, P, P, P, C.c_int, P, P],
    "jg_jagged_flash_attention_fwd_bwd_host": [P, I64, I32, I32, P, P, P, P, P, P, P, P, P, C.c_int, P],
    "jg_feature_interaction": [P, I64, I64, I64, I64, P, P, P, P, C.c_int, P, P],
    "jg_mlp_layer_forward": [I64, I64, I64, P, P, P, I32, P, P, C.c_int, P],
    "jg_mlp_layer_backward": [I64, I64, I64, P, P, P, I32, P, P, P, P, C.c_int, P],
}
OTHER = {
    "jg_last_error": ([], C.c_char_p),
    "jg_version": ([], C.c_char_p),
    "jg_launch_count": ([], C.c_int64),
    "jg_reset_launch_count": ([], None),
    "jg_scratch_counters": ([P, P], None),
    "jg_scratch_reset_peak": ([], None),
    "jg_scratch_raise_peak": ([I64], None),
    "jg_schedule_sq_offsets": ([P], P),
    "jg_attention_backward_workspace_size": ([I64, I64, I32, I32], C.c_int64),
    "jg_feature_interaction_workspace_size": ([I64, I64], C.c_int64),
}


class JaggedError(ValueError):
    """Raised for JG_INVALID_ARGUMENT (the reference's std::invalid_argument)."""


class JaggedDeviceError(RuntimeError):
    """Raised for CUDA errors, OOM and unsupported dtypes (no CPU fallback)."""


def load(path: str = LIB_PATH):
    """Load the shared library without touching the GPU (used by the CPU symbol test)."""
    if not os.path.exists(path):
        raise RuntimeError(f"{path} is missing: run `python -m paper_2409_15373_b200.build` (no CPU fallback)")
    lib = C.CDLL(path)
    for name, args in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = C.c_int
    for name, (args, res) in OTHER.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    return lib


def lib():
    global _lib
    if _lib is None:
        import torch

        if not torch.cuda.is_available():
            raise RuntimeError("libjagged_b200 needs a CUDA device (sm_100a); there is no CPU fallback")
        _lib = load()
    return _lib


def check(rc: int) -> None:
    if rc == 0:
        return
    msg = lib().jg_last_error().decode()
    if rc == 1:
        raise JaggedError(msg)
    raise JaggedDeviceError(f"{STATUS.get(rc, rc)}: {msg}")
