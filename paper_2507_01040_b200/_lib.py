"""Plain-ctypes view of the C-ABI (include/clifford_b200.h), for the tests
that check the boundary itself (every header symbol is exported, raw C
calls, status codes) -- the package calls the library through its PyTorch
operator registration instead (_ops.py, torch.ops.clifford_b200.*).
"""

from __future__ import annotations

import ctypes as C
import os

from .errors import STATUS_TO_ERROR, ConfigInvalid, MvkernelsError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CL_LIB_PATH") or os.path.join(_HERE, "lib", "libclifford_b200.so")  # override: A/B builds

_lib = None

EXPORTS = (
    "cl_validate_signature", "cl_blade_product", "cl_schedule_terms", "cl_basis_info", "cl_expand_kernel",
    "cl_conv_create", "cl_conv_gemm_flops", "cl_conv_plan_info", "cl_conv_out_side", "cl_conv_forward", "cl_conv_forward_host",
    "cl_conv_workspace_bytes", "cl_conv_time_kernel", "cl_conv_forward_ws", "cl_block_workspace_bytes", "cl_block_forward_ws",
    "cl_conv_destroy", "cl_linear_create", "cl_linear_forward", "cl_linear_forward_host",
    "cl_linear_destroy", "cl_act_create", "cl_act_forward", "cl_act_forward_host", "cl_act_preactivation", "cl_act_gather",
    "cl_act_kernel_count",
    "cl_act_destroy", "cl_block_create", "cl_block_forward", "cl_block_forward_host",
    "cl_block_destroy", "cl_block_time_conv2", "cl_last_error", "cl_launch_count", "cl_version",
)

P = C.c_void_p
I32P = C.POINTER(C.c_int32)


def load():
    """Load (once) and type the shared library."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"{LIB_PATH} is missing: build it with `python -m paper_2507_01040_b200.build` "
            "(the B200 path has no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    sig = {
        "cl_validate_signature": (C.c_int, [I32P, C.c_int]),
        "cl_blade_product": (C.c_int, [C.c_int, C.c_int, I32P, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
        "cl_schedule_terms": (C.c_int, [I32P, C.c_int]),
        "cl_basis_info": (C.c_int, [I32P, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int8)]),
        "cl_expand_kernel": (C.c_int, [I32P, C.c_int, P, C.c_int, C.c_int, C.c_int, P, P]),
        "cl_conv_create": (C.c_int, [I32P, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                     P, P, P, C.POINTER(P)]),
        "cl_conv_out_side": (C.c_int, [P, C.POINTER(C.c_int)]),
        "cl_conv_plan_info": (C.c_int, [I32P, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                        C.POINTER(C.c_int64)]),
        "cl_conv_gemm_flops": (C.c_int, [P, C.c_int64, C.POINTER(C.c_double), C.POINTER(C.c_double),
                                         C.POINTER(C.c_int)]),
        "cl_conv_forward": (C.c_int, [P, P, P, C.c_int64, P]),
        "cl_conv_forward_host": (C.c_int, [P, P, P, C.c_int64, P]),
        "cl_conv_workspace_bytes": (C.c_size_t, [P, C.c_int64]),
        "cl_conv_time_kernel": (C.c_int, [P, P, P, C.c_int64, C.c_int, P, C.POINTER(C.c_float)]),
        "cl_conv_forward_ws": (C.c_int, [P, P, P, C.c_int64, P, C.c_size_t, P]),
        "cl_block_workspace_bytes": (C.c_size_t, [P, C.c_int64]),
        "cl_block_forward_ws": (C.c_int, [P, P, P, C.c_int64, P, C.c_size_t, P]),
        "cl_conv_destroy": (None, [P]),
        "cl_linear_create": (C.c_int, [I32P, C.c_int, C.c_int, C.c_int, P, P, C.c_int, P, C.POINTER(P)]),
        "cl_linear_forward": (C.c_int, [P, P, P, C.c_int64, P]),
        "cl_linear_forward_host": (C.c_int, [P, P, P, C.c_int64, P]),
        "cl_linear_destroy": (None, [P]),
        "cl_act_create": (C.c_int, [I32P, C.c_int, C.c_int, I32P, C.c_int, C.c_int, P, P, P, C.POINTER(P)]),
        "cl_act_forward": (C.c_int, [P, P, P, C.c_int64, C.c_int64, P]),
        "cl_act_forward_host": (C.c_int, [P, P, P, C.c_int64, C.c_int64, P]),
        "cl_act_preactivation": (C.c_int, [P, P, P, C.c_int64, C.c_int64, P]),
        "cl_act_gather": (C.c_int, [P, P, P, C.c_int64, C.c_int64, P]),
        "cl_act_kernel_count": (C.c_int, [P]),
        "cl_act_destroy": (None, [P]),
        "cl_block_create": (C.c_int, [P, P, P, C.c_int, C.POINTER(P)]),
        "cl_block_forward": (C.c_int, [P, P, P, C.c_int64, P]),
        "cl_block_forward_host": (C.c_int, [P, P, P, C.c_int64, C.c_int64, P]),
        "cl_block_destroy": (None, [P]),
        "cl_block_time_conv2": (C.c_int, [P, P, P, C.c_int64, C.c_int, P, C.POINTER(C.c_float)]),
        "cl_last_error": (C.c_char_p, []),
        "cl_launch_count": (C.c_uint64, []),
        "cl_version": (C.c_char_p, []),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(status: int) -> None:
    """Raise the reference exception class for a non-zero C-ABI status."""
    if status == 0:
        return
    msg = load().cl_last_error().decode(errors="replace")
    cls = STATUS_TO_ERROR.get(abs(status), MvkernelsError)
    if ": " in msg:
        typ, rest = msg.split(": ", 1)
        if typ == "ValueError":
            raise ValueError(rest)
        msg = rest
    raise cls(msg)


def int32_array(values):
    arr = (C.c_int32 * max(1, len(values)))(*[int(v) for v in values])
    return arr


def launch_count() -> int:
    return int(load().cl_launch_count())


def require_cuda():
    import torch
    if not torch.cuda.is_available():
        raise ConfigInvalid("the B200 path needs a CUDA device (no CPU fallback)")
    return torch
