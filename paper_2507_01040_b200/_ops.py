"""The binding the package calls: libclifford_b200's C-ABI registered as
PyTorch operators, torch.ops.clifford_b200.* (csrc_torch/clifford_ops.cpp).

It replaces the paper's ctypes bindings: tensors go in, the
operators forward their data pointers and the current CUDA stream of their
device to the C-ABI, and a non-zero C-ABI status comes back as an error
message "clifford_b200[<status>] <Type>: <message>", re-raised here as the
reference's exception class (errors.py:4-56; ValueError where the reference
raises ValueError). There is deliberately no CPU fallback: without the
built extension, the library or a CUDA device, calls fail loudly.

CL_LIB_PATH selects another build of the C-ABI library (the diagnostic A/B
build, libclifford_b200_ab.so) before the first call.
"""

from __future__ import annotations

import os
import re

from .errors import STATUS_TO_ERROR, MvkernelsError

_HERE = os.path.dirname(os.path.abspath(__file__))
TORCH_OPS_PATH = os.path.join(_HERE, "lib", "libclifford_b200_torch.so")

_ops = None
_ERR = re.compile(r"clifford_b200\[(\d+)\] (?:([A-Za-z]+): )?([^\n]*)")


def lib_path() -> str:
    return os.environ.get("CL_LIB_PATH") or os.path.join(_HERE, "lib", "libclifford_b200.so")


def ops():
    """torch.ops.clifford_b200, loaded (once) on top of libclifford_b200.so."""
    global _ops
    if _ops is not None:
        return _ops
    import torch
    for path in (TORCH_OPS_PATH, lib_path()):
        if not os.path.exists(path):
            raise RuntimeError(f"{path} is missing: build it with `python -m paper_2507_01040_b200.build` "
                               "(the B200 path has no CPU fallback)")
    torch.ops.load_library(TORCH_OPS_PATH)
    o = torch.ops.clifford_b200
    call(o.load_library, lib_path())
    _ops = o
    return o


def call(fn, *args):
    """Run one operator; C-ABI failures become the reference's exceptions."""
    try:
        return fn(*args)
    except RuntimeError as e:
        m = _ERR.search(str(e))
        if not m:
            raise
        status, typ, msg = int(m.group(1)), m.group(2), m.group(3)
        if typ == "ValueError":
            raise ValueError(msg) from None
        raise STATUS_TO_ERROR.get(status, MvkernelsError)(msg) from None


def op(name: str, *args):
    """call(torch.ops.clifford_b200.<name>, *args)."""
    return call(getattr(ops(), name), *args)


def launch_count() -> int:
    """Kernels this process has launched through the library."""
    return int(op("launch_count"))


def destroyer(name: str):
    """A destroy callback for _device.Handle (no-op once the interpreter tears down)."""
    def destroy(h):
        try:
            getattr(ops(), name)(int(h))
        except Exception:
            pass
    return destroy
