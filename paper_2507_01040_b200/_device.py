"""Device-memory plumbing (PyTorch is used for allocation and streams only)."""

from __future__ import annotations

import contextlib

import numpy as np


class Handle:
    """Owns one C-ABI handle; destroyed with the Python object."""

    def __init__(self, ptr: int, destroy):
        self.ptr = ptr
        self._destroy = destroy

    def __del__(self):
        if self.ptr and self._destroy is not None:
            try:
                self._destroy(self.ptr)
            except Exception:
                pass
            self.ptr = 0


def require_cuda():
    import torch
    if not torch.cuda.is_available():
        from .errors import ConfigInvalid
        raise ConfigInvalid("the B200 path needs a CUDA device (no CPU fallback)")
    return torch


def host_view(a):
    """A zero-copy torch view of a C-contiguous float32 numpy array (host path)."""
    import torch
    return torch.from_numpy(a)


def torch_mod():
    import torch
    return torch


def is_cuda_tensor(x) -> bool:
    try:
        import torch
    except ImportError:
        return False
    return isinstance(x, torch.Tensor) and x.is_cuda


def is_cpu_tensor(x) -> bool:
    try:
        import torch
    except ImportError:
        return False
    return isinstance(x, torch.Tensor) and not x.is_cuda


_cuda_checked = False


def current_device() -> int:
    global _cuda_checked
    if not _cuda_checked:
        require_cuda()  # fail loudly without a GPU (no CPU fallback)
        _cuda_checked = True
    return torch_mod().cuda.current_device()


def stream_ptr(device=None) -> int:
    """cudaStream_t of torch's current stream (the raw query: a few hundred ns
    instead of building a Stream object per call)."""
    torch = torch_mod()
    raw = getattr(torch._C, "_cuda_getCurrentRawStream", None)
    if raw is not None:
        return raw(torch.cuda.current_device() if device is None else torch.device(device).index)
    return torch.cuda.current_stream(device).cuda_stream


_NULL_CTX = contextlib.nullcontext()


def on_device(device):
    """torch.cuda.device(device), or a no-op when it is already current."""
    torch = torch_mod()
    if device.index is None or device.index == torch.cuda.current_device():
        return _NULL_CTX
    return torch.cuda.device(device)


def device_input(x):
    """A CUDA tensor as the C-ABI takes it: fp32, contiguous, 16-byte aligned
    (a view with a 4-byte storage offset is copied rather than rejected)."""
    torch = torch_mod()
    if x.dtype == torch.float32 and x.is_contiguous() and x.data_ptr() % 16 == 0:
        return x
    y = x.float().contiguous()
    return y if y.data_ptr() % 16 == 0 else y.clone()


def to_device_f32(arr, device=None):
    """Contiguous fp32 CUDA copy of a numpy array / tensor."""
    torch = require_cuda()
    if isinstance(arr, torch.Tensor):
        return arr.detach().to(device=device or torch.cuda.current_device(), dtype=torch.float32).contiguous().clone()
    a = np.ascontiguousarray(arr, dtype=np.float32)
    return torch.from_numpy(a.copy()).to(device=device or torch.cuda.current_device())


def frozen_f32(arr) -> np.ndarray:
    """Private frozen fp32 copy (conv.py:70-74)."""
    if is_cuda_tensor(arr) or is_cpu_tensor(arr):
        arr = arr.detach().cpu().numpy()
    out = np.array(arr, dtype=np.float32, order="C", copy=True)
    out.flags.writeable = False
    return out
