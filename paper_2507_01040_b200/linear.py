"""Clifford linear layer on the B200.

Drop-in for linear.py:22-107 of the reference: `make_linear_layer(sig,
weight (N_B, C_out, C_in), bias (N_B, C_out))`, `linear_forward(x (B, C_in,
N_B), layer, variant)` and `linear_flops`. The layer runs on the same
tcgen05 implicit-GEMM kernel as the convolution (a 1x1 conv whose rows are
the samples, 128 samples per tile), in any of the four precision modes.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _device, _ops
from .algebra import Signature, schedule_flop_count
from .conv import PRECISIONS, _out, _out_np, check_variant
from .errors import ShapeMismatch

VARIANTS = ("b200",)
# The reference CPU implementations (conv.py:371-381 / activation.py:400-416 /
# linear.py:97-102) are not provided here: naming one is an error, so a harness
# that verifies variants against variant="reference" cannot silently compare
# the B200 path with itself.
REFERENCE_CPU_VARIANTS = ("reference", "gemm")


@dataclass(frozen=True, eq=False)
class LinearLayer:
    sig: Signature
    C_in: int
    C_out: int
    weight: np.ndarray  # (N_B, C_out, C_in) float32, frozen
    bias: np.ndarray    # (N_B, C_out) float32, frozen
    precision: str = "fp32"
    _handles: dict = field(default_factory=dict, repr=False)

    def handle(self) -> int:
        dev = _device.current_device()
        h = self._handles.get(dev)
        if h is None:
            torch = _device.torch_mod()
            w = torch.from_numpy(np.array(self.weight, dtype=np.float32))
            b = torch.from_numpy(np.array(self.bias, dtype=np.float32))
            ptr = _ops.op("linear_create", list(self.sig.g), self.C_in, self.C_out, w, b,
                          PRECISIONS[self.precision])
            h = _device.Handle(ptr, _ops.destroyer("conv_destroy"))
            self._handles[dev] = h
        return h.ptr


def make_linear_layer(sig: Signature, weight, bias, *, precision: str = "fp32") -> LinearLayer:
    """Checks of linear.py:32-47 (same exceptions)."""
    if not 1 <= sig.k <= 3:
        raise ShapeMismatch(f"linear layer supports k in {{1,2,3}}, got k={sig.k}")
    w = np.asarray(weight.detach().cpu().numpy() if hasattr(weight, "detach") else weight)
    b = np.asarray(bias.detach().cpu().numpy() if hasattr(bias, "detach") else bias)
    nb = sig.n_blades
    if w.ndim != 3 or w.shape[0] != nb:
        raise ShapeMismatch(f"weight shape {w.shape}, expected (N_B={nb}, C_out, C_in)")
    _, c_out, c_in = w.shape
    if b.shape != (nb, c_out):
        raise ShapeMismatch(f"bias shape {b.shape}, expected {(nb, c_out)}")
    if precision not in PRECISIONS:
        raise ValueError(f"unknown precision {precision!r}")
    return LinearLayer(sig, c_in, c_out, _device.frozen_f32(w), _device.frozen_f32(b), precision)


def linear_forward(x, layer: LinearLayer, variant: str = "b200", out=None):
    """(B, C_in, N_B) -> (B, C_out, N_B) (linear.py:97-102) on the B200."""
    check_variant(variant, "linear", REFERENCE_CPU_VARIANTS)
    nb = layer.sig.n_blades
    if x.ndim != 3 or x.shape[1] != layer.C_in or x.shape[2] != nb:
        raise ShapeMismatch(f"input shape {tuple(x.shape)}, expected (B, {layer.C_in}, {nb})")
    B = int(x.shape[0])
    shape = (B, layer.C_out, nb)
    if _device.is_cuda_tensor(x):
        with _device.on_device(x.device):
            xc = _device.device_input(x)
            y = _out(out, shape, x.device)
            _ops.op("conv_forward", layer.handle(), xc, B, y)  # cl_linear_forward == cl_conv_forward
        return y
    if _device.is_cpu_tensor(x):
        xc = x.float().contiguous()
        y = _out(out, shape, None, pinned=xc.is_pinned())
        _ops.op("conv_forward_host", layer.handle(), xc, B, y)
        return y
    xa = np.ascontiguousarray(x, dtype=np.float32)
    y = _out_np(out, shape)
    _ops.op("conv_forward_host", layer.handle(), _device.host_view(xa), B, _device.host_view(y))
    return y


def linear_flops(B: int, C_in: int, C_out: int, sig_or_layer) -> int:
    """B * C_out * (C_in * 2*terms + N_B) (linear.py:105-107)."""
    sig = getattr(sig_or_layer, "sig", sig_or_layer)
    return B * C_out * (C_in * schedule_flop_count(sig) + sig.n_blades)
