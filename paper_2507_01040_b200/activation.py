"""Multivector activation layer on the B200 (HBM-bound CUDA kernel).

Drop-in for activation.py:36-89 / :400-433 of the reference:
`make_activation_config(sig, agg_mode, kernel_indices, weight=None, bias=None)`
validates exactly like the reference and `activation_forward(x, cfg, variant)`
accepts the flat (B, C, N_B) form and the spatial (B, C, P, N_B) form that
the reference server folds to (B*P, C, N_B) (serve.py:108-117) -- here the
gate is computed per (b, c, p) in place, no fold is materialised. Any C and
any K <= N_B work (the reference's 'specialized' preconditions do not apply).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from enum import IntEnum

import numpy as np

from . import _device, _lib
from .algebra import Signature
from .conv import _out, _out_np, check_variant
from .errors import IndexOutOfRange, ModeConfigMismatch, ShapeMismatch

VARIANTS = ("b200",)
# The reference CPU implementations (conv.py:371-381 / activation.py:400-416 /
# linear.py:97-102) are not provided here: naming one is an error, so a harness
# that verifies variants against variant="reference" cannot silently compare
# the B200 path with itself.
REFERENCE_CPU_VARIANTS = ("reference", "hoisted", "packed", "specialized")


class AggMode(IntEnum):
    """Gate aggregation mode; values are part of the FFI contract (activation.py:36-41)."""

    LINEAR = 0
    SUM = 1
    MEAN = 2


@dataclass(frozen=True, eq=False)
class ActivationConfig:
    sig: Signature
    agg_mode: AggMode
    kernel_indices: tuple
    weight: np.ndarray | None = None  # (C, K) Linear only
    bias: np.ndarray | None = None    # (C,) Linear only
    _handles: dict = field(default_factory=dict, repr=False)

    @property
    def K(self) -> int:
        return len(self.kernel_indices)

    def handle(self, C_: int) -> int:
        """Device handle for C channels on the current device (cached)."""
        key = (_device.current_device(), C_)
        h = self._handles.get(key)
        if h is None:
            lib = _lib.load()
            w = b = None
            if self.agg_mode == AggMode.LINEAR:
                w = _device.to_device_f32(self.weight)
                b = _device.to_device_f32(self.bias)
            out = C.c_void_p()
            _lib.check(lib.cl_act_create(
                _lib.int32_array(self.sig.g), self.sig.k, int(self.agg_mode),
                _lib.int32_array(self.kernel_indices), self.K, C_,
                C.c_void_p(w.data_ptr()) if w is not None else None,
                C.c_void_p(b.data_ptr()) if b is not None else None,
                C.c_void_p(_device.stream_ptr()), C.byref(out)))
            h = _device.Handle(out.value, lib.cl_act_destroy)
            self._handles[key] = h
        return h.ptr


def make_activation_config(sig: Signature, agg_mode, kernel_indices, weight=None, bias=None) -> ActivationConfig:
    """Validation order and exceptions of activation.py:57-89."""
    agg_mode = AggMode(agg_mode)
    ki = tuple(int(i) for i in kernel_indices)
    nb = sig.n_blades
    if len(set(ki)) != len(ki):
        raise IndexOutOfRange(f"kernel indices {ki} contain duplicates")
    if not ki or any(i < 0 or i >= nb for i in ki):
        raise IndexOutOfRange(f"kernel indices {ki} outside [0, {nb})")
    if agg_mode == AggMode.LINEAR:
        if weight is None or bias is None:
            raise ModeConfigMismatch("Linear mode requires weight and bias")
        weight = _device.frozen_f32(weight)
        bias = _device.frozen_f32(bias)
        if weight.ndim != 2 or weight.shape[1] != len(ki):
            raise ShapeMismatch(f"weight shape {weight.shape}, expected (C, K={len(ki)})")
        if bias.shape != (weight.shape[0],):
            raise ShapeMismatch(f"bias shape {bias.shape}, expected ({weight.shape[0]},)")
    else:
        if weight is not None or bias is not None:
            raise ModeConfigMismatch(f"{agg_mode.name} mode forbids weight/bias")
    return ActivationConfig(sig, agg_mode, ki, weight, bias)


def _dims(x, cfg: ActivationConfig):
    nb = cfg.sig.n_blades
    if x.ndim == 3:
        B, C_, n = x.shape
        P = 1
    elif x.ndim == 4:
        B, C_, P, n = x.shape
    else:
        raise ShapeMismatch(f"input shape {tuple(x.shape)}, expected (B, C, {nb}) or (B, C, P, {nb})")
    if n != nb:
        raise ShapeMismatch(f"input shape {tuple(x.shape)}, expected (B, C, {nb})")
    if cfg.agg_mode == AggMode.LINEAR and cfg.weight.shape[0] != C_:
        raise ShapeMismatch(f"weight is for C={cfg.weight.shape[0]} channels, input has C={C_}")
    return B, C_, P


def activation_forward(x, cfg: ActivationConfig, variant: str = "b200", out=None):
    """Gated scaling of every multivector (activation.py:400-416 semantics)."""
    check_variant(variant, "activation", REFERENCE_CPU_VARIANTS)
    B, C_, P = _dims(x, cfg)
    lib = _lib.load()
    if _device.is_cuda_tensor(x):
        torch = _device.torch_mod()
        with _device.on_device(x.device):
            xc = _device.device_input(x)
            y = _out(out, tuple(xc.shape), x.device)
            _lib.check(lib.cl_act_forward(C.c_void_p(cfg.handle(C_)), C.c_void_p(xc.data_ptr()),
                                          C.c_void_p(y.data_ptr()), B, P, C.c_void_p(_device.stream_ptr())))
        return y
    if _device.is_cpu_tensor(x):
        torch = _device.torch_mod()
        xc = x.float().contiguous()
        y = _out(out, tuple(xc.shape), None, pinned=xc.is_pinned())
        _lib.check(lib.cl_act_forward_host(C.c_void_p(cfg.handle(C_)), C.c_void_p(xc.data_ptr()),
                                           C.c_void_p(y.data_ptr()), B, P, C.c_void_p(_device.stream_ptr())))
        return y
    xa = np.ascontiguousarray(x, dtype=np.float32)
    y = _out_np(out, xa.shape)
    _lib.check(lib.cl_act_forward_host(C.c_void_p(cfg.handle(C_)), C.c_void_p(xa.ctypes.data),
                                       C.c_void_p(y.ctypes.data), B, P, C.c_void_p(_device.stream_ptr())))
    return y


def activation_flops(B: int, C: int, n_blades: int, K: int, mode, sigmoid_cost: int = 30) -> int:
    """Cost model of activation.py:419-433."""
    mode = AggMode(mode)
    if mode == AggMode.LINEAR:
        per_bc = 2 * K + 1 + sigmoid_cost + n_blades
    elif mode == AggMode.SUM:
        per_bc = K - 1 + sigmoid_cost + n_blades
    else:
        per_bc = K - 1 + 1 + sigmoid_cost + n_blades
    return B * C * per_bc
