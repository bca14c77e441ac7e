"""Clifford basic block: conv1 -> multivector activation -> conv2 [+ residual].

Mirrors the block of the reference bindings (pkg/frontend/src/block.ts:24-35
BlockSpec, :134-148 referenceBlockForward) and adds the residual of BASELINE
configs 3/5 (D1: zero "same" padding so shapes match). On the B200
the activation runs inside conv1's epilogue and the residual inside conv2's
(one launch each; no standalone activation pass, no extra HBM round trip).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _device, _ops
from .activation import ActivationConfig, AggMode, make_activation_config
from .algebra import Signature
from .conv import ConvLayer, _out, _out_np, conv_flops, make_conv_layer
from .errors import ShapeMismatch
from .layout import Dims


@dataclass(frozen=True, eq=False)
class BasicBlock:
    conv1: ConvLayer
    act: ActivationConfig
    conv2: ConvLayer
    residual: bool = True
    _handles: dict = field(default_factory=dict, repr=False)

    @property
    def B(self) -> int:
        return self.conv1.dims.B

    def input_shape(self):
        return self.conv1.dims.input_shape()

    def output_shape(self):
        return self.conv2.output_shape()

    def flops(self) -> int:
        return conv_flops(self.conv1.dims, self.conv1) + conv_flops(self.conv2.dims, self.conv2)

    def handle(self) -> int:
        dev = _device.current_device()
        h = self._handles.get(dev)
        if h is None:
            ptr = _ops.op("block_create", self.conv1.handle(), self.act.handle(self.conv1.dims.C_out),
                          self.conv2.handle(), bool(self.residual))
            h = _device.Handle(ptr, _ops.destroyer("block_destroy"))
            self._handles[dev] = h
        return h.ptr


def make_basic_block(sig: Signature, B: int, C_in: int, C_mid: int, C_out: int, d_image: int,
                     filters1, bias1, mode, filters2, bias2, act_weight=None, act_bias=None,
                     d_filter1: int = 3, d_filter2: int = 3, kernel_indices=None,
                     padding: str = "same", residual: bool = True, precision: str = "fp32") -> BasicBlock:
    """Build a block from a block.ts-style spec (g, B, Cin, Cmid, Cout, dImage, dFilter1/2, mode)."""
    k = sig.k
    d1 = Dims(B, C_in, C_mid, d_image, d_filter1, k) if padding == "valid" else \
        Dims(B, C_in, C_mid, d_image, d_filter1, k)
    conv1 = make_conv_layer(d1, sig, filters1, bias1, precision=precision, padding=padding)
    d_mid = conv1.d_out
    d2 = Dims(B, C_mid, C_out, d_mid, d_filter2, k)
    conv2 = make_conv_layer(d2, sig, filters2, bias2, precision=precision, padding=padding)
    ki = tuple(range(sig.n_blades)) if kernel_indices is None else tuple(kernel_indices)
    mode = AggMode(mode)
    act = make_activation_config(sig, mode, ki,
                                 act_weight if mode == AggMode.LINEAR else None,
                                 act_bias if mode == AggMode.LINEAR else None)
    if residual:
        if C_out != C_in:
            raise ShapeMismatch("residual needs C_out == C_in")
        if (d_image - conv2.d_out) % 2 or conv2.d_out > d_image:
            raise ShapeMismatch("residual needs a centred crop of the input")
    return BasicBlock(conv1, act, conv2, residual)


def block_forward(x, blk: BasicBlock, chunk: int = 0, out=None):
    """y = conv2(act(conv1(x))) [+ x] (block.ts:134-148 + residual)."""
    if tuple(x.shape) != blk.input_shape():
        raise ShapeMismatch(f"input shape {tuple(x.shape)}, expected {blk.input_shape()}")
    B = blk.B
    if _device.is_cuda_tensor(x):
        with _device.on_device(x.device):
            xc = _device.device_input(x)
            y = _out(out, blk.output_shape(), x.device)
            _ops.op("block_forward", blk.handle(), xc, B, y)
        return y
    if _device.is_cpu_tensor(x):
        xc = x.float().contiguous()
        y = _out(out, blk.output_shape(), None, pinned=xc.is_pinned())
        _ops.op("block_forward_host", blk.handle(), xc, B, chunk, y)
        return y
    xa = np.ascontiguousarray(x, dtype=np.float32)
    y = _out_np(out, blk.output_shape())
    _ops.op("block_forward_host", blk.handle(), _device.host_view(xa), B, chunk, _device.host_view(y))
    return y
