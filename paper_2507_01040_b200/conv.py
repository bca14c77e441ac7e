"""Clifford convolution layer on the B200 tensor-core path.

Drop-in for the reference layer API (conv.py:77-140, :371-387): the same
`make_conv_layer(dims, sig, filters, bias, W=None, U=1)` constructor, the same
protocol layouts, `conv_forward(x, layer, variant)` and `conv_flops`. The
forward runs libclifford_b200.so's implicit-GEMM tcgen05 kernel; there is no
CPU path. Extensions (keyword-only): `precision` in {"fp32" (int8 digit slices,
exact accumulation), "3xtf32", "tf32", "bf16"} and `padding` in {"valid", "same"}.

Inputs: a CUDA torch tensor runs the device path and returns a CUDA tensor;
a numpy array (or CPU tensor) runs the host path of the C-ABI, which copies
in and out inside the call, and returns the same kind.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _device, _ops
from .algebra import Signature, schedule_flop_count
from .errors import ShapeMismatch
from .layout import Dims

PRECISIONS = {"fp32": 0, "tf32": 1, "bf16": 2, "3xtf32": 3}
PADDINGS = {"valid": 0, "same": 1}
VARIANTS = ("b200",)
# The reference CPU implementations (conv.py:371-381 / activation.py:400-416 /
# linear.py:97-102) are not provided here: naming one is an error, so a harness
# that verifies variants against variant="reference" cannot silently compare
# the B200 path with itself.
REFERENCE_CPU_VARIANTS = ("reference", "kernelized", "packed", "specialized")


def check_variant(variant, kind: str, cpu_variants) -> None:
    """ValueError for any variant but "b200" (the reference raises ValueError for
    unknown names, conv.py:381); its own CPU variant names get a message saying
    they are not implemented by this package."""
    if variant == "b200":
        return
    if variant in cpu_variants:
        raise ValueError(f"{kind} variant {variant!r} is a CPU implementation of the reference mvkernels "
                         f"package and is not provided by the B200 path (use 'b200')")
    raise ValueError(f"unknown {kind} variant {variant!r}")


@dataclass(frozen=True, eq=False)
class ConvLayer:
    dims: Dims
    sig: Signature
    filters: np.ndarray  # (N_B, C_in, C_out, d_filter^k) float32, frozen
    bias: np.ndarray     # (N_B, C_out) float32, frozen
    precision: str = "fp32"
    padding: str = "valid"
    W: int = 1
    U: int = 1
    _handles: dict = field(default_factory=dict, repr=False)

    @property
    def L(self) -> int:
        """Reference CPU packing width W*U (conv.py:95-97); unused by the B200 path."""
        return self.W * self.U

    @property
    def schedule(self):
        """The signature's FMA schedule (conv.py:131: schedule_for(sig))."""
        from .specialize import schedule_for
        return schedule_for(self.sig)

    @property
    def in_index(self) -> np.ndarray:
        """Valid-conv gather table (conv.py:136, layout.py:137-146), built on demand."""
        from .layout import gather_index_table
        return gather_index_table(self.dims)

    @property
    def pad(self) -> int:
        return (self.dims.d_filter - 1) // 2 if self.padding == "same" else 0

    @property
    def d_out(self) -> int:
        return self.dims.d_image + 2 * self.pad - self.dims.d_filter + 1

    def output_shape(self, B=None):
        B = self.dims.B if B is None else B
        return (B, self.dims.C_out, self.d_out ** self.dims.k, self.dims.n_blades)

    def handle(self) -> int:
        """The device handle on the current CUDA device (built once, cached)."""
        dev = _device.current_device()
        h = self._handles.get(dev)
        if h is None:
            f = _device.to_device_f32(self.filters)
            b = _device.to_device_f32(self.bias)
            ptr = _ops.op("conv_create", list(self.sig.g), self.dims.C_in, self.dims.C_out, self.dims.d_image,
                          self.dims.d_filter, PADDINGS[self.padding], PRECISIONS[self.precision], f, b)
            h = _device.Handle(ptr, _ops.destroyer("conv_destroy"))
            self._handles[dev] = h
        return h.ptr


def make_conv_layer(dims: Dims, sig: Signature, filters, bias, W: int | None = None, U: int = 1,
                    *, precision: str = "fp32", padding: str = "valid") -> ConvLayer:
    """Validate and freeze a layer (conv.py:101-140 checks, same exceptions)."""
    if sig.k != dims.k:
        raise ShapeMismatch(f"signature k={sig.k} does not match dims k={dims.k}")
    if not 1 <= dims.k <= 3:
        raise ShapeMismatch(f"convolution supports k in {{1,2,3}}, got k={dims.k}")
    f = filters.detach().cpu().numpy() if _device.is_cuda_tensor(filters) or _device.is_cpu_tensor(filters) else np.asarray(filters)
    b = bias.detach().cpu().numpy() if _device.is_cuda_tensor(bias) or _device.is_cpu_tensor(bias) else np.asarray(bias)
    if f.shape != dims.filters_shape():
        raise ShapeMismatch(f"filters shape {f.shape}, expected {dims.filters_shape()}")
    if b.shape != dims.bias_shape():
        raise ShapeMismatch(f"bias shape {b.shape}, expected {dims.bias_shape()}")
    W = 1 if W is None else W
    if W < 1 or U < 1:
        raise ShapeMismatch(f"W and U must be >= 1, got W={W} U={U}")
    if precision not in PRECISIONS:
        raise ValueError(f"unknown precision {precision!r}")
    if padding not in PADDINGS:
        raise ValueError(f"unknown padding {padding!r}")
    if padding == "same" and dims.d_filter % 2 == 0:
        raise ShapeMismatch("same padding needs an odd d_filter")
    return ConvLayer(dims, sig, _device.frozen_f32(f), _device.frozen_f32(b), precision, padding, W, U)


def _out(out, shape, device, pinned=False):
    """Validate a caller-provided output tensor or allocate one."""
    torch = _device.torch_mod()
    if out is None:
        if device is None:
            return torch.empty(shape, dtype=torch.float32, pin_memory=pinned)
        return torch.empty(shape, device=device, dtype=torch.float32)
    if tuple(out.shape) != tuple(shape) or out.dtype != torch.float32 or not out.is_contiguous():
        raise ShapeMismatch(f"out has shape {tuple(out.shape)}, expected contiguous float32 {tuple(shape)}")
    if (device is None) == out.is_cuda:
        raise ShapeMismatch("out must live on the same side (host/device) as the input")
    return out


def _out_np(out, shape):
    """Validate a caller-provided numpy output array (host path) or allocate one.
    The C-ABI writes straight into it, so shape, dtype and layout must be exact."""
    if out is None:
        return np.empty(shape, dtype=np.float32)
    if not isinstance(out, np.ndarray):
        raise ShapeMismatch(f"out must be a numpy array for numpy input, got {type(out).__name__}")
    if (tuple(out.shape) != tuple(shape) or out.dtype != np.float32 or not out.flags.c_contiguous
            or not out.flags.writeable):
        raise ShapeMismatch(f"out has shape {tuple(out.shape)} dtype {out.dtype}, expected writeable "
                            f"C-contiguous float32 {tuple(shape)}")
    return out


def _check_input(x, layer: ConvLayer):
    shape = tuple(x.shape)
    if shape != layer.dims.input_shape():
        raise ShapeMismatch(f"input shape {shape}, expected {layer.dims.input_shape()}")


def conv_forward(x, layer: ConvLayer, variant: str = "b200", out=None):
    """Protocol-to-protocol forward pass (conv.py:371-381) on the B200.

    `out` (optional) receives the result (a CUDA tensor for CUDA input, a
    CPU tensor / numpy array for host input)."""
    check_variant(variant, "conv", REFERENCE_CPU_VARIANTS)
    _check_input(x, layer)
    B = layer.dims.B
    if _device.is_cuda_tensor(x):
        with _device.on_device(x.device):
            xc = _device.device_input(x)
            y = _out(out, layer.output_shape(B), x.device)
            _ops.op("conv_forward", layer.handle(), xc, B, y)
        return y
    if _device.is_cpu_tensor(x):
        xc = x.float().contiguous()
        y = _out(out, layer.output_shape(B), None, pinned=xc.is_pinned())
        _ops.op("conv_forward_host", layer.handle(), xc, B, y)
        return y
    xa = np.ascontiguousarray(x, dtype=np.float32)
    y = _out_np(out, layer.output_shape(B))
    _ops.op("conv_forward_host", layer.handle(), _device.host_view(xa), B, _device.host_view(y))
    return y


def build_expanded_kernel(layer: ConvLayer):
    """(C_out*N_B, C_in*N_B, Q) real filter built on the device (conv.py:188-202)."""
    torch = _device.require_cuda()
    d = layer.dims
    nb = d.n_blades
    f = _device.to_device_f32(layer.filters)
    out = torch.empty((d.C_out * nb, d.C_in * nb, d.filter_positions), device=f.device, dtype=torch.float32)
    _ops.op("expand_kernel", list(layer.sig.g), f, d.C_in, d.C_out, d.filter_positions, out)
    return out


def conv_flops(dims: Dims, sig_or_layer, padding: str = "valid") -> int:
    """B * C_out * d_out^k * (C_in * Q * 2*terms + N_B) (conv.py:384-387). The
    second argument is the reference's OpSchedule (`layer.schedule`), a
    Signature, or a ConvLayer (whose padding then applies)."""
    if isinstance(sig_or_layer, ConvLayer):
        padding = sig_or_layer.padding
        sig_or_layer = sig_or_layer.sig
    pad = (dims.d_filter - 1) // 2 if padding == "same" else 0
    d_out = dims.d_image + 2 * pad - dims.d_filter + 1
    per_position = dims.C_in * dims.filter_positions * schedule_flop_count(sig_or_layer)
    return dims.B * dims.C_out * d_out ** dims.k * (per_position + dims.n_blades)
