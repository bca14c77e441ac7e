"""Bridge for the reference package's own dispatch: `variant="b200"` inside
mvkernels' `conv_forward` / `activation_forward` / `linear_forward`
(conv.py:371-381, activation.py:400-416, linear.py:97-102).

A maintainer adds one branch per dispatcher:

    if variant == "b200":
        from paper_2507_01040_b200.ref_bridge import conv_forward_b200
        return conv_forward_b200(x, layer)

and "b200" to bench.VARIANTS (bench.py:36-40); the reference's run_sweep
then verifies it against its own conv_reference before timing it
(bench.py:355-377) and parity_report covers it over all 36 signatures.

The functions take the reference's layer objects (duck-typed: the frozen
dataclasses of conv.py:77-98, activation.py:44-55, linear.py:22-29), build
the B200 layer once per reference layer (cached by identity, as the
reference layers are eq=False dataclasses) and run the host-buffer path of
the C-ABI: numpy in, numpy out, as the reference callers expect. Nothing
here computes on the CPU.
"""

from __future__ import annotations

import weakref

import numpy as np

from .activation import activation_forward, make_activation_config
from .algebra import Signature
from .conv import conv_forward, make_conv_layer
from .layout import Dims
from .linear import linear_forward, make_linear_layer

_cache: "weakref.WeakKeyDictionary" = weakref.WeakKeyDictionary()


def _sig(ref_sig) -> Signature:
    return Signature(tuple(int(v) for v in ref_sig.g))


def _ours(ref_obj, build):
    got = _cache.get(ref_obj)
    if got is None:
        got = build()
        _cache[ref_obj] = got
    return got


def conv_forward_b200(x, layer, precision: str = "fp32"):
    """conv_forward(x, layer, "b200") of the reference: x (B, C_in, d^k, N_B)."""
    d = layer.dims

    def build():
        dims = Dims(int(d.B), int(d.C_in), int(d.C_out), int(d.d_image), int(d.d_filter), int(d.k))
        return make_conv_layer(dims, _sig(layer.sig), np.asarray(layer.filters), np.asarray(layer.bias),
                               precision=precision)

    ours = _ours(layer, build)
    return conv_forward(np.ascontiguousarray(x, dtype=np.float32), ours)


def activation_forward_b200(x, cfg):
    """activation_forward(x, cfg, "b200") of the reference: x (B, C, N_B)
    (or the spatial (B, C, P, N_B) form, gated per position)."""
    def build():
        w = None if cfg.weight is None else np.asarray(cfg.weight)
        b = None if cfg.bias is None else np.asarray(cfg.bias)
        return make_activation_config(_sig(cfg.sig), int(cfg.agg_mode), tuple(cfg.kernel_indices), w, b)

    ours = _ours(cfg, build)
    return activation_forward(np.ascontiguousarray(x, dtype=np.float32), ours)


def linear_forward_b200(x, layer):
    """linear_forward(x, layer, "b200") of the reference: x (B, C_in, N_B)."""
    ours = _ours(layer, lambda: make_linear_layer(_sig(layer.sig), np.asarray(layer.weight),
                                                  np.asarray(layer.bias)))
    return linear_forward(np.ascontiguousarray(x, dtype=np.float32), ours)
