"""Signatures and blade products (host side of the reference algebra module,
algebra.py:26-63, :87-99, :116-145). Blade products come from the C-ABI
(`cl_blade_product`, through torch.ops.clifford_b200), i.e. the same integer
code that builds the device kernels; the Python side only validates and
shapes the results."""

from __future__ import annotations

from dataclasses import dataclass
from functools import lru_cache
from typing import Iterable

import numpy as np

from . import _ops
from .errors import DimensionMismatch, InvalidMetricValue, InvalidSignature


@dataclass(frozen=True)
class Signature:
    """Metric signature g of Cl_g(R^k), g_i in {-1, 0, +1} (algebra.py:26-46)."""

    g: tuple[int, ...]

    @property
    def k(self) -> int:
        return len(self.g)

    @property
    def n_blades(self) -> int:
        return 1 << len(self.g)

    def __str__(self) -> str:
        return "(" + ",".join(f"{v:+d}" for v in self.g) + ")"


def validate_signature(values: Iterable[float]) -> Signature:
    """algebra.py:49-63: InvalidMetricValue outside {-1,0,+1}, InvalidSignature if all zero."""
    g = []
    for v in values:
        if v not in (-1, 0, 1):
            raise InvalidMetricValue(f"metric value {v!r} not in {{-1, 0, +1}}")
        g.append(int(v))
    if not any(g):
        raise InvalidSignature(f"signature {tuple(g)} has no non-zero element")
    return Signature(tuple(g))


def blade_product(i_mask: int, j_mask: int, sig: Signature) -> tuple[int, int]:
    """(target, coeff) of e_I e_J via the C-ABI (algebra.py:87-99)."""
    t, c = _ops.op("blade_product", int(i_mask), int(j_mask), list(sig.g))
    return int(t), int(c)


@dataclass(frozen=True, eq=False)
class BladeProductTable:
    """Dense N_B x N_B blade product table (algebra.py:100-111): target[i, j] =
    i xor j, coeff[i, j] in {-1, 0, +1}; read-only arrays. Also unpacks as
    `target, coeff = table`."""

    sig: Signature
    target: np.ndarray
    coeff: np.ndarray

    def __iter__(self):
        return iter((self.target, self.coeff))


@lru_cache(maxsize=None)
def product_table(sig: Signature) -> BladeProductTable:
    """Cached blade product table from the C-ABI's integer code (algebra.py:114-129)."""
    nb = sig.n_blades
    tgt = np.empty((nb, nb), np.int64)
    cof = np.empty((nb, nb), np.int64)
    for i in range(nb):
        for j in range(nb):
            tgt[i, j], cof[i, j] = blade_product(i, j, sig)
    tgt.flags.writeable = False
    cof.flags.writeable = False
    return BladeProductTable(sig, tgt, cof)


@lru_cache(maxsize=None)
def cayley_tensor(sig: Signature) -> np.ndarray:
    """Structure tensor C[i, j, t] = coeff of blade t in e_I e_J (algebra.py:132-145);
    fp64, read-only. The device builds the expanded filter from the same table."""
    table = product_table(sig)
    nb = sig.n_blades
    cay = np.zeros((nb, nb, nb), dtype=np.float64)
    ii, jj = np.meshgrid(np.arange(nb), np.arange(nb), indexing="ij")
    cay[ii, jj, table.target] = table.coeff
    cay.flags.writeable = False
    return cay


def geometric_product(x, y, table: BladeProductTable) -> np.ndarray:
    """Geometric product of multivector arrays over their last (blade) axis,
    broadcasting the leading axes (algebra.py:155-173): accumulated in fp64,
    rounded once to the operands' common dtype; DimensionMismatch if a blade
    axis is not N_B. Host algebra helper (like the product table): the
    layers' products run on the device.

    out[..., i ^ j] += coeff[i, j] x[..., i] y[..., j], one blade row at a time."""
    x = np.asarray(x)
    y = np.asarray(y)
    nb = table.sig.n_blades
    for name, a in (("x", x), ("y", y)):
        if a.ndim == 0 or a.shape[-1] != nb:
            raise DimensionMismatch(f"{name} has blade axis {a.shape[-1] if a.ndim else '()'}, expected {nb}")
    out_dtype = np.result_type(x.dtype, y.dtype)
    xd = x.astype(np.float64, copy=False)
    yd = y.astype(np.float64, copy=False)
    out = np.zeros(np.broadcast_shapes(x.shape, y.shape), np.float64)
    for i in range(nb):
        for j in range(nb):
            c = int(table.coeff[i, j])
            if c:
                out[..., int(table.target[i, j])] += c * xd[..., i] * yd[..., j]
    return out.astype(out_dtype, copy=False)


def schedule_terms(sig: Signature) -> int:
    """Number of non-zero FMA terms of the signature schedule (specialize.py:49-63)."""
    return int(_ops.op("schedule_terms", list(sig.g)))


def schedule_flop_count(sig_or_schedule) -> int:
    """FLOPs of one geometric product (specialize.py:72-74). Takes the
    reference's OpSchedule (`specialize.schedule_for(sig)`) or a Signature."""
    terms = getattr(sig_or_schedule, "terms", None)
    if terms is not None:
        return 2 * len(terms)
    return 2 * schedule_terms(sig_or_schedule)


def all_valid_signatures(k_max: int = 3) -> list[Signature]:
    from itertools import product as iproduct
    return [Signature(g) for k in range(1, k_max + 1)
            for g in iproduct((-1, 0, 1), repeat=k) if any(g)]
