"""Signature-specialised FMA schedules (host side of specialize.py:24-74).

The schedule is the flat list of non-zero terms of the blade product table
(zero-metric terms dropped, signs folded into `negate`). On the B200 it is not
turned into generated CPU source: the same table drives the on-device kernel
construction (expand.cu), whose structurally zero blocks are exactly the
dropped terms, and `schedule_flop_count` defines the algorithmic FLOPs every
roofline number in this repo is quoted on.
"""

from __future__ import annotations

from dataclasses import dataclass
from functools import lru_cache

from .algebra import BladeProductTable, Signature, product_table, schedule_flop_count  # noqa: F401


@dataclass(frozen=True)
class FmaTerm:
    """out[out_blade] -+= a[a_blade] * b[b_blade] (specialize.py:24-31)."""

    out_blade: int
    a_blade: int
    b_blade: int
    negate: bool


@dataclass(frozen=True)
class OpSchedule:
    """Terms grouped by output blade, then a-operand blade, both ascending (specialize.py:34-46)."""

    sig: Signature
    terms: tuple[FmaTerm, ...]

    def __len__(self) -> int:
        return len(self.terms)


def build_schedule(table: BladeProductTable) -> OpSchedule:
    """One term per non-zero table entry; b = out xor a (specialize.py:49-63)."""
    nb = table.sig.n_blades
    terms = []
    for out in range(nb):
        for a in range(nb):
            b = out ^ a
            c = int(table.coeff[a, b])
            if c != 0:
                terms.append(FmaTerm(out, a, b, c < 0))
    return OpSchedule(table.sig, tuple(terms))


@lru_cache(maxsize=None)
def schedule_for(sig: Signature) -> OpSchedule:
    """Cached schedule of a signature (specialize.py:66-69)."""
    return build_schedule(product_table(sig))


def schedule_to_text(s: OpSchedule) -> str:
    """`out[t] += a[i] * b[j]` lines (specialize.py:104-118, index form)."""
    return "\n".join(f"out[{t.out_blade}] {'-=' if t.negate else '+='} a[{t.a_blade}] * b[{t.b_blade}]"
                     for t in s.terms)
