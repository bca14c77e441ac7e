"""Parity metrics of the reference harness (bench.py:74-96), re-exported so a
caller's `from mvkernels import max_rel_error` keeps working. These define
the tolerances the tests state; they are host numpy
arithmetic on results, not part of the device path."""

from __future__ import annotations

import numpy as np

from .errors import VerificationFailed


def _pair(a, b):
    a = np.asarray(a.detach().cpu().numpy() if hasattr(a, "detach") else a, dtype=np.float64)
    b = np.asarray(b.detach().cpu().numpy() if hasattr(b, "detach") else b, dtype=np.float64)
    if a.shape != b.shape:
        raise VerificationFailed(f"shape mismatch {a.shape} vs {b.shape}")
    return a, b


def max_rel_error(a, b, floor: float = 1e-2) -> float:
    """max |a - b| / (floor + max(|a|, |b|)) over all elements: relative with
    an absolute floor (the reference default 1e-2)."""
    a, b = _pair(a, b)
    if a.size == 0:
        return 0.0
    return float(np.max(np.abs(a - b) / (floor + np.maximum(np.abs(a), np.abs(b)))))


def max_abs_error(a, b) -> float:
    """max |a - b| over all elements (0 for empty arrays)."""
    a, b = _pair(a, b)
    return float(np.max(np.abs(a - b))) if a.size else 0.0
