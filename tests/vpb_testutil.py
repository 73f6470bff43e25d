"""Shared helpers for the test modules (imported by basename)."""

from __future__ import annotations

import numpy as np


def max_rel(a, b) -> float:
    """max|a-b| / max|b|: the north-star f-parity metric (pointwise relative
    error is ill-posed where f ~ 0)."""
    a = np.asarray(a)
    b = np.asarray(b)
    scale = float(np.max(np.abs(b)))
    return float(np.max(np.abs(a - b))) / (scale if scale > 0 else 1.0)
