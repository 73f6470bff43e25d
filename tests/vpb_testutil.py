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


def floored_rel(a, b, floor: float) -> float:
    """max |a-b| / max(|b|, floor * max|b|): a pointwise relative error that
    also constrains the velocity tails down to ``floor`` of the peak (where
    f ~ 1e-8 of its maximum a pure max-norm metric would allow large local
    relative errors).  Works on numpy arrays and torch tensors."""
    try:
        import torch

        if isinstance(a, torch.Tensor) or isinstance(b, torch.Tensor):
            a = torch.as_tensor(a)
            b = torch.as_tensor(b, device=a.device)
            babs = b.abs()
            den = torch.clamp(babs, min=floor * float(babs.max()))
            return float(((a - b).abs() / den).max())
    except ImportError:
        pass
    a = np.asarray(a)
    b = np.asarray(b)
    babs = np.abs(b)
    den = np.maximum(babs, floor * float(babs.max()))
    return float(np.max(np.abs(a - b) / den))


def torch_max_rel(a, b) -> float:
    """max_rel on device tensors (full-size states, no host copy)."""
    d = float((a - b).abs().max())
    s = float(b.abs().max())
    return d / (s if s > 0 else 1.0)
