"""Device plumbing: PyTorch supplies CUDA memory and streams, nothing else."""

from __future__ import annotations

import numpy as np
import torch

from . import _lib


def device() -> torch.device:
    """The CUDA device of the calling process; raises when there is none."""
    if not torch.cuda.is_available():
        raise _lib.VpbError(
            "vpb200 needs a CUDA device (B200, sm_100a); this build has no CPU fallback"
        )
    _lib.load()
    return torch.device("cuda", torch.cuda.current_device())


def stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def ptr(t) -> int | None:
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError("expected a CUDA tensor")
    return t.data_ptr()


def to_device(a, dtype=torch.float64) -> torch.Tensor:
    """Host array (or tensor) -> contiguous CUDA tensor."""
    if isinstance(a, torch.Tensor):
        return a.to(device=device(), dtype=dtype).contiguous()
    arr = np.ascontiguousarray(np.asarray(a))
    return torch.from_numpy(arr).to(device=device(), dtype=dtype)


def empty(n: int, dtype=torch.float64) -> torch.Tensor:
    return torch.empty(int(n), dtype=dtype, device=device())
