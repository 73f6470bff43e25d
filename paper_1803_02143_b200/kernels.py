"""Line-kernel backend registry (the reference's plugin API).

Mirrors ``slvp.kernels`` (/root/reference/pkg/src/slvp/kernels.py:17-72):
four entry points taking HOST NumPy arrays with the reference's argument
meaning.  The single backend here, ``"cuda"``, copies the lines to HBM,
runs the sm_100a kernel through the C ABI and copies the result back, so a
caller of the reference's FFI can switch to it unchanged.  ``threads`` and
``block`` are accepted and ignored (CPU scheduling knobs).

Unknown backend names raise ``ValueError`` exactly like the reference
(kernels.py:42-47); there is no CPU backend to fall back to.
"""

from __future__ import annotations

import os

import numpy as np
import torch

from . import _device, _lib


def _dev(a, dtype=torch.float64):
    arr = np.ascontiguousarray(a)
    return torch.from_numpy(arr).to(device=_device.device(), dtype=dtype)


class _CudaBackend:
    """H2D -> sm_100a kernel -> D2H, per call."""

    @staticmethod
    def dg_sweep_contig(lines, idx, a, b, q, alpha, ncells, nloc, threads):
        lines = np.ascontiguousarray(lines, dtype=np.float64)
        if lines.ndim != 2:
            raise ValueError("expected a (lines, n) array")
        L, n = lines.shape
        src = _dev(lines)
        out = torch.empty_like(src)
        ta, tb = _dev(a), _dev(b)
        tq = _dev(np.asarray(q, dtype=np.int64), torch.int64)
        tal = _dev(alpha)
        ti = _dev(np.asarray(idx, dtype=np.int64), torch.int64)
        lib = _lib.load()
        _lib.check(
            lib.vpb_dg_sweep_contig(src.data_ptr(), out.data_ptr(), L, n, ti.data_ptr(),
                                    ta.data_ptr(), tb.data_ptr(), tq.data_ptr(), tal.data_ptr(),
                                    int(tq.numel()), int(ncells), int(nloc), _device.stream()),
            "dg_sweep_contig",
        )
        return out.cpu().numpy()

    @staticmethod
    def dg_sweep_strided(view, idx, a, b, q, alpha, ncells, nloc, block, threads):
        n = view.shape[-1]
        out = _CudaBackend.dg_sweep_contig(
            np.ascontiguousarray(view).reshape(-1, n), idx, a, b, q, alpha, ncells, nloc, threads
        )
        view[...] = out.reshape(view.shape)

    @staticmethod
    def spline_sweep_contig(lines, idx, table, h, threads):
        lines = np.ascontiguousarray(lines, dtype=np.float64)
        if lines.ndim != 2:
            raise ValueError("expected a (lines, n) array")
        L, n = lines.shape
        src = _dev(lines)
        out = torch.empty_like(src)
        tt = _dev(np.asarray(table, dtype=np.float64))
        ti = _dev(np.asarray(idx, dtype=np.int64), torch.int64)
        lib = _lib.load()
        _lib.check(
            lib.vpb_spline_sweep_contig(src.data_ptr(), out.data_ptr(), L, n, ti.data_ptr(),
                                        tt.data_ptr(), int(tt.numel()), float(h),
                                        _device.stream()),
            "spline_sweep_contig",
        )
        return out.cpu().numpy()

    @staticmethod
    def spline_sweep_strided(view, idx, table, h, block, threads):
        n = view.shape[-1]
        out = _CudaBackend.spline_sweep_contig(
            np.ascontiguousarray(view).reshape(-1, n), idx, table, h, threads
        )
        view[...] = out.reshape(view.shape)


_BACKENDS = {"cuda": _CudaBackend}

_forced = os.environ.get("SLVP_BACKEND", "").strip().lower()
if _forced and _forced not in _BACKENDS:
    raise RuntimeError(f"SLVP_BACKEND must be one of {sorted(_BACKENDS)}, got {_forced!r}")
_active_name = _forced or "cuda"


def backend_name() -> str:
    return _active_name


def available_backends() -> tuple[str, ...]:
    return tuple(sorted(_BACKENDS))


def set_backend(name: str) -> None:
    global _active_name
    if name not in _BACKENDS:
        raise ValueError(f"unknown backend {name!r}; built: {sorted(_BACKENDS)}")
    _active_name = name


def spline_sweep_contig(lines, idx, table, h, threads):
    return _BACKENDS[_active_name].spline_sweep_contig(lines, idx, table, h, threads)


def spline_sweep_strided(view, idx, table, h, block, threads):
    return _BACKENDS[_active_name].spline_sweep_strided(view, idx, table, h, block, threads)


def dg_sweep_contig(lines, idx, a, b, q, alpha, ncells, nloc, threads):
    return _BACKENDS[_active_name].dg_sweep_contig(lines, idx, a, b, q, alpha, ncells, nloc,
                                                   threads)


def dg_sweep_strided(view, idx, a, b, q, alpha, ncells, nloc, block, threads):
    return _BACKENDS[_active_name].dg_sweep_strided(view, idx, a, b, q, alpha, ncells, nloc,
                                                    block, threads)
