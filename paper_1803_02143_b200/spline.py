"""Semi-Lagrangian cubic-spline advection on the device.

Mirrors ``slvp.spline`` (/root/reference/pkg/src/slvp/spline.py): each line
is interpolated by a periodic cubic B-spline (cyclic (1,4,1)/6 solve) and
evaluated at the foot points.  The solve and evaluation run in
``vpb_spline_sweep_axis`` / ``vpb_spline_sweep_contig`` and reproduce the
reference's compiled kernel operation for operation.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _device, _lib
from .dg import device_axis, reorder_table


def bspline_kernel(x, h: float) -> np.ndarray:
    """Centred cubic B-spline, support [-2h, 2h] (spline.py:20-36)."""
    if h <= 0.0:
        raise ValueError(f"spacing must be positive, got {h}")
    t = np.abs(np.asarray(x, dtype=float) / h)
    out = np.zeros_like(t)
    near = t <= 1.0
    far = ~near & (t <= 2.0)
    tn = t[near]
    out[near] = (4.0 - 6.0 * tn * tn + 3.0 * tn * tn * tn) / 6.0
    tf = 2.0 - t[far]
    out[far] = tf * tf * tf / 6.0
    return out


def advect_line_spline(line, shift: float, h: float) -> np.ndarray:
    """output_i = spline(line)(x_i - shift) for one periodic line (spline.py:81-88)."""
    line = np.ascontiguousarray(line, dtype=float)
    if line.ndim != 1 or line.size < 4:
        raise ValueError("line must be 1D with at least 4 samples")
    src = _device.to_device(line)
    out = torch.empty_like(src)
    idx = torch.zeros(1, dtype=torch.int64, device=src.device)
    table = _device.to_device(np.array([float(shift)]))
    lib = _lib.load()
    _lib.check(
        lib.vpb_spline_sweep_contig(src.data_ptr(), out.data_ptr(), 1, line.size, idx.data_ptr(),
                                    table.data_ptr(), 1, float(h), _device.stream()),
        "vpb_spline_sweep_contig",
    )
    return out.cpu().numpy()


class SplineAdvection:
    """Sweep kernel advecting spline lines by table-driven shifts (spline.py:91-110)."""

    def __init__(self, shift_table, table_axes, h: float, workers: int = 1):
        self.table_axes = tuple(table_axes)
        self.h = float(h)
        self.workers = int(workers)
        if self.h <= 0.0:
            raise ValueError(f"spacing must be positive, got {h}")
        self.table = np.ascontiguousarray(np.asarray(shift_table, dtype=float).ravel())
        self._dev: dict[int, torch.Tensor] = {}

    def run_device(self, grid, axis: int, src: torch.Tensor, dst: torch.Tensor, flag) -> None:
        if axis not in self._dev:
            self._dev[axis] = _device.to_device(reorder_table(grid, axis, self.table, self.table_axes))
        sweep_spline(grid, axis, src, dst, self._dev[axis], 1.0, self.h, flag)


def sweep_spline(grid, axis: int, src: torch.Tensor, dst: torch.Tensor, values: torch.Tensor,
                 scale: float, h: float, flag: torch.Tensor | None) -> None:
    lib = _lib.load()
    _lib.check(
        lib.vpb_spline_sweep_axis(device_axis(grid, axis), src.data_ptr(), dst.data_ptr(),
                                  _lib.dims(grid.dims4), values.data_ptr(), float(scale),
                                  float(h), None if flag is None else flag.data_ptr(),
                                  _device.stream()),
        "vpb_spline_sweep_axis",
    )


def sweep_spline2(grid, axis: int, src: torch.Tensor, dst: torch.Tensor, values: torch.Tensor,
                  scale: float, h: float, flag: torch.Tensor | None) -> None:
    """Two consecutive sweeps with the same shifts in one pass
    (``vpb_spline_sweep_axis2``; equal to two :func:`sweep_spline` calls up
    to round-off)."""
    lib = _lib.load()
    _lib.check(
        lib.vpb_spline_sweep_axis2(device_axis(grid, axis), src.data_ptr(), dst.data_ptr(),
                                   _lib.dims(grid.dims4), values.data_ptr(), float(scale),
                                   float(h), None if flag is None else flag.data_ptr(),
                                   _device.stream()),
        "vpb_spline_sweep_axis2",
    )


def sweep_spline2_density(grid, src: torch.Tensor, dst: torch.Tensor, values: torch.Tensor,
                          scale: float, h: float, flag: torch.Tensor | None, wv1: torch.Tensor,
                          part: torch.Tensor) -> None:
    """The x1 double sweep of :func:`sweep_spline2` with the density of its
    output as an epilogue (``vpb_spline_sweep_x1dbl_density``): ``part``
    receives per (v2, 32-row v1 block) partial sums of ``out * wv1``."""
    lib = _lib.load()
    _lib.check(
        lib.vpb_spline_sweep_x1dbl_density(src.data_ptr(), dst.data_ptr(), _lib.dims(grid.dims4),
                                           values.data_ptr(), float(scale), float(h),
                                           None if flag is None else flag.data_ptr(),
                                           wv1.data_ptr(), part.data_ptr(), _device.stream()),
        "vpb_spline_sweep_x1dbl_density",
    )


def double_sweep_ok(grid, axis: int) -> bool:
    """Whether :func:`sweep_spline2` supports this axis of the grid."""
    n = grid.dof(axis)
    return n % 16 == 0 and n >= 32
