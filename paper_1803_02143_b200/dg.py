"""Semi-Lagrangian discontinuous Galerkin advection on the device.

Mirrors ``slvp.dg`` (/root/reference/pkg/src/slvp/dg.py).  A shift
``s/h = q + alpha`` (alpha in [0, 1)) maps output cell ``i`` onto source
cells ``i-q-1`` and ``i-q`` through two (degree+1)^2 matrices; the
matrices are generated on the GPU (``vpb_dg_tables``) and the sweep runs in
``vpb_dg_sweep_axis`` / ``vpb_dg_sweep_contig``.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _device, _lib
from .grid import gauss_nodes  # noqa: F401  (re-exported, reference API)


@dataclass(frozen=True)
class ProjectionPair:
    """Update matrices for one constant shift (dg.py:85-96)."""

    a: np.ndarray
    b: np.ndarray
    cell_offset: int
    alpha: float


class DeviceTables:
    """Projection tables (A, B, q, alpha) resident in HBM."""

    def __init__(self, values: torch.Tensor, scale: float, h: float, degree: int):
        if h <= 0.0:
            raise ValueError(f"cell width must be positive, got {h}")
        if not 0 <= degree <= 8:
            raise ValueError(f"degree must be in [0, 8], got {degree}")
        p = degree + 1
        n = int(values.numel())
        dev = _device.device()
        self.order = p
        self.n = n
        self.a = torch.empty((n, p, p), dtype=torch.float64, device=dev)
        self.b = torch.empty((n, p, p), dtype=torch.float64, device=dev)
        self.q = torch.empty(n, dtype=torch.int64, device=dev)
        self.alpha = torch.empty(n, dtype=torch.float64, device=dev)
        self._k = None
        self.refresh(values, scale, h)

    def refresh(self, values: torch.Tensor, scale: float, h: float) -> None:
        """Regenerate in place from ``shift = values*scale`` (same length)."""
        lib = _lib.load()
        _lib.check(
            lib.vpb_dg_tables(values.data_ptr(), self.n, float(scale), float(h), self.order,
                              self.a.data_ptr(), self.b.data_ptr(), self.q.data_ptr(),
                              self.alpha.data_ptr(), _device.stream()),
            "vpb_dg_tables",
        )
        if self._k is not None:
            self._compose()

    def composed(self) -> torch.Tensor:
        """Two same-table sweeps as one three-cell stencil, per row:
        ``[AA, AB+BA, BB]`` (n, 3, p, p), for the merged x half steps of the
        "fast" arithmetic mode (``vpb_dg_sweep_xcomp``)."""
        if self._k is None:
            p = self.order
            self._k = torch.empty((self.n, 3, p, p), dtype=torch.float64, device=self.a.device)
            self._compose()
        return self._k

    def _compose(self) -> None:
        lib = _lib.load()
        _lib.check(
            lib.vpb_dg_compose_tables(self.a.data_ptr(), self.b.data_ptr(), self.n, self.order,
                                      self._k.data_ptr(), _device.stream()),
            "vpb_dg_compose_tables",
        )


def projection_pairs(shifts, h: float, degree: int):
    """Batch of update matrices (dg.py:99-152); returns host arrays."""
    if h <= 0.0:
        raise ValueError(f"cell width must be positive, got {h}")
    if not 0 <= degree <= 8:
        raise ValueError(f"degree must be in [0, 8], got {degree}")
    vals = _device.to_device(np.ascontiguousarray(np.asarray(shifts, dtype=float).ravel()))
    t = DeviceTables(vals, 1.0, h, degree)
    return t.a.cpu().numpy(), t.b.cpu().numpy(), t.q.cpu().numpy(), t.alpha.cpu().numpy()


def projection_pair(shift: float, h: float, degree: int) -> ProjectionPair:
    a, b, q, alpha = projection_pairs(np.array([shift]), h, degree)
    return ProjectionPair(a=a[0], b=b[0], cell_offset=int(q[0]), alpha=float(alpha[0]))


def advect_line_dg(line, shift: float, h: float, degree: int) -> np.ndarray:
    """Advect one periodic dG line by a constant shift (dg.py:161-175)."""
    line = np.ascontiguousarray(line, dtype=float)
    p = degree + 1
    if line.ndim != 1 or line.size % p:
        raise ValueError(f"line length {line.size} is not a multiple of {p}")
    src = _device.to_device(line)
    t = DeviceTables(_device.to_device(np.array([float(shift)])), 1.0, h, degree)
    out = torch.empty_like(src)
    idx = torch.zeros(1, dtype=torch.int64, device=src.device)
    lib = _lib.load()
    _lib.check(
        lib.vpb_dg_sweep_contig(src.data_ptr(), out.data_ptr(), 1, line.size, idx.data_ptr(),
                                t.a.data_ptr(), t.b.data_ptr(), t.q.data_ptr(),
                                t.alpha.data_ptr(), 1, line.size // p, p, _device.stream()),
        "vpb_dg_sweep_contig",
    )
    return out.cpu().numpy()


# ---------------------------------------------------------------------------
# Table layout: which transverse axes index a sweep's table on the device.
# ---------------------------------------------------------------------------
def device_axis(grid, axis: int) -> int:
    """Grid axis -> axis of the 4-D device geometry (1x1v grids skip x2/v2)."""
    if grid.ndim == 4:
        return axis
    return (0, 2)[axis]


def device_table_axes(grid, axis: int) -> tuple[int, ...]:
    """Grid axes whose index selects the table row on the device, slowest
    first (row-major).  x sweeps: the matching velocity axis; v sweeps:
    (x2, x1), i.e. row = ix2*n1 + ix1."""
    if grid.ndim == 4:
        return {0: (2,), 1: (3,), 2: (1, 0), 3: (1, 0)}[axis]
    return {0: (1,), 1: (0,)}[axis]


def reorder_table(grid, axis: int, table: np.ndarray, table_axes: tuple[int, ...]) -> np.ndarray:
    """Re-index a reference-order shift table (row-major over ``table_axes``,
    field.py:137-157) into the device order for ``axis``."""
    want = device_table_axes(grid, axis)
    for a in table_axes:
        if a not in want:
            raise ValueError(
                f"shift table over axes {table_axes} is not supported for a sweep along "
                f"axis {axis} (device tables index axes {want})"
            )
    sizes = [grid.dof(a) for a in want]
    coords = np.meshgrid(*[np.arange(s) for s in sizes], indexing="ij")
    ref_idx = np.zeros(sizes, dtype=np.int64)
    mult = 1
    for a in reversed(table_axes):
        ref_idx += mult * coords[want.index(a)]
        mult *= grid.dof(a)
    table = np.asarray(table, dtype=float).ravel()
    if table.size != mult:
        raise ValueError(f"shift table has {table.size} entries, expected {mult}")
    return table[ref_idx.ravel()]


class DGAdvection:
    """Sweep kernel advecting dG lines by table-driven shifts (dg.py:178-209).

    ``shift_table`` is indexed row-major over ``table_axes`` exactly as in
    the reference; it is re-indexed to the device order on first use for a
    given sweep axis.
    """

    def __init__(self, shift_table, table_axes, h: float, degree: int, workers: int = 1):
        self.table_axes = tuple(table_axes)
        self.h = float(h)
        self.degree = int(degree)
        self.workers = int(workers)
        if self.h <= 0.0:
            raise ValueError(f"cell width must be positive, got {h}")
        if not 0 <= self.degree <= 8:
            raise ValueError(f"degree must be in [0, 8], got {degree}")
        self._table = np.ascontiguousarray(np.asarray(shift_table, dtype=float).ravel())
        self._dev: dict[int, DeviceTables] = {}

    def tables_for(self, grid, axis: int) -> DeviceTables:
        if axis not in self._dev:
            vals = reorder_table(grid, axis, self._table, self.table_axes)
            self._dev[axis] = DeviceTables(_device.to_device(vals), 1.0, self.h, self.degree)
        return self._dev[axis]

    def run_device(self, grid, axis: int, src: torch.Tensor, dst: torch.Tensor, flag) -> None:
        t = self.tables_for(grid, axis)
        if grid.dg_degree != self.degree:
            raise ValueError("kernel degree does not match the grid")
        sweep_dg(grid, axis, src, dst, t, flag)


def sweep_dg(grid, axis: int, src: torch.Tensor, dst: torch.Tensor, t: DeviceTables,
             flag: torch.Tensor | None) -> None:
    lib = _lib.load()
    _lib.check(
        lib.vpb_dg_sweep_axis(device_axis(grid, axis), src.data_ptr(), dst.data_ptr(),
                              _lib.dims(grid.dims4), t.order, t.a.data_ptr(), t.b.data_ptr(),
                              t.q.data_ptr(), t.alpha.data_ptr(),
                              None if flag is None else flag.data_ptr(), _device.stream()),
        "vpb_dg_sweep_axis",
    )


def xplane_dg(grid, src: torch.Tensor, dst: torch.Tensor, t1: DeviceTables, t2: DeviceTables,
              flag1: torch.Tensor | None, flag2: torch.Tensor | None) -> None:
    """x1 then x2 sweep of a 2x2v field in one pass (``vpb_dg_sweep_xplane``)."""
    lib = _lib.load()
    _lib.check(
        lib.vpb_dg_sweep_xplane(src.data_ptr(), dst.data_ptr(), _lib.dims(grid.dims4), t1.order,
                                t1.a.data_ptr(), t1.b.data_ptr(), t1.q.data_ptr(),
                                t1.alpha.data_ptr(), t2.a.data_ptr(), t2.b.data_ptr(),
                                t2.q.data_ptr(), t2.alpha.data_ptr(),
                                None if flag1 is None else flag1.data_ptr(),
                                None if flag2 is None else flag2.data_ptr(), _device.stream()),
        "vpb_dg_sweep_xplane",
    )


def xplane2_dg(grid, src: torch.Tensor, dst: torch.Tensor, t1: DeviceTables, t2: DeviceTables,
               flags_a, flags_b) -> None:
    """Two consecutive x half steps (x1 x2 x1 x2, same tables) in one pass
    (``vpb_dg_sweep_xplane2``); ``flags_a`` / ``flags_b``: the (x1, x2) flag
    words of the first / second half step (or None)."""
    lib = _lib.load()
    fa = [None, None] if flags_a is None else [f.data_ptr() for f in flags_a]
    fb = [None, None] if flags_b is None else [f.data_ptr() for f in flags_b]
    _lib.check(
        lib.vpb_dg_sweep_xplane2(src.data_ptr(), dst.data_ptr(), _lib.dims(grid.dims4), t1.order,
                                 t1.a.data_ptr(), t1.b.data_ptr(), t1.q.data_ptr(),
                                 t1.alpha.data_ptr(), t2.a.data_ptr(), t2.b.data_ptr(),
                                 t2.q.data_ptr(), t2.alpha.data_ptr(), fa[0], fa[1], fb[0], fb[1],
                                 _device.stream()),
        "vpb_dg_sweep_xplane2",
    )


def xcomp_dg(grid, src: torch.Tensor, dst: torch.Tensor, t1: DeviceTables, t2: DeviceTables,
             flag: torch.Tensor | None) -> None:
    """Two consecutive x half steps (same tables) in one pass with composed
    three-cell stencils (``vpb_dg_sweep_xcomp``; equal to
    :func:`xplane2_dg` up to round-off).  ``flag``: any non-finite output."""
    lib = _lib.load()
    _lib.check(
        lib.vpb_dg_sweep_xcomp(src.data_ptr(), dst.data_ptr(), _lib.dims(grid.dims4), t1.order,
                               t1.composed().data_ptr(), t1.q.data_ptr(), t1.alpha.data_ptr(),
                               t2.composed().data_ptr(), t2.q.data_ptr(), t2.alpha.data_ptr(),
                               None if flag is None else flag.data_ptr(), _device.stream()),
        "vpb_dg_sweep_xcomp",
    )


def vplane_dg(grid, src: torch.Tensor, dst: torch.Tensor, t1: DeviceTables, t2: DeviceTables,
              flag1: torch.Tensor | None, flag2: torch.Tensor | None) -> None:
    """v1 then v2 sweep of a 2x2v field in one pass (``vpb_dg_sweep_vplane``)."""
    lib = _lib.load()
    _lib.check(
        lib.vpb_dg_sweep_vplane(src.data_ptr(), dst.data_ptr(), _lib.dims(grid.dims4), t1.order,
                                t1.a.data_ptr(), t1.b.data_ptr(), t1.q.data_ptr(),
                                t1.alpha.data_ptr(), t2.a.data_ptr(), t2.b.data_ptr(),
                                t2.q.data_ptr(), t2.alpha.data_ptr(),
                                None if flag1 is None else flag1.data_ptr(),
                                None if flag2 is None else flag2.data_ptr(), _device.stream()),
        "vpb_dg_sweep_vplane",
    )
