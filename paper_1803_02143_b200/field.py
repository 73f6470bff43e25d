"""Device-resident distribution function and line sweeps.

Mirrors ``slvp.field`` (/root/reference/pkg/src/slvp/field.py): a
:class:`DistributionField` owns one contiguous block plus a
:class:`LayoutDescriptor`; ``field.array`` is the logical view in grid
order.  Here the block is an HBM buffer (a CUDA tensor) and the physical
order is always the reference's canonical one, ``f[v2][v1][x2][x1]`` with
x1 fastest (field.py:67-76) -- the sweep kernels read every axis in place,
so neither of the reference's two strategies needs a transpose on the GPU.
Both strategy names are accepted and produce identical storage (the
reference requires them to agree bitwise, field.py:1-18).

``line_sweep`` (field.py:236-243) drives a fast sweep kernel
(:class:`~paper_1803_02143_b200.dg.DGAdvection` or
:class:`~paper_1803_02143_b200.spline.SplineAdvection`) over every line of
one axis.  Python per-line callables are a CPU concept and are rejected.

The VLF1 snapshot format (field.py:246-295) is kept byte-compatible.
"""

from __future__ import annotations

import struct
from dataclasses import dataclass
from pathlib import Path

import numpy as np
import torch

from . import _device
from .grid import DG, SPACE, SPLINE, VELOCITY, Axis, GridSpec

TRANSPOSE = "transpose"
STRIDED = "strided"
DEFAULT_STRATEGY = {SPLINE: TRANSPOSE, DG: STRIDED}


@dataclass(frozen=True)
class LayoutDescriptor:
    """Physical order of a field (field.py:38-76).

    ``dim_order`` lists grid axes slowest to fastest; the device storage is
    always canonical (reversed grid order).
    """

    strategy: str
    dim_order: tuple[int, ...]
    strides: tuple[int, ...]
    cache_block: int = 8

    def __post_init__(self) -> None:
        if self.strategy not in (TRANSPOSE, STRIDED):
            raise ValueError(f"unknown layout strategy {self.strategy!r}")
        if sorted(self.dim_order) != list(range(len(self.dim_order))):
            raise ValueError(f"dim_order {self.dim_order} is not a permutation")
        if self.cache_block < 1:
            raise ValueError(f"cache_block must be >= 1, got {self.cache_block}")

    @classmethod
    def for_grid(cls, grid: GridSpec, strategy: str, dim_order=None, cache_block: int = 8):
        canonical = tuple(reversed(range(grid.ndim)))
        if dim_order is not None and tuple(dim_order) != canonical:
            raise ValueError(
                f"device fields are stored in canonical order {canonical}; got {tuple(dim_order)}"
            )
        strides = [0] * grid.ndim
        acc = 1
        for a in reversed(canonical):
            strides[a] = acc
            acc *= grid.dof(a)
        return cls(strategy, canonical, tuple(strides), cache_block)


def _check_strategy(grid: GridSpec, strategy: str | None) -> str:
    s = strategy or DEFAULT_STRATEGY[grid.method]
    if s not in (TRANSPOSE, STRIDED):
        raise ValueError(f"unknown layout strategy {s!r}")
    return s


class DistributionField:
    """Grid function stored as one HBM block in canonical order."""

    def __init__(self, grid: GridSpec, layout: LayoutDescriptor, phys: torch.Tensor):
        expected = tuple(grid.dof(a) for a in layout.dim_order)
        if not isinstance(phys, torch.Tensor) or not phys.is_cuda:
            raise TypeError("device fields hold a CUDA tensor")
        if tuple(phys.shape) != expected:
            raise ValueError(f"storage shape {tuple(phys.shape)} does not match layout {expected}")
        if phys.dtype != torch.float64 or not phys.is_contiguous():
            raise ValueError("field storage must be contiguous float64")
        self.grid = grid
        self.layout = layout
        self._phys = phys

    # -- construction ----------------------------------------------------
    @classmethod
    def zeros(cls, grid: GridSpec, strategy: str | None = None, cache_block: int = 8):
        layout = LayoutDescriptor.for_grid(grid, _check_strategy(grid, strategy), cache_block=cache_block)
        phys = torch.zeros(tuple(grid.dof(a) for a in layout.dim_order), dtype=torch.float64,
                           device=_device.device())
        return cls(grid, layout, phys)

    @classmethod
    def empty(cls, grid: GridSpec, strategy: str | None = None, cache_block: int = 8):
        layout = LayoutDescriptor.for_grid(grid, _check_strategy(grid, strategy), cache_block=cache_block)
        phys = torch.empty(tuple(grid.dof(a) for a in layout.dim_order), dtype=torch.float64,
                           device=_device.device())
        return cls(grid, layout, phys)

    @classmethod
    def from_values(cls, grid: GridSpec, values, strategy: str | None = None, cache_block: int = 8):
        """Build from values in logical (grid-axis) order (host array or tensor)."""
        field = cls.empty(grid, strategy, cache_block)
        if isinstance(values, torch.Tensor):
            src = values.to(device=field._phys.device, dtype=torch.float64)
        else:
            src = torch.from_numpy(np.asarray(values, dtype=np.float64)).to(field._phys.device)
        field.array[...] = src
        return field

    # -- views -----------------------------------------------------------
    @property
    def data(self) -> torch.Tensor:
        """Flat view of the storage (canonical order)."""
        return self._phys.reshape(-1)

    @property
    def array(self) -> torch.Tensor:
        """Logical view with axes in grid order (a strided CUDA tensor view)."""
        return self._phys.permute(*reversed(range(self.grid.ndim)))

    def numpy(self) -> np.ndarray:
        """Host copy in logical order."""
        return self.array.cpu().numpy()

    def copy(self) -> "DistributionField":
        return DistributionField(self.grid, self.layout, self._phys.clone())

    def _swap(self, phys: torch.Tensor) -> torch.Tensor:
        old = self._phys
        self._phys = phys
        return old


def lead_shape_of(field: DistributionField, axis: int) -> tuple[int, ...]:
    return tuple(field.grid.dof(a) for a in range(field.grid.ndim) if a != axis)


def _sweep(field: DistributionField, axis: int, kernel, consume: bool) -> DistributionField:
    """One sweep along ``axis`` (field.py:166-202) on the device."""
    grid = field.grid
    if not 0 <= axis < grid.ndim:
        raise ValueError(f"axis {axis} out of range for {grid.ndim} axes")
    if not hasattr(kernel, "run_device"):
        raise TypeError(
            "device sweeps take a DGAdvection or SplineAdvection kernel; "
            "per-line Python callables are not supported on the GPU"
        )
    other = tuple(a for a in range(grid.ndim) if a != axis)
    for a in getattr(kernel, "table_axes", ()):
        if a not in other:
            raise ValueError(f"table axis {a} is not transverse to the sweep")
    target = field if consume else field.copy()
    out = torch.empty_like(target._phys)
    kernel.run_device(grid, axis, target._phys, out, None)
    target._swap(out)
    return target


def line_sweep(field: DistributionField, axis: int, kernel) -> DistributionField:
    """Apply a sweep kernel to every line along ``axis``; input untouched."""
    return _sweep(field, axis, kernel, consume=False)


# --- VLF1 snapshots (field.py:246-295), byte-compatible ---------------------
_MAGIC = b"VLF1"
_KIND = {SPACE: 0, VELOCITY: 1}
_KIND_BACK = {0: SPACE, 1: VELOCITY}
_METHOD = {SPLINE: 0, DG: 1}
_METHOD_BACK = {0: SPLINE, 1: DG}


def write_snapshot(field: DistributionField, path) -> None:
    grid = field.grid
    head = bytearray(_MAGIC) + struct.pack("<I", grid.ndim)
    for ax in grid.axes:
        head += struct.pack("<ddIB", ax.lower, ax.upper, ax.count, _KIND[ax.kind])
    head += struct.pack("<BB", _METHOD[grid.method], grid.dg_degree)
    payload = field.data.cpu().numpy().astype("<f8", copy=False)  # canonical == VLF1 order
    target = Path(path)
    target.parent.mkdir(parents=True, exist_ok=True)
    with open(target, "wb") as fh:
        fh.write(bytes(head))
        fh.write(payload.tobytes())


def read_snapshot(path) -> DistributionField:
    blob = Path(path).read_bytes()
    if blob[:4] != _MAGIC:
        raise ValueError(f"{path}: not a VLF1 snapshot")
    (ndim,) = struct.unpack_from("<I", blob, 4)
    pos = 8
    rec = struct.calcsize("<ddIB")
    axes = []
    for _ in range(ndim):
        lo, hi, count, kind = struct.unpack_from("<ddIB", blob, pos)
        pos += rec
        axes.append(Axis(lo, hi, count, _KIND_BACK[kind]))
    mcode, degree = struct.unpack_from("<BB", blob, pos)
    pos += 2
    grid = GridSpec(tuple(axes), _METHOD_BACK[mcode], degree if mcode == 1 else 0)
    payload = np.frombuffer(blob, dtype="<f8", offset=pos)
    if payload.size != grid.total_dof:
        raise ValueError(f"{path}: payload has {payload.size} values, expected {grid.total_dof}")
    layout = LayoutDescriptor.for_grid(grid, DEFAULT_STRATEGY[grid.method])
    phys = torch.from_numpy(payload.astype(np.float64)).to(_device.device())
    return DistributionField(grid, layout, phys.reshape(tuple(grid.dof(a) for a in layout.dim_order)))
