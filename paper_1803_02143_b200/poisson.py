"""Charge density, spectral field solve and electric energy on the device.

Mirrors ``slvp.poisson`` (/root/reference/pkg/src/slvp/poisson.py):

* density  rho(x) = sum_v f w_v1 w_v2                          (poisson.py:85-95)
* dG grids collapse rho to cell centres with the Lagrange weights at xi=1/2
  along each space axis, transform, divide by |k|^2 (k=0 dropped), form
  E_d = -i k_d phi (even-count Nyquist k zeroed), and evaluate the
  trigonometric interpolant back at the Gauss nodes     (poisson.py:106-196)
* spline grids transform and inverse-transform on the points.

On the GPU every transform is a dense complex matrix product; the matrices
(G = DFT o collapse, M = node evaluation, K_d = -i k_d/|k|^2) are built
once per grid on the host and uploaded, then ``vpb_field_solve`` chains
four small complex GEMMs.  The neutrality warning (poisson.py:143-160) is
raised from a device-computed weighted mean.
"""

from __future__ import annotations

import warnings
from dataclasses import dataclass
from functools import lru_cache

import numpy as np
import torch

from . import _device, _lib
from .grid import DG, GridSpec, gauss_nodes


def _lagrange_row(nodes: np.ndarray, x: float) -> np.ndarray:
    """Lagrange basis on ``nodes`` evaluated at ``x`` (product form)."""
    out = np.empty(nodes.size)
    for j in range(nodes.size):
        num = 1.0
        den = 1.0
        for k in range(nodes.size):
            if k != j:
                num *= x - nodes[k]
                den *= nodes[j] - nodes[k]
        out[j] = num / den
    return out


def _dft_matrix(count: int, sign: float) -> np.ndarray:
    """exp(sign*2*pi*i*(j*k mod count)/count), argument reduced for accuracy."""
    j = np.arange(count)
    phase = (np.outer(j, j) % count) / count
    return np.exp(sign * 2j * np.pi * phase)


@dataclass
class FieldGeometry:
    """Host-built transform matrices for one grid, resident on the device."""

    grid: GridSpec
    n1: int
    n2: int
    c1: int
    c2: int
    ncomp: int
    tensors: dict
    struct: _lib.FieldGeom
    struct_c: _lib.FieldGeom | None = None  # cell-centre input variant (dG)
    volume: float = 0.0

    @property
    def work_len(self) -> int:
        return int(_lib.load().vpb_field_work_len(self.struct))


def _axis_mats(grid: GridSpec, axis: int):
    """(G [c x n], M [n x c], k-vector, count) for one space axis."""
    ax = grid.axes[axis]
    count = ax.count
    if grid.method == DG:
        p = grid.dg_degree + 1
        nodes, _ = gauss_nodes(p)
        mid = _lagrange_row(nodes, 0.5)
        fwd = _dft_matrix(count, -1.0)
        g = (fwd[:, :, None] * mid[None, None, :]).reshape(count, count * p)
        offsets = (np.arange(count)[:, None] + nodes[None, :] - 0.5).ravel()
        modes = np.fft.fftfreq(count) * count
        m = np.exp(2j * np.pi * np.outer(offsets, modes) / count) / count
    else:
        g = _dft_matrix(count, -1.0)
        m = _dft_matrix(count, 1.0) / count
    kvec = 2.0 * np.pi * np.fft.fftfreq(count, d=ax.h)
    return g, m, kvec, count


@lru_cache(maxsize=32)
def field_geometry(grid: GridSpec, device_index: int) -> FieldGeometry:
    g1, m1, k1, c1 = _axis_mats(grid, 0)
    if grid.ndim_x == 2:
        g2, m2, k2, c2 = _axis_mats(grid, 1)
    else:
        g2 = np.ones((1, 1), dtype=complex)
        m2 = np.ones((1, 1), dtype=complex)
        k2 = np.zeros(1)
        c2 = 1
    ksq = k1[:, None] ** 2 + k2[None, :] ** 2
    inv = np.zeros_like(ksq)
    np.divide(1.0, ksq, out=inv, where=ksq > 0.0)
    kd = []
    for kv, count in ((k1, c1), (k2, c2)):
        kv = kv.copy()
        if count % 2 == 0:
            kv[count // 2] = 0.0
        kd.append(kv)
    comps = [(-1j * kd[0][:, None]) * inv]
    if grid.ndim_x == 2:
        comps.append((-1j * kd[1][None, :]) * inv)
    kmul = np.stack(comps)

    dev = _device.device()

    def cplx(a):
        t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.complex128)).to(dev)
        return t

    wx1 = grid.axis_weights(0)
    wx2 = grid.axis_weights(1) if grid.ndim_x == 2 else np.ones(1)
    volume = 1.0
    for a in grid.space_axes:
        volume *= grid.axes[a].upper - grid.axes[a].lower
    tensors = {
        "g1": cplx(g1), "g2": cplx(g2), "m1": cplx(m1), "m2": cplx(m2), "kmul": cplx(kmul),
        "wx1": _device.to_device(wx1), "wx2": _device.to_device(wx2),
        # product weights in device layout [x2][x1]
        "wx": _device.to_device((wx2[:, None] * wx1[None, :]).ravel()),
    }
    n1 = grid.dof(0)
    n2 = grid.dof(1) if grid.ndim_x == 2 else 1
    st = _lib.FieldGeom(
        n1, n2, c1, c2, len(comps),
        tensors["g1"].data_ptr(), tensors["g2"].data_ptr(), tensors["m1"].data_ptr(),
        tensors["m2"].data_ptr(), tensors["kmul"].data_ptr(), tensors["wx1"].data_ptr(),
        tensors["wx2"].data_ptr(), volume, 0, 0,
    )
    geo = FieldGeometry(grid, n1, n2, c1, c2, len(comps), tensors, st)
    geo.volume = volume
    if grid.method == DG and grid.ndim_x == 2:
        # same solve fed with the density already collapsed to cell centres
        # (produced by the fused x-plane pass): G = plain DFT on the C grid
        nodes, _ = gauss_nodes(grid.dg_degree + 1)
        tensors["f1"] = cplx(_dft_matrix(c1, -1.0))
        tensors["f2"] = cplx(_dft_matrix(c2, -1.0))
        tensors["mid"] = _device.to_device(_lagrange_row(nodes, 0.5))
        geo.struct_c = _lib.FieldGeom(
            n1, n2, c1, c2, len(comps),
            tensors["f1"].data_ptr(), tensors["f2"].data_ptr(), tensors["m1"].data_ptr(),
            tensors["m2"].data_ptr(), tensors["kmul"].data_ptr(), tensors["wx1"].data_ptr(),
            tensors["wx2"].data_ptr(), volume, c1, c2,
        )
    return geo


def geometry(grid: GridSpec) -> FieldGeometry:
    return field_geometry(grid, torch.cuda.current_device())


# ---------------------------------------------------------------------------
# Public API (poisson.py)
# ---------------------------------------------------------------------------
@dataclass(frozen=True)
class DensityField:
    """Spatial density; ``values`` has logical shape (dof(x1)[, dof(x2)])."""

    grid: GridSpec
    values: object  # torch CUDA tensor view or host array


@dataclass(frozen=True)
class ElectricField:
    """Per-direction field components on the spatial dof grid."""

    grid: GridSpec
    components: tuple


def _logical_x(grid: GridSpec, flat: torch.Tensor):
    """Device [x2][x1] buffer -> logical (n1, n2) (or (n1,)) view."""
    if grid.ndim_x == 1:
        return flat
    return flat.view(grid.dof(1), grid.dof(0)).t()


def _device_x(grid: GridSpec, values) -> torch.Tensor:
    """Logical (n1, n2) values -> contiguous device [x2][x1] buffer."""
    if isinstance(values, torch.Tensor):
        t = values.to(device=_device.device(), dtype=torch.float64)
    else:
        t = torch.from_numpy(np.asarray(values, dtype=np.float64)).to(_device.device())
    if grid.ndim_x == 2:
        t = t.t()
    return t.contiguous().reshape(-1)


class _Scratch:
    """Per-grid device work buffers (density partials, transform scratch)."""

    def __init__(self, grid: GridSpec):
        lib = _lib.load()
        d = _lib.dims(grid.dims4)
        self.wv1 = _device.to_device(grid.axis_weights(grid.ndim_x))
        self.wv2 = _device.to_device(grid.axis_weights(3) if grid.ndim == 4 else np.ones(1))
        self.dens_work = _device.empty(lib.vpb_density_work_len(d))
        self.geom = geometry(grid)
        self.field_work = _device.empty(self.geom.work_len)
        self.stats = _device.empty(4)


@lru_cache(maxsize=32)
def _scratch_cached(grid: GridSpec, device_index: int) -> _Scratch:
    return _Scratch(grid)


def scratch(grid: GridSpec) -> _Scratch:
    return _scratch_cached(grid, torch.cuda.current_device())


def density_into(field_data: torch.Tensor, grid: GridSpec, rho: torch.Tensor) -> None:
    s = scratch(grid)
    lib = _lib.load()
    _lib.check(
        lib.vpb_density(field_data.data_ptr(), _lib.dims(grid.dims4), s.wv1.data_ptr(),
                        s.wv2.data_ptr(), rho.data_ptr(), s.dens_work.data_ptr(),
                        _device.stream()),
        "vpb_density",
    )


def solve_into(rho: torch.Tensor, grid: GridSpec, e: torch.Tensor, stats, flag,
               centred: bool = False) -> None:
    """Field from a nodal density, or (``centred``) from the density already
    collapsed to cell centres by the fused x-plane pass."""
    s = scratch(grid)
    lib = _lib.load()
    geo = s.geom.struct_c if centred else s.geom.struct
    _lib.check(
        lib.vpb_field_solve(rho.data_ptr(), geo, e.data_ptr(),
                            None if stats is None else stats.data_ptr(),
                            s.field_work.data_ptr(), None if flag is None else flag.data_ptr(),
                            _device.stream()),
        "vpb_field_solve",
    )


def compute_density(field) -> DensityField:
    grid = field.grid
    rho = _device.empty(grid.dims4[0] * grid.dims4[1])
    density_into(field.data, grid, rho)
    return DensityField(grid, _logical_x(grid, rho))


def _warn_if_not_neutral(mean: float) -> None:
    if abs(mean - 1.0) > 1e-3:
        warnings.warn(
            f"density mean {mean:.9g} deviates from the unit background; "
            "the k=0 mode is dropped regardless",
            RuntimeWarning,
            stacklevel=3,
        )


def solve_poisson(density: DensityField, dft=None) -> ElectricField:
    """Field from a density.  ``dft`` is accepted for API compatibility; the
    device transforms are always the dense (DirectDFT-equivalent) ones."""
    grid = density.grid
    rho = _device_x(grid, density.values)
    geom = geometry(grid)
    e = _device.empty(geom.ncomp * geom.n1 * geom.n2)
    stats = _device.empty(1)
    solve_into(rho, grid, e, stats, None)
    _warn_if_not_neutral(float(stats.cpu()[0]))
    nx = geom.n1 * geom.n2
    comps = tuple(_logical_x(grid, e[d * nx:(d + 1) * nx]) for d in range(geom.ncomp))
    return ElectricField(grid, comps)


def electric_energy(efield: ElectricField) -> float:
    """0.5 * integral of |E|^2 over space (poisson.py:199-217)."""
    grid = efield.grid
    geom = geometry(grid)
    e = torch.cat([_device_x(grid, c) for c in efield.components])
    out = _device.empty(1)
    lib = _lib.load()
    _lib.check(
        lib.vpb_electric_energy(e.data_ptr(), len(efield.components), geom.n1 * geom.n2,
                                geom.tensors["wx"].data_ptr(), out.data_ptr(), _device.stream()),
        "vpb_electric_energy",
    )
    return float(out.cpu()[0])


__all__ = [
    "DensityField",
    "ElectricField",
    "compute_density",
    "solve_poisson",
    "electric_energy",
]
