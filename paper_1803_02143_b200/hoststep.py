"""Strang steps of a distribution function that lives in HOST memory.

The reference keeps f in host memory between steps
(/root/reference/pkg/src/slvp/field.py:79-134: a NumPy array) and its
``strang_step`` (driver.py:245-265) returns a host field.  A user who keeps
that contract with this package pays one host->device and one device->host
copy of f per step (2 x 8 B/dof over PCIe).  :func:`host_steps` pipelines
those copies against the device work block by block along v2, the
outermost axis of the canonical layout (a block of v2 rows is one
contiguous byte range of f, on the host and on the device):

    step m   H2D(b) -> opening x half step of block b
             density, field solve, v-shift tables, v1 v2 sweeps (whole f)
             closing x half step of block b -> D2H(b)
    step m+1 H2D(b) waits only for step m's D2H(b)

so the device->host copy of block b+1 (step m) and the host->device copy of
block b (step m+1) run at the same time in the two PCIe directions, and
the x passes of a block overlap the copies of the others.  x half steps are
local to one (v1, v2) plane, so the per-block x passes are the whole-field
kernels on a sub-range of planes (x2 tables offset to the block's first
v2 row); every dof sees exactly the arithmetic of :func:`strang_step` with
the density computed by its own pass (``vpb_density``), i.e. the result is
bitwise that of the step chain with the unfused density.

There is no host compute: every sweep is an sm_100a kernel.
"""

from __future__ import annotations

from dataclasses import dataclass
from functools import lru_cache

import numpy as np
import torch

from . import _device
from .dg import xplane_dg, sweep_dg
from .driver import check_steps, step_state
from .field import DistributionField
from .grid import DG, GridSpec
from .poisson import density_into, solve_into
from .spline import sweep_spline


class HostField:
    """f in pinned host memory, canonical order (VLF1 payload order,
    field.py:246-251): the host-resident counterpart of
    :class:`DistributionField`."""

    def __init__(self, grid: GridSpec, data: torch.Tensor):
        if data.is_cuda or data.dtype != torch.float64 or data.numel() != grid.total_dof:
            raise ValueError("HostField holds a host float64 tensor of grid.total_dof values")
        if not data.is_pinned():
            data = data.pin_memory()
        self.grid = grid
        self.data = data.reshape(-1)

    @classmethod
    def from_field(cls, field: DistributionField) -> "HostField":
        host = torch.empty(field.grid.total_dof, dtype=torch.float64, pin_memory=True)
        host.copy_(field.data)
        return cls(field.grid, host)

    @classmethod
    def from_values(cls, grid: GridSpec, values) -> "HostField":
        """From values in logical (grid-axis) order."""
        host = torch.empty(grid.total_dof, dtype=torch.float64, pin_memory=True)
        phys = np.asarray(values, dtype=np.float64).transpose(*reversed(range(grid.ndim)))
        host.numpy().reshape(phys.shape)[...] = phys
        return cls(grid, host)

    def logical(self) -> np.ndarray:
        """Logical-order view of the host storage (no copy)."""
        shape = tuple(reversed(self.grid.dofs))
        return self.data.numpy().reshape(shape).transpose(*reversed(range(self.grid.ndim)))

    def to_device(self) -> DistributionField:
        field = DistributionField.empty(self.grid)
        field.data.copy_(self.data)
        return field


@dataclass
class _BlockGrid:
    """A v2 block of a 2x2v grid as the device geometry the sweep entry
    points take (dims4 with nv2 replaced by the block's row count)."""

    grid: GridSpec
    rows: int

    @property
    def dims4(self):
        d = self.grid.dims4
        return (d[0], d[1], d[2], self.rows)

    @property
    def ndim(self):
        return self.grid.ndim


class _TabRows:
    """Rows [r0, r1) of x-sweep projection tables (a view, no copy)."""

    def __init__(self, t, r0: int, r1: int):
        self.order = t.order
        self.a, self.b = t.a[r0:r1], t.b[r0:r1]
        self.q, self.alpha = t.q[r0:r1], t.alpha[r0:r1]


class HostStepper:
    """Device buffers, copy streams and events of the pipelined host-field
    step for one grid (cached per grid and device)."""

    def __init__(self, grid: GridSpec, blocks: int = 16):
        self.grid = grid
        self.st = step_state(grid)
        dev = _device.device()
        n = grid.total_dof
        self.a = torch.empty(n, dtype=torch.float64, device=dev)
        # second buffer: the step state's scratch copy (driver.StepState.buf,
        # re-read at every steps() call since device-resident steps swap it
        # with their field's storage), so a host-field step needs 2 copies of
        # f on the device, not 3 (config 5: 110 GB instead of 165 GB)
        self.b = self.st.buf
        nv2 = grid.dims4[3]
        nb = max(1, min(int(blocks), nv2))
        edges = [round(i * nv2 / nb) for i in range(nb + 1)]
        self.rows = [(edges[i], edges[i + 1]) for i in range(nb) if edges[i + 1] > edges[i]]
        self.plane = grid.dims4[0] * grid.dims4[1] * grid.dims4[2]
        self.h2d = torch.cuda.Stream(device=dev)
        self.d2h = torch.cuda.Stream(device=dev)
        nb = len(self.rows)
        self.h2d_done = [torch.cuda.Event() for _ in range(nb)]
        self.d2h_done = [torch.cuda.Event() for _ in range(nb)]
        self.closed = [torch.cuda.Event() for _ in range(nb)]
        self.fused_x = self.st.fused_x
        self._bgrid = {}

    def _span(self, k: int) -> slice:
        r0, r1 = self.rows[k]
        return slice(r0 * self.plane, r1 * self.plane)

    def _bg(self, k: int) -> _BlockGrid:
        r0, r1 = self.rows[k]
        g = self._bgrid.get(r1 - r0)
        if g is None:
            g = self._bgrid[r1 - r0] = _BlockGrid(self.grid, r1 - r0)
        return g

    def _x_half(self, k: int, tau: float, fl, slot: int) -> torch.Tensor:
        """x half step of block k from ``self.a``; returns the buffer holding
        the result (``self.b`` for the fused pass, ``self.a`` for two sweeps)."""
        st, grid = self.st, self.grid
        s = self._span(k)
        r0, r1 = self.rows[k]
        bg = self._bg(k)
        if grid.method == DG:
            t1 = st.x_tables(0, tau)
            t2 = _TabRows(st.x_tables(1, tau), r0, r1)
            if self.fused_x:
                xplane_dg(bg, self.a[s], self.b[s], t1, t2, fl[slot:slot + 1],
                          fl[slot + 1:slot + 2])
                return self.b
            sweep_dg(bg, 0, self.a[s], self.b[s], t1, fl[slot:slot + 1])
            sweep_dg(bg, 1, self.b[s], self.a[s], t2, fl[slot + 1:slot + 2])
            return self.a
        v1 = st.x_tables(0, tau)
        v2 = st.x_tables(1, tau)[r0:r1]
        sweep_spline(bg, 0, self.a[s], self.b[s], v1, 0.5 * tau, grid.axes[0].h,
                     fl[slot:slot + 1])
        sweep_spline(bg, 1, self.b[s], self.a[s], v2, 0.5 * tau, grid.axes[1].h,
                     fl[slot + 1:slot + 2])
        return self.a

    def _velocity(self, src: torch.Tensor, tau: float, fl, m: int, stats) -> torch.Tensor:
        """density -> field solve -> v1, v2 sweeps of the whole field, from
        ``src``; returns the buffer holding the result."""
        st, grid = self.st, self.grid
        density_into(src, grid, st.rho)
        solve_into(st.rho, grid, st.e, stats[m], fl[2:3])
        dst = self.a if src is self.b else self.b
        if grid.method == DG:
            from .dg import vplane_dg

            t1 = st.v_tables(0, tau)
            t2 = st.v_tables(1, tau)
            if st.fused_v:
                vplane_dg(grid, src, dst, t1, t2, fl[3:4], fl[4:5])
                return dst
            sweep_dg(grid, 2, src, dst, t1, fl[3:4])
            sweep_dg(grid, 3, dst, src, t2, fl[4:5])
            return src
        h1, h2 = grid.axes[2].h, grid.axes[3].h
        sweep_spline(grid, 2, src, dst, st.v_tables(0, tau), tau, h1, fl[3:4])
        sweep_spline(grid, 3, dst, src, st.v_tables(1, tau), tau, h2, fl[4:5])
        return src

    def steps(self, host: HostField, tau: float, nsteps: int,
              first_step: int | None = None) -> None:
        """``nsteps`` Strang steps of ``host`` in place (see the module doc)."""
        if host.grid != self.grid:
            raise ValueError("host field is on another grid")
        if nsteps <= 0:
            return
        if self.grid.ndim != 4:
            raise ValueError("host_steps supports 2x2v grids")
        comp = torch.cuda.current_stream()
        st = self.st
        self.b = st.buf
        dev = self.a.device
        flags = torch.zeros((nsteps, st.flags.numel()), dtype=torch.int32, device=dev)
        stats = torch.zeros((nsteps, st.stats.numel()), dtype=torch.float64, device=dev)
        entry = torch.cuda.Event()
        entry.record(comp)
        nb = len(self.rows)
        hd = host.data
        for m in range(nsteps):
            fl = flags[m]
            # H2D of every block (after its D2H of the previous step)
            with torch.cuda.stream(self.h2d):
                for k in range(nb):
                    self.h2d.wait_event(self.d2h_done[k] if m else entry)
                    s = self._span(k)
                    self.a[s].copy_(hd[s], non_blocking=True)
                    self.h2d_done[k].record(self.h2d)
            # opening x half step, block by block as the blocks arrive
            for k in range(nb):
                comp.wait_event(self.h2d_done[k])
                out = self._x_half(k, tau, fl, 0)
            if out is self.a:
                mid = self._velocity(self.a, tau, fl, m, stats)
            else:
                mid = self._velocity(self.b, tau, fl, m, stats)
            if mid is not self.a:  # the x passes read from self.a
                self.a.copy_(mid)
            # closing x half step and D2H, block by block
            for k in range(nb):
                out = self._x_half(k, tau, fl, 5)
                self.closed[k].record(comp)
                with torch.cuda.stream(self.d2h):
                    self.d2h.wait_event(self.closed[k])
                    s = self._span(k)
                    hd[s].copy_(out[s], non_blocking=True)
                    self.d2h_done[k].record(self.d2h)
        for k in range(nb):
            comp.wait_event(self.d2h_done[k])
        check_steps(st, flags, stats, first_step, tau)


@lru_cache(maxsize=4)
def _stepper(grid: GridSpec, device_index: int, blocks: int) -> HostStepper:
    return HostStepper(grid, blocks)


def host_steps(host: HostField, tau: float, nsteps: int = 1, blocks: int = 16,
               first_step: int | None = None) -> HostField:
    """``nsteps`` Strang steps (driver.py:245-265 each) of a host-resident
    field, in place, with the PCIe copies pipelined against the device work
    (module doc).  Returns ``host``; its memory holds the state after the
    last step when the call returns."""
    stepper = _stepper(host.grid, torch.cuda.current_device(), int(blocks))
    stepper.steps(host, tau, nsteps, first_step)
    return host
