"""Time integration on the device: problems, initial data, Strang step, run loop.

Mirrors ``slvp.driver`` (/root/reference/pkg/src/slvp/driver.py).  One
``strang_step`` (driver.py:245-265) is, for a 2x2v grid,

    x1(tau/2) x2(tau/2) | rho -> E | v1(tau) v2(tau) | x1(tau/2) x2(tau/2)

entirely in HBM: six sweep kernels ping-ponging between the field's buffer
and one scratch buffer, the density reduction, four small transform GEMMs,
and on-device table generation for the E-dependent velocity shifts.  The
reference's per-sub-step ``isfinite(sum(f))`` checks (driver.py:209-211)
become flag words set by each kernel's epilogue; they are read back once
per step and the first flagged sub-step is raised as :class:`SubstepError`
with the reference's exact message.  (Unlike the reference, the remaining
sub-steps of a failing step still execute before the error is raised.)
"""

from __future__ import annotations

import math
import os
from dataclasses import dataclass
from functools import lru_cache

import numpy as np
import torch

from . import _device, _lib
from .dg import DeviceTables, sweep_dg, vplane_dg, xcomp_dg, xplane2_dg, xplane_dg
from .field import DEFAULT_STRATEGY, DistributionField, LayoutDescriptor, write_snapshot
from .grid import DG, SPACE, SPLINE, VELOCITY, Axis, GridSpec, gauss_nodes
from .poisson import (
    ElectricField,
    _device_x,
    _lagrange_row,
    _warn_if_not_neutral,
    density_into,
    geometry,
    scratch,
    solve_into,
)
from .spline import double_sweep_ok, sweep_spline, sweep_spline2, sweep_spline2_density


# Fused x1+x2 plane sweeps and fused v1+v2 column sweeps (set False to run
# the sweeps separately; the results are bitwise identical either way).
FUSE_X = True
FUSE_V = True
# Density as an epilogue of the opening x pass (dG): saves the 8 B/dof read
# of the standalone density pass.  VPB_FUSE_RHO=0/1 overrides the default.
FUSE_RHO = os.environ.get("VPB_FUSE_RHO", "1") != "0"

# Arithmetic of the merged x half steps (closing x1 x2 of step m + opening
# x1 x2 of step m+1 in one pass, see enqueue_steps):
#   "fast"  (default) -- x1 x2 x1 x2 = (x1 x1)(x2 x2) applied as one composed
#           three-cell stencil per axis with fused multiply-adds
#           (vpb_dg_sweep_xcomp): HBM-bound; equal to the sweep chain up to
#           round-off (~1e-16 relative per step, far inside the 1e-12 bar);
#   "exact" -- the four sweeps chained with the reference's rounding
#           (vpb_dg_sweep_xplane2): advance() is then bitwise K strang_step
#           calls.
# Every other pass keeps the reference's operation order in both modes.
# VPB_ARITH=exact|fast overrides the default; see set_arithmetic().
_ARITH_MODES = ("fast", "exact")
ARITH = os.environ.get("VPB_ARITH", "fast")
# spline density fused into the merged x pass ("fast" arithmetic only)
SPLINE_RHO = os.environ.get("VPB_SPLINE_RHO", "1") != "0"
if ARITH not in _ARITH_MODES:
    raise ValueError(f"VPB_ARITH must be one of {_ARITH_MODES}, got {ARITH!r}")


def set_arithmetic(mode: str) -> str:
    """Select the merged-x-pass arithmetic ("fast" or "exact"); returns the
    previous mode."""
    global ARITH
    if mode not in _ARITH_MODES:
        raise ValueError(f"unknown arithmetic mode {mode!r}; expected one of {_ARITH_MODES}")
    prev, ARITH = ARITH, mode
    return prev


def arithmetic() -> str:
    return ARITH


class SubstepError(RuntimeError):
    """Non-finite values after a sub-step (driver.py:31-38)."""

    def __init__(self, substep: str, time: float | None = None):
        self.substep = substep
        self.time = time
        at = "" if time is None else f" at t={time:g}"
        super().__init__(f"non-finite values after sub-step '{substep}'{at}")


@dataclass(frozen=True)
class ProblemSpec:
    """Benchmark problem: extents and initial-data parameters (driver.py:41-58)."""

    name: str
    x_extents: tuple
    v_extents: tuple
    epsilon: float
    wavenumber: float
    drift: float = 0.0

    @property
    def ndim_x(self) -> int:
        return len(self.x_extents)

    @property
    def ndim(self) -> int:
        return 2 * self.ndim_x


_FOUR_PI = 4.0 * math.pi
_TEN_PI = 10.0 * math.pi

_PROBLEMS = {
    # driver.py:61-84
    "landau2d": ProblemSpec("landau2d", ((0.0, _FOUR_PI),), ((-6.0, 6.0),), 0.5, 0.5),
    "landau4d": ProblemSpec("landau4d", ((0.0, _FOUR_PI),) * 2, ((-6.0, 6.0),) * 2, 0.5, 0.5),
    "twostream4d": ProblemSpec(
        "twostream4d", ((0.0, _TEN_PI),) * 2, ((-6.0, 6.0),) * 2, 1e-3, 0.2, drift=2.4
    ),
    # BASELINE.json config 3: beams along v1 only, additive perturbation
    # (1/2pi) * 0.5[e^{-(v1-d)^2/2} + e^{-(v1+d)^2/2}] e^{-v2^2/2} (1 + eps cos k x1 + eps cos k x2)
    "twostream4d_baseline": ProblemSpec(
        "twostream4d_baseline", ((0.0, _TEN_PI),) * 2, ((-6.0, 6.0),) * 2, 1e-3, 0.2, drift=2.4
    ),
}


def problem_spec(name: str) -> ProblemSpec:
    try:
        return _PROBLEMS[name]
    except KeyError:
        known = ", ".join(sorted(_PROBLEMS))
        raise ValueError(f"unknown problem {name!r} (known: {known})") from None


def parse_method(name: str) -> tuple[str, int]:
    """"spline" -> (spline, 0); "dg<order>" -> (dg, order-1) (driver.py:95-107)."""
    if name == "spline":
        return SPLINE, 0
    if name.startswith("dg") and name[2:].isdigit():
        order = int(name[2:])
        if 1 <= order <= 9:
            return DG, order - 1
    raise ValueError(f"unknown method {name!r} (expected 'spline' or 'dg<order>')")


def method_label(grid: GridSpec) -> str:
    return "spline" if grid.method == SPLINE else f"dg{grid.dg_degree + 1}"


def make_grid(problem: ProblemSpec, method: str, dofs, dg_order: int = 0) -> GridSpec:
    """Grid targeting ``dofs`` points per axis (driver.py:114-144)."""
    if isinstance(dofs, int):
        dofs = (dofs,) * problem.ndim
    if len(dofs) != problem.ndim:
        raise ValueError(f"expected {problem.ndim} dof values, got {len(dofs)}")
    if method == DG:
        if not 1 <= dg_order <= 9:
            raise ValueError("dg_order must be in 1..9")
        counts = [max(4, round(d / dg_order)) for d in dofs]
    elif method == SPLINE:
        counts = list(dofs)
    else:
        raise ValueError(f"unknown method {method!r}")
    axes = [Axis(lo, hi, counts[i], SPACE) for i, (lo, hi) in enumerate(problem.x_extents)]
    axes += [
        Axis(lo, hi, counts[problem.ndim_x + i], VELOCITY)
        for i, (lo, hi) in enumerate(problem.v_extents)
    ]
    return GridSpec(tuple(axes), method, dg_order - 1 if method == DG else 0)


def initial_value(problem: ProblemSpec, point) -> float:
    """Pointwise initial distribution (driver.py:147-164)."""
    eps, k = problem.epsilon, problem.wavenumber
    if problem.name == "landau2d":
        x, v = point
        return (1.0 + eps * math.cos(k * x)) * math.exp(-0.5 * v * v) / math.sqrt(2.0 * math.pi)
    if problem.name == "landau4d":
        x1, x2, v1, v2 = point
        return (1.0 + eps * (math.cos(k * x1) + math.cos(k * x2))) * math.exp(
            -0.5 * (v1 * v1 + v2 * v2)) / (2.0 * math.pi)
    d = problem.drift
    x1, x2, v1, v2 = point
    if problem.name == "twostream4d":
        g1 = math.exp(-0.5 * (v1 - d) ** 2) + math.exp(-0.5 * (v1 + d) ** 2)
        g2 = math.exp(-0.5 * (v2 - d) ** 2) + math.exp(-0.5 * (v2 + d) ** 2)
        return (1.0 + eps * math.cos(k * x1) * math.cos(k * x2)) * g1 * g2 / (8.0 * math.pi)
    if problem.name == "twostream4d_baseline":
        g1 = 0.5 * (math.exp(-0.5 * (v1 - d) ** 2) + math.exp(-0.5 * (v1 + d) ** 2))
        g2 = math.exp(-0.5 * v2 * v2)
        return (1.0 + eps * (math.cos(k * x1) + math.cos(k * x2))) * g1 * g2 / (2.0 * math.pi)
    raise ValueError(f"unknown problem {problem.name!r}")


def separable_factors(problem: ProblemSpec, grid: GridSpec):
    """(g1, g2, space) with f[iv2][iv1][ix2][ix1] = (g2*g1)*space, computed by
    the same NumPy expressions as the reference broadcast (driver.py:182-198),
    so the device product is bitwise the reference's initial state."""
    eps, k = problem.epsilon, problem.wavenumber
    pts = [grid.axis_points(a) for a in range(grid.ndim)]
    root = math.sqrt(2.0 * math.pi)
    if problem.name == "landau2d":
        space = 1.0 + eps * np.cos(k * pts[0])
        g1 = np.exp(-0.5 * pts[1] ** 2) / root
        return g1, np.ones(1), space
    if problem.name == "landau4d":
        space = 1.0 + eps * (np.cos(k * pts[1])[:, None] + np.cos(k * pts[0])[None, :])
        g1 = np.exp(-0.5 * pts[2] ** 2) / root
        g2 = np.exp(-0.5 * pts[3] ** 2) / root
        return g1, g2, space
    d = problem.drift
    if problem.name == "twostream4d":
        space = np.cos(k * pts[1])[:, None] * np.cos(k * pts[0])[None, :]
        space = (1.0 + eps * space) / (8.0 * math.pi)
        g1 = np.exp(-0.5 * (pts[2] - d) ** 2) + np.exp(-0.5 * (pts[2] + d) ** 2)
        g2 = np.exp(-0.5 * (pts[3] - d) ** 2) + np.exp(-0.5 * (pts[3] + d) ** 2)
        return g1, g2, space
    if problem.name == "twostream4d_baseline":
        space = 1.0 + eps * (np.cos(k * pts[1])[:, None] + np.cos(k * pts[0])[None, :])
        g1 = 0.5 * (np.exp(-0.5 * (pts[2] - d) ** 2) + np.exp(-0.5 * (pts[2] + d) ** 2)) / root
        g2 = np.exp(-0.5 * pts[3] ** 2) / root
        return g1, g2, space
    raise ValueError(f"unknown problem {problem.name!r}")


def initialize(problem: ProblemSpec, grid: GridSpec, strategy: str | None = None,
               cache_block: int = 8) -> DistributionField:
    """Sample the initial distribution on the device (driver.py:167-206)."""
    if grid.ndim != problem.ndim:
        raise ValueError(f"grid is {grid.ndim}-dimensional, problem needs {problem.ndim}")
    g1, g2, space = separable_factors(problem, grid)
    field = DistributionField.empty(grid, strategy, cache_block)
    lib = _lib.load()
    dg1, dg2 = _device.to_device(g1), _device.to_device(g2)
    dsp = _device.to_device(np.ascontiguousarray(space).ravel())
    _lib.check(
        lib.vpb_fill_separable(field.data.data_ptr(), _lib.dims(grid.dims4), dg1.data_ptr(),
                               dg2.data_ptr(), dsp.data_ptr(), _device.stream()),
        "vpb_fill_separable",
    )
    return field


# ---------------------------------------------------------------------------
# Per-grid step state
# ---------------------------------------------------------------------------
class StepState:
    """Scratch buffers, cached x tables and flag words for one grid."""

    def __init__(self, grid: GridSpec):
        self.grid = grid
        dev = _device.device()
        n = grid.total_dof
        self.buf = torch.empty(n, dtype=torch.float64, device=dev)
        self.geom = geometry(grid)
        nx = self.geom.n1 * self.geom.n2
        self.nx = nx
        self.rho = torch.empty(nx, dtype=torch.float64, device=dev)
        self.e = torch.empty(self.geom.ncomp * nx, dtype=torch.float64, device=dev)
        self.flags = torch.zeros(8, dtype=torch.int32, device=dev)
        self.stats = torch.zeros(4, dtype=torch.float64, device=dev)
        self.flags_host = torch.zeros(8, dtype=torch.int32).pin_memory()
        self.stats_host = torch.zeros(4, dtype=torch.float64).pin_memory()
        self.vpoints = [_device.to_device(grid.axis_points(a)) for a in grid.velocity_axes]
        self._xtab: dict = {}
        self._vtab: list = [None] * grid.ndim_x
        d = grid.ndim_x
        names = ["x"] if d == 1 else ["x1", "x2"]
        vnames = ["v"] if d == 1 else ["v1", "v2"]
        self.names = (
            [f"{x} half (open)" for x in names] + ["field solve"] + [f"{v} full" for v in vnames]
            + [f"{x} half (close)" for x in names]
        )
        # both x sweeps of a half step in one pass (bitwise-identical result)
        self.fused_x = (grid.method == DG and grid.ndim == 4
                        and (grid.dof(0) * grid.order) % 2 == 0 and FUSE_X)
        # both v sweeps in one pass (bitwise-identical result)
        self.fused_v = grid.method == DG and grid.ndim == 4 and FUSE_V
        # spline: merged x half steps as one double sweep per x axis ("fast")
        self.spline_x2 = grid.method == SPLINE and all(
            double_sweep_ok(grid, d) for d in range(grid.ndim_x))
        lib = _lib.load()
        self.diag_work = torch.empty(int(lib.vpb_diag_work_len(_lib.dims(grid.dims4))),
                                     dtype=torch.float64, device=dev)
        self.diag_out = torch.zeros(8, dtype=torch.float64, device=dev)
        self.diag_host = torch.zeros(8, dtype=torch.float64).pin_memory()
        wv = [grid.axis_weights(a) for a in grid.velocity_axes]
        vsq = [grid.axis_points(a) ** 2 for a in grid.velocity_axes]
        if d == 1:
            wv.append(np.ones(1))
            vsq.append(np.zeros(1))
        self.wv1, self.wv2 = (_device.to_device(w) for w in wv)
        self.v1sq, self.v2sq = (_device.to_device(v) for v in vsq)
        # density as an epilogue of the opening fused x pass (dG, 2x2v)
        self.fused_rho = self.fused_x and FUSE_RHO and self.geom.struct_c is not None
        if self.fused_rho:
            n = int(lib.vpb_dg_xplane_density_work_len(_lib.dims(grid.dims4), grid.order))
            if n <= 0:
                self.fused_rho = False
            else:
                self.rho_work = torch.empty(n, dtype=torch.float64, device=dev)
                self.rho_work2 = None  # double x pass work, allocated on first use
                self.rho_work3 = None  # composed x pass work, allocated on first use
                self.rc = torch.empty(grid.axes[0].count * grid.axes[1].count,
                                      dtype=torch.float64, device=dev)
                # host constants of the epilogue: centre Lagrange weights and
                # the space quadrature weights of one cell per axis
                p = grid.order
                nodes, _ = gauss_nodes(p)
                self.dens_mid = np.ascontiguousarray(_lagrange_row(nodes, 0.5))
                cells = []
                for a in (0, 1):
                    w = np.asarray(grid.axis_weights(a), dtype=np.float64)
                    cell = np.ascontiguousarray(w[:p])
                    if not np.array_equal(w.reshape(-1, p), np.broadcast_to(cell, (w.size // p, p))):
                        self.fused_rho = False  # non-uniform cells: keep the separate density
                    cells.append(cell)
                self.dens_w1, self.dens_w2 = cells

        # spline ("fast"): density as an epilogue of the merged pass's x1
        # double sweep (vpb_spline_sweep_x1dbl_density; the x2 double sweep
        # runs first), partial sums per 32-row v1 block reduced by vpb_density
        self.spline_rho = False
        if (self.spline_x2 and grid.ndim == 4 and SPLINE_RHO
                and os.environ.get("VPB_SPLINE_ROWS") is None
                and grid.dof(0) % 8 == 0 and grid.dof(0) >= 64):
            plen = int(lib.vpb_spline_density_part_len(_lib.dims(grid.dims4)))
            if plen > 0:
                self.spline_rho = True
                d4 = grid.dims4
                self.spart_dims = (d4[0], d4[1], d4[2] // 32, d4[3])
                self.spart = torch.empty(plen, dtype=torch.float64, device=dev)
                self.spart_w1 = torch.ones(d4[2] // 32, dtype=torch.float64, device=dev)
                self.spart_work = torch.empty(
                    int(lib.vpb_density_work_len(_lib.dims(self.spart_dims))),
                    dtype=torch.float64, device=dev)

    def x_tables(self, d: int, tau: float):
        """Tables for the half x-sweep along space axis d: shift = v_d * (tau/2)."""
        key = (d, float(tau))
        tab = self._xtab.get(key)
        if tab is None:
            grid = self.grid
            h = grid.axes[d].h
            if grid.method == DG:
                tab = DeviceTables(self.vpoints[d], 0.5 * tau, h, grid.dg_degree)
            else:
                tab = self.vpoints[d]
            if len(self._xtab) > 16:
                self._xtab.clear()
            self._xtab[key] = tab
        return tab

    def v_tables(self, d: int, tau: float):
        """Tables for the v-sweep along velocity axis d: shift = E_d * tau."""
        grid = self.grid
        e_d = self.e[d * self.nx:(d + 1) * self.nx]
        h = grid.axes[grid.ndim_x + d].h
        if grid.method != DG:
            return e_d
        tab = self._vtab[d]
        if tab is None:
            tab = DeviceTables(e_d, tau, h, grid.dg_degree)
            self._vtab[d] = tab
        else:
            tab.refresh(e_d, tau, h)
        return tab


@lru_cache(maxsize=16)
def _state_cached(grid: GridSpec, device_index: int) -> StepState:
    return StepState(grid)


def step_state(grid: GridSpec) -> StepState:
    return _state_cached(grid, torch.cuda.current_device())


def _sweep_into(state: StepState, axis: int, src, dst, tab, scale: float, flag) -> None:
    grid = state.grid
    if grid.method == DG:
        sweep_dg(grid, axis, src, dst, tab, flag)
    else:
        h = grid.axes[axis].h
        sweep_spline(grid, axis, src, dst, tab, scale, h, flag)


def enqueue_step(field: DistributionField, tau: float, state: StepState | None = None,
                 timer=None) -> None:
    """Queue one Strang step on the current stream (no host synchronisation).

    Flags and the density mean land in ``state.flags`` / ``state.stats``.
    ``timer(label)`` (optional) is called before each sub-step kernel group
    and once with ``None`` at the end; bench.py uses it to bracket kernels
    with CUDA events.
    """
    st = state or step_state(field.grid)
    enqueue_steps(field, tau, 1, st, st.flags.view(1, -1), st.stats.view(1, -1), timer)


def enqueue_steps(field: DistributionField, tau: float, nsteps: int, st: StepState,
                  flags: torch.Tensor, stats: torch.Tensor, timer=None,
                  merge: bool = True, moments: torch.Tensor | None = None) -> None:
    """Queue ``nsteps`` Strang steps (driver.py:245-265 each).

    ``flags[m]`` / ``stats[m]`` receive step m's flag words (slots as
    ``st.names``) and density mean.  With ``merge`` (and the fused x pass),
    the closing x half step of step m and the opening one of step m+1 run as
    one HBM pass; the state between the two steps is then never written to
    HBM.  "exact" arithmetic: ``vpb_dg_sweep_xplane2``, four sweeps chained
    in registers and shared memory, bitwise equal to running them
    separately; "fast" (default): ``vpb_dg_sweep_xcomp``, composed
    three-cell stencils, equal up to round-off.

    ``moments`` (8 doubles, needs ``st.fused_rho``): the closing pass of the
    last step also produces the diagnostics of the final state
    (driver.py:279-316; fresh ρ -> E of that state): moments[0..4] = mass,
    l1, l2^2, kinetic, electric energy and moments[5] = its density mean.
    """
    grid = field.grid
    mark = timer or (lambda label: None)
    flags.zero_()
    half = 0.5 * tau
    nx = grid.ndim_x
    field_k, v_k, close_k = nx, nx + 1, 2 * nx + 1
    xn = ["x"] if nx == 1 else ["x1", "x2"]
    vn = ["v"] if nx == 1 else ["v1", "v2"]

    def swap(out) -> None:
        st.buf = field._swap(out.view(field._phys.shape)).view(-1)

    def sweep(axis: int, tab, scale: float, label: str, flag) -> None:
        out = st.buf
        mark(label)
        _sweep_into(st, axis, field._phys.view(-1), out, tab, scale, flag)
        swap(out)

    def x_half(fl, k: int, with_density: bool, stats_row) -> None:
        """_advect_space(tau/2) (driver.py:220-228) into flag slots k, k+1."""
        if st.fused_x:
            out = st.buf
            t1, t2 = st.x_tables(0, tau), st.x_tables(1, tau)
            if with_density:
                # x1+x2 sweeps with the cell-centre density of the result as an
                # epilogue (compute_density + centre collapse, poisson.py:85-139)
                mark("sweep_x12_rho")
                xplane_density_dg(grid, field._phys.view(-1), out, t1, t2, fl[k:k + 1],
                                  fl[k + 1:k + 2], st, stats_row)
            else:
                mark("sweep_x12")
                xplane_dg(grid, field._phys.view(-1), out, t1, t2, fl[k:k + 1], fl[k + 1:k + 2])
            swap(out)
            return
        for d in range(nx):
            sweep(d, st.x_tables(d, tau), half, f"sweep_{xn[d]}", fl[k + d:k + d + 1])

    def x_double(fl_a, fl_b, with_density: bool, stats_row) -> None:
        """Closing x half step of one step + opening one of the next, one pass."""
        out = st.buf
        t1, t2 = st.x_tables(0, tau), st.x_tables(1, tau)
        fa = (fl_a[close_k:close_k + 1], fl_a[close_k + 1:close_k + 2])
        fb = (fl_b[0:1], fl_b[1:2])
        if ARITH == "fast":
            # composed stencils: intermediate states never exist, so a
            # non-finite output is reported against the pass's first sub-step
            # (inputs are checked by the producing pass, so only an overflow
            # inside this pass can land here)
            if with_density:
                mark("sweep_x12x12_rho")
                xcomp_density_dg(grid, field._phys.view(-1), out, t1, t2, fa[0], st, stats_row)
            else:
                mark("sweep_x12x12")
                xcomp_dg(grid, field._phys.view(-1), out, t1, t2, fa[0])
            swap(out)
            return
        if with_density:
            mark("sweep_x12x12_rho")
            xplane2_density_dg(grid, field._phys.view(-1), out, t1, t2, fa, fb, st, stats_row)
        else:
            mark("sweep_x12x12")
            xplane2_dg(grid, field._phys.view(-1), out, t1, t2, fa, fb)
        swap(out)

    def x_double_spline(fl, with_density: bool) -> None:
        """Spline: closing x half step of one step + opening one of the next
        as one double sweep per x axis (vpb_spline_sweep_axis2); a
        non-finite result is reported against the closing sub-step.  With
        ``with_density`` the x2 double sweep runs first (the two axes'
        operators commute) and the x1 one carries the density epilogue
        (st.rho of the next step, compute_density poisson.py:85-95)."""
        lib = _lib.load()
        for d in ((1, 0) if with_density else range(nx)):
            out = st.buf
            if with_density and d == 0:
                mark("sweep_x1x2_rho")
                sweep_spline2_density(grid, field._phys.view(-1), out, st.x_tables(0, tau),
                                      half, grid.axes[0].h, fl[close_k:close_k + 1], st.wv1,
                                      st.spart)
                swap(out)
                mark("density")
                _lib.check(lib.vpb_density(st.spart.data_ptr(), _lib.dims(st.spart_dims),
                                           st.spart_w1.data_ptr(), st.wv2.data_ptr(),
                                           st.rho.data_ptr(), st.spart_work.data_ptr(),
                                           _device.stream()), "vpb_density")
                continue
            mark(f"sweep_{xn[d]}x2")
            sweep_spline2(grid, d, field._phys.view(-1), out, st.x_tables(d, tau), half,
                          grid.axes[d].h, fl[close_k + d:close_k + d + 1])
            swap(out)

    rho_ready = set()  # steps whose density the merged spline pass produced

    def field_solve_of(m: int) -> None:
        fl = flags[m]
        if st.fused_rho:
            mark("field_solve")
            solve_into(st.rc, grid, st.e, None, fl[field_k:field_k + 1], centred=True)
        else:
            if m not in rho_ready:
                mark("density")
                density_into(field.data, grid, st.rho)  # compute_density  poisson.py:85-95
            mark("field_solve")
            solve_into(st.rho, grid, st.e, stats[m], fl[field_k:field_k + 1])  # solve_poisson

    def field_and_velocity(m: int) -> None:
        field_solve_of(m)
        fl = flags[m]
        if st.fused_v:  # _advect_velocity(tau) in one pass  driver.py:231-242
            mark("tables_v12")
            t1 = st.v_tables(0, tau)
            t2 = st.v_tables(1, tau)
            out = st.buf
            mark("sweep_v12")
            vplane_dg(grid, field._phys.view(-1), out, t1, t2, fl[v_k:v_k + 1],
                      fl[v_k + 1:v_k + 2])
            swap(out)
        else:
            for d in range(nx):  # _advect_velocity(tau)  driver.py:231-242
                mark(f"tables_{vn[d]}")
                tab = st.v_tables(d, tau)
                sweep(nx + d, tab, tau, f"sweep_{vn[d]}", fl[v_k + d:v_k + d + 1])

    def x_close_with_moments(fl) -> None:
        out = st.buf
        t1, t2 = st.x_tables(0, tau), st.x_tables(1, tau)
        mark("sweep_x12_diag")
        xplane_moments_dg(grid, field._phys.view(-1), out, t1, t2, fl[close_k:close_k + 1],
                          fl[close_k + 1:close_k + 2], st, moments)
        swap(out)
        mark("diag_field")
        solve_into(st.rc, grid, st.e, None, None, centred=True)
        lib = _lib.load()
        _lib.check(lib.vpb_electric_energy(st.e.data_ptr(), st.geom.ncomp, st.nx,
                                           st.geom.tensors["wx"].data_ptr(),
                                           moments[4:5].data_ptr(), _device.stream()),
                   "vpb_electric_energy")

    if moments is not None and not (st.fused_x and st.fused_rho):
        raise ValueError("fused diagnostics need the fused x pass with the density epilogue")
    x_half(flags[0], 0, st.fused_rho, stats[0])  # "open" of step 0
    for m in range(nsteps):
        field_and_velocity(m)
        if m + 1 == nsteps:
            if moments is not None:
                x_close_with_moments(flags[m])
            else:
                x_half(flags[m], close_k, False, None)  # "close" of the last step
        elif merge and st.fused_x:
            x_double(flags[m], flags[m + 1], st.fused_rho, stats[m + 1])
        elif merge and st.spline_x2 and ARITH == "fast":
            x_double_spline(flags[m], st.spline_rho)
            if st.spline_rho:
                rho_ready.add(m + 1)
        else:
            x_half(flags[m], close_k, False, None)
            x_half(flags[m + 1], 0, st.fused_rho, stats[m + 1])
    mark(None)


def xplane_density_dg(grid, src, dst, t1, t2, flag1, flag2, st: StepState, stats) -> None:
    """Fused x pass whose epilogue writes the cell-centre density of its
    output to ``st.rc`` and the neutrality mean to ``stats[0]``."""
    lib = _lib.load()
    g = st.geom
    _lib.check(
        lib.vpb_dg_sweep_xplane_density(
            src.data_ptr(), dst.data_ptr(), _lib.dims(grid.dims4), t1.order, t1.a.data_ptr(),
            t1.b.data_ptr(), t1.q.data_ptr(), t1.alpha.data_ptr(), t2.a.data_ptr(),
            t2.b.data_ptr(), t2.q.data_ptr(), t2.alpha.data_ptr(), flag1.data_ptr(),
            flag2.data_ptr(), st.wv1.data_ptr(), st.wv2.data_ptr(),
            st.dens_mid.ctypes.data, st.dens_w1.ctypes.data, st.dens_w2.ctypes.data,
            g.volume, st.rho_work.data_ptr(), st.rc.data_ptr(),
            stats.data_ptr(), _device.stream()),
        "vpb_dg_sweep_xplane_density",
    )


def xplane_moments_dg(grid, src, dst, t1, t2, flag1, flag2, st: StepState, moments) -> None:
    """Fused x pass with the density epilogue (-> st.rc) and the diagnostics
    moments of its output (-> moments[0..3], its mean -> moments[5])."""
    lib = _lib.load()
    g = st.geom
    _lib.check(
        lib.vpb_dg_sweep_xplane_moments(
            src.data_ptr(), dst.data_ptr(), _lib.dims(grid.dims4), t1.order, t1.a.data_ptr(),
            t1.b.data_ptr(), t1.q.data_ptr(), t1.alpha.data_ptr(), t2.a.data_ptr(),
            t2.b.data_ptr(), t2.q.data_ptr(), t2.alpha.data_ptr(), flag1.data_ptr(),
            flag2.data_ptr(), st.wv1.data_ptr(), st.wv2.data_ptr(),
            st.dens_mid.ctypes.data, st.dens_w1.ctypes.data, st.dens_w2.ctypes.data,
            st.v1sq.data_ptr(), st.v2sq.data_ptr(), g.volume, st.rho_work.data_ptr(),
            st.rc.data_ptr(), moments[5:6].data_ptr(), moments.data_ptr(), _device.stream()),
        "vpb_dg_sweep_xplane_moments",
    )


def xplane2_density_dg(grid, src, dst, t1, t2, fa, fb, st: StepState, stats) -> None:
    """Two x half steps in one pass with the density epilogue on the result."""
    lib = _lib.load()
    g = st.geom
    if st.rho_work2 is None:
        n = int(lib.vpb_dg_xplane2_density_work_len(_lib.dims(grid.dims4), grid.order))
        if n <= 0:
            raise _lib.VpbError("cannot plan the double x pass")
        st.rho_work2 = torch.empty(n, dtype=torch.float64, device=_device.device())
    _lib.check(
        lib.vpb_dg_sweep_xplane2_density(
            src.data_ptr(), dst.data_ptr(), _lib.dims(grid.dims4), t1.order, t1.a.data_ptr(),
            t1.b.data_ptr(), t1.q.data_ptr(), t1.alpha.data_ptr(), t2.a.data_ptr(),
            t2.b.data_ptr(), t2.q.data_ptr(), t2.alpha.data_ptr(), fa[0].data_ptr(),
            fa[1].data_ptr(), fb[0].data_ptr(), fb[1].data_ptr(), st.wv1.data_ptr(),
            st.wv2.data_ptr(), st.dens_mid.ctypes.data, st.dens_w1.ctypes.data,
            st.dens_w2.ctypes.data, g.volume, st.rho_work2.data_ptr(), st.rc.data_ptr(),
            stats.data_ptr(), _device.stream()),
        "vpb_dg_sweep_xplane2_density",
    )


def xcomp_density_dg(grid, src, dst, t1, t2, flag, st: StepState, stats) -> None:
    """Merged x half steps with composed stencils and the density epilogue."""
    lib = _lib.load()
    g = st.geom
    if st.rho_work3 is None:
        n = int(lib.vpb_dg_xcomp_density_work_len(_lib.dims(grid.dims4), grid.order))
        if n <= 0:
            raise _lib.VpbError("cannot plan the composed x pass")
        st.rho_work3 = torch.empty(n, dtype=torch.float64, device=_device.device())
    _lib.check(
        lib.vpb_dg_sweep_xcomp_density(
            src.data_ptr(), dst.data_ptr(), _lib.dims(grid.dims4), t1.order,
            t1.composed().data_ptr(), t1.q.data_ptr(), t1.alpha.data_ptr(),
            t2.composed().data_ptr(), t2.q.data_ptr(), t2.alpha.data_ptr(), flag.data_ptr(),
            st.wv1.data_ptr(), st.wv2.data_ptr(), st.dens_mid.ctypes.data,
            st.dens_w1.ctypes.data, st.dens_w2.ctypes.data, g.volume,
            st.rho_work3.data_ptr(), st.rc.data_ptr(), stats.data_ptr(), _device.stream()),
        "vpb_dg_sweep_xcomp_density",
    )


def check_step(state: StepState, time_label: float | None) -> None:
    """Read the step's flags (one D2H + sync) and raise / warn like the reference."""
    state.flags_host.copy_(state.flags, non_blocking=True)
    state.stats_host.copy_(state.stats, non_blocking=True)
    torch.cuda.current_stream().synchronize()
    flags = state.flags_host.numpy()
    _warn_if_not_neutral(float(state.stats_host[0]))
    for k, name in enumerate(state.names):
        if flags[k]:
            raise SubstepError(name, time_label)


class StepGraph:
    """Repeated Strang steps of one field replayed from CUDA graphs.

    The device work of :func:`enqueue_step` (sweeps, tables, density, field
    solve) is captured once; every :meth:`step` replays it and performs the
    same per-step non-finite check as :func:`strang_step`.  The field's two
    buffers ping-pong, so when a step swaps an odd number of times two graphs
    are captured (one per parity).  Results are bitwise those of
    ``strang_step(field, tau, consume=True)``.
    """

    def __init__(self, field: DistributionField, tau: float):
        self.field = field
        self.tau = float(tau)
        self.st = step_state(field.grid)
        # eager warm-up: caches x tables, allocates v tables, sets kernel attributes
        enqueue_step(field, tau, self.st)
        check_step(self.st, None)
        self.graphs = []
        self.bufs = []  # (field buffer, scratch buffer) before each graph
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        for _ in range(2):
            self.bufs.append((field._phys, self.st.buf))
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=side):
                enqueue_step(field, tau, self.st)
            self.graphs.append(g)
            if field._phys is self.bufs[0][0]:
                break  # even number of swaps: one graph suffices
        torch.cuda.current_stream().wait_stream(side)
        # capture executed nothing: restore the pre-capture buffer roles
        field._phys, self.st.buf = self.bufs[0]
        self.parity = 0

    def step(self, time_label: float | None = None) -> DistributionField:
        self.graphs[self.parity].replay()
        nxt = (self.parity + 1) % len(self.graphs)  # one graph: roles unchanged
        self.field._phys, self.st.buf = self.bufs[nxt]
        self.parity = nxt
        check_step(self.st, time_label)
        return self.field


class AdvanceGraph:
    """Blocks of ``nsteps`` merged Strang steps (:func:`advance` with
    ``consume=True``) replayed from CUDA graphs -- the reference's ``run``
    loop between two records (driver.py:371-377) repeats the same block, and
    on small, L2-resident grids the host-side launch cost of the block's
    kernels exceeds their device time.

    The block is captured once per buffer parity (like :class:`StepGraph`);
    :meth:`advance` replays it and then performs the same non-finite checks
    and neutrality warnings as :func:`advance`.  Results are bitwise those of
    ``advance(field, tau, nsteps, consume=True)``.
    """

    def __init__(self, field: DistributionField, tau: float, nsteps: int):
        if nsteps <= 0:
            raise ValueError("nsteps must be positive")
        self.field = field
        self.tau = float(tau)
        self.nsteps = int(nsteps)
        self.st = step_state(field.grid)
        dev = _device.device()
        self.flags = torch.zeros((nsteps, self.st.flags.numel()), dtype=torch.int32, device=dev)
        self.stats = torch.zeros((nsteps, self.st.stats.numel()), dtype=torch.float64,
                                 device=dev)
        # eager warm-up block: caches x tables, allocates the scratch of every
        # pass, sets kernel attributes (nothing may allocate during capture)
        enqueue_steps(field, tau, nsteps, self.st, self.flags, self.stats)
        check_steps(self.st, self.flags, self.stats, None, tau)
        self.graphs = []
        self.bufs = []
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        for _ in range(2):
            self.bufs.append((field._phys, self.st.buf))
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=side):
                enqueue_steps(field, tau, nsteps, self.st, self.flags, self.stats)
            self.graphs.append(g)
            if field._phys is self.bufs[0][0]:
                break  # even number of swaps per block: one graph suffices
        torch.cuda.current_stream().wait_stream(side)
        field._phys, self.st.buf = self.bufs[0]  # capture executed nothing
        self.parity = 0

    def replay(self) -> None:
        """Queue one block (no host synchronisation, no checks)."""
        self.graphs[self.parity].replay()
        nxt = (self.parity + 1) % len(self.graphs)
        self.field._phys, self.st.buf = self.bufs[nxt]
        self.parity = nxt

    def advance(self, first_step: int | None = None) -> DistributionField:
        """One block of ``nsteps`` steps; raises / warns like :func:`advance`."""
        self.replay()
        check_steps(self.st, self.flags, self.stats, first_step, self.tau)
        return self.field


def strang_step(field: DistributionField, tau: float, workers: int = 1, consume: bool = False,
                time_label: float | None = None) -> DistributionField:
    """Advance by one Strang step of size tau (driver.py:245-265).

    ``workers`` is the reference's CPU thread count; it has no effect here.
    """
    work = field if consume else field.copy()
    st = step_state(work.grid)
    enqueue_step(work, tau, st)
    check_step(st, time_label)
    return work


def advance(field: DistributionField, tau: float, nsteps: int, consume: bool = False,
            first_step: int | None = None, record_time: float | None = None):
    """``nsteps`` Strang steps (driver.py:245-265 each, the reference's
    ``run`` loop between records, driver.py:371-377).

    Adjacent x half steps of consecutive steps share one HBM pass
    (:func:`enqueue_steps`), so the states between the steps are never
    written out; use :func:`strang_step` when every intermediate state is
    needed.  What the result equals depends on the arithmetic mode
    (:func:`set_arithmetic`):

    * ``"exact"``: bitwise ``nsteps`` :func:`strang_step` calls, with the
      same errors and warnings;
    * ``"fast"`` (default): the closing x half step of step m and the
      opening one of step m+1 are applied as composed three-cell stencils
      per x axis, so the result equals the strang_step chain up to
      round-off (tests: <= 1e-13 of max|f| against the chain, <= 1e-12 per
      step against the reference).  The intermediate states are never
      formed, so a non-finite value CREATED inside a merged pass (an
      overflow of finite inputs) is reported as the closing ``x1 half
      (close)`` of step m, where the reference might name step m+1's
      ``x1 half (open)``; non-finite inputs are caught by the pass that
      produced them, as in the reference.

    Non-finite checks and neutrality warnings are evaluated after the last
    step, in step order; with ``first_step`` the errors carry the time label
    ``(first_step + m) * tau`` of step m (as run() labels them).

    With ``record_time`` the result is ``(field, DiagnosticsRecord)``: the
    diagnostics of the final state (== ``diagnostics(field, record_time)``
    up to summation order), computed by the closing x pass itself when the
    fused path is available (no extra read of f).
    """
    if nsteps < 0:
        raise ValueError("nsteps must be non-negative")
    work = field if consume else field.copy()
    if nsteps == 0:
        return work
    st = step_state(work.grid)
    dev = _device.device()
    flags = torch.zeros((nsteps, st.flags.numel()), dtype=torch.int32, device=dev)
    stats = torch.zeros((nsteps, st.stats.numel()), dtype=torch.float64, device=dev)
    fused_record = record_time is not None and st.fused_x and st.fused_rho
    moments = torch.zeros(8, dtype=torch.float64, device=dev) if fused_record else None
    enqueue_steps(work, tau, nsteps, st, flags, stats, moments=moments)
    check_steps(st, flags, stats, first_step, tau)
    if record_time is None:
        return work
    if not fused_record:
        return work, diagnostics(work, record_time)
    v = moments.cpu().numpy()
    _warn_if_not_neutral(float(v[5]))
    mass, l1, l2sq, kin, ee = (float(x) for x in v[:5])
    return work, DiagnosticsRecord(
        time=float(record_time), electric_energy=ee, mass=mass, l1_norm=l1,
        l2_norm=float(math.sqrt(max(l2sq, 0.0))), kinetic_energy=kin, total_energy=kin + ee)


def check_steps(st: StepState, flags: torch.Tensor, stats: torch.Tensor,
                first_step: int | None, tau: float) -> None:
    """Flags / means of several steps (one D2H + sync), raised in step order."""
    fh = flags.cpu().numpy()
    sh = stats.cpu().numpy()
    for m in range(fh.shape[0]):
        _warn_if_not_neutral(float(sh[m, 0]))
        for k, name in enumerate(st.names):
            if fh[m, k]:
                raise SubstepError(name, None if first_step is None else (first_step + m) * tau)


@dataclass(frozen=True)
class DiagnosticsRecord:
    time: float
    electric_energy: float
    mass: float
    l1_norm: float
    l2_norm: float
    kinetic_energy: float
    total_energy: float


def enqueue_diagnostics(field: DistributionField, st: StepState, e: torch.Tensor | None,
                        stats: torch.Tensor | None) -> None:
    grid = field.grid
    if e is None:
        density_into(field.data, grid, st.rho)
        solve_into(st.rho, grid, st.e, stats, None)
        e = st.e
    lib = _lib.load()
    _lib.check(
        lib.vpb_diagnostics(field.data.data_ptr(), _lib.dims(grid.dims4),
                            st.geom.tensors["wx"].data_ptr(), st.wv1.data_ptr(),
                            st.wv2.data_ptr(), st.v1sq.data_ptr(), st.v2sq.data_ptr(),
                            e.data_ptr(), st.geom.ncomp, st.diag_out.data_ptr(),
                            st.diag_work.data_ptr(), _device.stream()),
        "vpb_diagnostics",
    )


def diagnostics(field: DistributionField, time: float = 0.0,
                efield: ElectricField | None = None) -> DiagnosticsRecord:
    """Conserved quantities (driver.py:279-316), computed on the device."""
    grid = field.grid
    st = step_state(grid)
    e = None
    if efield is not None:
        e = torch.cat([_device_x(grid, c) for c in efield.components])
    stats = st.diag_out[5:6]
    enqueue_diagnostics(field, st, e, stats if e is None else None)
    st.diag_host.copy_(st.diag_out, non_blocking=True)
    torch.cuda.current_stream().synchronize()
    v = st.diag_host.numpy().copy()
    if e is None:
        _warn_if_not_neutral(float(v[5]))
    mass, l1, l2sq, kin, ee = (float(x) for x in v[:5])
    return DiagnosticsRecord(
        time=float(time),
        electric_energy=ee,
        mass=mass,
        l1_norm=l1,
        l2_norm=float(math.sqrt(max(l2sq, 0.0))),
        kinetic_energy=kin,
        total_energy=kin + ee,
    )


@dataclass(frozen=True)
class RunConfig:
    problem: ProblemSpec
    grid: GridSpec
    tau: float
    t_end: float
    layout: str | None = None
    cache_block: int = 8
    workers: int = 1
    diag_every: int = 1
    snapshot_times: tuple = ()
    snapshot_stem: str | None = None


def _steps_for(t: float, tau: float) -> int:
    m = round(t / tau)
    if abs(m * tau - t) > 1e-9 * max(1.0, abs(t)):
        raise ValueError(f"time {t} is not an integer multiple of tau={tau}")
    return m


def run(config: RunConfig):
    """Run to t_end with diagnostics and snapshots (driver.py:341-378)."""
    if config.tau <= 0.0:
        raise ValueError("tau must be positive")
    if config.t_end < 0.0:
        raise ValueError("t_end must be non-negative")
    if config.diag_every < 1 or config.workers < 1:
        raise ValueError("diag_every and workers must be >= 1")
    nsteps = _steps_for(config.t_end, config.tau)
    snap_at: dict[int, float] = {}
    for t in config.snapshot_times:
        m = _steps_for(float(t), config.tau)
        if not 0 <= m <= nsteps:
            raise ValueError(f"snapshot time {t} outside [0, t_end]")
        snap_at[m] = float(t)

    field = initialize(config.problem, config.grid, strategy=config.layout,
                       cache_block=config.cache_block)
    records = [diagnostics(field, time=0.0)]
    snapshots: list = []

    def capture(t: float) -> None:
        copy = field.copy()
        snapshots.append((t, copy))
        if config.snapshot_stem is not None:
            write_snapshot(copy, f"{config.snapshot_stem}_t{t:g}.vlf")

    if 0 in snap_at:
        capture(0.0)
    # the states the loop must observe: diagnostics records and snapshots;
    # the steps in between run through advance() (merged x half steps)
    stops = sorted({m for m in range(1, nsteps + 1) if m % config.diag_every == 0}
                   | {m for m in snap_at if m > 0} | ({nsteps} if nsteps else set()))
    done = 0
    for m in stops:
        t = m * config.tau
        if m % config.diag_every == 0:
            field, rec = advance(field, config.tau, m - done, consume=True, first_step=done + 1,
                                 record_time=t)
            records.append(rec)
        else:
            field = advance(field, config.tau, m - done, consume=True, first_step=done + 1)
        done = m
        if m in snap_at:
            capture(snap_at[m])
    return records, snapshots


__all__ = [
    "DEFAULT_STRATEGY",
    "LayoutDescriptor",
    "SubstepError",
    "ProblemSpec",
    "problem_spec",
    "parse_method",
    "method_label",
    "make_grid",
    "initial_value",
    "initialize",
    "strang_step",
    "advance",
    "DiagnosticsRecord",
    "diagnostics",
    "RunConfig",
    "run",
]
