"""Kernel-level parity of the sm_100a path against the oracle and the
reference's golden vectors.  Runs on the B200 box: ``pytest -m gpu``.

Bars: integer/index outputs (q, alpha, whole-cell copies) bitwise; sweeps
bitwise against the reference's compiled kernels when fed the same tables;
generated tables within 1e-14 of the reference's; reductions and the field
solve within 1e-12 relative (fp64 round-off of a different summation order).
"""

from __future__ import annotations

import ctypes

import numpy as np
import pytest
import torch

import paper_1803_02143_b200 as vpb
from oracle import core
from paper_1803_02143_b200 import _device, _lib, kernels
from paper_1803_02143_b200 import dg as vdg
from vpb_testutil import max_rel

pytestmark = pytest.mark.gpu


def ogrid(grid):
    return core.OGrid(tuple(a.lower for a in grid.axes), tuple(a.upper for a in grid.axes),
                      tuple(a.count for a in grid.axes), grid.method, grid.dg_degree)


def dev(a, dtype=torch.float64):
    return torch.from_numpy(np.ascontiguousarray(a)).to("cuda", dtype)


# ---------------------------------------------------------------------------
# K3 tables
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("h", [0.7, 0.5, 1.0])
@pytest.mark.parametrize("deg", [0, 1, 2, 3, 4])
def test_tables_match_reference_projection_pairs(golden, h, deg):
    z = golden("kernels")
    a, b, q, al = vpb.projection_pairs(z["pp_shifts"], h, deg)
    tag = f"pp_h{h}_d{deg}"
    assert np.array_equal(q, z[tag + "_q"])
    assert np.array_equal(al, z[tag + "_alpha"])
    assert np.abs(a - z[tag + "_a"]).max() <= 1e-14
    assert np.abs(b - z[tag + "_b"]).max() <= 1e-14


def test_tables_degree_eight_and_identity_cases():
    pair = vpb.projection_pair(4.0, 1.0, 8)
    assert pair.alpha == 0.0 and pair.cell_offset == 4
    assert np.all(pair.a == 0.0) and np.array_equal(pair.b, np.eye(9))
    # constants and mass are preserved (test_dg.py:178-185 of the reference)
    for degree in (0, 1, 2, 3, 5, 8):
        for alpha in (0.1, 0.3, 0.5, 0.9):
            pr = vpb.projection_pair(alpha, 1.0, degree)
            ones = np.ones(degree + 1)
            _, w = vpb.gauss_nodes(degree + 1)
            np.testing.assert_allclose((pr.a + pr.b) @ ones, ones, atol=1e-13)
            np.testing.assert_allclose(w @ (pr.a + pr.b), w, atol=1e-13)
    with pytest.raises(ValueError):
        vpb.projection_pair(0.1, -1.0, 2)
    with pytest.raises(ValueError):
        vpb.projection_pair(0.1, 1.0, 9)


# ---------------------------------------------------------------------------
# Plugin API (kernels.py entry points) vs the reference's compiled kernels
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("p", [1, 2, 3, 4])
@pytest.mark.parametrize("C", [4, 9, 16])
def test_plugin_dg_sweep_contig_bitwise(golden, p, C):
    z = golden("kernels")
    tag = f"dg_p{p}_c{C}"
    a, b, q, al = core.projection_pairs(z[tag + "_table"], 0.4, p - 1)
    out = kernels.dg_sweep_contig(z[tag + "_lines"], z[tag + "_idx"], a, b, q, al, C, p, 1)
    assert np.array_equal(out, z[tag + "_out"])


@pytest.mark.parametrize("p", [2, 3])
def test_plugin_dg_sweep_strided_in_place(golden, p):
    z = golden("kernels")
    tag = f"dg_p{p}_c16"
    lines = z[tag + "_lines"]
    a, b, q, al = core.projection_pairs(z[tag + "_table"], 0.4, p - 1)
    # a (4, 4, 4, n) strided view whose last axis is the line
    base = np.ascontiguousarray(lines.reshape(4, 4, 4, -1).transpose(3, 0, 1, 2))
    view = np.moveaxis(base, 0, -1)
    kernels.dg_sweep_strided(view, z[tag + "_idx"], a, b, q, al, 16, p, 8, 1)
    assert np.array_equal(view.reshape(64, -1), z[tag + "_out"])


@pytest.mark.parametrize("n", [4, 16, 48, 128])
def test_plugin_spline_sweep_contig_bitwise(golden, n):
    z = golden("kernels")
    tag = f"sp_n{n}"
    out = kernels.spline_sweep_contig(z[tag + "_lines"], z[tag + "_idx"], z[tag + "_table"],
                                      0.25, 1)
    assert np.array_equal(out, z[tag + "_out"])


def test_c_abi_strided_entry_points_on_device_views():
    """vpb_*_sweep_strided update a genuinely strided device view in place."""
    lib = _lib.load()
    rng = np.random.default_rng(11)
    p, C = 3, 8
    n = p * C
    host = rng.standard_normal((n, 5, 6, 7))
    base = dev(host)
    view = base.permute(1, 2, 3, 0)  # last axis = line, strides (42, 7, 1, 210)
    shape = (ctypes.c_int64 * 4)(*view.shape)
    strides = (ctypes.c_int64 * 4)(*view.stride())
    table = rng.uniform(-2, 2, 5)
    a, b, q, al = core.projection_pairs(table, 1.0, p - 1)
    idx = rng.integers(0, 5, 5 * 6 * 7).astype(np.int64)
    da, db, dq, dal, di = dev(a), dev(b), dev(q, torch.int64), dev(al), dev(idx, torch.int64)
    _lib.check(lib.vpb_dg_sweep_strided(view.data_ptr(), shape, strides, di.data_ptr(),
                                        da.data_ptr(), db.data_ptr(), dq.data_ptr(),
                                        dal.data_ptr(), 5, C, p, _device.stream()), "strided")
    lines = np.ascontiguousarray(np.moveaxis(host, 0, -1)).reshape(-1, n)
    ref = core.dg_lines(lines, idx, a, b, q, al, C, p)
    got = view.cpu().numpy().reshape(-1, n)
    assert np.array_equal(got, ref)
    # spline, same view geometry
    base2 = dev(host)
    view2 = base2.permute(1, 2, 3, 0)
    tab = dev(rng.uniform(-5, 5, 5))
    _lib.check(lib.vpb_spline_sweep_strided(view2.data_ptr(), shape, strides, di.data_ptr(),
                                            tab.data_ptr(), 5, 0.5, _device.stream()), "sp")
    ref2 = core.spline_lines(lines, idx, tab.cpu().numpy(), 0.5)
    assert np.array_equal(view2.cpu().numpy().reshape(-1, n), ref2)


# ---------------------------------------------------------------------------
# Canonical-layout axis sweeps, fed the oracle's (= reference's) tables
# ---------------------------------------------------------------------------
REF_AXES = {0: (2,), 1: (3,), 2: (0, 1), 3: (0, 1)}


@pytest.mark.parametrize("order", [1, 2, 3, 4])
@pytest.mark.parametrize("axis", [0, 1, 2, 3])
def test_dg_axis_sweep_bitwise(order, axis):
    prob = vpb.problem_spec("landau4d")
    dofs = tuple(order * c for c in (4, 5, 6, 7))
    grid = vpb.make_grid(prob, "dg", dofs, dg_order=order)
    og = ogrid(grid)
    rng = np.random.default_rng(100 * order + axis)
    vals = rng.standard_normal(grid.dofs)
    h = grid.axes[axis].h
    nt = int(np.prod([grid.dof(a) for a in REF_AXES[axis]]))
    shifts = rng.uniform(-2.5, 2.5, nt) * h
    shifts[: max(1, nt // 7)] = np.round(shifts[: max(1, nt // 7)] / h) * h  # alpha == 0 rows
    ref = core.sweep(vals, og, axis, shifts, REF_AXES[axis], h, strategy="strided")
    a, b, q, al = core.projection_pairs(shifts, h, order - 1)
    perm = vdg.reorder_table(grid, axis, np.arange(nt, dtype=float), REF_AXES[axis]).astype(int)
    src = vpb.DistributionField.from_values(grid, vals)
    dst = torch.empty_like(src.data)
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")
    lib = _lib.load()
    # keep the tables referenced: only raw pointers cross the ABI
    da, db = dev(a[perm]), dev(b[perm])
    dq, dal = dev(q[perm], torch.int64), dev(al[perm])
    _lib.check(lib.vpb_dg_sweep_axis(axis, src.data.data_ptr(), dst.data_ptr(),
                                     _lib.dims(grid.dims4), order, da.data_ptr(), db.data_ptr(),
                                     dq.data_ptr(), dal.data_ptr(), flag.data_ptr(),
                                     _device.stream()),
               "sweep")
    got = dst.view(src._phys.shape).permute(3, 2, 1, 0).cpu().numpy()
    assert np.array_equal(got, ref)
    assert int(flag.item()) == 0


@pytest.mark.parametrize("axis", [0, 1, 2, 3])
def test_spline_axis_sweep_bitwise(axis):
    prob = vpb.problem_spec("landau4d")
    grid = vpb.make_grid(prob, "spline", (16, 12, 20, 8))
    og = ogrid(grid)
    rng = np.random.default_rng(7 + axis)
    vals = rng.standard_normal(grid.dofs)
    h = grid.axes[axis].h
    nt = int(np.prod([grid.dof(a) for a in REF_AXES[axis]]))
    shifts = rng.uniform(-6.0, 6.0, nt) * h
    shifts[0] = 0.0
    shifts[1 % nt] = 3 * h
    ref = core.sweep(vals, og, axis, shifts, REF_AXES[axis], h)
    values = dev(vdg.reorder_table(grid, axis, shifts, REF_AXES[axis]))
    src = vpb.DistributionField.from_values(grid, vals)
    dst = torch.empty_like(src.data)
    lib = _lib.load()
    _lib.check(lib.vpb_spline_sweep_axis(axis, src.data.data_ptr(), dst.data_ptr(),
                                         _lib.dims(grid.dims4), values.data_ptr(), 1.0, h, None,
                                         _device.stream()), "spline")
    got = dst.view(src._phys.shape).permute(3, 2, 1, 0).cpu().numpy()
    assert np.array_equal(got, ref)


def test_line_sweep_api_matches_oracle():
    prob = vpb.problem_spec("landau2d")
    grid = vpb.make_grid(prob, "dg", 32, dg_order=4)
    og = ogrid(grid)
    rng = np.random.default_rng(7)
    vals = rng.standard_normal(grid.dofs)
    shifts = rng.uniform(-2.0, 2.0, grid.dof(1))
    h = grid.axes[0].h
    kern = vpb.DGAdvection(shifts, (1,), h, grid.dg_degree)
    outs = []
    for strategy in ("transpose", "strided"):
        f = vpb.DistributionField.from_values(grid, vals, strategy=strategy)
        outs.append(vpb.line_sweep(f, 0, kern).numpy())
        assert np.array_equal(f.numpy(), vals)  # input untouched
    assert np.array_equal(outs[0], outs[1])
    ref = core.sweep(vals, og, 0, shifts, (1,), h)
    assert max_rel(outs[0], ref) <= 1e-14


def test_sweep_flags_non_finite_output():
    grid = vpb.make_grid(vpb.problem_spec("landau4d"), "dg", 12, dg_order=3)
    vals = np.ones(grid.dofs)
    vals[3, 4, 5, 6] = np.nan
    f = vpb.DistributionField.from_values(grid, vals)
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")
    t = vdg.DeviceTables(dev(np.full(12, 0.37)), 1.0, grid.axes[0].h, 2)
    out = torch.empty_like(f.data)
    for axis in range(4):
        flag.zero_()
        vdg.sweep_dg(grid, axis, f.data, out, t if axis < 2 else
                     vdg.DeviceTables(dev(np.full(144, 0.2)), 1.0, grid.axes[axis].h, 2), flag)
        assert int(flag.item()) == 1, axis


# ---------------------------------------------------------------------------
# Moments, field solve, diagnostics, initial data
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("method,order,dofs", [("dg", 3, 24), ("dg", 2, 16), ("spline", 0, 16)])
def test_density_field_solve_and_diagnostics_vs_oracle(method, order, dofs):
    prob = vpb.problem_spec("landau4d")
    grid = vpb.make_grid(prob, method, dofs, dg_order=order)
    og = ogrid(grid)
    f = vpb.initialize(prob, grid)
    ref = core.initialize("landau4d", og)
    assert np.array_equal(f.numpy(), ref)  # bitwise initial state
    rho = vpb.compute_density(f)
    rho_ref = core.compute_density(ref, og)
    assert max_rel(rho.values.cpu().numpy(), rho_ref) <= 1e-14
    e = vpb.solve_poisson(rho)
    e_ref, _ = core.solve_poisson(rho_ref, og)
    for d in range(2):
        assert np.abs(e.components[d].cpu().numpy() - e_ref[d]).max() <= 1e-13
    assert vpb.electric_energy(e) == pytest.approx(core.electric_energy(e_ref, og), rel=1e-12)
    rec = vpb.diagnostics(f)
    rref = core.diagnostics(ref, og)
    for k, v in rref.items():
        assert getattr(rec, k) == pytest.approx(v, rel=1e-12, abs=1e-300), k


def test_density_of_maxwellian_and_zero():
    grid = vpb.GridSpec((vpb.Axis(0, 4 * np.pi, 4, "space"), vpb.Axis(0, 4 * np.pi, 4, "space"),
                         vpb.Axis(-6, 6, 64, "velocity"), vpb.Axis(-6, 6, 64, "velocity")),
                        "spline")
    v1 = grid.axis_points(2)
    v2 = grid.axis_points(3)
    mx = np.exp(-0.5 * (v1[:, None] ** 2 + v2[None, :] ** 2)) / (2 * np.pi)
    vals = np.broadcast_to(mx[None, None], (4, 4, 64, 64))
    rho = vpb.compute_density(vpb.DistributionField.from_values(grid, vals)).values.cpu().numpy()
    assert np.abs(rho - 1.0).max() <= 1e-7
    z = vpb.compute_density(vpb.DistributionField.zeros(grid)).values.cpu().numpy()
    assert np.array_equal(z, np.zeros((4, 4)))


def test_poisson_closed_forms():
    grid = vpb.GridSpec((vpb.Axis(0, 10 * np.pi, 40, "space"), vpb.Axis(0, 10 * np.pi, 40, "space"),
                         vpb.Axis(-6, 6, 4, "velocity"), vpb.Axis(-6, 6, 4, "velocity")), "spline")
    eps, k = 1e-3, 0.2
    x1 = grid.axis_points(0)[:, None]
    x2 = grid.axis_points(1)[None, :]
    rho = 1.0 + eps * np.cos(k * x1) * np.cos(k * x2)
    e = vpb.solve_poisson(vpb.DensityField(grid, rho))
    assert vpb.electric_energy(e) == pytest.approx(25 * np.pi ** 2 * eps ** 2 / (4 * k * k), rel=1e-11)
    e1 = (eps / (2 * k)) * np.sin(k * x1) * np.cos(k * x2)
    assert np.abs(e.components[0].cpu().numpy() - e1).max() <= 1e-12
    with pytest.warns(RuntimeWarning, match="unit background"):
        vpb.solve_poisson(vpb.DensityField(grid, np.full((40, 40), 1.5)))


def test_poisson_dg_coupling_single_mode_1d():
    grid = vpb.GridSpec((vpb.Axis(0, 4 * np.pi, 64, "space"), vpb.Axis(-6, 6, 4, "velocity")),
                        "dg", 5)
    x = grid.axis_points(0)
    e = vpb.solve_poisson(vpb.DensityField(grid, 1.0 + 0.5 * np.cos(0.5 * x)))
    assert np.abs(e.components[0].cpu().numpy() - np.sin(0.5 * x)).max() <= 1e-11


@pytest.mark.parametrize("axis,dofs", [
    (a, d) for a in (0, 1, 2, 3) for d in ((32, 64, 48, 128), (128, 32, 64, 48))]
    + [(0, (64, 16, 8, 8)), (0, (256, 8, 8, 4)), (0, (96, 16, 8, 4))])
def test_spline_pcr_axis_sweep_matches_reference_solver(axis, dofs):
    """Product spline sweeps use parallel cyclic reduction when the line length
    allows (n % 16 == 0, n >= 32); they agree with the reference's Thomas +
    Sherman-Morrison solve to round-off (<= 1e-14 of max|f|)."""
    prob = vpb.problem_spec("landau4d")
    grid = vpb.make_grid(prob, "spline", dofs)
    og = ogrid(grid)
    rng = np.random.default_rng(70 + axis)
    vals = rng.standard_normal(grid.dofs)
    h = grid.axes[axis].h
    nt = int(np.prod([grid.dof(a) for a in REF_AXES[axis]]))
    shifts = rng.uniform(-6.0, 6.0, nt) * h
    shifts[0] = 0.0
    ref = core.sweep(vals, og, axis, shifts, REF_AXES[axis], h)
    values = dev(vdg.reorder_table(grid, axis, shifts, REF_AXES[axis]))
    src = vpb.DistributionField.from_values(grid, vals)
    dst = torch.empty_like(src.data)
    lib = _lib.load()
    _lib.check(lib.vpb_spline_sweep_axis(axis, src.data.data_ptr(), dst.data_ptr(),
                                         _lib.dims(grid.dims4), values.data_ptr(), 1.0, h, None,
                                         _device.stream()), "spline")
    got = dst.view(src._phys.shape).permute(3, 2, 1, 0).cpu().numpy()
    assert max_rel(got, ref) <= 1e-14
