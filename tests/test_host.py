"""Host-side logic of the product package (no GPU needed).

Geometry, problem catalogue, table re-indexing, initial-data factors and
the transform matrices that parameterise the device field solve are all
checked against the oracle here; the kernels themselves are checked in the
``gpu``-marked suites.
"""

from __future__ import annotations

import math

import numpy as np
import pytest

import paper_1803_02143_b200 as vpb
from oracle import core
from paper_1803_02143_b200 import dg as vdg
from paper_1803_02143_b200 import driver, poisson
from paper_1803_02143_b200.grid import SPACE, VELOCITY


def ogrid(grid):
    return core.OGrid(tuple(a.lower for a in grid.axes), tuple(a.upper for a in grid.axes),
                      tuple(a.count for a in grid.axes), grid.method, grid.dg_degree)


@pytest.mark.parametrize("method,order", [("spline", 0), ("dg", 2), ("dg", 3), ("dg", 4)])
def test_points_and_weights_match_oracle(method, order):
    grid = vpb.make_grid(vpb.problem_spec("landau4d"), method, 24, dg_order=order)
    og = ogrid(grid)
    for a in range(4):
        assert np.array_equal(grid.axis_points(a), og.points(a))
        assert np.array_equal(grid.axis_weights(a), og.weights(a))


def test_problem_catalogue_and_methods():
    # test_driver.py:36-72 of the reference
    assert vpb.problem_spec("landau4d").ndim == 4
    ts = vpb.problem_spec("twostream4d")
    assert (ts.epsilon, ts.wavenumber, ts.drift) == (1e-3, 0.2, 2.4)
    with pytest.raises(ValueError):
        vpb.problem_spec("bump_on_tail")
    assert vpb.parse_method("spline") == ("spline", 0)
    assert vpb.parse_method("dg4") == ("dg", 3)
    for bad in ("dg0", "dg10", "cubic", "dg", "DG4"):
        with pytest.raises(ValueError):
            vpb.parse_method(bad)
    prob = vpb.problem_spec("landau4d")
    assert all(ax.count == 16 for ax in vpb.make_grid(prob, "dg", 64, dg_order=4).axes)
    assert vpb.make_grid(prob, "dg", 64, dg_order=6).axes[0].count == 11
    with pytest.raises(ValueError):
        vpb.make_grid(prob, "dg", 64)
    with pytest.raises(ValueError):
        vpb.make_grid(prob, "spline", (64, 64))


def test_axis_validation():
    with pytest.raises(ValueError):
        vpb.Axis(1.0, 0.0, 8, SPACE)
    with pytest.raises(ValueError):
        vpb.Axis(0.0, 1.0, 3, SPACE)
    with pytest.raises(ValueError):
        vpb.GridSpec((vpb.Axis(0, 1, 8, VELOCITY), vpb.Axis(0, 1, 8, SPACE)), "spline")


def test_baseline_config_grids():
    """BASELINE.json configs map onto these grids (degree-2 = dg_order 3)."""
    prob = vpb.problem_spec("landau4d")
    cfg1 = vpb.make_grid(prob, "dg", 48, dg_order=3)
    assert cfg1.dofs == (48,) * 4 and cfg1.axes[0].count == 16
    cfg2 = vpb.make_grid(prob, "dg", 192, dg_order=3)
    assert cfg2.total_dof == 192 ** 4
    cfg3 = vpb.make_grid(vpb.problem_spec("twostream4d_baseline"), "dg", 128, dg_order=2)
    assert cfg3.axes[0].count == 64 and cfg3.axes[0].upper == pytest.approx(10 * math.pi)
    cfg5 = vpb.make_grid(prob, "dg", 288, dg_order=3)
    assert cfg5.axes[0].count == 96


@pytest.mark.parametrize("prob", ["landau4d", "twostream4d", "twostream4d_baseline", "landau2d"])
@pytest.mark.parametrize("method,order", [("spline", 0), ("dg", 3)])
def test_separable_factors_reproduce_initial_data_bitwise(prob, method, order):
    problem = vpb.problem_spec(prob)
    dofs = 12 if problem.ndim == 4 else 24
    grid = vpb.make_grid(problem, method, dofs, dg_order=order)
    g1, g2, space = driver.separable_factors(problem, grid)
    # the device kernel computes (g2[iv2] * g1[iv1]) * space[x]
    phys = (g2[:, None] * g1[None, :]).reshape(-1)[:, None] * np.asarray(space).reshape(-1)[None, :]
    n = grid.dims4
    logical = phys.reshape(n[3], n[2], n[1], n[0]).transpose(3, 2, 1, 0)
    ref = core.initialize(prob, ogrid(grid))
    assert np.array_equal(logical.reshape(ref.shape), ref)


def test_initial_value_spot_checks():
    four = vpb.problem_spec("landau4d")
    assert vpb.initial_value(four, (0.0, 0.0, 0.0, 0.0)) == pytest.approx(1.0 / math.pi, rel=1e-14)
    stream = vpb.problem_spec("twostream4d")
    expected = (1.001 / (8.0 * math.pi)) * 4.0 * math.exp(-5.76)
    assert vpb.initial_value(stream, (0.0, 0.0, 0.0, 0.0)) == pytest.approx(expected, rel=1e-13)
    base = vpb.problem_spec("twostream4d_baseline")
    want = (1.002 / (2 * math.pi)) * math.exp(-2.88) * 1.0
    assert vpb.initial_value(base, (0.0, 0.0, 0.0, 0.0)) == pytest.approx(want, rel=1e-13)


@pytest.mark.parametrize("axis", [0, 1, 2, 3])
def test_reorder_table_matches_reference_line_indexing(axis):
    grid = vpb.make_grid(vpb.problem_spec("landau4d"), "dg", (6, 9, 12, 15), dg_order=3)
    og = ogrid(grid)
    ref_axes = {0: (2,), 1: (3,), 2: (0, 1), 3: (0, 1)}[axis]
    nt = int(np.prod([grid.dof(a) for a in ref_axes]))
    table = np.arange(nt, dtype=float) * 1.5 + 0.25
    dev = vdg.reorder_table(grid, axis, table, ref_axes)
    # per line: the reference's table entry
    ref_line = table[core.table_index(og, axis, ref_axes)]
    lead = tuple(grid.dof(a) for a in range(4) if a != axis)
    ref_line = ref_line.reshape(lead)
    # device row for each line
    want = vdg.device_table_axes(grid, axis)
    coords = np.meshgrid(*[np.arange(s) for s in lead], indexing="ij")
    other = [a for a in range(4) if a != axis]
    row = np.zeros(lead, dtype=np.int64)
    mult = 1
    for a in reversed(want):
        row += mult * coords[other.index(a)]
        mult *= grid.dof(a)
    assert np.array_equal(dev[row], ref_line)


def test_reorder_table_rejects_foreign_axes():
    grid = vpb.make_grid(vpb.problem_spec("landau4d"), "dg", 12, dg_order=3)
    with pytest.raises(ValueError):
        vdg.reorder_table(grid, 0, np.zeros(12), (1,))


@pytest.mark.parametrize("method,order,dofs", [("dg", 3, 24), ("dg", 2, 16), ("spline", 0, 16),
                                               ("dg", 4, 20)])
def test_transform_matrices_reproduce_reference_solve(method, order, dofs):
    """E = Re(M1 (K .* (G1 R G2^T)) M2^T) with the host-built matrices equals
    the reference's FFT solve (poisson.py:123-196) to round-off."""
    grid = vpb.make_grid(vpb.problem_spec("landau4d"), method, dofs, dg_order=order)
    og = ogrid(grid)
    rng = np.random.default_rng(3)
    x1 = grid.axis_points(0)[:, None]
    x2 = grid.axis_points(1)[None, :]
    rho = 1.0 + 0.3 * np.cos(0.5 * x1) * np.cos(x2) + 0.1 * np.sin(0.5 * x1 + 1.5 * x2)
    rho = rho + 1e-3 * rng.standard_normal(rho.shape)
    ref, _ = core.solve_poisson(rho, og)
    g1, m1, k1, c1 = poisson._axis_mats(grid, 0)
    g2, m2, k2, c2 = poisson._axis_mats(grid, 1)
    ksq = k1[:, None] ** 2 + k2[None, :] ** 2
    inv = np.zeros_like(ksq)
    np.divide(1.0, ksq, out=inv, where=ksq > 0)
    kd = [k1.copy(), k2.copy()]
    for kv, c in zip(kd, (c1, c2)):
        if c % 2 == 0:
            kv[c // 2] = 0.0
    rhat = g1 @ rho @ g2.T
    for d in range(2):
        kk = (-1j * (kd[0][:, None] if d == 0 else kd[1][None, :])) * inv
        e = (m1 @ (kk * rhat) @ m2.T).real
        assert np.abs(e - ref[d]).max() <= 1e-12 * max(1.0, np.abs(ref[d]).max())


def test_cli_free_api_surface_matches_reference_names():
    # names of /root/reference/pkg/src/slvp/__init__.py:11-91 on the hot path
    for name in ("Axis", "GridSpec", "DistributionField", "LayoutDescriptor", "DGAdvection",
                 "SplineAdvection", "DensityField", "ElectricField", "DiagnosticsRecord",
                 "ProblemSpec", "RunConfig", "SubstepError", "advect_line_dg",
                 "advect_line_spline", "available_backends", "backend_name", "set_backend",
                 "compute_density", "diagnostics", "electric_energy", "gauss_nodes",
                 "initialize", "line_sweep", "make_grid", "problem_spec", "projection_pair",
                 "read_snapshot", "run", "solve_poisson", "strang_step", "write_snapshot"):
        assert hasattr(vpb, name), name


def test_backend_registry_contract():
    assert vpb.available_backends() == ("cuda",)
    assert vpb.backend_name() == "cuda"
    with pytest.raises(ValueError, match="unknown backend 'fortran'"):
        vpb.set_backend("fortran")
    vpb.set_backend("cuda")


def test_substep_error_message():
    err = vpb.SubstepError("x1 half (open)", 0.1)
    assert str(err) == "non-finite values after sub-step 'x1 half (open)' at t=0.1"
    assert str(vpb.SubstepError("field solve")) == "non-finite values after sub-step 'field solve'"


def test_diagnostics_csv_and_meta_match_the_reference_cli_format(tmp_path):
    from paper_1803_02143_b200 import records
    from paper_1803_02143_b200.driver import DiagnosticsRecord

    recs = [DiagnosticsRecord(0.0, 1.0 / 3.0, 2.0, 2.5, 0.1, 1e-300, 1.0 / 3.0 + 1e-300),
            DiagnosticsRecord(0.05, 2.5e-7, 39.47841760435743, 39.4784176043574, 3.0, 1.5, 1.5)]
    out = tmp_path / "sub" / "run.csv"
    records.write_diagnostics_csv(out, recs)
    lines = out.read_text().split("\n")
    assert lines[0] == "time,electric_energy,mass,l1_norm,l2_norm,kinetic_energy,total_energy"
    for rec, line in zip(recs, lines[1:3]):
        assert line == ",".join(format(float(v), ".17g") for v in (
            rec.time, rec.electric_energy, rec.mass, rec.l1_norm, rec.l2_norm,
            rec.kinetic_energy, rec.total_energy))
    assert lines[2].startswith("0.050000000000000003,2.4999999999999999e-07,39.478417604357432,")
    assert lines[-1] == "" and len(lines) == 4
    records.write_meta(out, "run cfg.toml", {"tau": "0.05", "grid": "dg"}, ["synthetic"])
    meta = out.with_suffix(".meta").read_text().split("\n")
    assert meta[:3] == [f"version = {vpb.__version__}", "command = run cfg.toml", "backend = cuda"]
    assert meta[3:6] == ["grid = dg", "tau = 0.05", "note = synthetic"]


def test_bench_accounting_helpers():
    """bench.py: sweeps per launch of each kernel group label, per-config
    step defaults, and the committed ncu traffic lookup."""
    import importlib.util
    import json
    from pathlib import Path

    root = Path(__file__).resolve().parents[1]
    spec = importlib.util.spec_from_file_location("bench_mod", root / "bench.py")
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    assert bench.sweeps_per_launch("sweep_x12x12_rho") == 4
    assert bench.sweeps_per_launch("sweep_v12") == 2
    assert bench.sweeps_per_launch("sweep_x1x2") == 2
    assert bench.sweeps_per_launch("sweep_x1") == 1
    assert {k: v["nsteps"] for k, v in bench.CONFIGS.items()} == {
        "cfg1": 20, "cfg2": 100, "cfg3": 200, "cfg4": 50, "cfg5": 20}
    traffic = json.loads((root / "profiles" / "traffic.json").read_text())
    got = bench.load_traffic("cfg2", "sweep_x12x12_rho")
    assert got == float(traffic["cfg2"]["sweep_x12x12_rho"]["dram_bytes_per_launch"])
    assert bench.load_traffic("cfg2", "no_such_kernel") is None
