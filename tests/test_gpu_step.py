"""Step-level parity of the device Strang step against the reference.

North-star bars (BASELINE.json): per-step max relative error in f <= 1e-12,
electric-energy series within 1e-10 relative, mass conserved to 1e-13.
Runs on the B200 box: ``pytest -m gpu``.
"""

from __future__ import annotations

import math

import numpy as np
import pytest
import torch

import paper_1803_02143_b200 as vpb
from oracle import core
from paper_1803_02143_b200 import driver
from vpb_testutil import max_rel

pytestmark = pytest.mark.gpu

F_TOL = 1e-12
EE_TOL = 1e-10
MASS_TOL = 1e-13

STEP_CASES = [
    ("landau4d_dg3", "landau4d", "dg", 12, 3, 0.1),
    ("landau4d_dg4", "landau4d", "dg", 16, 4, 0.1),
    ("landau4d_spline", "landau4d", "spline", 12, 0, 0.1),
    ("twostream_dg2", "twostream4d_baseline", "dg", 12, 2, 0.1),
    ("twostream_ref_dg3", "twostream4d", "dg", 12, 3, 0.1),
    ("landau2d_dg4", "landau2d", "dg", 32, 4, 0.1),
    ("landau2d_spline", "landau2d", "spline", 32, 0, 0.1),
]
KEYS = ("time", "electric_energy", "mass", "l1_norm", "l2_norm", "kinetic_energy", "total_energy")


@pytest.mark.parametrize("tag,prob,method,dofs,order,tau", STEP_CASES)
def test_steps_match_reference_golden(golden, tag, prob, method, dofs, order, tau):
    z = golden("steps")
    states, recs = z[tag + "_f"], z[tag + "_rec"]
    problem = vpb.problem_spec(prob)
    grid = vpb.make_grid(problem, method, dofs, dg_order=order)
    field = vpb.initialize(problem, grid)
    assert np.array_equal(field.numpy(), states[0])
    for m in range(1, states.shape[0]):
        field = vpb.strang_step(field, tau, consume=True)
        assert max_rel(field.numpy(), states[m]) <= F_TOL, (tag, m)
        rec = vpb.diagnostics(field, m * tau)
        ee_ref = recs[m][1]
        assert abs(rec.electric_energy - ee_ref) <= EE_TOL * abs(ee_ref), (tag, m)
        for k, ref in zip(KEYS, recs[m]):
            assert getattr(rec, k) == pytest.approx(ref, rel=1e-11), (tag, m, k)


def _oracle_run(prob, method, dofs, order, tau, nsteps):
    og = core.make_grid(prob, method, dofs, order)
    f = core.initialize(prob, og)
    for _ in range(nsteps):
        f = core.strang_step(f, og, tau)
        yield f, og


def test_config1_parity_20_steps(golden):
    """BASELINE config 1: Landau 4D, 16^4 cells, degree 2, dt=0.1, 20 steps.
    f per step vs the live oracle (bitwise-pinned to the reference), EE and
    mass series vs the reference's own series."""
    z = golden("series")
    recs, sums = z["cfg1_rec"], z["cfg1_sums"]
    problem = vpb.problem_spec("landau4d")
    grid = vpb.make_grid(problem, "dg", 48, dg_order=3)
    field = vpb.initialize(problem, grid)
    rec0 = vpb.diagnostics(field, 0.0)
    m0 = rec0.mass
    worst = 0.0
    for m, (ref, _) in enumerate(_oracle_run("landau4d", "dg", 48, 3, 0.1, 20), start=1):
        field = vpb.strang_step(field, 0.1, consume=True, time_label=m * 0.1)
        got = field.numpy()
        err = max_rel(got, ref)
        worst = max(worst, err)
        assert err <= F_TOL, (m, err)
        np.testing.assert_allclose([got.sum(), (got * got).sum(), np.abs(got).max()],
                                   sums[m - 1], rtol=1e-12)
        rec = vpb.diagnostics(field, m * 0.1)
        assert abs(rec.electric_energy - recs[m][1]) <= EE_TOL * abs(recs[m][1]), m
        assert abs(rec.mass - m0) <= MASS_TOL * m0, m
    print(f"config1 worst per-step max-rel error in f: {worst:.3e}")


@pytest.mark.parametrize("tag,prob,method,dofs,order,nsteps", [
    ("cfg3_small", "twostream4d_baseline", "dg", 32, 2, 20),
    ("cfg4_small", "landau4d", "spline", 32, 0, 10),
])
def test_reduced_configs_energy_series(golden, tag, prob, method, dofs, order, nsteps):
    z = golden("series")
    recs = z[tag + "_rec"]
    problem = vpb.problem_spec(prob)
    grid = vpb.make_grid(problem, method, dofs, dg_order=order)
    field = vpb.initialize(problem, grid)
    m0 = vpb.diagnostics(field).mass
    for m in range(1, nsteps + 1):
        field = vpb.strang_step(field, 0.1, consume=True)
        rec = vpb.diagnostics(field, m * 0.1)
        assert abs(rec.electric_energy - recs[m][1]) <= EE_TOL * abs(recs[m][1]), (tag, m)
        assert abs(rec.mass - m0) <= MASS_TOL * abs(m0) * 10, (tag, m)


def test_run_loop_records_and_snapshots(tmp_path):
    prob = vpb.problem_spec("landau4d")
    grid = vpb.make_grid(prob, "dg", 12, dg_order=3)
    cfg = vpb.RunConfig(problem=prob, grid=grid, tau=0.1, t_end=0.5, snapshot_times=(0.0, 0.3),
                        snapshot_stem=str(tmp_path / "snap"), diag_every=2)
    records, snaps = vpb.run(cfg)
    np.testing.assert_allclose([r.time for r in records], [0.0, 0.2, 0.4], atol=1e-12)
    assert [t for t, _ in snaps] == [0.0, 0.3]
    assert (tmp_path / "snap_t0.vlf").exists() and (tmp_path / "snap_t0.3.vlf").exists()
    back = vpb.read_snapshot(tmp_path / "snap_t0.3.vlf")
    assert np.array_equal(back.numpy(), snaps[1][1].numpy())
    with pytest.raises(ValueError):
        vpb.run(vpb.RunConfig(problem=prob, grid=grid, tau=0.1, t_end=0.25))


def test_run_is_deterministic_and_strategy_independent():
    prob = vpb.problem_spec("landau4d")
    grid = vpb.make_grid(prob, "dg", 24, dg_order=3)
    outs = []
    for strategy in ("strided", "transpose", "strided"):
        f = vpb.initialize(prob, grid, strategy=strategy)
        for _ in range(3):
            f = vpb.strang_step(f, 0.1, consume=True)
        outs.append(f.numpy())
    assert np.array_equal(outs[0], outs[1]) and np.array_equal(outs[0], outs[2])


def test_step_without_consume_leaves_input():
    prob = vpb.problem_spec("landau4d")
    grid = vpb.make_grid(prob, "spline", 12)
    f = vpb.initialize(prob, grid)
    before = f.numpy()
    g = vpb.strang_step(f, 0.1)
    assert np.array_equal(f.numpy(), before)
    assert not np.array_equal(g.numpy(), before)


def test_step_reports_first_nonfinite_substep():
    prob = vpb.problem_spec("landau4d")
    grid = vpb.make_grid(prob, "spline", 8)
    f = vpb.initialize(prob, grid)
    f.array[0, 0, 0, 0] = math.inf
    with pytest.raises(vpb.SubstepError, match="x1 half"):
        vpb.strang_step(f, 0.1)
    two = vpb.problem_spec("landau2d")
    g2 = vpb.make_grid(two, "dg", 16, dg_order=2)
    f2 = vpb.initialize(two, g2)
    f2.array[3, 3] = math.nan
    with pytest.raises(vpb.SubstepError, match=r"sub-step 'x half \(open\)' at t=0\.1"):
        vpb.strang_step(f2, 0.1, time_label=0.1)


def test_step_reports_broken_field_solve(monkeypatch):
    prob = vpb.problem_spec("landau4d")
    grid = vpb.make_grid(prob, "dg", 12, dg_order=3)
    f = vpb.initialize(prob, grid)
    real = driver.solve_into

    def poisoned(rho, grid_, e, stats, flag, **kw):
        real(rho, grid_, e, stats, flag, **kw)
        e.fill_(math.nan)
        if flag is not None:
            flag.fill_(1)

    monkeypatch.setattr(driver, "solve_into", poisoned)
    with pytest.raises(vpb.SubstepError, match="field solve"):
        vpb.strang_step(f, 0.1)


def test_identity_without_field():
    flat = vpb.ProblemSpec("landau4d", ((0.0, 4 * math.pi),) * 2, ((-6.0, 6.0),) * 2, 0.0, 0.5)
    grid = vpb.make_grid(flat, "dg", 16, dg_order=4)
    before = vpb.initialize(flat, grid)
    after = vpb.strang_step(before, 0.1)
    scale = np.abs(before.numpy()).max()
    assert np.abs(after.numpy() - before.numpy()).max() <= 1e-13 * scale


def test_dg_l2_norm_never_grows():
    prob = vpb.problem_spec("landau4d")
    grid = vpb.make_grid(prob, "dg", 24, dg_order=3)
    f = vpb.initialize(prob, grid)
    vals = [vpb.diagnostics(f).l2_norm]
    for _ in range(5):
        f = vpb.strang_step(f, 0.1, consume=True)
        vals.append(vpb.diagnostics(f).l2_norm)
    assert all(c <= p * (1 + 1e-12) for p, c in zip(vals, vals[1:]))


# ---- reference kernel-test mirrors (per-line API) -------------------------
@pytest.mark.parametrize("m", [2, -3, 8, -11])
def test_advect_whole_cell_shift_rolls_bitwise(m):
    rng = np.random.default_rng(50 + abs(m))
    line = rng.standard_normal(8 * 4)
    out = vpb.advect_line_dg(line, m * 0.5, 0.5, 3)
    assert np.array_equal(out, np.roll(line.reshape(8, 4), m, axis=0).ravel())


def test_advect_near_integer_and_constants_and_mass():
    rng = np.random.default_rng(53)
    line = rng.standard_normal(32)
    out = vpb.advect_line_dg(line, -3 * 0.7, 0.7, 3)
    assert np.abs(out - np.roll(line.reshape(8, 4), -3, axis=0).ravel()).max() <= 1e-12
    for degree in range(4):
        out = vpb.advect_line_dg(np.full(6 * (degree + 1), 2.5), 0.213, 0.5, degree)
        np.testing.assert_allclose(out, 2.5, rtol=1e-13)
    for seed in range(5):
        r = np.random.default_rng(700 + seed)
        degree = int(r.integers(0, 4))
        line = r.standard_normal(8 * (degree + 1))
        shift = float(r.uniform(-5, 5))
        _, w = vpb.gauss_nodes(degree + 1)
        mass = lambda v: float(w @ v.reshape(8, -1).T @ np.ones(8))  # noqa: E731
        out = vpb.advect_line_dg(line, shift, 1.0, degree)
        assert abs(mass(out) - mass(line)) <= 1e-12 * max(1.0, abs(mass(line)))
    with pytest.raises(ValueError):
        vpb.advect_line_dg(np.ones(7), 0.1, 1.0, 1)


@pytest.mark.parametrize("m", [1, 3, -2, 13, -45])
def test_spline_integer_shift_is_circular(m):
    rng = np.random.default_rng(400 + abs(m))
    u = rng.standard_normal(16)
    out = vpb.advect_line_spline(u, m * 0.3, 0.3)
    assert np.abs(out - np.roll(u, m)).max() <= 1e-13 * np.abs(u).max()


def test_spline_line_sum_and_wrap_and_symbol():
    for seed in range(5):
        r = np.random.default_rng(900 + seed)
        u = r.standard_normal(48)
        out = vpb.advect_line_spline(u, float(r.uniform(-20, 20)), 0.2)
        assert abs(out.sum() - u.sum()) <= 1e-12 * max(1.0, abs(u.sum()))
    u = np.random.default_rng(17).standard_normal(16)
    base = vpb.advect_line_spline(u, 1.3, 0.5)
    assert np.abs(base - vpb.advect_line_spline(u, 1.3 + 7 * 8.0, 0.5)).max() <= 1e-11
    n = 32
    x = np.arange(n)
    for mode in range(n):
        re = vpb.advect_line_spline(np.cos(2 * np.pi * mode * x / n), 0.37, 1.0)
        im = vpb.advect_line_spline(np.sin(2 * np.pi * mode * x / n), 0.37, 1.0)
        assert np.sqrt(re ** 2 + im ** 2).max() <= 1.0 + 1e-12


def test_plugin_entry_points_with_torch_current_stream():
    """The step runs on torch's current stream (side stream honoured)."""
    prob = vpb.problem_spec("landau4d")
    grid = vpb.make_grid(prob, "dg", 12, dg_order=3)
    ref = vpb.strang_step(vpb.initialize(prob, grid), 0.1).numpy()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        f = vpb.initialize(prob, grid)
        g = vpb.strang_step(f, 0.1)
        got = g.numpy()
    assert np.array_equal(got, ref)


@pytest.mark.parametrize("order,dofs", [(3, (24, 18, 12, 15)), (2, (16, 12, 8, 10)),
                                        (4, (16, 20, 12, 8)), (1, (12, 10, 8, 6))])
def test_fused_x_planes_bitwise_equal_to_separate_sweeps(monkeypatch, order, dofs):
    """vpb_dg_sweep_xplane == x1 sweep then x2 sweep, bit for bit, over steps."""
    prob = vpb.problem_spec("landau4d")
    grid = vpb.make_grid(prob, "dg", dofs, dg_order=order)
    outs = []
    monkeypatch.setattr(driver, "FUSE_RHO", False)  # same density path in both runs
    for fused in (False, True):
        monkeypatch.setattr(driver, "FUSE_X", fused)
        driver._state_cached.cache_clear()
        f = vpb.initialize(prob, grid)
        for _ in range(3):
            f = vpb.strang_step(f, 0.37, consume=True)
        assert driver.step_state(grid).fused_x == fused
        outs.append(f.numpy())
    driver._state_cached.cache_clear()
    assert np.array_equal(outs[0], outs[1])


@pytest.mark.parametrize("order,dofs", [(3, (24, 18, 12, 15)), (2, (16, 12, 8, 10)),
                                        (4, (16, 20, 12, 8)), (1, (12, 10, 8, 6))])
def test_fused_v_columns_bitwise_equal_to_separate_sweeps(monkeypatch, order, dofs):
    """vpb_dg_sweep_vplane == v1 sweep then v2 sweep, bit for bit, over steps."""
    prob = vpb.problem_spec("landau4d")
    grid = vpb.make_grid(prob, "dg", dofs, dg_order=order)
    outs = []
    for fused in (False, True):
        monkeypatch.setattr(driver, "FUSE_V", fused)
        driver._state_cached.cache_clear()
        f = vpb.initialize(prob, grid)
        for _ in range(3):
            f = vpb.strang_step(f, 0.37, consume=True)
        assert driver.step_state(grid).fused_v == fused
        outs.append(f.numpy())
    driver._state_cached.cache_clear()
    assert np.array_equal(outs[0], outs[1])


@pytest.mark.parametrize("order,dofs", [(3, (24, 18, 12, 15)), (2, (16, 12, 8, 10)),
                                        (4, (16, 20, 12, 8))])
def test_density_epilogue_matches_separate_density(monkeypatch, order, dofs):
    """The opening x pass's cell-centre density epilogue replaces compute_density +
    collapse; only the summation order changes (<= 1e-14 after several steps)."""
    prob = vpb.problem_spec("landau4d")
    grid = vpb.make_grid(prob, "dg", dofs, dg_order=order)
    outs, e = [], []
    for fused in (False, True):
        monkeypatch.setattr(driver, "FUSE_RHO", fused)
        driver._state_cached.cache_clear()
        f = vpb.initialize(prob, grid)
        for _ in range(4):
            f = vpb.strang_step(f, 0.37, consume=True)
        st = driver.step_state(grid)
        assert st.fused_rho == fused
        outs.append(f.numpy())
        e.append(st.e.cpu().numpy())
    driver._state_cached.cache_clear()
    assert max_rel(outs[1], outs[0]) <= 1e-14
    assert max_rel(e[1], e[0]) <= 1e-13


def test_density_epilogue_keeps_neutrality_warning(monkeypatch):
    prob = vpb.problem_spec("landau4d")
    grid = vpb.make_grid(prob, "dg", 12, dg_order=3)
    monkeypatch.setattr(driver, "FUSE_RHO", True)
    driver._state_cached.cache_clear()
    f = vpb.DistributionField.from_values(grid, np.full(grid.dofs, 0.25))
    assert driver.step_state(grid).fused_rho
    with pytest.warns(RuntimeWarning, match="unit background"):
        vpb.strang_step(f, 0.1)
    driver._state_cached.cache_clear()


@pytest.mark.parametrize("prob,method,dofs,order", [
    ("landau4d", "dg", 24, 3), ("landau4d", "spline", 16, 0), ("landau2d", "dg", 32, 4),
    ("twostream4d_baseline", "dg", 16, 2)])
def test_step_graph_replays_bitwise_equal_to_eager_steps(prob, method, dofs, order):
    problem = vpb.problem_spec(prob)
    grid = vpb.make_grid(problem, method, dofs, dg_order=order)
    f_eager = vpb.initialize(problem, grid)
    f_graph = vpb.initialize(problem, grid)
    for _ in range(1):  # StepGraph's constructor performs one eager step
        f_eager = vpb.strang_step(f_eager, 0.1, consume=True)
    g = driver.StepGraph(f_graph, 0.1)
    for m in range(4):
        f_eager = vpb.strang_step(f_eager, 0.1, consume=True)
        g.step()
        assert np.array_equal(f_graph.numpy(), f_eager.numpy()), m
    f_graph.data[7] = math.nan
    with pytest.raises(vpb.SubstepError):
        g.step()


@pytest.mark.parametrize("prob,method,dofs,order,k", [
    ("landau4d", "dg", 24, 3, 3), ("landau4d", "dg", 24, 3, 2), ("landau4d", "spline", 16, 0, 3),
    ("landau2d", "dg", 32, 4, 3), ("twostream4d_baseline", "dg", 16, 2, 4)])
def test_advance_graph_replays_bitwise_equal_to_advance(prob, method, dofs, order, k):
    """driver.AdvanceGraph: K-step blocks of advance() from CUDA graphs
    (both buffer parities when a block swaps an odd number of times)."""
    problem = vpb.problem_spec(prob)
    grid = vpb.make_grid(problem, method, dofs, dg_order=order)
    f_eager = vpb.initialize(problem, grid)
    f_graph = vpb.initialize(problem, grid)
    f_eager = vpb.advance(f_eager, 0.1, k, consume=True)  # the constructor's eager block
    g = vpb.AdvanceGraph(f_graph, 0.1, k)
    for b in range(3):
        f_eager = vpb.advance(f_eager, 0.1, k, consume=True)
        assert g.advance() is f_graph
        assert np.array_equal(f_graph.numpy(), f_eager.numpy()), b
    f_graph.data[7] = math.nan
    with pytest.raises(vpb.SubstepError):
        g.advance(first_step=4 * k)


def test_fused_v_reports_nonfinite_field_in_v1():
    prob = vpb.problem_spec("landau4d")
    grid = vpb.make_grid(prob, "dg", 12, dg_order=3)
    f = vpb.initialize(prob, grid)
    st = driver.step_state(grid)
    assert st.fused_v
    out = torch.empty_like(f.data)
    flags = torch.zeros(2, dtype=torch.int32, device="cuda")
    e = torch.full((144,), 0.3, dtype=torch.float64, device="cuda")
    t1 = driver.DeviceTables(e, 0.1, grid.axes[2].h, 2)
    t2 = driver.DeviceTables(e, 0.1, grid.axes[3].h, 2)
    bad = f.data.clone()
    bad[1000] = math.inf
    driver.vplane_dg(grid, bad, out, t1, t2, flags[0:1], flags[1:2])
    assert flags.tolist() == [1, 1]


def test_fused_x_reports_nonfinite_in_x1_and_x2():
    prob = vpb.problem_spec("landau4d")
    grid = vpb.make_grid(prob, "dg", 12, dg_order=3)
    f = vpb.initialize(prob, grid)
    f.array[5, 6, 7, 8] = math.nan
    with pytest.raises(vpb.SubstepError, match=r"x1 half \(open\)"):
        vpb.strang_step(f, 0.1)


# ---------------------------------------------------------------------------
# merged x half steps of consecutive steps (vpb_dg_sweep_xplane2, advance)
# ---------------------------------------------------------------------------
ADVANCE_CASES = [
    (3, (24, 18, 12, 15), 0.37),    # one output chunk per plane
    (3, (192, 24, 6, 6), 0.37),     # G = 1: many chunks per plane
    (3, (192, 24, 6, 6), 2.9),      # |q| of several cells, wrapped loads
    (2, (128, 22, 4, 6), 0.37),     # G = 2 with a partial last chunk
    (2, (128, 22, 4, 6), 5.0),
    (4, (16, 20, 12, 8), 0.37),
    (1, (12, 10, 8, 6), 0.37),
    (3, (24, 18, 15, 12), 0.37),    # v1 = 0 plane: alpha == 0 (exact shift) along x1
    (2, (16, 12, 6, 10), 0.0),      # tau = 0: every row an exact shift
    (5, (20, 15, 10, 10), 0.37),    # high orders (register spills in the fused passes)
    (7, (28, 14, 14, 7), 0.6),
    (9, (18, 18, 9, 9), 0.37),
]


@pytest.mark.parametrize("order,dofs,tau", ADVANCE_CASES)
def test_advance_bitwise_equal_to_strang_steps(monkeypatch, order, dofs, tau):
    """"exact" arithmetic: K steps with merged x half steps == K separate
    strang_step calls, bit for bit (separate density pass in both, so every
    reduction is the same)."""
    prob = vpb.problem_spec("landau4d")
    grid = vpb.make_grid(prob, "dg", dofs, dg_order=order)
    monkeypatch.setattr(driver, "FUSE_RHO", False)
    monkeypatch.setattr(driver, "ARITH", "exact")
    driver._state_cached.cache_clear()
    f1 = vpb.initialize(prob, grid)
    for _ in range(4):
        f1 = vpb.strang_step(f1, tau, consume=True)
    f2 = vpb.advance(vpb.initialize(prob, grid), tau, 4)
    assert driver.step_state(grid).fused_x
    driver._state_cached.cache_clear()
    assert np.array_equal(f1.numpy(), f2.numpy())


@pytest.mark.parametrize("order,dofs,tau", ADVANCE_CASES)
def test_advance_fast_arithmetic_matches_strang_steps(monkeypatch, order, dofs, tau):
    """"fast" arithmetic (composed three-cell stencils, vpb_dg_sweep_xcomp):
    K merged steps == K strang_step calls up to round-off."""
    prob = vpb.problem_spec("landau4d")
    grid = vpb.make_grid(prob, "dg", dofs, dg_order=order)
    monkeypatch.setattr(driver, "FUSE_RHO", False)
    monkeypatch.setattr(driver, "ARITH", "fast")
    driver._state_cached.cache_clear()
    f1 = vpb.initialize(prob, grid)
    for _ in range(4):
        f1 = vpb.strang_step(f1, tau, consume=True)
    f2 = vpb.advance(vpb.initialize(prob, grid), tau, 4)
    driver._state_cached.cache_clear()
    a, b = f1.numpy(), f2.numpy()
    assert max_rel(b, a) <= 1e-14
    if tau == 0.0:
        assert np.array_equal(a, b)  # exact shifts stay copies
    # mass: the composed projections conserve it like the separate ones
    m1, m2 = vpb.diagnostics(f1).mass, vpb.diagnostics(f2).mass
    assert abs(m2 - m1) <= 1e-14 * abs(m1)


def test_composed_tables_are_the_matrix_products():
    prob = vpb.problem_spec("landau4d")
    grid = vpb.make_grid(prob, "dg", (24, 18, 15, 12), dg_order=3)
    st = driver.step_state(grid)
    for d in (0, 1):
        t = st.x_tables(d, 0.37)
        a, b = t.a.cpu().numpy(), t.b.cpu().numpy()
        k = t.composed().cpu().numpy()
        np.testing.assert_allclose(k[:, 0], a @ a, rtol=0, atol=1e-15)
        np.testing.assert_allclose(k[:, 1], a @ b + b @ a, rtol=0, atol=1e-15)
        np.testing.assert_allclose(k[:, 2], b @ b, rtol=0, atol=1e-15)


@pytest.mark.parametrize("arith", ["fast", "exact"])
@pytest.mark.parametrize("order,dofs,tau", ADVANCE_CASES[:5])
def test_advance_with_density_epilogues(monkeypatch, order, dofs, tau, arith):
    """With the density folded into the x passes only the density summation
    order (and, for "fast", the composed stencils' rounding) differs between
    the single and the merged pass."""
    prob = vpb.problem_spec("landau4d")
    grid = vpb.make_grid(prob, "dg", dofs, dg_order=order)
    monkeypatch.setattr(driver, "FUSE_RHO", True)
    monkeypatch.setattr(driver, "ARITH", arith)
    driver._state_cached.cache_clear()
    f1 = vpb.initialize(prob, grid)
    for _ in range(4):
        f1 = vpb.strang_step(f1, tau, consume=True)
    f2 = vpb.advance(vpb.initialize(prob, grid), tau, 4)
    assert driver.step_state(grid).fused_rho
    driver._state_cached.cache_clear()
    assert max_rel(f2.numpy(), f1.numpy()) <= 1e-13


@pytest.mark.parametrize("arith", ["fast", "exact"])
def test_advance_config1_parity_vs_oracle(monkeypatch, arith):
    """BASELINE config 1, 10 merged steps vs the oracle: north-star bar."""
    monkeypatch.setattr(driver, "ARITH", arith)
    prob, method, dofs, order, tau = "landau4d", "dg", 48, 3, 0.1
    for ref, _ in _oracle_run(prob, method, dofs, order, tau, 10):
        pass
    problem = vpb.problem_spec(prob)
    grid = vpb.make_grid(problem, method, dofs, dg_order=order)
    f = vpb.advance(vpb.initialize(problem, grid), tau, 10)
    assert max_rel(f.numpy(), ref) <= F_TOL


def test_double_x_pass_flags_every_substep():
    prob = vpb.problem_spec("landau4d")
    grid = vpb.make_grid(prob, "dg", (192, 24, 6, 6), dg_order=3)
    f = vpb.initialize(prob, grid)
    st = driver.step_state(grid)
    bad = f.data.clone()
    bad[12345] = math.nan
    out = torch.empty_like(bad)
    flags = torch.zeros(4, dtype=torch.int32, device="cuda")
    t1, t2 = st.x_tables(0, 0.37), st.x_tables(1, 0.37)
    driver.xplane2_dg(grid, bad, out, t1, t2, (flags[0:1], flags[1:2]), (flags[2:3], flags[3:4]))
    assert flags.tolist() == [1, 1, 1, 1]
    flags.zero_()
    driver.xplane2_dg(grid, f.data, out, t1, t2, (flags[0:1], flags[1:2]),
                      (flags[2:3], flags[3:4]))
    assert flags.tolist() == [0, 0, 0, 0]


def test_composed_x_pass_flags_nonfinite_output():
    prob = vpb.problem_spec("landau4d")
    grid = vpb.make_grid(prob, "dg", (192, 24, 6, 6), dg_order=3)
    f = vpb.initialize(prob, grid)
    st = driver.step_state(grid)
    bad = f.data.clone()
    bad[12345] = math.nan
    out = torch.empty_like(bad)
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")
    t1, t2 = st.x_tables(0, 0.37), st.x_tables(1, 0.37)
    driver.xcomp_dg(grid, bad, out, t1, t2, flag)
    assert flag.item() == 1
    flag.zero_()
    driver.xcomp_dg(grid, f.data, out, t1, t2, flag)
    assert flag.item() == 0


def test_advance_reports_first_nonfinite_substep_with_time_label():
    prob = vpb.problem_spec("landau4d")
    grid = vpb.make_grid(prob, "dg", 24, dg_order=3)
    f = vpb.initialize(prob, grid)
    f.array[5, 6, 7, 8] = math.nan
    with pytest.raises(vpb.SubstepError, match=r"x1 half \(open\)") as err:
        vpb.advance(f, 0.1, 3, first_step=4)
    assert "0.4" in str(err.value)


def test_run_with_sparse_diagnostics_matches_every_step_records():
    prob = vpb.problem_spec("landau4d")
    grid = vpb.make_grid(prob, "dg", 24, dg_order=3)
    cfg1 = vpb.RunConfig(problem=prob, grid=grid, tau=0.1, t_end=0.6, diag_every=1)
    cfg3 = vpb.RunConfig(problem=prob, grid=grid, tau=0.1, t_end=0.6, diag_every=3,
                         snapshot_times=(0.5,))
    rec1, _ = vpb.run(cfg1)
    rec3, snaps = vpb.run(cfg3)
    assert [r.time for r in rec3] == pytest.approx([0.0, 0.3, 0.6])
    for r in rec3:
        r1 = next(x for x in rec1 if abs(x.time - r.time) < 1e-12)
        for k in KEYS[1:]:
            assert getattr(r, k) == pytest.approx(getattr(r1, k), rel=1e-12, abs=1e-300), k
    assert snaps[0][0] == pytest.approx(0.5)


@pytest.mark.parametrize("order,dofs", [(3, (24, 18, 12, 15)), (2, (128, 22, 4, 6)),
                                        (3, (192, 24, 6, 6))])
def test_advance_record_matches_diagnostics_of_the_final_state(order, dofs):
    """The closing pass's diagnostics epilogue == diagnostics() of the state."""
    prob = vpb.problem_spec("landau4d")
    grid = vpb.make_grid(prob, "dg", dofs, dg_order=order)
    f, rec = vpb.advance(vpb.initialize(prob, grid), 0.37, 3, record_time=1.11)
    assert driver.step_state(grid).fused_rho
    ref = vpb.diagnostics(f, 1.11)
    assert rec.time == ref.time
    for k in KEYS[1:]:
        assert getattr(rec, k) == pytest.approx(getattr(ref, k), rel=1e-12, abs=1e-300), k


@pytest.mark.parametrize("prob,method,dofs,order", [
    ("landau4d", "spline", 16, 0), ("landau2d", "dg", 32, 4), ("landau2d", "spline", 32, 0)])
def test_advance_without_fused_x_pass_equals_strang_steps(monkeypatch, prob, method, dofs,
                                                          order):
    """Grids without the fused x pass (spline, 1x1v) run advance() as plain
    steps ("exact" arithmetic): bitwise the strang_step loop, records via
    diagnostics()."""
    monkeypatch.setattr(driver, "ARITH", "exact")
    problem = vpb.problem_spec(prob)
    grid = vpb.make_grid(problem, method, dofs, dg_order=order)
    f1 = vpb.initialize(problem, grid)
    for _ in range(3):
        f1 = vpb.strang_step(f1, 0.1, consume=True)
    f2, rec = vpb.advance(vpb.initialize(problem, grid), 0.1, 3, record_time=0.3)
    assert np.array_equal(f1.numpy(), f2.numpy())
    ref = vpb.diagnostics(f1, 0.3)
    for k in KEYS:
        assert getattr(rec, k) == getattr(ref, k), k


# ---------------------------------------------------------------------------
# spline: merged x half steps as one double sweep per axis (vpb_spline_sweep_axis2)
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("prob,dofs,tau", [
    ("landau4d", (32, 64, 32, 48), 0.1),      # rows kernel NPT 1, strided tiles
    ("landau4d", (128, 32, 48, 32), 0.37),    # NPT 4, |shift| of several points
    ("landau4d", (256, 48, 32, 32), 0.1),     # NPT 8, density epilogue (one v1 block)
    ("landau4d", (64, 32, 96, 16), 0.37),     # density epilogue over three v1 blocks
    ("landau2d", (64, 96), 0.2),              # 1x1v: contiguous x
])
def test_spline_double_sweep_advance_matches_strang_steps(monkeypatch, prob, dofs, tau):
    monkeypatch.setattr(driver, "ARITH", "fast")
    problem = vpb.problem_spec(prob)
    grid = vpb.make_grid(problem, "spline", dofs)
    driver._state_cached.cache_clear()
    assert driver.step_state(grid).spline_x2
    f1 = vpb.initialize(problem, grid)
    for _ in range(4):
        f1 = vpb.strang_step(f1, tau, consume=True)
    f2 = vpb.advance(vpb.initialize(problem, grid), tau, 4)
    driver._state_cached.cache_clear()
    a, b = f1.numpy(), f2.numpy()
    assert max_rel(b, a) <= 1e-13


@pytest.mark.parametrize("dofs", [(64, 32, 64, 16), (128, 32, 32, 8), (96, 32, 32, 16)])
def test_spline_x1_double_sweep_density_epilogue(dofs):
    """vpb_spline_sweep_x1dbl_density: the x1 double sweep with the density
    of its output as an epilogue equals the plain double sweep (the lines run
    on other lanes, so a line's start point, and with it the rounding, may
    differ) and vpb_density of that output."""
    from paper_1803_02143_b200 import _device, _lib
    from paper_1803_02143_b200.poisson import density_into
    from paper_1803_02143_b200.spline import sweep_spline2, sweep_spline2_density
    prob = vpb.problem_spec("landau4d")
    grid = vpb.make_grid(prob, "spline", dofs)
    f = vpb.initialize(prob, grid)
    rng = np.random.default_rng(11)
    f.data.copy_(torch.from_numpy(rng.standard_normal(f.data.numel())))
    st = driver.step_state(grid)
    assert st.spline_rho
    vals, h = st.vpoints[0], grid.axes[0].h
    d1 = torch.empty_like(f.data)
    sweep_spline2(grid, 0, f.data, d1, vals, 0.37, h, None)
    rho1 = torch.empty(grid.dof(0) * grid.dof(1), dtype=torch.float64, device="cuda")
    density_into(d1, grid, rho1)
    d2 = torch.full_like(f.data, float("nan"))
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")
    st.spart.fill_(float("nan"))
    sweep_spline2_density(grid, f.data, d2, vals, 0.37, h, flag, st.wv1, st.spart)
    rho2 = torch.empty_like(rho1)
    lib = _lib.load()
    _lib.check(lib.vpb_density(st.spart.data_ptr(), _lib.dims(st.spart_dims),
                               st.spart_w1.data_ptr(), st.wv2.data_ptr(), rho2.data_ptr(),
                               st.spart_work.data_ptr(), _device.stream()), "vpb_density")
    assert flag.item() == 0
    a, b = d1.cpu().numpy(), d2.cpu().numpy()
    assert np.isfinite(b).all()
    assert np.max(np.abs(a - b)) <= 1e-14 * np.max(np.abs(a))
    r1, r2 = rho1.cpu().numpy(), rho2.cpu().numpy()
    assert np.max(np.abs(r1 - r2)) <= 1e-13 * np.max(np.abs(r1))
    # deterministic: a second run is bitwise the same
    d3 = torch.empty_like(f.data)
    part2 = st.spart.clone()
    sweep_spline2_density(grid, f.data, d3, vals, 0.37, h, flag, st.wv1, st.spart)
    assert torch.equal(d2, d3) and torch.equal(part2, st.spart)


def test_spline_density_epilogue_advance_equals_separate_density(monkeypatch):
    """advance() with the spline density epilogue against the same merged
    passes with the standalone density pass (VPB_SPLINE_RHO=0 semantics)."""
    monkeypatch.setattr(driver, "ARITH", "fast")
    problem = vpb.problem_spec("landau4d")
    grid = vpb.make_grid(problem, "spline", (64, 32, 64, 32))
    driver._state_cached.cache_clear()
    assert driver.step_state(grid).spline_rho
    f1 = vpb.advance(vpb.initialize(problem, grid), 0.2, 5)
    monkeypatch.setattr(driver, "SPLINE_RHO", False)
    driver._state_cached.cache_clear()
    assert not driver.step_state(grid).spline_rho
    f2 = vpb.advance(vpb.initialize(problem, grid), 0.2, 5)
    driver._state_cached.cache_clear()
    assert max_rel(f1.numpy(), f2.numpy()) <= 1e-13


@pytest.mark.parametrize("axis", [0, 1, 2, 3])
def test_spline_double_sweep_equals_two_sweeps(axis):
    _double_vs_two(axis)


def test_spline_double_sweep_rows_kernel_equals_two_sweeps(monkeypatch):
    """The warp-per-line rows kernel variant of the contiguous-axis double
    sweep (VPB_SPLINE_DBL_ROWS; read once per process, so run in a child)."""
    import subprocess
    import sys
    code = ("import sys; sys.path.insert(0, 'tests'); import test_gpu_step as t; "
            "t._double_vs_two(0)")
    env = dict(__import__("os").environ, VPB_SPLINE_DBL_ROWS="1")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]


def _contig_tile_digest():
    """sha256 of the contiguous-axis spline sweeps of one random field: the
    single sweep, the double sweep and the double sweep with the density
    epilogue (f and the partial densities), on full and on partial tiles."""
    import hashlib
    from paper_1803_02143_b200.spline import sweep_spline, sweep_spline2, sweep_spline2_density
    h = hashlib.sha256()
    for dofs in ((128, 32, 32, 8), (72, 24, 32, 4), (64, 20, 5, 4)):
        prob = vpb.problem_spec("landau4d")
        grid = vpb.make_grid(prob, "spline", dofs)
        f = vpb.initialize(prob, grid)
        rng = np.random.default_rng(31)
        f.data.copy_(torch.from_numpy(rng.standard_normal(f.data.numel())))
        st = driver.step_state(grid)
        vals, hx = st.vpoints[0], grid.axes[0].h
        flag = torch.zeros(1, dtype=torch.int32, device="cuda")
        out = torch.empty_like(f.data)
        sweep_spline(grid, 0, f.data, out, vals, 0.41, hx, flag)
        h.update(out.cpu().numpy().tobytes())
        if grid.dof(0) % 16 == 0:
            sweep_spline2(grid, 0, f.data, out, vals, 0.41, hx, flag)
            h.update(out.cpu().numpy().tobytes())
        if st.spline_rho:
            sweep_spline2_density(grid, f.data, out, vals, 0.41, hx, flag, st.wv1, st.spart)
            h.update(out.cpu().numpy().tobytes())
            h.update(st.spart.cpu().numpy().tobytes())
        assert flag.item() == 0
    return h.hexdigest()


def test_spline_contiguous_tiles_tma_equals_per_lane_copies():
    """The fused contiguous-axis sweeps load their [32 lines][n + 2] tile by
    one TMA tensor copy whose box is two points wider than the tensor (the
    zero-filled padding columns give the row pitch); VPB_SPLINE_CONTIG_TMA=0
    selects one bulk copy per line.  Both must give the same bits (the
    switch is read once per process, so each side runs in a child)."""
    import subprocess
    import sys
    code = ("import sys; sys.path.insert(0, 'tests'); import test_gpu_step as t; "
            "print('DIGEST', t._contig_tile_digest())")
    got = {}
    for tma in ("1", "0"):
        env = dict(__import__("os").environ, VPB_SPLINE_CONTIG_TMA=tma)
        r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True,
                           text=True, timeout=300)
        assert r.returncode == 0, r.stderr[-2000:]
        got[tma] = [ln for ln in r.stdout.splitlines() if ln.startswith("DIGEST")][-1]
    assert got["1"] == got["0"]


def _double_vs_two(axis):
    from paper_1803_02143_b200.spline import sweep_spline, sweep_spline2
    prob = vpb.problem_spec("landau4d")
    grid = vpb.make_grid(prob, "spline", (64, 32, 48, 32))
    f = vpb.initialize(prob, grid)
    rng = np.random.default_rng(5)
    f.data.copy_(torch.from_numpy(rng.standard_normal(f.data.numel())))
    st = driver.step_state(grid)
    if axis < 2:
        vals, scale = st.vpoints[axis], 0.37
    else:
        n = grid.dof(0) * grid.dof(1)
        vals = torch.from_numpy(rng.uniform(-3, 3, n)).cuda()
        scale = 0.3
    h = grid.axes[axis].h
    t1 = torch.empty_like(f.data)
    t2 = torch.empty_like(f.data)
    sweep_spline(grid, axis, f.data, t1, vals, scale, h, None)
    sweep_spline(grid, axis, t1, t2, vals, scale, h, None)
    d = torch.empty_like(f.data)
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")
    sweep_spline2(grid, axis, f.data, d, vals, scale, h, flag)
    assert flag.item() == 0
    a, b = t2.cpu().numpy(), d.cpu().numpy()
    assert np.max(np.abs(a - b)) <= 1e-13 * np.max(np.abs(a))
