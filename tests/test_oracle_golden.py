"""Pin the oracle (CPU restatement) against the reference's golden vectors.

Two kinds of pins:
* the reference test-suite's own frozen known answers, restated here with
  the file:line they come from;
* fixtures produced by running the reference itself
  (tests/golden/make_golden.py).
The oracle must reproduce the reference bitwise wherever the reference is
deterministic arithmetic (line kernels, tables, whole steps).
"""

from __future__ import annotations

import math

import numpy as np
import pytest

from oracle import core

# /root/reference/pkg/tests/test_dg.py:15-24
A_DEG2_ALPHA03 = [
    [-0.04775999999999975, 0.26338571037849795, 0.7403701912436376],
    [0.02228393101343877, -0.09690000000000026, 0.16461606898656156],
    [-0.00789019124363636, 0.035654289621501356, -0.04776000000000041],
]
B_DEG2_ALPHA03 = [
    [0.12375999999999918, -0.10915984515372924, 0.029403943531594486],
    [0.6163249032210805, 0.3619000000000008, -0.06822490322108057],
    [-0.08988394353159262, 0.9861198451537293, 0.12376000000000027],
]
# /root/reference/pkg/tests/test_spline.py:15
IMPULSE_N4 = [1.7499999999999998, -0.5, 0.25, -0.5]
# /root/reference/pkg/tests/test_driver.py:27-32
LANDAU2D_MASS = 12.56637058956352
LANDAU4D_KINETIC = 157.9136582806675


def test_frozen_projection_matrices():
    a, b, q, al = core.projection_pairs(np.array([0.3]), 1.0, 2)
    np.testing.assert_allclose(a[0], A_DEG2_ALPHA03, rtol=0, atol=1e-10)
    np.testing.assert_allclose(b[0], B_DEG2_ALPHA03, rtol=0, atol=1e-10)
    assert q[0] == 0 and al[0] == pytest.approx(0.3, abs=1e-15)


def test_frozen_impulse_spline():
    got = core.cyclic_solve_lines(np.array([[1.0, 0.0, 0.0, 0.0]]))[0]
    np.testing.assert_allclose(got, IMPULSE_N4, rtol=0, atol=1e-13)


def test_frozen_landau_mass_and_kinetic():
    g2 = core.make_grid("landau2d", "spline", 64)
    rec = core.diagnostics(core.initialize("landau2d", g2), g2)
    assert rec["mass"] == pytest.approx(LANDAU2D_MASS, abs=1e-6)
    g4 = core.make_grid("landau4d", "spline", 32)
    rec = core.diagnostics(core.initialize("landau4d", g4), g4)
    assert rec["kinetic_energy"] == pytest.approx(LANDAU4D_KINETIC, abs=1e-4)
    # initial EE 8 pi^2 (test_driver.py:273-279)
    assert rec["electric_energy"] == pytest.approx(8.0 * math.pi ** 2, rel=1e-6)


def test_electric_energy_closed_form_twostream():
    # poisson test: 25 pi^2 eps^2/(4 k^2) for rho = 1 + eps cos(k x1) cos(k x2)
    # (/root/reference/pkg/tests/test_poisson.py:216-223)
    eps, k = 1e-3, 0.2
    g = core.OGrid((0.0, 0.0, -6.0, -6.0), (10 * math.pi, 10 * math.pi, 6.0, 6.0),
                   (40, 40, 4, 4), "spline")
    x1 = g.points(0)[:, None]
    x2 = g.points(1)[None, :]
    rho = 1.0 + eps * np.cos(k * x1) * np.cos(k * x2)
    comps, _ = core.solve_poisson(rho, g)
    assert core.electric_energy(comps, g) == pytest.approx(25 * math.pi ** 2 * eps ** 2 / (4 * k * k),
                                                           rel=1e-11)


def test_projection_pairs_bitwise_vs_reference(golden):
    z = golden("kernels")
    shifts = z["pp_shifts"]
    for h in (0.7, 0.5, 1.0):
        for deg in range(0, 5):
            tag = f"pp_h{h}_d{deg}"
            a, b, q, al = core.projection_pairs(shifts, h, deg)
            assert np.array_equal(a, z[tag + "_a"]), tag
            assert np.array_equal(b, z[tag + "_b"]), tag
            assert np.array_equal(q, z[tag + "_q"]), tag
            assert np.array_equal(al, z[tag + "_alpha"]), tag


@pytest.mark.parametrize("n", [4, 5, 16, 48, 128, 288])
def test_spline_factors_bitwise_vs_reference(golden, n):
    mult, denom, z, sden = core.spline_factors(n)
    got = np.concatenate([mult, denom, z, [sden]])
    assert np.array_equal(got, golden("kernels")[f"fac{n}"])


@pytest.mark.parametrize("p", [1, 2, 3, 4])
@pytest.mark.parametrize("C", [4, 9, 16])
def test_dg_lines_bitwise_vs_reference(golden, p, C):
    z = golden("kernels")
    tag = f"dg_p{p}_c{C}"
    a, b, q, al = core.projection_pairs(z[tag + "_table"], 0.4, p - 1)
    args = (z[tag + "_lines"], z[tag + "_idx"], a, b, q, al, C, p)
    ref = z[tag + "_out"]
    assert np.array_equal(core.dg_lines(*args), ref)
    assert np.array_equal(core.dg_lines_numpy(*args), ref)


@pytest.mark.parametrize("n", [4, 16, 48, 128])
def test_spline_lines_bitwise_vs_reference(golden, n):
    z = golden("kernels")
    tag = f"sp_n{n}"
    lines, idx, tab = z[tag + "_lines"], z[tag + "_idx"], z[tag + "_table"]
    ref = z[tag + "_out"]
    assert np.array_equal(core.spline_lines(lines, idx, tab, 0.25), ref)
    assert np.array_equal(core.spline_lines_numpy(lines, tab[idx], 0.25), ref)


STEP_CASES = [
    ("landau4d_dg3", "landau4d", "dg", 12, 3, 0.1),
    ("landau4d_dg4", "landau4d", "dg", 16, 4, 0.1),
    ("landau4d_spline", "landau4d", "spline", 12, 0, 0.1),
    ("twostream_dg2", "twostream4d_baseline", "dg", 12, 2, 0.1),
    ("twostream_ref_dg3", "twostream4d", "dg", 12, 3, 0.1),
    ("landau2d_dg4", "landau2d", "dg", 32, 4, 0.1),
    ("landau2d_spline", "landau2d", "spline", 32, 0, 0.1),
]

REC_KEYS = ("time", "electric_energy", "mass", "l1_norm", "l2_norm", "kinetic_energy",
            "total_energy")


@pytest.mark.parametrize("tag,prob,method,dofs,order,tau", STEP_CASES)
def test_oracle_steps_match_reference(golden, tag, prob, method, dofs, order, tau):
    z = golden("steps")
    states = z[tag + "_f"]
    recs = z[tag + "_rec"]
    grid = core.make_grid(prob, method, dofs, order)
    f = core.initialize(prob, grid)
    assert np.array_equal(f, states[0])
    for m in range(1, states.shape[0]):
        f = core.strang_step(f, grid, tau)
        assert np.array_equal(f, states[m]), (tag, m)
        rec = core.diagnostics(f, grid, m * tau)
        np.testing.assert_allclose([rec[k] for k in REC_KEYS], recs[m], rtol=1e-14, atol=0)


def test_oracle_config1_series_matches_reference(golden):
    """BASELINE config 1 (48^4, dG p=3, dt=0.1): first 5 of 20 steps bitwise,
    diagnostics to 1e-14 (the full series is checked on the GPU box)."""
    z = golden("series")
    recs = z["cfg1_rec"]
    sums = z["cfg1_sums"]
    grid = core.make_grid("landau4d", "dg", 48, 3)
    f = core.initialize("landau4d", grid)
    for m in range(1, 6):
        f = core.strang_step(f, grid, 0.1)
        got = [float(np.sum(f)), float(np.sum(f * f)), float(np.max(np.abs(f)))]
        np.testing.assert_allclose(got, sums[m - 1], rtol=1e-15, atol=0)
        rec = core.diagnostics(f, grid, m * 0.1)
        np.testing.assert_allclose([rec[k] for k in REC_KEYS], recs[m], rtol=1e-14, atol=0)


def test_markstein_division_identity():
    """The CUDA spline kernel divides by the factor denominators with a
    reciprocal + two FMAs; that sequence must equal IEEE division."""
    lib = core.clib()
    assert lib is not None
    dens = []
    for n in (4, 5, 16, 48, 128, 288, 1024):
        _, denom, _, sden = core.spline_factors(n)
        dens.extend(denom.tolist())
        dens.append(sden)
    dens = np.unique(np.array(dens))
    assert lib.oracle_check_markstein(dens.ctypes.data, dens.size, 20000, 12345) == 0
    rnd = np.random.default_rng(5).uniform(0.5, 16.0, 2000)
    assert lib.oracle_check_markstein(rnd.ctypes.data, rnd.size, 2000, 777) == 0
