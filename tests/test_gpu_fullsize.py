"""BASELINE configurations at their full sizes: size-independent properties.

The oracle cannot step 1.4e9-6.9e9 dofs in test time, so at the sizes
bench.py measures these tests check what holds at any size:
mass conservation (every dG projection and every periodic spline sweep
conserves the weighted sum; 1e-13 bar), the L2 norm never growing (dG
projections are L2 contractions), and the "fast" merged x passes agreeing
with the "exact" four-sweep chain that reproduces the reference's rounding
(the oracle parity of "exact" is pinned on the small grids of
test_gpu_step.py).  Runs on the B200 box: ``pytest -m gpu``.
"""

from __future__ import annotations

import gc

import pytest
import torch

import paper_1803_02143_b200 as vpb
from paper_1803_02143_b200 import driver

pytestmark = pytest.mark.gpu

MASS_TOL = 1e-13

# BASELINE.json configs: (problem, method, dofs per axis, dg_order, dt)
CFG = {
    "cfg2": ("landau4d", "dg", 192, 3, 0.05),
    "cfg3": ("twostream4d_baseline", "dg", 128, 2, 0.1),
    "cfg4": ("landau4d", "spline", 128, 0, 0.1),
    "cfg5": ("landau4d", "dg", 288, 3, 0.05),
}


@pytest.fixture(autouse=True)
def _free_device_memory():
    yield
    driver._state_cached.cache_clear()
    gc.collect()
    torch.cuda.empty_cache()


def _grid(name):
    prob, method, dofs, order, tau = CFG[name]
    problem = vpb.problem_spec(prob)
    return problem, vpb.make_grid(problem, method, dofs, dg_order=order), tau


@pytest.mark.parametrize("name", ["cfg2", "cfg3", "cfg4"])
def test_fast_merged_steps_match_exact_chain_and_conserve_mass(monkeypatch, name):
    problem, grid, tau = _grid(name)
    f0 = vpb.initialize(problem, grid)
    d0 = vpb.diagnostics(f0, 0.0)
    monkeypatch.setattr(driver, "ARITH", "exact")
    fe = vpb.advance(f0, tau, 3)
    monkeypatch.setattr(driver, "ARITH", "fast")
    ff = vpb.advance(f0, tau, 3)
    del f0
    # f: max-norm relative difference of the two arithmetics after 3 steps
    diff = torch.max(torch.abs(ff.data - fe.data)).item()
    scale = torch.max(torch.abs(fe.data)).item()
    assert diff <= 1e-13 * scale, (name, diff / scale)
    for f in (fe, ff):
        d = vpb.diagnostics(f, 3 * tau)
        assert abs(d.mass - d0.mass) <= MASS_TOL * abs(d0.mass), (name, d.mass, d0.mass)
        if grid.method == "dg":
            assert d.l2_norm <= d0.l2_norm * (1 + 1e-14)


def test_config5_steps_conserve_mass_and_l2():
    """Config 5 (288^4 = 6.9e9 dofs, 55 GB per copy): two merged steps in
    place (f + one scratch copy = 110 GB of HBM)."""
    problem, grid, tau = _grid("cfg5")
    f = vpb.initialize(problem, grid)
    d0 = vpb.diagnostics(f, 0.0)
    f, rec = vpb.advance(f, tau, 2, consume=True, record_time=2 * tau)
    assert abs(rec.mass - d0.mass) <= MASS_TOL * abs(d0.mass)
    assert rec.l2_norm <= d0.l2_norm * (1 + 1e-14)
    # the closing pass's diagnostics epilogue agrees with a separate reduction
    d = vpb.diagnostics(f, 2 * tau)
    assert rec.electric_energy == pytest.approx(d.electric_energy, rel=1e-12)
    assert rec.mass == pytest.approx(d.mass, rel=1e-13)
