"""host_steps(): Strang steps of a field held in pinned host memory with the
PCIe copies pipelined per v2 block (paper_1803_02143_b200/hoststep.py).

Per-block x passes are the whole-field kernels on a sub-range of (v1, v2)
planes and the density is the standalone ``vpb_density`` pass, so the
result must be BITWISE the strang_step chain with the unfused density
(driver.FUSE_RHO off), for any block count."""

from __future__ import annotations

import numpy as np
import pytest

import paper_1803_02143_b200 as vpb
from paper_1803_02143_b200 import driver
from vpb_testutil import max_rel

pytestmark = pytest.mark.gpu


def _chain(f0, tau, nsteps, fuse_rho):
    old = driver.FUSE_RHO
    driver.FUSE_RHO = fuse_rho
    driver._state_cached.cache_clear()
    try:
        f = f0
        for _ in range(nsteps):
            f = vpb.strang_step(f, tau)
        return f.numpy()
    finally:
        driver.FUSE_RHO = old
        driver._state_cached.cache_clear()


CASES = [
    ("landau4d", "dg", (24, 18, 12, 12), 3),
    ("landau4d", "dg", (16, 12, 10, 8), 2),
    ("twostream4d_baseline", "dg", (16, 16, 16, 16), 2),
    ("landau4d", "spline", (32, 24, 16, 16), 0),
]


@pytest.mark.parametrize("prob,method,dofs,order", CASES)
@pytest.mark.parametrize("blocks", [1, 3, 16, 1000])
def test_host_steps_bitwise_equal_to_step_chain(prob, method, dofs, order, blocks):
    problem = vpb.problem_spec(prob)
    grid = vpb.make_grid(problem, method, dofs, dg_order=order)
    f0 = vpb.initialize(problem, grid)
    ref = _chain(f0, 0.3, 3, fuse_rho=False)
    host = vpb.HostField.from_field(f0)
    out = vpb.host_steps(host, 0.3, 3, blocks=blocks)
    assert out is host
    got = host.logical()
    assert np.array_equal(got, ref)
    # and equal to the default (fused-density) chain up to round-off
    assert max_rel(got, _chain(f0, 0.3, 3, fuse_rho=True)) <= 1e-14


def test_host_steps_repeated_calls_and_from_values():
    problem = vpb.problem_spec("landau4d")
    grid = vpb.make_grid(problem, "dg", (24, 18, 12, 12), dg_order=3)
    f0 = vpb.initialize(problem, grid)
    host = vpb.HostField.from_values(grid, f0.numpy())
    assert np.array_equal(host.logical(), f0.numpy())
    vpb.host_steps(host, 0.2, 2, blocks=4)
    vpb.host_steps(host, 0.2, 1, blocks=4)
    assert np.array_equal(host.logical(), _chain(f0, 0.2, 3, fuse_rho=False))
    dev = host.to_device()
    assert np.array_equal(dev.numpy(), host.logical())


def test_host_steps_reports_nonfinite_substep():
    problem = vpb.problem_spec("landau4d")
    grid = vpb.make_grid(problem, "dg", (24, 18, 12, 12), dg_order=3)
    host = vpb.HostField.from_field(vpb.initialize(problem, grid))
    host.data[777] = float("nan")
    with pytest.raises(vpb.SubstepError, match=r"x1 half \(open\)"):
        vpb.host_steps(host, 0.2, 2, blocks=4, first_step=5)
