"""Guard-band checks of every sweep / reduction kernel family (a stand-in for
compute-sanitizer memcheck / initcheck, which is closed on this GPU pool).

Each kernel runs on a field embedded in a larger allocation:

    [ guard | payload | guard ]     guard = 64 doubles (512 B, keeps TMA / bulk alignment)

* source guards hold NaN: a read outside the payload that reaches an output
  makes it non-finite (and raises the kernel's non-finite flag);
* destination guards hold a sentinel: any write outside the payload changes it;
* the destination payload starts as NaN: an output the kernel never writes
  stays NaN (initcheck-like);
* the result equals the same kernel on a plain allocation bitwise, twice
  (run-to-run determinism of the RED / slab reductions and the mbarrier rings).
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

import paper_1803_02143_b200 as vpb
from paper_1803_02143_b200 import driver
from paper_1803_02143_b200.dg import sweep_dg, vplane_dg, xcomp_dg, xplane2_dg, xplane_dg
from paper_1803_02143_b200.poisson import density_into
from paper_1803_02143_b200.spline import double_sweep_ok, sweep_spline, sweep_spline2

pytestmark = pytest.mark.gpu

G = 64
SENT = 12345.0


def guarded(n: int, fill: float, payload: torch.Tensor | None = None):
    big = torch.full((n + 2 * G,), float("nan"), dtype=torch.float64, device="cuda")
    big[:G] = fill
    big[G + n:] = fill
    if payload is not None:
        big[G:G + n] = payload
    return big, big[G:G + n]


def run_guarded(n, src_data, launch):
    """launch(src, dst) on guarded buffers; returns the payload (host)."""
    sbig, src = guarded(n, float("nan"), src_data)
    dbig, dst = guarded(n, SENT)
    launch(src, dst)
    torch.cuda.synchronize()
    d = dbig.cpu().numpy()
    assert np.all(d[:G] == SENT) and np.all(d[G + n:] == SENT), "write outside the payload"
    out = d[G:G + n]
    assert np.all(np.isfinite(out)), "unwritten output or a read of a NaN guard"
    s = sbig.cpu().numpy()
    assert np.all(np.isnan(s[:G])) and np.all(np.isnan(s[G + n:])), "source guard modified"
    return out


def check_family(n, src_data, launch):
    a = run_guarded(n, src_data, launch)
    b = run_guarded(n, src_data, launch)
    plain_src = src_data.clone()
    plain_dst = torch.empty_like(plain_src)
    launch(plain_src, plain_dst)
    torch.cuda.synchronize()
    assert np.array_equal(a, b), "not deterministic"
    assert np.array_equal(a, plain_dst.cpu().numpy())


GRIDS = [("landau4d", "dg", (24, 18, 12, 12), 3), ("landau4d", "dg", (16, 12, 10, 8), 2),
         ("landau4d", "dg", (20, 16, 12, 12), 4),
         # composed x pass with output staging (BST) over many ring chunks per
         # plane: 4 cells per chunk (96 x1 dofs) and config 2's 2 cells (192)
         ("landau4d", "dg", (96, 96, 6, 6), 3), ("landau4d", "dg", (192, 48, 6, 6), 3)]


def _field(prob, method, dofs, order, tau=0.7, steps=1):
    problem = vpb.problem_spec(prob)
    grid = vpb.make_grid(problem, method, dofs, dg_order=order)
    f = vpb.initialize(problem, grid)
    for _ in range(steps):
        f = vpb.strang_step(f, tau, consume=True)  # E != 0, non-trivial v tables
    return grid, f


@pytest.mark.parametrize("prob,method,dofs,order", GRIDS)
def test_dg_sweeps_and_fused_passes_stay_in_bounds(prob, method, dofs, order):
    grid, f = _field(prob, method, dofs, order)
    st = driver.step_state(grid)
    n = grid.total_dof
    tau = 0.7
    tx = [st.x_tables(d, tau) for d in range(2)]
    tv = [st.v_tables(d, tau) for d in range(2)]
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")
    for axis, tab in ((0, tx[0]), (1, tx[1]), (2, tv[0]), (3, tv[1])):
        check_family(n, f.data, lambda s, d, a=axis, t=tab: sweep_dg(grid, a, s, d, t, flag))
    if st.fused_x:
        check_family(n, f.data, lambda s, d: xplane_dg(grid, s, d, tx[0], tx[1], flag, flag))
        check_family(n, f.data, lambda s, d: xplane2_dg(grid, s, d, tx[0], tx[1], None, None))
        check_family(n, f.data, lambda s, d: xcomp_dg(grid, s, d, tx[0], tx[1], flag))
        stats = torch.zeros(4, dtype=torch.float64, device="cuda")

        def xcomp_rho(s, d):
            driver.xcomp_density_dg(grid, s, d, tx[0], tx[1], flag, st, stats)

        check_family(n, f.data, xcomp_rho)
        rc1 = st.rc.clone()
        check_family(n, f.data, xcomp_rho)
        assert torch.equal(rc1, st.rc), "density epilogue not deterministic"
    check_family(n, f.data, lambda s, d: vplane_dg(grid, s, d, tv[0], tv[1], flag, flag))
    assert int(flag.item()) == 0


@pytest.mark.parametrize("dofs", [(32, 24, 16, 16), (64, 32, 32, 16)])
def test_spline_sweeps_stay_in_bounds(dofs):
    grid, f = _field("landau4d", "spline", dofs, 0)
    st = driver.step_state(grid)
    n = grid.total_dof
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")
    for axis in range(4):
        vals = st.x_tables(axis, 0.3) if axis < 2 else st.v_tables(axis - 2, 0.3)
        scale = 0.15 if axis < 2 else 0.3
        h = grid.axes[axis].h
        check_family(n, f.data,
                     lambda s, d, a=axis, v=vals, c=scale, hh=h: sweep_spline(grid, a, s, d, v, c,
                                                                              hh, flag))
        if axis < 2 and double_sweep_ok(grid, axis):
            check_family(n, f.data,
                         lambda s, d, a=axis, v=vals, hh=h: sweep_spline2(grid, a, s, d, v, 0.15,
                                                                          hh, flag))
    assert int(flag.item()) == 0


@pytest.mark.parametrize("prob,method,dofs,order", GRIDS + [("landau4d", "spline",
                                                             (32, 24, 16, 16), 0)])
def test_density_reduction_in_bounds_and_deterministic(prob, method, dofs, order):
    grid, f = _field(prob, method, dofs, order)
    n = grid.total_dof
    nx = grid.dims4[0] * grid.dims4[1]
    sbig, src = guarded(n, float("nan"), f.data)
    outs = []
    for _ in range(2):
        rbig, rho = guarded(nx, SENT)
        density_into(src, grid, rho)
        torch.cuda.synchronize()
        r = rbig.cpu().numpy()
        assert np.all(r[:G] == SENT) and np.all(r[G + nx:] == SENT)
        assert np.all(np.isfinite(r[G:G + nx]))
        outs.append(r[G:G + nx])
    assert np.array_equal(outs[0], outs[1])


def test_plugin_line_kernels_in_bounds():
    """The plugin entry points (reference FFI) on guarded device lines."""
    from paper_1803_02143_b200 import _device, _lib

    rng = np.random.default_rng(3)
    L, n, p = 37, 24, 3
    lines = torch.from_numpy(rng.standard_normal(L * n)).cuda()
    idx = torch.from_numpy(rng.integers(0, 5, L).astype(np.int64)).cuda()
    shifts = rng.uniform(-3, 3, 5) * 0.5
    a, b, q, al = (torch.from_numpy(np.ascontiguousarray(x)).cuda()
                   for x in vpb.projection_pairs(shifts, 0.5, p - 1))
    lib = _lib.load()

    def dg(s, d):
        _lib.check(lib.vpb_dg_sweep_contig(s.data_ptr(), d.data_ptr(), L, n, idx.data_ptr(),
                                           a.data_ptr(), b.data_ptr(), q.data_ptr(),
                                           al.data_ptr(), 5, n // p, p, _device.stream()), "dg")

    tab = torch.from_numpy(shifts).cuda()

    def sp(s, d):
        _lib.check(lib.vpb_spline_sweep_contig(s.data_ptr(), d.data_ptr(), L, n, idx.data_ptr(),
                                               tab.data_ptr(), 5, 0.5, _device.stream()), "sp")

    check_family(L * n, lines, dg)
    check_family(L * n, lines, sp)
