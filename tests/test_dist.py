"""Multi-GPU layer, exercised on CPU: decomposition, halo widths and message
pattern, ρ assembly, flag/diagnostic reductions.

The local compute is the oracle (tests/dist_oracle_ops.py), so these tests
check the sharding logic itself: a sharded Strang step must reproduce the
unsharded oracle step.  Two-rank runs use torch.distributed with gloo over
127.0.0.1; the 4 x 2 layout of 8 GPUs runs in-process (VirtualComm).
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import paper_1803_02143_b200 as vpb
from dist_oracle_ops import NumpyOps
from oracle import core
from paper_1803_02143_b200 import dist
from vpb_testutil import max_rel

PROB = "landau4d"
DOFS = (24, 18, 12, 12)  # dg_order 3: 8 x 6 x 4 x 4 cells
ORDER = 3
TAU = 0.4  # large enough that x shifts reach |q| = 1


def grids():
    grid = vpb.make_grid(vpb.problem_spec(PROB), "dg", DOFS, dg_order=ORDER)
    og = core.OGrid(tuple(a.lower for a in grid.axes), tuple(a.upper for a in grid.axes),
                    tuple(a.count for a in grid.axes), grid.method, grid.dg_degree)
    return grid, og


def oracle_run(nsteps):
    grid, og = grids()
    f = core.initialize(PROB, og)
    for _ in range(nsteps):
        f = core.strang_step(f, og, TAU)
    return f, core.diagnostics(f, og, nsteps * TAU)


def test_process_grid_and_cell_split():
    assert dist.process_grid(1) == (1, 1)
    assert dist.process_grid(2) == (2, 1)
    assert dist.process_grid(4) == (4, 1)
    assert dist.process_grid(8) == (4, 2)
    cells = [dist.split_cells(10, 3, r) for r in range(3)]
    assert cells == [(0, 4), (4, 7), (7, 10)]
    grid, _ = grids()
    dec = dist.Decomposition(grid, 4, 2)
    assert dec.world == 8
    assert dec.local_dims(0) == (6, 9, 12, 12)
    assert dec.neighbours(0, 0) == (6, 2)  # x1 left/right of rank (0, 0)
    assert dec.neighbours(1, 1) == (0, 0)  # x2 neighbours wrap on a 2-wide axis
    with pytest.raises(ValueError):
        dist.Decomposition(grid, 9, 1)


def test_halo_widths_are_one_sided():
    assert dist.halo_widths(np.array([0, 0])) == (1, 0)
    assert dist.halo_widths(np.array([-1, 0])) == (1, 1)
    assert dist.halo_widths(np.array([-2, -1])) == (0, 2)
    assert dist.halo_widths(np.array([1, 3])) == (4, 0)
    assert dist.halo_widths(np.array([], dtype=np.int64)) == (0, 0)


@pytest.mark.parametrize("p1,p2", [(2, 1), (1, 2), (4, 2), (3, 1), (2, 3)])
def test_virtual_sharded_step_matches_unsharded_oracle(p1, p2):
    grid, og = grids()
    dec = dist.Decomposition(grid, p1, p2)
    solver = dist.ShardedSolver(grid, dec, dist.VirtualComm(dec.world), range(dec.world),
                                ops=NumpyOps(), device=torch.device("cpu"))
    solver.scatter(core.initialize(PROB, og))
    for m in range(2):
        solver.step(TAU, time_label=(m + 1) * TAU)
    ref, rec = oracle_run(2)
    assert max_rel(solver.gather(), ref) <= 1e-14
    got = solver.diagnostics(2 * TAU)
    for k in ("mass", "l1_norm", "l2_norm", "kinetic_energy", "electric_energy"):
        assert got[k] == pytest.approx(rec[k], rel=1e-12), k


def test_x_shifts_need_halos_in_this_setup():
    grid, _ = grids()
    q1 = core.projection_pairs(grid.axis_points(2) * (0.5 * TAU), grid.axes[0].h, ORDER - 1)[2]
    wl, wr = dist.halo_widths(q1)
    assert wl >= 1 and wr >= 1  # both directions are exercised


def test_sharded_step_reports_nonfinite_on_every_shard():
    grid, og = grids()
    dec = dist.Decomposition(grid, 2, 1)
    solver = dist.ShardedSolver(grid, dec, dist.VirtualComm(2), range(2), ops=NumpyOps(),
                                device=torch.device("cpu"))
    f = core.initialize(PROB, og).copy()
    f[20, 3, 4, 5] = np.nan  # lives on rank 1
    solver.scatter(f)
    with pytest.raises(vpb.SubstepError, match=r"x1 half \(open\)"):
        solver.step(TAU)


@pytest.mark.parametrize("p1,tau", [(2, TAU), (4, TAU), (2, 1.3)])
def test_virtual_sharded_advance_matches_oracle_steps(p1, tau):
    """advance(): x1 halo exchange + merged three-cell stencil passes with the
    density epilogue (oracle restatement of the kernels) vs oracle steps."""
    grid, og = grids()
    dec = dist.Decomposition(grid, p1, 1)
    solver = dist.ShardedSolver(grid, dec, dist.VirtualComm(dec.world), range(dec.world),
                                ops=NumpyOps(), device=torch.device("cpu"))
    assert solver._stencil_ready()
    solver.scatter(core.initialize(PROB, og))
    solver.advance(tau, 3)
    f = core.initialize(PROB, og)
    for _ in range(3):
        f = core.strang_step(f, og, tau)
    assert max_rel(solver.gather(), f) <= 1e-13


@pytest.mark.parametrize("p1,p2,tau", [(2, 2, TAU), (4, 2, TAU), (2, 3, 0.25)])
def test_virtual_sharded_advance_x1x2_matches_oracle_steps(p1, p2, tau):
    """x1 x x2 process grids (the 4 x 2 layout at 8 GPUs): advance() runs the
    stencil passes with x1 halos, then x2 halos carrying the corner cells
    (vpb_dg_sweep_xstencil2; oracle restatement), against oracle steps."""
    calls = []

    class Counting(NumpyOps):
        def xstencil2(self, *a, **k):
            calls.append(a[8])  # qmul
            return super().xstencil2(*a, **k)

    grid, og = grids()
    dec = dist.Decomposition(grid, p1, p2)
    solver = dist.ShardedSolver(grid, dec, dist.VirtualComm(dec.world), range(dec.world),
                                ops=Counting(), device=torch.device("cpu"))
    assert solver._stencil_ready(tau)
    solver.scatter(core.initialize(PROB, og))
    solver.advance(tau, 3)
    assert calls, "the x1 x x2 stencil path did not run"
    f = core.initialize(PROB, og)
    for _ in range(3):
        f = core.strang_step(f, og, tau)
    assert max_rel(solver.gather(), f) <= 1e-13


@pytest.mark.parametrize("blocks", [2, 3, 100])
def test_pipelined_halo_blocks_match_one_exchange(blocks):
    """advance() with the halo exchange and stencil pass pipelined in blocks
    of v2 rows (comm/compute overlap) equals the one-exchange
    pass up to the summation order of the density partials."""
    grid, og = grids()
    out = []
    for nb in (1, blocks):
        dec = dist.Decomposition(grid, 2, 1)
        solver = dist.ShardedSolver(grid, dec, dist.VirtualComm(dec.world), range(dec.world),
                                    ops=NumpyOps(), device=torch.device("cpu"))
        solver.halo_blocks = nb
        solver.scatter(core.initialize(PROB, og))
        solver.advance(TAU, 3)
        out.append(solver.gather())
    assert max_rel(out[1], out[0]) <= 1e-14


@pytest.mark.parametrize("p1", [3, 5])
def test_virtual_sharded_advance_uneven_split_falls_back_to_step(p1):
    """8 x1 cells over 3 / 5 ranks: shards of 2-3 / 1-2 cells.  Odd local dof
    rows (3 cells * 3 * 3) miss the stencil kernel's 16-byte precondition and
    the single half step's halo may exceed a 1-cell shard: advance() must
    run the per-sweep halo path, not raise."""
    grid, og = grids()
    dec = dist.Decomposition(grid, p1, 1)
    solver = dist.ShardedSolver(grid, dec, dist.VirtualComm(dec.world), range(dec.world),
                                ops=NumpyOps(), device=torch.device("cpu"))
    assert not solver._stencil_ready(TAU)
    solver.scatter(core.initialize(PROB, og))
    solver.advance(TAU, 2)
    f = core.initialize(PROB, og)
    for _ in range(2):
        f = core.strang_step(f, og, TAU)
    assert max_rel(solver.gather(), f) <= 1e-13


def test_stencil_ready_checks_halo_fit():
    """Even 2-cell shards (4 ranks x 2 cells) meet the row precondition, but
    a shift of several cells needs a wider halo than a shard: not ready."""
    grid, og = grids()
    dec = dist.Decomposition(grid, 4, 1)
    solver = dist.ShardedSolver(grid, dec, dist.VirtualComm(dec.world), range(dec.world),
                                ops=NumpyOps(), device=torch.device("cpu"))
    assert solver._stencil_ready(TAU)
    assert not solver._stencil_ready(12.0)


def _advance_worker(rank, world, port, outdir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as tdist

    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        grid, og = grids()
        dec = dist.Decomposition(grid, world, 1)
        solver = dist.ShardedSolver(grid, dec, dist.TorchComm(), [rank], ops=NumpyOps(),
                                    device=torch.device("cpu"))
        solver.scatter(core.initialize(PROB, og))
        solver.advance(TAU, 3)
        np.save(os.path.join(outdir, f"a{rank}.npy"), solver.local_logical(rank))
    finally:
        tdist.destroy_process_group()


def test_two_rank_gloo_sharded_advance_equals_in_process(tmp_path):
    """The TorchComm path of advance() (halo send/recv, centred-density
    all-gather, flag / mean reductions) == the in-process VirtualComm run."""
    port = _free_port()
    mp.start_processes(_advance_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True,
                       start_method="spawn")
    grid, og = grids()
    dec = dist.Decomposition(grid, 2, 1)
    solver = dist.ShardedSolver(grid, dec, dist.VirtualComm(2), range(2), ops=NumpyOps(),
                                device=torch.device("cpu"))
    solver.scatter(core.initialize(PROB, og))
    solver.advance(TAU, 3)
    for r in range(2):
        assert np.array_equal(np.load(tmp_path / f"a{r}.npy"), solver.local_logical(r))


def _advance2d_worker(rank, world, port, p1, p2, outdir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as tdist

    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        grid, og = grids()
        dec = dist.Decomposition(grid, p1, p2)
        solver = dist.ShardedSolver(grid, dec, dist.TorchComm(), [rank], ops=NumpyOps(),
                                    device=torch.device("cpu"))
        assert solver._stencil_ready(TAU)
        solver.scatter(core.initialize(PROB, og))
        solver.advance(TAU, 3)
        np.save(os.path.join(outdir, f"a{rank}.npy"), solver.local_logical(rank))
    finally:
        tdist.destroy_process_group()


def test_four_rank_gloo_x1x2_advance_equals_in_process(tmp_path):
    """2 x 2 process grid over gloo: the x1 then x2 halo exchanges of the
    stencil passes (6 x2 messages per rank, corners included) through
    TorchComm == the in-process VirtualComm run."""
    port = _free_port()
    mp.start_processes(_advance2d_worker, args=(4, port, 2, 2, str(tmp_path)), nprocs=4,
                       join=True, start_method="spawn")
    grid, og = grids()
    dec = dist.Decomposition(grid, 2, 2)
    solver = dist.ShardedSolver(grid, dec, dist.VirtualComm(4), range(4), ops=NumpyOps(),
                                device=torch.device("cpu"))
    solver.scatter(core.initialize(PROB, og))
    solver.advance(TAU, 3)
    for r in range(4):
        assert np.array_equal(np.load(tmp_path / f"a{r}.npy"), solver.local_logical(r))


# ---- two real processes over gloo ---------------------------------------
def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, p1, p2, outdir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as tdist

    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        grid, og = grids()
        dec = dist.Decomposition(grid, p1, p2)
        solver = dist.ShardedSolver(grid, dec, dist.TorchComm(), [rank], ops=NumpyOps(),
                                    device=torch.device("cpu"))
        solver.scatter(core.initialize(PROB, og))
        for _ in range(2):
            solver.step(TAU)
        rec = solver.diagnostics(2 * TAU)
        np.save(os.path.join(outdir, f"f{rank}.npy"), solver.local_logical(rank))
        np.save(os.path.join(outdir, f"d{rank}.npy"),
                np.array([rec["mass"], rec["electric_energy"], rec["l2_norm"]]))
    finally:
        tdist.destroy_process_group()


@pytest.mark.parametrize("p1,p2", [(2, 1), (1, 2)])
def test_two_rank_gloo_sharded_step(tmp_path, p1, p2):
    port = _free_port()
    mp.start_processes(_worker, args=(2, port, p1, p2, str(tmp_path)), nprocs=2, join=True,
                       start_method="spawn")
    grid, _ = grids()
    dec = dist.Decomposition(grid, p1, p2)
    ref, rec = oracle_run(2)
    for r in range(2):
        got = np.load(tmp_path / f"f{r}.npy")
        assert max_rel(got, dec.local_slice(r, ref)) <= 1e-14 * 10
        d = np.load(tmp_path / f"d{r}.npy")
        assert d[0] == pytest.approx(rec["mass"], rel=1e-12)
        assert d[1] == pytest.approx(rec["electric_energy"], rel=1e-12)
        assert d[2] == pytest.approx(rec["l2_norm"], rel=1e-12)


# ---- cubic-spline field: all-to-all reshards ----------------------------------
SP_DOFS = (16, 12, 10, 9)
SP_TAU = 0.3


def spline_grids():
    grid = vpb.make_grid(vpb.problem_spec(PROB), "spline", SP_DOFS)
    og = core.OGrid(tuple(a.lower for a in grid.axes), tuple(a.upper for a in grid.axes),
                    tuple(a.count for a in grid.axes), grid.method, grid.dg_degree)
    return grid, og


def spline_oracle_run(nsteps):
    grid, og = spline_grids()
    f = core.initialize(PROB, og)
    for _ in range(nsteps):
        f = core.strang_step(f, og, SP_TAU)
    return f, core.diagnostics(f, og, nsteps * SP_TAU)


@pytest.mark.parametrize("world", [2, 3])
def test_virtual_spline_sharded_step_matches_unsharded_oracle(world):
    grid, og = spline_grids()
    solver = dist.SplineShardedSolver(grid, dist.VirtualComm(world), range(world), world,
                                      ops=NumpyOps(), device=torch.device("cpu"))
    solver.scatter(core.initialize(PROB, og))
    for _ in range(2):
        solver.step(SP_TAU)
    ref, rec = spline_oracle_run(2)
    assert max_rel(solver.gather(), ref) <= 1e-13
    d = solver.diagnostics(2 * SP_TAU)
    for k in ("mass", "electric_energy", "l2_norm", "kinetic_energy"):
        assert d[k] == pytest.approx(rec[k], rel=1e-12), k


def test_spline_sharded_step_reports_nonfinite():
    grid, og = spline_grids()
    solver = dist.SplineShardedSolver(grid, dist.VirtualComm(2), range(2), 2, ops=NumpyOps(),
                                      device=torch.device("cpu"))
    f = core.initialize(PROB, og).copy()
    f[3, 4, 5, 7] = np.inf  # v2 index 7 lives on rank 1
    solver.scatter(f)
    with pytest.raises(vpb.SubstepError, match=r"x1 half \(open\)"):
        solver.step(SP_TAU)


def _spline_worker(rank, world, port, outdir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as tdist

    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        grid, og = spline_grids()
        solver = dist.SplineShardedSolver(grid, dist.TorchComm(), [rank], world, ops=NumpyOps(),
                                          device=torch.device("cpu"))
        solver.scatter(core.initialize(PROB, og))
        for _ in range(2):
            solver.step(SP_TAU)
        v0, v1 = solver.vr[rank]
        np.save(os.path.join(outdir, f"s{rank}.npy"), solver.gather()[:, :, :, v0:v1])
        rec = solver.diagnostics(2 * SP_TAU)
        np.save(os.path.join(outdir, f"sd{rank}.npy"),
                np.array([rec["mass"], rec["electric_energy"], rec["l2_norm"]]))
    finally:
        tdist.destroy_process_group()


def test_two_rank_gloo_spline_sharded_step(tmp_path):
    port = _free_port()
    mp.start_processes(_spline_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True,
                       start_method="spawn")
    ref, rec = spline_oracle_run(2)
    grid, _ = spline_grids()
    for r in range(2):
        v0, v1 = dist.split_cells(grid.dims4[3], 2, r)
        got = np.load(tmp_path / f"s{r}.npy")
        assert max_rel(got, ref[:, :, :, v0:v1]) <= 1e-13
        d = np.load(tmp_path / f"sd{r}.npy")
        assert d[0] == pytest.approx(rec["mass"], rel=1e-12)
        assert d[1] == pytest.approx(rec["electric_energy"], rel=1e-12)
        assert d[2] == pytest.approx(rec["l2_norm"], rel=1e-12)


# ---- velocity-sharded dG (VShardedSolver, the paper's decomposition) -------
VDOFS = (24, 18, 12, 24)  # dg_order 3: 8 x 6 x 4 x 8 cells


def vgrids():
    grid = vpb.make_grid(vpb.problem_spec(PROB), "dg", VDOFS, dg_order=ORDER)
    og = core.OGrid(tuple(a.lower for a in grid.axes), tuple(a.upper for a in grid.axes),
                    tuple(a.count for a in grid.axes), grid.method, grid.dg_degree)
    return grid, og


@pytest.mark.parametrize("world", [2, 3, 4])
def test_virtual_vsharded_advance_matches_oracle_steps(world):
    """v2 slabs with H-cell halos: local x passes, density partials summed in
    rank order, v2 halo exchange + non-periodic v pass, vs oracle steps."""
    grid, og = vgrids()
    solver = dist.VShardedSolver(grid, dist.VirtualComm(world), range(world), world,
                                 ops=NumpyOps(), device=torch.device("cpu"))
    f0 = core.initialize(PROB, og)
    solver.scatter(f0)
    assert np.array_equal(solver.gather(), f0)
    solver.advance(TAU, 3)
    f = f0
    for _ in range(3):
        f = core.strang_step(f, og, TAU)
    assert max_rel(solver.gather(), f) <= 1e-13
    got = solver.diagnostics(3 * TAU)
    ref = core.diagnostics(f, og, 3 * TAU)
    for k in ("mass", "l1_norm", "l2_norm", "kinetic_energy", "electric_energy"):
        assert got[k] == pytest.approx(ref[k], rel=1e-12), k


@pytest.mark.parametrize("world", [2, 3])
def test_virtual_vsharded_peer_halos_match_exchanged_halos(world):
    """peer_halos: the v pass reads the neighbours' boundary rows in place
    (the NVLink peer-memory variant) -- the same result as the NCCL-filled
    halo rows (bitwise when the exchanged variant does not split its x pass
    into boundary and interior blocks, else up to the density partials'
    summation order)."""
    grid, og = vgrids()
    out = []
    for peer in (False, True):
        solver = dist.VShardedSolver(grid, dist.VirtualComm(world), range(world), world,
                                     ops=NumpyOps(), device=torch.device("cpu"), peer_halos=peer)
        solver.scatter(core.initialize(PROB, og))
        solver.advance(TAU, 3)
        out.append(solver.gather())
    if world == 3:  # shards of 3, 3, 2 cells: no boundary/interior split
        assert np.array_equal(out[0], out[1])
    assert max_rel(out[1], out[0]) <= 1e-14


def test_vsharded_rejects_shards_narrower_than_the_halo():
    grid, _ = vgrids()
    with pytest.raises(ValueError, match="narrower than"):
        dist.VShardedSolver(grid, dist.VirtualComm(8), range(8), 8, ops=NumpyOps(),
                            device=torch.device("cpu"), halo_cells=2)


def test_vsharded_halo_overflow_raises():
    grid, og = vgrids()
    solver = dist.VShardedSolver(grid, dist.VirtualComm(2), range(2), 2, ops=NumpyOps(),
                                 device=torch.device("cpu"), halo_cells=2)
    solver.scatter(core.initialize(PROB, og))
    with pytest.raises(RuntimeError, match="v2 halo"):
        solver.advance(40.0, 1)  # |E tau / h_v| far beyond two cells


def _vadvance_worker(rank, world, port, outdir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as tdist

    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        grid, og = vgrids()
        solver = dist.VShardedSolver(grid, dist.TorchComm(), [rank], world, ops=NumpyOps(),
                                     device=torch.device("cpu"))
        solver.scatter(core.initialize(PROB, og))
        solver.advance(TAU, 3)
        np.save(os.path.join(outdir, f"v{rank}.npy"), solver.local_logical(rank))
        d = solver.diagnostics(3 * TAU)
        np.save(os.path.join(outdir, f"vd{rank}.npy"), np.array([d["mass"], d["electric_energy"]]))
    finally:
        tdist.destroy_process_group()


def test_two_rank_gloo_vsharded_advance_equals_in_process(tmp_path):
    port = _free_port()
    mp.spawn(_vadvance_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    grid, og = vgrids()
    solver = dist.VShardedSolver(grid, dist.VirtualComm(2), range(2), 2, ops=NumpyOps(),
                                 device=torch.device("cpu"))
    solver.scatter(core.initialize(PROB, og))
    solver.advance(TAU, 3)
    for r in range(2):
        assert np.array_equal(np.load(tmp_path / f"v{r}.npy"), solver.local_logical(r))
    d = solver.diagnostics(3 * TAU)
    for r in range(2):
        m, ee = np.load(tmp_path / f"vd{r}.npy")
        assert m == d["mass"] and ee == d["electric_energy"]
