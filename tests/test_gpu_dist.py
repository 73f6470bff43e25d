"""Sharded (multi-GPU) path on ONE B200: shards live in one process and the
halo "messages" are device copies (VirtualComm), so the halo pack / halo
sweep kernels and the ρ assembly are checked against the unsharded step
without running ranks that wait on each other on a single GPU."""

from __future__ import annotations

import numpy as np
import pytest
import torch

import paper_1803_02143_b200 as vpb
from paper_1803_02143_b200 import dist
from paper_1803_02143_b200.dg import DeviceTables, sweep_dg
from vpb_testutil import max_rel

pytestmark = pytest.mark.gpu

DOFS = (48, 36, 24, 24)  # dg_order 3: 16 x 12 x 8 x 8 cells
TAU = 0.4


def setup(p1, p2):
    prob = vpb.problem_spec("landau4d")
    grid = vpb.make_grid(prob, "dg", DOFS, dg_order=3)
    dec = dist.Decomposition(grid, p1, p2)
    solver = dist.ShardedSolver(grid, dec, dist.VirtualComm(dec.world), range(dec.world))
    f0 = vpb.initialize(prob, grid)
    solver.scatter(f0.numpy())
    return prob, grid, solver, f0


@pytest.mark.parametrize("axis", [0, 1])
@pytest.mark.parametrize("p", [2, 4])
def test_halo_sweep_bitwise_equal_to_unsharded_sweep(axis, p):
    p1, p2 = (p, 1) if axis == 0 else (1, 2 if p == 2 else 3)
    prob, grid, solver, f0 = setup(p1, p2)
    solver._x_sweep(axis, TAU, 0)
    tab, _ = solver.x_tables(axis, TAU)
    out = torch.empty_like(f0.data)
    sweep_dg(grid, axis, f0.data, out, tab, None)
    ref = out.view(f0._phys.shape).permute(3, 2, 1, 0).cpu().numpy()
    assert np.array_equal(solver.gather(), ref)


@pytest.mark.parametrize("p1,p2", [(1, 1), (2, 1), (1, 2), (4, 2)])
def test_sharded_steps_match_single_gpu_step(p1, p2):
    prob, grid, solver, f0 = setup(p1, p2)
    f = f0
    for m in range(3):
        solver.step(TAU)
        f = vpb.strang_step(f, TAU, consume=True)
        assert max_rel(solver.gather(), f.numpy()) <= 1e-13, m
    got = solver.diagnostics(3 * TAU)
    rec = vpb.diagnostics(f, 3 * TAU)
    for k in ("mass", "l1_norm", "l2_norm", "kinetic_energy", "electric_energy"):
        assert got[k] == pytest.approx(getattr(rec, k), rel=1e-12), k


@pytest.mark.parametrize("p1,tau", [(2, TAU), (4, TAU), (2, 1.7), (4, 0.0)])
def test_sharded_advance_with_merged_stencil_passes_matches_single_gpu(p1, tau):
    """x1-sharded advance(): x1 halo exchange + the three-cell stencil kernel
    (single x half steps and merged pairs, density epilogue) against the
    single-GPU advance() in the same ("fast") arithmetic."""
    prob, grid, solver, f0 = setup(p1, 1)
    assert solver._stencil_ready()
    solver.advance(tau, 4)
    f = vpb.advance(f0, tau, 4)
    assert max_rel(solver.gather(), f.numpy()) <= 1e-13
    got = solver.diagnostics(4 * tau)
    rec = vpb.diagnostics(f, 4 * tau)
    for k in ("mass", "l1_norm", "l2_norm", "kinetic_energy", "electric_energy"):
        assert got[k] == pytest.approx(getattr(rec, k), rel=1e-12), k


@pytest.mark.parametrize("p1,p2,tau", [(2, 2, TAU), (4, 2, TAU), (2, 2, 1.7), (4, 3, TAU),
                                        (2, 2, 0.0)])
def test_sharded_advance_x1x2_stencil_passes_match_single_gpu(p1, p2, tau):
    """x1 x x2 process grids (the north-star 4 x 2 layout at 8 GPUs):
    advance() runs vpb_dg_sweep_xstencil2 -- x1 halos, then x2 halos with
    the corner cells -- with the density epilogue, against the single-GPU
    advance() ("fast" arithmetic)."""
    prob, grid, solver, f0 = setup(p1, p2)
    assert solver._stencil_ready(tau)
    calls = []
    orig = solver.ops.xstencil2
    solver.ops.xstencil2 = lambda *a, **k: (calls.append(1), orig(*a, **k))[1]
    solver.advance(tau, 4)
    assert calls
    f = vpb.advance(f0, tau, 4)
    assert max_rel(solver.gather(), f.numpy()) <= 1e-13
    got = solver.diagnostics(4 * tau)
    rec = vpb.diagnostics(f, 4 * tau)
    for k in ("mass", "l1_norm", "l2_norm", "kinetic_energy", "electric_energy"):
        assert got[k] == pytest.approx(getattr(rec, k), rel=1e-12), k


@pytest.mark.parametrize("p1", [3, 5])
def test_sharded_advance_uneven_split_falls_back_to_halo_sweeps(p1):
    """Uneven x1 splits (16 cells over 3 or 5 ranks: shards of 5-6 / 3-4
    cells, some with an odd dof row of 5*3*3 values) miss the stencil
    kernel's 16-byte row precondition: advance() must take the per-sweep
    halo path instead of raising (the reference has no such restriction)."""
    prob, grid, solver, f0 = setup(p1, 1)
    assert not solver._stencil_ready(TAU)
    solver.advance(TAU, 3)
    f = vpb.advance(f0, TAU, 3)
    assert max_rel(solver.gather(), f.numpy()) <= 1e-13


def test_sharded_advance_reports_nonfinite_substep():
    prob, grid, solver, f0 = setup(2, 1)
    sh = solver.shards[1]
    sh.f[1234] = float("nan")
    with pytest.raises(vpb.SubstepError, match=r"x1 half \(open\)"):
        solver.advance(TAU, 3, first_step=2)


def test_sharded_initialize_is_the_shard_of_the_global_initial_state():
    prob, grid, solver, f0 = setup(4, 2)
    solver.initialize(prob)
    assert np.array_equal(solver.gather(), f0.numpy())


# ---- velocity sharding: v2 slabs, v2 halos, vpb_dg_sweep_vplane_v2halo ----------
@pytest.mark.parametrize("world,tau", [(2, TAU), (4, TAU), (3, 0.9)])
def test_vsharded_advance_matches_single_gpu_advance(world, tau):
    """VShardedSolver on one GPU (VirtualComm): local x passes on v2 slabs
    (tables offset to the slab), density partials, v2 halo exchange and the
    non-periodic halo v pass, against the single-GPU advance()."""
    prob = vpb.problem_spec("landau4d")
    grid = vpb.make_grid(prob, "dg", DOFS, dg_order=3)
    solver = dist.VShardedSolver(grid, dist.VirtualComm(world), range(world), world)
    f0 = vpb.initialize(prob, grid)
    solver.initialize(prob)
    assert np.array_equal(solver.gather(), f0.numpy())
    solver.advance(tau, 4)
    f = vpb.advance(f0, tau, 4)
    assert max_rel(solver.gather(), f.numpy()) <= 1e-13
    got = solver.diagnostics(4 * tau)
    rec = vpb.diagnostics(f, 4 * tau)
    for k in ("mass", "l1_norm", "l2_norm", "kinetic_energy", "electric_energy"):
        assert got[k] == pytest.approx(getattr(rec, k), rel=1e-12), k


@pytest.mark.parametrize("world", [2, 3])
def test_vsharded_peer_halos_match_exchanged_halos(world):
    """peer_halos=True: the v pass reads the neighbours' boundary rows in
    place through per-region tensor maps (vpb_dg_sweep_vplane_v2peer; on a
    multi-GPU box the neighbours' buffers are CUDA IPC mappings over NVLink)
    -- against the exchanged-halo solver and the single-GPU advance()."""
    prob = vpb.problem_spec("landau4d")
    grid = vpb.make_grid(prob, "dg", DOFS, dg_order=3)
    out = []
    for peer in (False, True):
        solver = dist.VShardedSolver(grid, dist.VirtualComm(world), range(world), world,
                                     peer_halos=peer)
        solver.initialize(prob)
        solver.advance(TAU, 4)
        out.append(solver.gather())
    f = vpb.advance(vpb.initialize(prob, grid), TAU, 4)
    assert max_rel(out[1], f.numpy()) <= 1e-13
    assert max_rel(out[1], out[0]) <= 1e-14


def _ipc_child(args, q):
    import torch as _t
    from torch.multiprocessing.reductions import rebuild_cuda_tensor

    t = rebuild_cuda_tensor(*args)
    q.put((float(t.sum()), float(t[7])))


def test_cuda_ipc_mapping_used_for_peer_halos():
    """The plumbing VShardedSolver._map_peers uses on a multi-GPU box (each
    rank maps its neighbours' buffers with torch's CUDA IPC reductions): a
    second process maps this process's buffer and reads it."""
    import torch.multiprocessing as tmp
    from torch.multiprocessing.reductions import reduce_tensor

    t = torch.arange(1000, dtype=torch.float64, device="cuda")
    args = reduce_tensor(t)[1]
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    proc = ctx.Process(target=_ipc_child, args=(args, q))
    proc.start()
    got = q.get(timeout=120)
    proc.join(timeout=60)
    assert got == (float(t.sum()), 7.0)


def test_vsharded_v2halo_pass_bitwise_equal_to_fused_v_pass():
    """The halo-fed v pass of each slab is bitwise the single-GPU fused v
    pass restricted to the slab (same operations, same order)."""
    from paper_1803_02143_b200 import driver
    from paper_1803_02143_b200.dg import vplane_dg

    prob = vpb.problem_spec("landau4d")
    grid = vpb.make_grid(prob, "dg", DOFS, dg_order=3)
    f = vpb.strang_step(vpb.initialize(prob, grid), TAU)  # E != 0
    st = driver.step_state(grid)
    tv = [st.v_tables(d, TAU) for d in range(2)]
    out = torch.empty_like(f.data)
    vplane_dg(grid, f.data, out, tv[0], tv[1], None, None)
    ref = out.view(f._phys.shape).permute(3, 2, 1, 0).cpu().numpy()
    solver = dist.VShardedSolver(grid, dist.VirtualComm(2), range(2), 2)
    solver.scatter(f.numpy())
    solver.e.copy_(st.e)
    flags = {r: (torch.zeros(1, dtype=torch.int32, device="cuda"),
                 torch.zeros(1, dtype=torch.int32, device="cuda")) for r in range(2)}
    hflag = torch.zeros(1, dtype=torch.int32, device="cuda")
    solver._v_pass(TAU, flags, hflag, lambda label: None)
    assert int(hflag.item()) == 0
    assert np.array_equal(solver.gather(), ref)


# ---- spline: all-to-all reshards (vpb_slab_copy + grouped send/recv) ----------
SP_DOFS = (64, 48, 32, 24)


def spline_setup(world):
    prob = vpb.problem_spec("landau4d")
    grid = vpb.make_grid(prob, "spline", SP_DOFS)
    solver = dist.SplineShardedSolver(grid, dist.VirtualComm(world), range(world), world)
    f0 = vpb.initialize(prob, grid)
    solver.scatter(f0.numpy())
    return prob, grid, solver, f0


@pytest.mark.parametrize("world", [2, 3, 8])
def test_spline_reshard_round_trip_is_exact(world):
    prob, grid, solver, f0 = spline_setup(world)
    before = solver.gather()
    solver._a_to_b()
    # layout B of every rank is the x2 slab of the global field
    ref = f0.numpy()
    for s in range(world):
        x0, x1 = solver.xr[s]
        d = solver.dims_b(s)
        got = solver.b[s][0].view(d[3], d[2], d[1], d[0]).permute(3, 2, 1, 0).cpu().numpy()
        assert np.array_equal(got, ref[:, x0:x1])
    for r in range(world):
        solver.a[r][0].zero_()
    solver._b_to_a()
    assert np.array_equal(solver.gather(), before)


@pytest.mark.parametrize("world", [2, 4, 8])
def test_spline_sharded_steps_match_single_gpu_step(world):
    prob, grid, solver, f0 = spline_setup(world)
    f = f0
    for m in range(3):
        solver.step(TAU)
        f = vpb.strang_step(f, TAU, consume=True)
        assert max_rel(solver.gather(), f.numpy()) <= 1e-13, m
    got = solver.diagnostics(3 * TAU)
    rec = vpb.diagnostics(f, 3 * TAU)
    for k in ("mass", "l1_norm", "l2_norm", "kinetic_energy", "electric_energy"):
        assert got[k] == pytest.approx(getattr(rec, k), rel=1e-12), k


def test_spline_sharded_initialize_is_the_slab_of_the_global_initial_state():
    prob, grid, solver, f0 = spline_setup(4)
    solver.initialize(prob)
    assert np.array_equal(solver.gather(), f0.numpy())
