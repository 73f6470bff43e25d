"""Exercise every kernel family of libvpb200.so on small grids, for
compute-sanitizer (memcheck / racecheck / synccheck / initcheck).

    compute-sanitizer --tool racecheck python scripts/sanitize.py [family ...]

Families: dg (strang_step p=2,3 + diagnostics), advance (fast + exact merged
x passes with the density epilogue), graph (StepGraph replay), spline
(strang_step + advance: recursive-filter tiles, rows kernel, double sweeps),
plugin (the four plugin entry points: Thomas/Markstein kernel, dg rows/cols),
dist (x1-sharded halo sweeps and the halo stencil pass, spline all-to-all
slab copies, through VirtualComm on one device), e2e (host-field stepper).
Each family prints one line; the script exits non-zero on a parity failure.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import paper_1803_02143_b200 as vpb  # noqa: E402
from paper_1803_02143_b200 import dist  # noqa: E402


def rel(a, b):
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


def fam_dg():
    prob = vpb.problem_spec("landau4d")
    for order, dofs in ((2, (16, 12, 10, 8)), (3, (24, 18, 12, 12))):
        grid = vpb.make_grid(prob, "dg", dofs, dg_order=order)
        f = vpb.initialize(prob, grid)
        for _ in range(2):
            f = vpb.strang_step(f, 0.3, consume=True)
        rec = vpb.diagnostics(f, 0.6)
        print(f"dg order {order}: EE {rec.electric_energy:.6g}")


def fam_advance():
    prob = vpb.problem_spec("landau4d")
    grid = vpb.make_grid(prob, "dg", (24, 18, 12, 12), dg_order=3)
    f0 = vpb.initialize(prob, grid)
    ref = f0
    for _ in range(3):
        ref = vpb.strang_step(ref, 0.3)
    for mode in ("fast", "exact"):
        vpb.set_arithmetic(mode)
        got = vpb.advance(f0, 0.3, 3)
        e = rel(got.numpy(), ref.numpy())
        print(f"advance {mode}: rel {e:.2e}")
        assert e <= 1e-13
    vpb.set_arithmetic("fast")


def fam_graph():
    prob = vpb.problem_spec("landau4d")
    grid = vpb.make_grid(prob, "dg", (24, 18, 12, 12), dg_order=3)
    f = vpb.initialize(prob, grid)
    g = vpb.StepGraph(f, 0.3)
    for _ in range(2):
        out = g.step()
    print(f"graph: sum {float(out.data.sum()):.6g}")


def fam_spline():
    prob = vpb.problem_spec("landau4d")
    grid = vpb.make_grid(prob, "spline", (32, 24, 16, 16))
    f0 = vpb.initialize(prob, grid)
    f = f0
    for _ in range(2):
        f = vpb.strang_step(f, 0.3)
    g = vpb.advance(f0, 0.3, 2)
    e = rel(g.numpy(), f.numpy())
    print(f"spline: advance vs steps rel {e:.2e}")
    assert e <= 1e-12


def fam_plugin():
    from paper_1803_02143_b200.kernels import _CudaBackend as cb

    rng = np.random.default_rng(1)
    lines = rng.standard_normal((37, 24))
    idx = rng.integers(0, 5, 37).astype(np.int64)
    shifts = rng.uniform(-3, 3, 5) * 0.5
    a, b, q, al = vpb.projection_pairs(shifts, 0.5, 3)
    out = cb.dg_sweep_contig(lines, idx, a, b, q, al, 8, 3, 1)
    view = rng.standard_normal((5, 6, 24))
    cb.dg_sweep_strided(view, np.zeros(30, np.int64), a, b, q, al, 8, 3, 8, 1)
    sp = cb.spline_sweep_contig(lines, idx, shifts, 0.5, 1)
    print(f"plugin: {out.sum():.6g} {sp.sum():.6g}")


def fam_dist():
    prob = vpb.problem_spec("landau4d")
    grid = vpb.make_grid(prob, "dg", (48, 36, 24, 24), dg_order=3)
    f0 = vpb.initialize(prob, grid)
    for p1, p2, how in ((2, 1, "advance"), (2, 2, "step"), (4, 2, "advance")):
        dec = dist.Decomposition(grid, p1, p2)
        solver = dist.ShardedSolver(grid, dec, dist.VirtualComm(dec.world), range(dec.world))
        solver.scatter(f0.numpy())
        if how == "advance":
            solver.advance(0.4, 2)
            ref = vpb.advance(f0, 0.4, 2)
        else:
            solver.step(0.4)
            ref = vpb.strang_step(f0, 0.4)
        e = rel(solver.gather(), ref.numpy())
        print(f"dist {p1}x{p2} {how}: rel {e:.2e}")
        assert e <= 1e-13
    sgrid = vpb.make_grid(prob, "spline", (32, 24, 16, 16))
    sf = vpb.initialize(prob, sgrid)
    ss = dist.SplineShardedSolver(sgrid, dist.VirtualComm(2), range(2), 2)
    ss.scatter(sf.numpy())
    ss.step(0.3)
    e = rel(ss.gather(), vpb.strang_step(sf, 0.3).numpy())
    print(f"dist spline 2: rel {e:.2e}")
    assert e <= 1e-13


def fam_e2e():
    from paper_1803_02143_b200 import hoststep

    prob = vpb.problem_spec("landau4d")
    grid = vpb.make_grid(prob, "dg", (24, 18, 12, 12), dg_order=3)
    f0 = vpb.initialize(prob, grid)
    host = hoststep.HostField.from_field(f0)
    stepper = hoststep.HostStepper(grid, blocks=3)
    stepper.steps(host, 0.3, 2)
    ref = vpb.strang_step(vpb.strang_step(f0, 0.3), 0.3)
    e = rel(host.logical(), ref.numpy())
    print(f"e2e: rel {e:.2e}")
    assert e == 0.0


FAMILIES = {
    "dg": fam_dg,
    "advance": fam_advance,
    "graph": fam_graph,
    "spline": fam_spline,
    "plugin": fam_plugin,
    "dist": fam_dist,
    "e2e": fam_e2e,
}


def main(argv):
    names = argv or list(FAMILIES)
    for n in names:
        FAMILIES[n]()
    torch.cuda.synchronize()
    print("sanitize: all families ran")


if __name__ == "__main__":
    main(sys.argv[1:])
