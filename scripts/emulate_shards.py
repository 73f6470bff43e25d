"""Per-rank compute time of the sharded dG step, emulated on ONE GPU.

All W shards of ShardedSolver live in this process (VirtualComm: halo
"messages" are device copies), so running advance() executes every shard's
kernels back to back on one B200.  total / W estimates one rank's compute
time per step on a W-GPU box (each shard's kernels still fill the GPU); NCCL
time is NOT included -- the halo bytes per step and rank are printed so the
NVLink share can be estimated.  This is a projection, not a multi-GPU
measurement.

    python scripts/emulate_shards.py --config cfg2 --worlds 1 2 4 8 --steps 5
    python scripts/emulate_shards.py --config cfg5 --worlds 2 4 8 --vshard

--vshard runs VShardedSolver (velocity-direction sharding, the paper's own
choice) the same way: every shard's x passes
(local, whole (x1, x2) planes), v2 halo copies and halo-fed v pass back to
back on one GPU, total / W per rank.
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

CFG = {"cfg2": ("landau4d", 192, 3, 0.05), "cfg3": ("twostream4d_baseline", 128, 2, 0.1),
       "cfg5": ("landau4d", 288, 3, 0.05)}


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--worlds", type=int, nargs="+", default=[1, 2, 4, 8])
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--vshard", action="store_true", help="v2-slab sharding (see doc)")
    ap.add_argument("--grid2d", default=None,
                    help="x-sharded process grid P1xP2 (e.g. 4x2): one run of that layout")
    args = ap.parse_args()
    import gc

    import numpy as np
    import torch

    import paper_1803_02143_b200 as vpb
    from paper_1803_02143_b200 import dist, driver

    prob, dofs, order, tau = CFG[args.config]
    problem = vpb.problem_spec(prob)
    grid = vpb.make_grid(problem, "dg", dofs, dg_order=order)
    N = grid.total_dof
    if args.grid2d:
        p1, p2 = (int(x) for x in args.grid2d.split("x"))
        w = p1 * p2
        dec = dist.Decomposition(grid, p1, p2)
        solver = dist.ShardedSolver(grid, dec, dist.VirtualComm(w), range(w))
        solver.initialize(problem)
        ready = solver._stencil_ready(tau)
        merged = ready and solver._merged_halo_fits(tau)
        solver.advance(tau, 2)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        solver._halo_bytes = 0
        e0.record()
        solver.advance(tau, args.steps)
        e1.record()
        torch.cuda.synchronize()
        per_rank = e0.elapsed_time(e1) / args.steps / w
        print(json.dumps({"config": args.config, "world": w, "layout": f"x1 x x2 {p1}x{p2}",
                          "stencil_passes": ready, "merged_pass": merged,
                          "per_rank_compute_ms_per_step": per_rank,
                          "projected_dof_per_s_compute_only": N / (per_rank * 1e-3),
                          "halo_bytes_per_rank_per_step": int(solver._halo_bytes
                                                              / args.steps / w),
                          "cells_per_shard": [grid.axes[0].count // p1,
                                              grid.axes[1].count // p2]}), flush=True)
        return
    for w in args.worlds:
        if args.vshard:
            solver = dist.VShardedSolver(grid, dist.VirtualComm(w), range(w), w)
            solver.initialize(problem)
            solver.advance(tau, 2)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            solver._halo_bytes = 0
            e0.record()
            solver.advance(tau, args.steps)
            e1.record()
            torch.cuda.synchronize()
            per_rank = e0.elapsed_time(e1) / args.steps / w
            print(json.dumps({"config": args.config, "world": w, "layout": f"v2 x{w}",
                              "per_rank_compute_ms_per_step": per_rank,
                              "projected_dof_per_s_compute_only": N / (per_rank * 1e-3),
                              "v2_cells_per_rank": solver.cr[0][1] - solver.cr[0][0],
                              "halo_cells_per_side": solver.H,
                              "halo_bytes_per_rank_per_step": int(solver._halo_bytes
                                                                  / args.steps / w),
                              "rho_allgather_bytes": 8 * (grid.axes[0].count
                                                          * grid.axes[1].count)}), flush=True)
            del solver
            driver._state_cached.cache_clear()
            gc.collect()
            torch.cuda.empty_cache()
            continue
        if w == 1:
            f = vpb.initialize(problem, grid)
            f = vpb.advance(f, tau, 2, consume=True)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            f = vpb.advance(f, tau, args.steps, consume=True)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / args.steps
            print(json.dumps({"config": args.config, "world": 1, "ms_per_step": ms,
                              "dof_per_s": N / (ms * 1e-3)}), flush=True)
            del f
        else:
            dec = dist.Decomposition(grid, w, 1)
            solver = dist.ShardedSolver(grid, dec, dist.VirtualComm(w), range(w))
            solver.initialize(problem)
            assert solver._stencil_ready() and solver._merged_halo_fits(tau)
            solver.advance(tau, 2)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            solver.advance(tau, args.steps)
            e1.record()
            torch.cuda.synchronize()
            total = e0.elapsed_time(e1) / args.steps
            _, _, tabs = solver._stencil_setup(tau)
            wl, wr = tabs[2][2], tabs[2][3]
            halo_bytes = (wl + wr) * order * grid.dof(1) * grid.dof(2) * grid.dof(3) * 8
            per_rank = total / w
            print(json.dumps({"config": args.config, "world": w, "layout": f"x1 x{w}",
                              "all_shards_ms_per_step": total,
                              "per_rank_compute_ms_per_step": per_rank,
                              "projected_dof_per_s_compute_only": N / (per_rank * 1e-3),
                              "halo_cells_left_right": [wl, wr],
                              "halo_bytes_per_rank_per_step": int(halo_bytes),
                              "x1_cells_per_shard": grid.axes[0].count // w}), flush=True)
            del solver
        driver._state_cached.cache_clear()
        gc.collect()
        torch.cuda.empty_cache()
        _ = np


if __name__ == "__main__":
    main()
