"""Prototype: the dG step with the v pass and the merged x pass split into
blocks of v2 cells on two streams, so the x pass of block b (latency-bound)
overlaps the v pass of block b+1 (HBM-bound).  Times K steady-state steps
(field solve -> v pass blocks -> merged x pass blocks with density partials)
against advance() on the same grid.

    python scripts/proto_overlap.py --config cfg2 --blocks 1 2 4 8 --steps 20
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

GRIDS = {"cfg2": ("landau4d", 192, 3, 0.05), "cfg3": ("twostream4d_baseline", 128, 2, 0.1),
         "small": ("landau4d", (48, 48, 48, 48), 3, 0.05)}


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--blocks", type=int, nargs="+", default=[1, 2, 4, 8])
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--check", action="store_true")
    args = ap.parse_args()
    import torch

    import paper_1803_02143_b200 as vpb
    from paper_1803_02143_b200 import dist
    from paper_1803_02143_b200.grid import gauss_nodes
    from paper_1803_02143_b200.poisson import _lagrange_row

    prob_name, dofs, order, tau = GRIDS[args.config]
    prob = vpb.problem_spec(prob_name)
    grid = vpb.make_grid(prob, "dg", dofs, dg_order=order)
    ops = dist.CudaOps()
    p = order
    n1, n2, nv1, nv2 = grid.dims4
    C2 = nv2 // p
    row = n1 * n2 * nv1
    dev = torch.device("cuda")
    w = [torch.as_tensor(grid.axis_weights(a), dtype=torch.float64).to(dev) for a in range(4)]
    wv1, wv2 = w[2], w[3]
    vpts = [torch.as_tensor(grid.axis_points(a), dtype=torch.float64).to(dev) for a in (2, 3)]
    t1 = ops.tables(vpts[0], 0.5 * tau, grid.axes[0].h, grid.dg_degree)
    t2 = ops.tables(vpts[1], 0.5 * tau, grid.axes[1].h, grid.dg_degree)
    nodes, _ = gauss_nodes(p)
    mid = np.ascontiguousarray(_lagrange_row(nodes, 0.5))
    wc = [np.ascontiguousarray(np.asarray(grid.axis_weights(a))[:p]) for a in (0, 1)]
    ax = grid.axes
    volume = (ax[0].upper - ax[0].lower) * (ax[1].upper - ax[1].lower)
    nx = n1 * n2
    e = torch.empty(2 * nx, dtype=torch.float64, device=dev)
    fl = torch.zeros(8, dtype=torch.int32, device=dev)
    hflag = torch.zeros(1, dtype=torch.int32, device=dev)
    s0 = torch.cuda.current_stream()
    s1 = torch.cuda.Stream()

    f0 = vpb.initialize(prob, grid)
    out = {"config": args.config, "steps": args.steps}

    # reference: advance() (open + K-1 merged + close) timed as the bench does
    a = vpb.advance(f0, tau, 3)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record()
    a = vpb.advance(f0, tau, args.steps)
    ev[1].record()
    torch.cuda.synchronize()
    out["advance_ms_per_step"] = ev[0].elapsed_time(ev[1]) / args.steps

    def run(nb: int, steps: int, bufs: list, rc: torch.Tensor):
        """bufs = [v input, v output / x input, x output]; rotated every step,
        so the x pass of block b waits only for the v pass of block b."""
        edges = [round(i * C2 / nb) for i in range(nb + 1)]
        blocks = [(edges[i], edges[i + 1]) for i in range(nb)]
        evv = [torch.cuda.Event() for _ in range(nb)]
        evx = torch.cuda.Event()
        for m in range(steps):
            A, B, C = bufs
            ops.field_solve_centred(grid, rc, e, fl[2:3])
            tv = [ops.tables(e[d * nx:(d + 1) * nx], tau, grid.axes[2 + d].h, grid.dg_degree)
                  for d in range(2)]
            for b, (c0, c1) in enumerate(blocks):
                dims = (n1, n2, nv1, (c1 - c0) * p)
                ops.vplane_v2peer(A, C2, (c0 - 1) % C2, A, C2, c0, A, C2, c1 % C2, 1,
                                  B[c0 * p * row:c1 * p * row], dims, p, tv[0], tv[1],
                                  fl[3:4], fl[4:5], hflag)
                evv[b].record(s0)
            parts = []
            with torch.cuda.stream(s1):
                for b, (c0, c1) in enumerate(blocks):
                    s1.wait_event(evv[b])
                    dims = (n1, n2, nv1, (c1 - c0) * p)
                    work = torch.empty(ops.xpass_work(dims, p, 2), dtype=torch.float64,
                                       device=dev)
                    rcb = torch.empty((n1 // p) * (n2 // p), dtype=torch.float64, device=dev)
                    stb = torch.zeros(4, dtype=torch.float64, device=dev)
                    wv2b = wv2[c0 * p:c1 * p].contiguous()
                    dens = (wv1, wv2b, mid, wc[0], wc[1], volume, work, rcb, stb)
                    ops.xpass_rows(B[c0 * p * row:c1 * p * row], C[c0 * p * row:c1 * p * row],
                                   dims, p, t1, t2, c0 * p, 2, fl[5:6], fl[6:7], dens)
                    parts.append(rcb)
                tot = parts[0].clone()
                for r in parts[1:]:
                    tot += r
                rc.copy_(tot)
                evx.record(s1)
            s0.wait_event(evx)
            bufs[:] = [C, A, B]

    for nb in args.blocks:
        A = f0.data.clone()
        bufs = [A, torch.empty_like(A), torch.empty_like(A)]
        rc = torch.empty((n1 // p) * (n2 // p), dtype=torch.float64, device=dev)
        # opening x pass with the density (whole field), as advance() does
        work = torch.empty(ops.xpass_work((n1, n2, nv1, nv2), p, 1), dtype=torch.float64,
                           device=dev)
        stb = torch.zeros(4, dtype=torch.float64, device=dev)
        ops.xpass_rows(f0.data, A, (n1, n2, nv1, nv2), p, t1, t2, 0, 1, fl[0:1], fl[1:2],
                       (wv1, wv2, mid, wc[0], wc[1], volume, work, rc, stb))
        run(nb, 3, bufs, rc)  # warm-up
        torch.cuda.synchronize()
        ev[0].record()
        run(nb, args.steps, bufs, rc)
        ev[1].record()
        torch.cuda.synchronize()
        out[f"blocks{nb}_ms_per_step"] = ev[0].elapsed_time(ev[1]) / args.steps
        out[f"blocks{nb}_hflag"] = int(hflag.item())
        del bufs, A
        torch.cuda.empty_cache()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
