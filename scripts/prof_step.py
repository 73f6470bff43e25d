"""Run a few device Strang steps for profiling (ncu launch lists / --set full).

    python scripts/prof_step.py --method dg --order 3 --dofs 192 192 48 48 --steps 2
"""

from __future__ import annotations

import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--problem", default="landau4d")
    ap.add_argument("--method", default="dg")
    ap.add_argument("--order", type=int, default=3)
    ap.add_argument("--dofs", type=int, nargs=4, default=[192, 192, 48, 48])
    ap.add_argument("--tau", type=float, default=0.05)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--advance", action="store_true", help="advance() (merged x passes)")
    args = ap.parse_args()
    import torch

    import paper_1803_02143_b200 as vpb

    prob = vpb.problem_spec(args.problem)
    grid = vpb.make_grid(prob, args.method, tuple(args.dofs), dg_order=args.order)
    f = vpb.initialize(prob, grid)
    if args.advance:
        f = vpb.advance(f, args.tau, args.steps, consume=True)
    else:
        for _ in range(args.steps):
            f = vpb.strang_step(f, args.tau, consume=True)
    torch.cuda.synchronize()
    print("ok", grid.dofs)


if __name__ == "__main__":
    main()
