"""Time the composed merged-x pass (vpb_dg_sweep_xcomp_density) alone on a
BASELINE grid; launch parameters come from VPB_XCOMP_* in the environment.

    python scripts/tune_xcomp.py --config cfg5 [--reps 5]
"""

from __future__ import annotations

import argparse
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

GRIDS = {"cfg2": (192, 3, 0.05), "cfg3": (128, 2, 0.1), "cfg5": (288, 3, 0.05)}


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--nodens", action="store_true")
    args = ap.parse_args()
    import torch

    import paper_1803_02143_b200 as vpb
    from paper_1803_02143_b200 import driver

    dofs, order, tau = GRIDS[args.config]
    prob = vpb.problem_spec("landau4d")
    grid = vpb.make_grid(prob, "dg", dofs, dg_order=order)
    f = vpb.initialize(prob, grid)
    st = driver.step_state(grid)
    t1, t2 = st.x_tables(0, tau), st.x_tables(1, tau)
    out = st.buf
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")
    stats = torch.zeros(4, dtype=torch.float64, device="cuda")

    def once(a, b):
        if args.nodens:
            driver.xcomp_dg(grid, a, b, t1, t2, flag)
        else:
            driver.xcomp_density_dg(grid, a, b, t1, t2, flag, st, stats)

    src = f.data
    once(src, out)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.reps + 1)]
    ev[0].record()
    for r in range(args.reps):
        once(src, out) if r % 2 == 0 else once(out, src)
        ev[r + 1].record()
    torch.cuda.synchronize()
    ms = sorted(ev[r].elapsed_time(ev[r + 1]) for r in range(args.reps))
    n = grid.total_dof
    med = ms[len(ms) // 2]
    print(json.dumps({"config": args.config, "env": {k: v for k, v in os.environ.items()
                                                      if k.startswith("VPB_XCOMP")},
                      "ms_med": med, "ms_min": ms[0], "frac": 16 * n / (med * 1e-3) / 6449.4e9}))


if __name__ == "__main__":
    main()
