"""Per-label device time of the velocity-sharded advance() with all W shards
in one process (VirtualComm), i.e. where the emulated per-rank time goes.

    python scripts/vshard_breakdown.py --config cfg2 --world 8 --steps 5
"""
import argparse
import json
import sys
from collections import defaultdict
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

CFG = {"cfg2": ("landau4d", 192, 3, 0.05), "cfg5": ("landau4d", 288, 3, 0.05),
       "cfg3": ("twostream4d_baseline", 128, 2, 0.1)}


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--world", type=int, default=8)
    ap.add_argument("--steps", type=int, default=5)
    args = ap.parse_args()
    import torch

    import paper_1803_02143_b200 as vpb
    from paper_1803_02143_b200 import dist

    prob, dofs, order, tau = CFG[args.config]
    problem = vpb.problem_spec(prob)
    grid = vpb.make_grid(problem, "dg", dofs, dg_order=order)
    w = args.world
    solver = dist.VShardedSolver(grid, dist.VirtualComm(w), range(w), w)
    solver.initialize(problem)
    solver.advance(tau, 2)
    torch.cuda.synchronize()
    labels, evs = [], []

    def mark(label):
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        evs.append(e)
        labels.append(label)

    solver.advance(tau, args.steps, timer=mark)
    torch.cuda.synchronize()
    tot = defaultdict(float)
    for i in range(len(evs) - 1):
        if labels[i] is not None:
            tot[labels[i]] += evs[i].elapsed_time(evs[i + 1])
    all_ms = evs[0].elapsed_time(evs[-1])
    print(json.dumps({"config": args.config, "world": w, "steps": args.steps,
                      "per_rank_ms_per_step": all_ms / args.steps / w,
                      "per_rank_ms_by_label": {k: v / args.steps / w for k, v in
                                               sorted(tot.items(), key=lambda kv: -kv[1])}}))


if __name__ == "__main__":
    main()
