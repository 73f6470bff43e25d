"""Digest (sha256) of one composed merged-x pass with the density epilogue
(vpb_dg_sweep_xcomp_density) on a few grids: compare two builds of the
library bitwise (VPB_LIB=... python scripts/xcomp_digest.py)."""

from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

GRIDS = [((192, 192, 96, 48), 3, 0.05), ((288, 288, 24, 24), 3, 0.05),
         ((128, 128, 64, 32), 2, 0.1), ((60, 40, 20, 16), 4, 0.3)]


def main() -> None:
    import torch

    import paper_1803_02143_b200 as vpb
    from paper_1803_02143_b200 import driver

    prob = vpb.problem_spec("landau4d")
    out = {}
    for dofs, order, tau in GRIDS:
        grid = vpb.make_grid(prob, "dg", dofs, dg_order=order)
        f = vpb.initialize(prob, grid)
        st = driver.step_state(grid)
        t1, t2 = st.x_tables(0, tau), st.x_tables(1, tau)
        flag = torch.zeros(1, dtype=torch.int32, device="cuda")
        stats = torch.zeros(4, dtype=torch.float64, device="cuda")
        dst = st.buf
        driver.xcomp_density_dg(grid, f.data, dst, t1, t2, flag, st, stats)
        torch.cuda.synchronize()
        h = hashlib.sha256(dst.cpu().numpy().tobytes())
        h.update(st.rc.cpu().numpy().tobytes())
        h.update(stats.cpu().numpy().tobytes())
        out["x".join(map(str, dofs)) + f"_p{order}"] = h.hexdigest()[:16]
    print(json.dumps(out))


if __name__ == "__main__":
    main()
