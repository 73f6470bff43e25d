"""Warm-in-loop vs isolated time of the composed merged x pass, with the SM
clock sampled (nvidia-smi, 50 ms) inside each phase.

A  the x pass alone, back to back (same tables, ping-pong buffers)
B  v pass -> x pass, back to back (the steady state of advance())
C  v pass -> 256 MB L2-flush write -> x pass (dirty v-pass lines written back first)
D  200 ms idle -> v pass -> x pass (the pair from a cool, unthrottled start)

    python scripts/xcomp_gap.py [cfg2|cfg3|cfg5]
"""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1803_02143_b200 as vpb  # noqa: E402
from paper_1803_02143_b200 import driver  # noqa: E402
from paper_1803_02143_b200.dg import vplane_dg  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
dofs = {"cfg2": 192, "cfg5": 288, "cfg3": 128}[cfg]
order = 2 if cfg == "cfg3" else 3
prob = vpb.problem_spec("twostream4d_baseline" if cfg == "cfg3" else "landau4d")
grid = vpb.make_grid(prob, "dg", dofs, dg_order=order)
tau = 0.1 if cfg == "cfg3" else 0.05
f = vpb.initialize(prob, grid)
st = driver.step_state(grid)
f = vpb.advance(f, tau, 3, consume=True)
t1, t2 = st.x_tables(0, tau), st.x_tables(1, tau)
flag = torch.zeros(1, dtype=torch.int32, device="cuda")
stats = torch.zeros(4, dtype=torch.float64, device="cuda")
src, dst = f.data, st.buf
flush = torch.empty(256 << 17, dtype=torch.float64, device="cuda")  # 256 MB


def xpass():
    global src, dst
    driver.xcomp_density_dg(grid, src, dst, t1, t2, flag, st, stats)
    src, dst = dst, src


def vpass():
    global src, dst
    vplane_dg(grid, src, dst, st.v_tables(0, tau), st.v_tables(1, tau), None, None)
    src, dst = dst, src


def phase(pre, reps, idle=0.0):
    clk = bench.ClockSampler(0).start()
    ts = []
    clk.begin()
    for _ in range(reps):
        if idle:
            torch.cuda.synchronize()
            time.sleep(idle)
        pre()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        xpass()
        e1.record()
        ts.append((e0, e1))
    torch.cuda.synchronize()
    clk.end()
    clk.stop()
    v = sorted(a.elapsed_time(b) for a, b in ts)
    return {"median_ms": v[len(v) // 2], "min_ms": v[0], "max_ms": v[-1],
            "clocks": clk.summary()}


res = {
    "A_isolated_back_to_back": phase(lambda: None, 30),
    "B_after_vpass": phase(vpass, 30),
    "C_after_vpass_and_l2_flush": phase(lambda: (vpass(), flush.fill_(1.0)), 30),
    "D_cool_start_then_vpass": phase(vpass, 15, idle=0.2),
}
print(json.dumps(res, indent=1))
