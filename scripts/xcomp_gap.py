"""Warm-in-loop vs isolated time of the composed merged x pass (config 2).

A: the x pass alone, back to back (same tables, ping-pong buffers);
B: inside advance() (after the v pass, as in the bench);
C: v pass -> 256 MB L2-flush write -> x pass (dirty L2 lines of the v pass
   written back before the x pass starts).
SM clocks are sampled by nvidia-smi around each phase."""
import json
import subprocess
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

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


def clk():
    try:
        return subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw",
                               "--format=csv,noheader,nounits"], capture_output=True,
                              text=True).stdout.strip()
    except OSError:
        return None


def timed(fn, reps):
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        fn(pre=True)
        e0.record()
        fn(pre=False)
        e1.record()
        ts.append((e0, e1))
    torch.cuda.synchronize()
    v = sorted(a.elapsed_time(b) for a, b in ts)
    return {"median_ms": v[len(v) // 2], "min_ms": v[0], "max_ms": v[-1], "clk": clk()}


def xpass(pre):
    global src, dst
    if pre:
        return
    driver.xcomp_density_dg(grid, src, dst, t1, t2, flag, st, stats)
    src, dst = dst, src


def vx(pre):
    global src, dst
    if pre:
        tv1, tv2 = st.v_tables(0, tau), st.v_tables(1, tau)
        vplane_dg(grid, src, dst, tv1, tv2, None, None)
        src, dst = dst, src
        return
    xpass(False)


def vflushx(pre):
    if pre:
        vx(True)
        flush.fill_(1.0)
        return
    xpass(False)


res = {"A_isolated_back_to_back": timed(xpass, 20), "B_after_vpass": timed(vx, 20),
       "C_after_vpass_and_l2_flush": timed(vflushx, 20)}
print(json.dumps(res, indent=1))
