"""Where the e2e step time goes: one host_steps() step at config 2 with
timing events around every copy and pass (timeline in ms from the start)."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_1803_02143_b200 as vpb  # noqa: E402
from paper_1803_02143_b200 import hoststep  # noqa: E402

blocks = int(sys.argv[1]) if len(sys.argv) > 1 else 16
prob = vpb.problem_spec("landau4d")
grid = vpb.make_grid(prob, "dg", 192, dg_order=3)
host = vpb.HostField.from_field(vpb.initialize(prob, grid))
vpb.host_steps(host, 0.05, 2, blocks=blocks)
stp = hoststep._stepper(grid, torch.cuda.current_device(), blocks)
# swap the done-events for timing events and add start events
T = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
nb = len(stp.rows)
stp.h2d_done = [T() for _ in range(nb)]
stp.d2h_done = [T() for _ in range(nb)]
stp.closed = [T() for _ in range(nb)]
torch.cuda.synchronize()
t0 = T()
t0.record()
vpb.host_steps(host, 0.05, 3, blocks=blocks)
t1 = T()
t1.record()
torch.cuda.synchronize()
rel = lambda e: t0.elapsed_time(e)  # noqa: E731
print(json.dumps({
    "blocks": nb, "total_ms_3_steps": rel(t1),
    "last_step_h2d_done": [round(rel(e), 2) for e in stp.h2d_done],
    "last_step_closed": [round(rel(e), 2) for e in stp.closed],
    "last_step_d2h_done": [round(rel(e), 2) for e in stp.d2h_done],
}))
