"""host_steps() call time against the step count at config 2: the
increment between K and 2K steps is the steady-state e2e step; the rest is
the call's unoverlapped fill (first H2D) and drain (last D2H)."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_1803_02143_b200 as vpb  # noqa: E402

blocks = int(sys.argv[1]) if len(sys.argv) > 1 else 16
prob = vpb.problem_spec("landau4d")
grid = vpb.make_grid(prob, "dg", 192, dg_order=3)
host = vpb.HostField.from_field(vpb.initialize(prob, grid))
vpb.host_steps(host, 0.05, 1, blocks=blocks)
out = {"blocks": blocks}
for k in (1, 5, 10, 20):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    vpb.host_steps(host, 0.05, k, blocks=blocks)
    e1.record()
    torch.cuda.synchronize()
    out[f"k{k}_ms"] = e0.elapsed_time(e1)
out["steady_ms_per_step"] = (out["k20_ms"] - out["k10_ms"]) / 10
out["fill_drain_ms"] = out["k20_ms"] - 20 * out["steady_ms_per_step"]
print(json.dumps(out))
