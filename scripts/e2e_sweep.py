"""host_steps() e2e at config 2 for several block counts (ms per step)."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_1803_02143_b200 as vpb  # noqa: E402

prob = vpb.problem_spec("landau4d")
grid = vpb.make_grid(prob, "dg", 192, dg_order=3)
host = vpb.HostField.from_field(vpb.initialize(prob, grid))
out = {}
for blocks in [int(b) for b in (sys.argv[1:] or ["2", "4", "8", "16", "32", "64"])]:
    vpb.host_steps(host, 0.05, 1, blocks=blocks)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    vpb.host_steps(host, 0.05, 3, blocks=blocks)
    e1.record()
    torch.cuda.synchronize()
    out[blocks] = e0.elapsed_time(e1) / 3
    print(blocks, out[blocks], flush=True)
    from paper_1803_02143_b200 import hoststep
    hoststep._stepper.cache_clear()
    torch.cuda.empty_cache()
print(json.dumps(out))
