"""PCIe ceiling for the e2e path: pinned host <-> HBM copy bandwidth one
direction at a time and both directions at once (two streams)."""
import json
import sys

import torch

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 1 << 30  # doubles per buffer
h1 = torch.empty(n, dtype=torch.float64, pin_memory=True)
h2 = torch.empty(n, dtype=torch.float64, pin_memory=True)
h1.fill_(1.0)
h2.fill_(2.0)
d1 = torch.empty(n, dtype=torch.float64, device="cuda")
d2 = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fn()
    for s in (s1, s2):
        torch.cuda.current_stream().wait_stream(s)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e-3


def h2d():
    with torch.cuda.stream(s1):
        s1.wait_stream(torch.cuda.current_stream())
        d1.copy_(h1, non_blocking=True)


def d2h():
    with torch.cuda.stream(s2):
        s2.wait_stream(torch.cuda.current_stream())
        h2.copy_(d2, non_blocking=True)


def both():
    h2d()
    d2h()


res = {}
for name, fn in (("h2d", h2d), ("d2h", d2h), ("both", both)):
    fn()
    t = min(timed(fn) for _ in range(3))
    res[name + "_gbs_per_direction"] = 8 * n / t / 1e9
print(json.dumps(res))
