"""Host link bandwidth of this box: pinned H2D alone, D2H alone, and both at once on two streams
(1.5 GB each, the size of one cfg4 step's particle state)."""
import json
import time

import torch

N = 1536 * 1024 * 1024 // 4
dev_a = torch.empty(N, device="cuda")
dev_b = torch.empty(N, device="cuda")
host_a = torch.empty(N).pin_memory()
host_b = torch.empty(N).pin_memory()
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
nbytes = N * 4


def run(h2d, d2h):
    torch.cuda.synchronize()
    t = time.perf_counter()
    if h2d:
        with torch.cuda.stream(s1):
            dev_a.copy_(host_a, non_blocking=True)
    if d2h:
        with torch.cuda.stream(s2):
            host_b.copy_(dev_b, non_blocking=True)
    torch.cuda.synchronize()
    return time.perf_counter() - t


run(True, True)
out = {}
for name, a, b in (("h2d", True, False), ("d2h", False, True), ("both", True, True)):
    ts = [run(a, b) for _ in range(3)]
    t = min(ts)
    out[name] = {"ms": round(t * 1e3, 2), "GBps_per_direction": round(nbytes / t / 1e9, 1)}
print(json.dumps(out))
