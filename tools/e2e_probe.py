"""Host-side timing of the pipelined end-to-end loop (diagnostic): per step, how long each public
call blocks the host, and the wall time per step."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_07853_b200 import mpl, scenes  # noqa: E402

sc = scenes.by_name(sys.argv[1] if len(sys.argv) > 1 else "cfg4", 32)
ctx = mpl.from_scene(sc, 0)
host = [torch.from_numpy(np.ascontiguousarray(a)).to(torch.float32).pin_memory() for a in (sc.x, sc.v, sc.F, sc.G, sc.vol)]
mat = torch.from_numpy(np.ascontiguousarray(sc.mat)).pin_memory()
n = sc.n_particles
outs = [torch.empty((n, w), dtype=torch.float32).pin_memory() for w in (3, 3, 9, 9)]
print("pinned:", [h.is_pinned() for h in host], flush=True)
# copy bandwidths alone
d = [torch.empty_like(h, device="cuda") for h in host]
torch.cuda.synchronize()
t = time.perf_counter()
for a, b in zip(d, host):
    a.copy_(b, non_blocking=True)
torch.cuda.synchronize()
th = time.perf_counter() - t
t = time.perf_counter()
for a, b in zip(d, host):
    b.copy_(a, non_blocking=True)
torch.cuda.synchronize()
td = time.perf_counter() - t
nb = sum(h.numel() * 4 for h in host)
print(f"H2D {nb/th/1e9:.1f} GB/s ({th*1e3:.1f} ms), D2H {nb/td/1e9:.1f} GB/s ({td*1e3:.1f} ms)", flush=True)
s1 = torch.cuda.Stream()
s2 = torch.cuda.Stream()
torch.cuda.synchronize()
t = time.perf_counter()
with torch.cuda.stream(s1):
    for a, b in zip(d, host):
        a.copy_(b, non_blocking=True)
with torch.cuda.stream(s2):
    for a, b in zip(d, host):
        b.copy_(a, non_blocking=True)
torch.cuda.synchronize()
print(f"H2D + D2H concurrently: {(time.perf_counter()-t)*1e3:.1f} ms", flush=True)
del d
for mode in ("stage+readback", "stage only", "readback only"):
    stage = mode != "readback only"
    rb = mode != "stage only"
    if stage:
        ctx.stage_particles(*host, mat)
    T = []
    t_all = time.perf_counter()
    for i in range(4):
        r = {}
        if not stage:
            t = time.perf_counter(); ctx.set_particles(*host, mat); r["set"] = time.perf_counter() - t
        t = time.perf_counter(); ctx.resample(sc.dt); r["resample"] = time.perf_counter() - t
        t = time.perf_counter()
        if stage and i < 3:
            ctx.stage_particles(*host, mat)
        r["stage"] = time.perf_counter() - t
        t = time.perf_counter(); st = ctx.newton_step(sc.solver); r["newton"] = time.perf_counter() - t
        t = time.perf_counter(); ctx.transfer_to_particles(sc.dt); r["transfer"] = time.perf_counter() - t
        t = time.perf_counter()
        if rb:
            ctx.get_particles_async(*outs)
        r["get_async"] = time.perf_counter() - t
        T.append({k: round(v * 1e3, 2) for k, v in r.items()})
    t = time.perf_counter(); ctx.stage_wait(); w = time.perf_counter() - t
    print(f"{mode}: total {(time.perf_counter()-t_all)*1e3:.1f} ms for 4 steps, final wait {w*1e3:.1f} ms", flush=True)
    for x in T:
        print("  ", x, flush=True)
