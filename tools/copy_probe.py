"""Does a small D2H copy wait behind a large D2H copy on another stream?  (pageable vs pinned
destination, large copy whole vs in 16 MB chunks; and a kernel-written mapped-memory read)."""
import time

import torch

N = 1500 * 1024 * 1024 // 4
dev = torch.empty(N, device="cuda")
host = torch.empty(N).pin_memory()
small_dev = torch.ones(16, device="cuda")
s_big = torch.cuda.Stream()
s_main = torch.cuda.current_stream()


def big(chunked):
    with torch.cuda.stream(s_big):
        if chunked:
            CH = 4 * 1024 * 1024
            for o in range(0, N, CH):
                host[o:o + CH].copy_(dev[o:o + CH], non_blocking=True)
        else:
            host.copy_(dev, non_blocking=True)


for chunked in (False, True):
    for pinned in (False, True):
        torch.cuda.synchronize()
        big(chunked)
        time.sleep(0.002)
        dst = torch.empty(16).pin_memory() if pinned else torch.empty(16)
        t = time.perf_counter()
        dst.copy_(small_dev, non_blocking=pinned)
        torch.cuda.current_stream().synchronize()
        lat = time.perf_counter() - t
        torch.cuda.synchronize()
        print(f"big D2H {'chunked' if chunked else 'whole  '}: small D2H to {'pinned  ' if pinned else 'pageable'} waited {lat*1e3:.2f} ms", flush=True)
torch.cuda.synchronize()
t = time.perf_counter()
big(False)
torch.cuda.synchronize()
print(f"big D2H alone {(time.perf_counter()-t)*1e3:.1f} ms", flush=True)
