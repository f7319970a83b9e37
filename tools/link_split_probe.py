"""Host-link probe: one 504 MB D2H / H2D (the C2 slab) as 1, 2 or 4 concurrent
cudaMemcpyAsync chunks on separate streams (separate copy engines), one direction alone
and both at once; GB/s from CUDA events (best of 5)."""
import json

import torch

dev = torch.device("cuda:0")
N = 504_102_912
host = torch.empty(N, dtype=torch.uint8, pin_memory=True)
host2 = torch.empty(N, dtype=torch.uint8, pin_memory=True)
d = torch.empty(N, dtype=torch.uint8, device=dev)
d2 = torch.empty(N, dtype=torch.uint8, device=dev)
streams = [torch.cuda.Stream(dev) for _ in range(8)]


def run(k, directions):
    best = None
    for _ in range(5):
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        ends = []
        for di, dirn in enumerate(directions):
            for i in range(k):
                s = streams[di * 4 + i]
                s.wait_event(e0)
                lo, hi = N * i // k, N * (i + 1) // k
                with torch.cuda.stream(s):
                    if dirn == "d2h":
                        host[lo:hi].copy_(d[lo:hi], non_blocking=True)
                    else:
                        d2[lo:hi].copy_(host2[lo:hi], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(s)
                ends.append(ev)
        for ev in ends:
            torch.cuda.current_stream().wait_event(ev)
        e1.record()
        e1.synchronize()
        t = e0.elapsed_time(e1) / 1e3
        best = t if best is None else min(best, t)
    return {"chunks": k, "directions": directions, "ms": round(best * 1e3, 2),
            "gbs_per_direction": round(N / best / 1e9, 1)}


for dirs in (["d2h"], ["h2d"], ["d2h", "h2d"]):
    for k in (1, 2, 4):
        print(json.dumps(run(k, dirs)), flush=True)
