"""D2H interference vs issue granularity: the HBM-bound compute loop (LayerNorm + GeLU at
C2) beside back-to-back D2H of 504 MB issued as one cudaMemcpyAsync or as chunks of
64 / 16 / 4 MB on the same copy stream; link GB/s of each issue pattern alone.  (The
batched-copy driver call measured in round 1 is closed on this GPU pool and was removed.)"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2503_01328_b200.runtime import native  # noqa: E402

dev = torch.device("cuda:0")
bf = dict(device=dev, dtype=torch.bfloat16)
s, h = 4096, 2048
x, y = torch.randn(s, h, **bf), torch.empty(s, h, **bf)
f, g = torch.randn(s, 4 * h, **bf), torch.empty(s, 4 * h, **bf)
gam, bet = torch.ones(h, device=dev), torch.zeros(h, device=dev)
N = 504_102_912
hd = torch.empty(N, dtype=torch.uint8, pin_memory=True)
dd = torch.empty(N, dtype=torch.uint8, device=dev)
cs, s1 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)


def d2h(chunk):
    with torch.cuda.stream(s1):
        if chunk is None:
            hd.copy_(dd, non_blocking=True)
        else:
            for lo in range(0, N, chunk):
                hi = min(N, lo + chunk)
                hd[lo:hi].copy_(dd[lo:hi], non_blocking=True)


def link(chunk):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s1)
    d2h(chunk)
    e1.record(s1)
    e1.synchronize()
    return round(N / (e0.elapsed_time(e1) / 1e3) / 1e9, 1)


def compute(bg_chunk="none", n=100):
    torch.cuda.synchronize()
    if bg_chunk != "none":
        for _ in range(6):
            d2h(bg_chunk)
    with torch.cuda.stream(cs):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(cs)
        for _ in range(n):
            native.layernorm_fwd(x, gam, bet, y)
            native.gelu_fwd(f, g)
        e1.record(cs)
    torch.cuda.synchronize()
    return round(e0.elapsed_time(e1) * 1e3 / n, 2)


compute()
out = {"alone_us": compute()}
for c in (None, 64 << 20, 16 << 20, 4 << 20):
    key = "whole" if c is None else f"{c >> 20}MB"
    out[key] = {"link_gbs": link(c), "compute_us": compute(c)}
print(json.dumps(out))
