"""Does host-link DMA slow the compute stream's launches?  A chain of N short
pass-like CUDA graphs (each ~0.4 ms of GEMM) runs on one stream, alone and while a
copy stream moves pinned host memory H2D, D2H, or both.  Reports per-launch gap
(stream time minus kernel time) for eager launches, per-pass graphs, and the whole
chain captured as ONE graph."""
import json
import time

import torch

dev = torch.device("cuda:0")
torch.cuda.set_device(dev)
a = torch.randn(4096, 2048, device=dev, dtype=torch.bfloat16)
w = torch.randn(2048, 2048, device=dev, dtype=torch.bfloat16)
outs = [torch.empty(4096, 2048, device=dev, dtype=torch.bfloat16) for _ in range(4)]
N = 200
comp = torch.cuda.Stream(dev)
c_h2d = torch.cuda.Stream(dev)
c_d2h = torch.cuda.Stream(dev)
host = torch.empty(512 << 20, dtype=torch.uint8).pin_memory()
host2 = torch.empty(512 << 20, dtype=torch.uint8).pin_memory()
dbuf = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
dbuf2 = torch.empty(512 << 20, dtype=torch.uint8, device=dev)


def body(i):
    for j in range(4):
        torch.mm(a, w, out=outs[j])


# per-pass graphs
graphs = []
with torch.cuda.stream(comp):
    for i in range(4):
        body(i)
    torch.cuda.synchronize()
    for i in range(8):
        g = torch.cuda.CUDAGraph()
        g.capture_begin()
        body(i)
        g.capture_end()
        graphs.append(g)
    ev_between = [torch.cuda.Event() for _ in range(N)]
    whole = torch.cuda.CUDAGraph()
    whole.capture_begin()
    for i in range(N):
        body(i)
    whole.capture_end()
torch.cuda.synchronize()


def run(kind):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(comp):
        s.record()
        if kind == "eager":
            for i in range(N):
                body(i)
                ev_between[i].record()
        elif kind == "graphs":
            for i in range(N):
                graphs[i % 8].replay()
                ev_between[i].record()
        else:
            whole.replay()
        e.record()
    return s, e


def copies(mode, reps):
    for _ in range(reps):
        if mode in ("h2d", "both"):
            with torch.cuda.stream(c_h2d):
                dbuf.copy_(host, non_blocking=True)
        if mode in ("d2h", "both"):
            with torch.cuda.stream(c_d2h):
                host2.copy_(dbuf2, non_blocking=True)


res = {}
for kind in ("eager", "graphs", "whole"):
    for mode in ("none", "h2d", "d2h", "both"):
        ts = []
        for rep in range(3):
            torch.cuda.synchronize()
            copies(mode, 16)  # ~150 ms of link traffic per direction
            s, e = run(kind)
            torch.cuda.synchronize()
            ts.append(s.elapsed_time(e))
        res[f"{kind}/{mode}"] = round(min(ts), 3)
        print(kind, mode, res[f"{kind}/{mode}"], "ms for", N, "passes", flush=True)
print(json.dumps(res))
