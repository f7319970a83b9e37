"""Does concurrent host-link DMA slow the compute stream?  A C2-shaped compute loop
(PROBE_KIND=mix: fc1 GEMM + GeLU + LayerNorm; gemm: the tcgen05 GEMM alone; hbm: the
HBM-bound LayerNorm + GeLU alone; ln / gelu / lnbwd: one kernel; libppo_b200 kernels) timed alone and
while D2H and H2D of 504 MB slabs run back to back on two copy streams (CUDA events on
the compute stream, best of 5 of 50 iterations)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2503_01328_b200.runtime import native  # noqa: E402

dev = torch.device("cuda:0")
bf = dict(device=dev, dtype=torch.bfloat16)
s, h = 4096, 2048
a, w, f, g = torch.randn(s, h, **bf), torch.randn(4 * h, h, **bf), torch.empty(s, 4 * h, **bf), torch.empty(s, 4 * h, **bf)
x, y = torch.randn(s, h, **bf), torch.randn(s, h, **bf)
gam, bet = torch.ones(h, device=dev), torch.zeros(h, device=dev)
z = torch.zeros(4 * h, device=dev)
N = 504_102_912
hd, hh = torch.empty(N, dtype=torch.uint8, pin_memory=True), torch.empty(N, dtype=torch.uint8, pin_memory=True)
dd, dh = torch.empty(N, dtype=torch.uint8, device=dev), torch.empty(N, dtype=torch.uint8, device=dev)
cs, s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev), torch.cuda.Stream(dev)


KIND = os.environ.get("PROBE_KIND", "mix")


def step():
    if KIND in ("mix", "gemm"):
        native.gemm_tn_gelu(a, w, g, f, z)
    if KIND in ("mix", "hbm", "ln"):
        native.layernorm_fwd(x, gam, bet, y)
    if KIND in ("mix", "hbm", "gelu"):
        native.gelu_fwd(f, g)
    if KIND == "lnbwd":
        native.layernorm_bwd(x, gam, y, x, a, z[:h], z[h:2 * h], drop_out=None, p=0.0)


def timed(n=50):
    with torch.cuda.stream(cs):
        for _ in range(3):
            step()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(cs)
        for _ in range(n):
            step()
        e1.record(cs)
    return e0, e1, n


out = {}
for mode in ("alone", "with_duplex_dma", "with_d2h_dma", "with_h2d_dma") * 2:
    torch.cuda.synchronize()
    if mode != "alone":
        for _ in range(8):
            if mode in ("with_duplex_dma", "with_d2h_dma"):
                with torch.cuda.stream(s1):
                    hd.copy_(dd, non_blocking=True)
            if mode in ("with_duplex_dma", "with_h2d_dma"):
                with torch.cuda.stream(s2):
                    dh.copy_(hh, non_blocking=True)
    e0, e1, n = timed()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / n
    out[mode] = min(out.get(mode, 1e9), us)
print(json.dumps({"kind": KIND, "compute_step_us": {k: round(v, 2) for k, v in out.items()},
                  "slowdown_pct": {k: round(100 * (v / out["alone"] - 1), 2) for k, v in out.items() if k != "alone"}}))
