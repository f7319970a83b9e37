"""Probe: SM-driven host-link copies (tools/probes/smcopy.cu: a kernel storing to mapped
pinned memory for D2H, loading from it for H2D) vs the copy engines -- link GB/s alone
and the slowdown of an HBM-bound compute loop (LayerNorm + GeLU at C2) running beside
each.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared -Xcompiler -fPIC
-o tools/probes/libsmcopy.so tools/probes/smcopy.cu"""
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2503_01328_b200.runtime import native  # noqa: E402

lib = ctypes.CDLL(os.path.join(ROOT, "tools", "probes", "libsmcopy.so"))
lib.smcopy.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_int, ctypes.c_void_p]
dev = torch.device("cuda:0")
bf = dict(device=dev, dtype=torch.bfloat16)
s, h = 4096, 2048
x, y = torch.randn(s, h, **bf), torch.empty(s, h, **bf)
f, g = torch.randn(s, 4 * h, **bf), torch.empty(s, 4 * h, **bf)
gam, bet = torch.ones(h, device=dev), torch.zeros(h, device=dev)
N = 504_102_912
hd = torch.empty(N, dtype=torch.uint8, pin_memory=True)  # pinned => mapped (UVA): device can address it
hh = torch.empty(N, dtype=torch.uint8, pin_memory=True)
dd, dh = torch.empty(N, dtype=torch.uint8, device=dev), torch.empty(N, dtype=torch.uint8, device=dev)
cs, s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev), torch.cuda.Stream(dev)


def ce(direction, st):
    with torch.cuda.stream(st):
        (hd.copy_(dd, non_blocking=True) if direction == "d2h" else dh.copy_(hh, non_blocking=True))


def sm(direction, st, blocks):
    if direction == "d2h":
        lib.smcopy(dd.data_ptr(), hd.data_ptr(), N, blocks, 512, st.cuda_stream)
    else:
        lib.smcopy(hh.data_ptr(), dh.data_ptr(), N, blocks, 512, st.cuda_stream)


def link_gbs(fn):
    best = 1e9
    for _ in range(3):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s1)
        fn()
        e1.record(s1)
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1) / 1e3)
    return round(N / best / 1e9, 1)


def compute_us(bg=None, n=100):
    torch.cuda.synchronize()
    if bg:
        for _ in range(6):
            bg()
    with torch.cuda.stream(cs):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(cs)
        for _ in range(n):
            native.layernorm_fwd(x, gam, bet, y)
            native.gelu_fwd(f, g)
        e1.record(cs)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / n


compute_us()  # warm-up (first launches, occupancy queries)
out = {"compute_alone_us": round(compute_us(), 2)}
out["ce_d2h_gbs"] = link_gbs(lambda: ce("d2h", s1))
out["compute_with_ce_duplex_us"] = round(compute_us(lambda: (ce("d2h", s1), ce("h2d", s2))), 2)
for blocks in (8, 16, 32):
    out[f"sm{blocks}_d2h_gbs"] = link_gbs(lambda: sm("d2h", s1, blocks))
    out[f"sm{blocks}_h2d_gbs"] = link_gbs(lambda: sm("h2d", s1, blocks))
    out[f"compute_with_sm{blocks}_duplex_us"] = round(compute_us(lambda: (sm("d2h", s1, blocks), sm("h2d", s2, blocks))), 2)
print(json.dumps(out))
