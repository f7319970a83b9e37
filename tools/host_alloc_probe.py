"""Host-link probe: D2H / H2D of one 504 MB C2 slab into cudaHostAlloc memory with the
portable / write-combined / default flags (CUDA events, best of 5)."""
import json, ctypes
import torch
from cuda.bindings import runtime as rt

dev = torch.device("cuda:0")
torch.cuda.init()
N = 504_102_912
d = torch.empty(N, dtype=torch.uint8, device=dev)
d2 = torch.empty(N, dtype=torch.uint8, device=dev)

def alloc(flags):
    err, p = rt.cudaHostAlloc(N, flags)
    assert err == rt.cudaError_t.cudaSuccess, err
    return p

def bench(hp, direction, other=None):
    s = torch.cuda.current_stream()
    best = 1e9
    for _ in range(5):
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        if direction == "d2h":
            rt.cudaMemcpyAsync(hp, d.data_ptr(), N, rt.cudaMemcpyKind.cudaMemcpyDeviceToHost, s.cuda_stream)
        else:
            rt.cudaMemcpyAsync(d2.data_ptr(), hp, N, rt.cudaMemcpyKind.cudaMemcpyHostToDevice, s.cuda_stream)
        e1.record(); e1.synchronize()
        best = min(best, e0.elapsed_time(e1) / 1e3)
    return round(N / best / 1e9, 1)

for name, flags in (("portable", rt.cudaHostAllocPortable), ("portable+writecombined", rt.cudaHostAllocPortable | rt.cudaHostAllocWriteCombined), ("default", rt.cudaHostAllocDefault)):
    hp = alloc(flags)
    ctypes.memset(hp, 1, N)
    print(json.dumps({"host_alloc": name, "d2h_gbs": bench(hp, "d2h"), "h2d_gbs": bench(hp, "h2d")}), flush=True)
    rt.cudaFreeHost(hp)
