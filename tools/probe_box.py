"""One-off probe of the GPU box: host link bandwidth, topology, attention backends."""
import json, os, subprocess, time
import torch

out = {}
def sh(c):
    try:
        return subprocess.run(c, shell=True, capture_output=True, text=True, timeout=60).stdout
    except Exception as e:
        return str(e)
out["nproc"] = sh("nproc").strip()
out["lscpu"] = sh("lscpu | head -20")
out["topo"] = sh("nvidia-smi topo -m")
out["smi"] = sh("nvidia-smi --query-gpu=name,pci.bus_id,pcie.link.gen.max,pcie.link.width.max,memory.total --format=csv")
out["numa"] = sh("numactl -H 2>/dev/null || ls /sys/devices/system/node")
dev = torch.device("cuda:0")
torch.cuda.init()
def bw(n_bytes, direction, pinned=True, reps=5):
    h = torch.empty(n_bytes, dtype=torch.uint8, pin_memory=pinned)
    d = torch.empty(n_bytes, dtype=torch.uint8, device=dev)
    s = torch.cuda.Stream()
    best = 0
    for _ in range(reps):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            e0.record(s)
            if direction == "d2h":
                h.copy_(d, non_blocking=True)
            else:
                d.copy_(h, non_blocking=True)
            e1.record(s)
        e1.synchronize()
        best = max(best, n_bytes / (e0.elapsed_time(e1) * 1e-3) / 1e9)
    return best
for n in (1 << 20, 16 << 20, 256 << 20, 1 << 30):
    out[f"d2h_{n>>20}MiB"] = bw(n, "d2h")
    out[f"h2d_{n>>20}MiB"] = bw(n, "h2d")
# bidirectional
n = 512 << 20
h1 = torch.empty(n, dtype=torch.uint8, pin_memory=True); h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d1 = torch.empty(n, dtype=torch.uint8, device=dev); d2 = torch.empty(n, dtype=torch.uint8, device=dev)
s1 = torch.cuda.Stream(); s2 = torch.cuda.Stream()
torch.cuda.synchronize(); t = time.perf_counter()
for _ in range(3):
    with torch.cuda.stream(s1): h1.copy_(d1, non_blocking=True)
    with torch.cuda.stream(s2): d2.copy_(h2, non_blocking=True)
torch.cuda.synchronize(); dt = time.perf_counter() - t
out["bidir_total_GBs"] = 3 * 2 * n / dt / 1e9
# attention backends
q = torch.randn(1, 16, 4096, 128, device=dev, dtype=torch.bfloat16)
for name, fn in [("flash", lambda: torch.ops.aten._scaled_dot_product_flash_attention(q, q, q, 0.0, True, False, scale=None)),
                 ("cudnn", lambda: torch.ops.aten._scaled_dot_product_cudnn_attention(q, q, q, None, True, 0.0, True, False)),
                 ("efficient", lambda: torch.ops.aten._scaled_dot_product_efficient_attention(q, q, q, None, True, 0.0, True))]:
    try:
        r = fn(); torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10): r = fn()
        e1.record(); e1.synchronize()
        ms = e0.elapsed_time(e1) / 10
        fl = 4 * 16 * 4096 * 4096 * 128 / 2
        out[f"attn_{name}"] = {"ok": True, "ms": ms, "tflops_causal": fl / ms / 1e9}
    except Exception as e:
        out[f"attn_{name}"] = {"ok": False, "err": str(e)[:300]}
# GEMM
a = torch.randn(4096, 2048, device=dev, dtype=torch.bfloat16); b = torch.randn(2048, 8192, device=dev, dtype=torch.bfloat16)
for _ in range(3): c = a @ b
torch.cuda.synchronize()
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20): c = a @ b
e1.record(); e1.synchronize()
ms = e0.elapsed_time(e1) / 20
out["gemm_4096x2048x8192_tflops"] = 2 * 4096 * 2048 * 8192 / ms / 1e9
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/probe_box.json", "w"), indent=1)
print(json.dumps({k: v for k, v in out.items() if k not in ("lscpu", "topo")}, indent=1))
print(out["topo"]); print(out["lscpu"])
