"""Per-kernel HBM roofline check of libppo_b200 at a transformer shape (default C2:
s=4096, h=2048).  Each launch is timed alone with CUDA events after an L2 flush
(a 256 MB write), median of N reps; GB/s = algorithmic bytes / time."""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2503_01328_b200.runtime import native  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--s", type=int, default=4096)
ap.add_argument("--h", type=int, default=2048)
ap.add_argument("--heads", type=int, default=16)
ap.add_argument("--reps", type=int, default=20)
a = ap.parse_args()
s, h = a.s, a.h
dev = torch.device("cuda:0")
bf = dict(device=dev, dtype=torch.bfloat16)
x, y, z, w, u = (torch.randn(s, h, **bf) for _ in range(5))
f4, g4 = torch.randn(s, 4 * h, **bf), torch.randn(s, 4 * h, **bf)
gam, bet = torch.ones(h, device=dev), torch.zeros(h, device=dev)
dg, db = torch.zeros(h, device=dev), torch.zeros(h, device=dev)
slab = torch.empty(64 << 20, dtype=torch.uint8, device=dev)
lse = torch.randn(a.heads, s, device=dev)
flush = torch.ones(64 << 20, dtype=torch.int32, device=dev)  # 256 MB, read (clean) between reps
peak = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6650.0
E = 2 * s * h  # bytes of one [s, h] bf16 tensor

cases = {
    "layernorm_fwd": (lambda: native.layernorm_fwd(x, gam, bet, y), 2 * E),
    "residual_dropout_ln_fwd": (lambda: native.residual_dropout_ln_fwd(x, y, z, gam, bet, w, 0.1, 42, 1), 4 * E),
    "residual_dropout_fwd(no ln)": (lambda: native.residual_dropout_ln_fwd(x, y, z, None, None, None, 0.1, 42, 1), 3 * E),
    "layernorm_bwd(resid+drop)": (lambda: native.layernorm_bwd(x, gam, y, z, w, dg, db, drop_out=u, p=0.1, drop_seed=4, drop_offset=5), 5 * E),
    "layernorm_bwd(plain)": (lambda: native.layernorm_bwd(x, gam, y, None, w, dg, db), 3 * E),
    "gelu_fwd": (lambda: native.gelu_fwd(f4, g4), 2 * 4 * E),
    "gelu_bwd": (lambda: native.gelu_bwd(f4, g4, f4.new_empty(f4.shape), g4), 4 * 4 * E),
    "dropout": (lambda: native.dropout(x, y, 0.1, 42, 3), 2 * E),
    "pack(o+lse)": (lambda: native.pack([(x, 0, 1, E, 0), (lse, E, 1, 4 * a.heads * s, 0)], slab), 2 * (E + 4 * a.heads * s)),
}
res = {}
for name, (fn, nbytes) in cases.items():
    fn()
    ts = []
    for _ in range(a.reps):
        flush.sum()
        torch.cuda._sleep(200_000)  # keep the GPU busy while the host enqueues: time the kernel, not the launch
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    us = statistics.median(ts)
    res[name] = {"us": round(us, 2), "GBps": round(nbytes / us / 1e3, 1), "frac": round(nbytes / us / 1e3 / peak, 3)}
    print(f"{name:32s} {us:8.2f} us  {nbytes / us / 1e3:8.1f} GB/s  {nbytes / us / 1e3 / peak:6.1%} of {peak:.0f}")
os.makedirs("gpurun_out", exist_ok=True)
json.dump({"shape": {"s": s, "h": h}, "peak_gbs": peak, "kernels": res}, open(f"gpurun_out/kbench_s{s}_h{h}.json", "w"), indent=1)
