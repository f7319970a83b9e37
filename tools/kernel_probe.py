"""Recompute/pack kernels at a transformer shape, timed exactly as bench.py does
(graph replay of 16 launches over rotating inputs larger than L2, CUDA events on the
replay stream).  PPO_LN_VPL=2|4|8 overrides the forward kernels' vectors per lane
(A/B runs; the TMA-staged LayerNorm variant this tool once compared was removed).

usage: python tools/kernel_probe.py [--s 4096 --h 2048 --heads 16]"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2503_01328_b200.runtime import native  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--s", type=int, default=4096)
ap.add_argument("--h", type=int, default=2048)
ap.add_argument("--heads", type=int, default=16)
a = ap.parse_args()
dev = torch.device("cuda:0")
torch.cuda.set_device(dev)
peak, kind, _ = bench.measured_peaks()
res = bench.measure_kernels(a.s, a.h, a.heads, dev, torch, native)
out = {k: {"us": round(v["avg_us"], 2), "GBps": round(v["bytes_per_launch"] / v["avg_us"] / 1e3, 1),
           "frac": round(v["bytes_per_launch"] / v["avg_us"] / 1e3 / peak, 3)} for k, v in res.items()}
print(json.dumps({"ln_vpl": os.environ.get("PPO_LN_VPL", "default"), "s": a.s, "h": a.h, "peak_gbs": peak,
                  "peak_source": kind, "kernels": out}))
