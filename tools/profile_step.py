"""One iteration of the bench workload (C2 rank 0, full offload) for ncu captures.

Usage (under gpurun): ncu ... python tools/profile_step.py [--policy full|none] [--iters 1]
"""
import argparse
import os
import sys
from fractions import Fraction

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2503_01328_b200 import PassCosts, build_1f1b, plan_slots  # noqa: E402
from paper_2503_01328_b200.runtime.executor import execute  # noqa: E402
from paper_2503_01328_b200.runtime.model import ModelConfig  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--policy", default="full")
ap.add_argument("--iters", type=int, default=1)
ap.add_argument("--warmup", type=int, default=0)
ap.add_argument("--schedule", default="1f1b", choices=("1f1b", "gis-h", "po"))
# fixed backends: the measured per-shape choice ("auto") is meaningless under a profiler
ap.add_argument("--gemm", default="best", choices=("auto", "best", "tcgen05", "cublas"))
ap.add_argument("--attn", default="cudnn", choices=("auto", "tcgen05", "cudnn"))
a = ap.parse_args()
cfg = ModelConfig(n_layers=24, hidden=2048, heads=16, seq=4096, vocab=50304)
costs = PassCosts(Fraction(447), Fraction(1045), Fraction(0), Fraction(32))  # measured per layer (us)
if a.schedule == "1f1b":
    sched = build_1f1b(8, 3, 32, costs)
else:  # split backward at v = 3 (1-layer chunks), as in the bench
    from paper_2503_01328_b200 import build_gis_h, build_po, measured_pass_costs

    c1 = measured_pass_costs(0.42e-3, 0.6e-3, 0.4e-3, 30e-6)
    sched = (build_gis_h if a.schedule == "gis-h" else build_po)(8, 3, 32, c1)
plan = plan_slots(sched, (0,), Fraction(17750)) if a.policy == "full" and a.schedule == "1f1b" else None
res = execute(sched, plan, model=cfg, mode="emulate", rank=0, iters=a.iters, warmup=a.warmup, gemm=a.gemm, attn=a.attn)
print("iteration ms", [round(x * 1e3, 2) for x in res.iteration_seconds])
if a.iters > 1 or a.warmup:
    import statistics

    tr = res.trace
    comp = sorted((p for p in tr.passes if p.kind.value in ("F", "B", "W")), key=lambda p: p.start)
    for kind in ("F", "B"):
        ds = [float(p.duration) * 1e3 for p in comp if p.kind.value == kind]
        print(kind, "n", len(ds), "median ms", round(statistics.median(ds), 4), "sum ms", round(sum(ds), 2))
    gaps = [float(b.start - (a_.start + a_.duration)) * 1e3 for a_, b in zip(comp, comp[1:])]
    print("gaps between passes: sum ms", round(sum(gaps), 2), "max", round(max(gaps), 3))
    print("first pass start ms", round(float(comp[0].start) * 1e3, 3), "last end ms",
          round(float(comp[-1].start + comp[-1].duration) * 1e3, 3))
