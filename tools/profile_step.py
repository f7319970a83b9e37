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
a = ap.parse_args()
cfg = ModelConfig(n_layers=24, hidden=2048, heads=16, seq=4096, vocab=50304)
costs = PassCosts(Fraction(447), Fraction(1045), Fraction(0), Fraction(32))  # measured per layer (us)
sched = build_1f1b(8, 3, 32, costs)
plan = plan_slots(sched, (0,), Fraction(17750)) if a.policy == "full" else None
res = execute(sched, plan, model=cfg, mode="emulate", rank=0, iters=a.iters, warmup=a.warmup)
print("iteration ms", [round(x * 1e3, 2) for x in res.iteration_seconds])
