"""A/B of programmatic dependent launch (PPO_PDL=1 vs 0) on the bench workload: C2 rank 0
(3 layers of h=2048, s=4096, 1F1B over PP=8, m=32), one CUDA graph per iteration, the
no-offload and full-offload policies; each arm in its own process, arms alternated.

    python tools/pdl_ab.py [--rounds 2] [--iters 8]
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
from fractions import Fraction

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def one(policy, iters, warmup):
    from paper_2503_01328_b200 import PassCosts, build_1f1b, plan_slots
    from paper_2503_01328_b200.runtime.executor import execute
    from paper_2503_01328_b200.runtime.model import ModelConfig

    cfg = ModelConfig(n_layers=24, hidden=2048, heads=16, seq=4096, vocab=50304)
    costs = PassCosts(Fraction(447), Fraction(1045), Fraction(0), Fraction(32))
    sched = build_1f1b(8, 3, 32, costs)
    plan = plan_slots(sched, (0,), Fraction(17750)) if policy == "full" else None
    res = execute(sched, plan, model=cfg, mode="emulate", rank=0, iters=iters, warmup=warmup,
                  iteration_graph=True, stream_mode="dual" if policy == "full" else "single")
    ms = [x * 1e3 for x in res.iteration_seconds]
    return {"policy": policy, "pdl": os.environ.get("PPO_PDL", "0"), "median_ms": round(statistics.median(ms), 3),
            "min_ms": round(min(ms), 3), "loss": res.losses[-1]}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rounds", type=int, default=2)
    ap.add_argument("--iters", type=int, default=8)
    ap.add_argument("--policies", default="none")
    ap.add_argument("--modes", default="0,1,2,3", help="PPO_PDL values: bit 0 our kernels, bit 1 CUTLASS GEMMs")
    ap.add_argument("--one", default=None, help=argparse.SUPPRESS)
    a = ap.parse_args()
    if a.one:
        print(json.dumps(one(a.one, a.iters, 3)))
        return
    for _ in range(a.rounds):
        for pol in a.policies.split(","):
            for pdl in a.modes.split(","):
                p = subprocess.run([sys.executable, __file__, "--one", pol, "--iters", str(a.iters)],
                                   env=dict(os.environ, PPO_PDL=pdl), capture_output=True, text=True)
                print(p.stdout.strip().splitlines()[-1] if p.returncode == 0 else p.stderr[-3000:], flush=True)


if __name__ == "__main__":
    main()
