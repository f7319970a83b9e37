"""Kernel timeline of one replayed bench iteration (C2 rank 0, emulated boundary),
from CUPTI via torch.profiler: device busy vs wall span, idle gaps between kernels on
the compute stream and what ends them, device time per kernel family.  nsys is not in
the image; this is the timeline the copy/compute overlap and launch-gap questions need.

usage: python tools/iteration_timeline.py [--schedule 1f1b|gis-h|po] [--policy none|full]
"""
import argparse
import json
import os
import statistics
import sys
from fractions import Fraction

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2503_01328_b200 as po  # noqa: E402
from paper_2503_01328_b200.runtime import executor as ex  # noqa: E402
from paper_2503_01328_b200.runtime.model import ModelConfig  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--schedule", default="gis-h", choices=("1f1b", "gis-h", "po"))
ap.add_argument("--policy", default="none", choices=("none", "full"))
ap.add_argument("--json", default=None)
a = ap.parse_args()

cfg = ModelConfig(n_layers=24, hidden=2048, heads=16, seq=4096, vocab=50304)
if a.schedule == "1f1b":
    sched = po.build_1f1b(8, 3, 32, po.measured_pass_costs(0.35e-3, 0.8e-3, 0.0, 30e-6))
    plan = po.plan_slots(sched, (0,), Fraction(18, 1000)) if a.policy == "full" else None
else:
    c1 = po.measured_pass_costs(0.39e-3, 0.53e-3, 0.35e-3, 30e-6)
    sched = (po.build_gis_h if a.schedule == "gis-h" else po.build_po)(8, 3, 32, c1)
    plan = None
res = ex.execute(sched, plan, model=cfg, mode="emulate", rank=0, iters=2, warmup=1, iteration_graph=True)
print("iteration ms", [round(1e3 * x, 2) for x in res.iteration_seconds])
res.close()

from torch.profiler import ProfilerActivity, profile  # noqa: E402

tokens = torch.randint(0, cfg.vocab, (32, cfg.seq + 1), generator=torch.Generator().manual_seed(0))
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    r2 = ex.execute(sched, plan, model=cfg, mode="emulate", rank=0, iters=1, warmup=1, iteration_graph=True,
                    tokens=tokens)
    torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type.name == "CUDA" and e.time_range.end > e.time_range.start]
# keep the last iteration: the window of the final replay = the last len(kernels-per-iteration)
evs.sort(key=lambda e: e.time_range.start)
span_end = evs[-1].time_range.end
it_s = r2.iteration_seconds[-1] * 1e6
lo = span_end - it_s * 1.02
win = [e for e in evs if e.time_range.start >= lo]
busy = 0.0
gaps = []
prev = None
for e in win:
    if prev is not None:
        g = e.time_range.start - prev.time_range.end
        if g > 0:
            gaps.append((g, prev.name[:50], e.name[:50]))
    if prev is None or e.time_range.end > prev.time_range.end:
        prev = e
    busy += e.time_range.end - e.time_range.start
fam = {}
for e in win:
    k = e.name.split("<")[0].split("(")[0][:60]
    f = fam.setdefault(k, [0, 0.0])
    f[0] += 1
    f[1] += e.time_range.end - e.time_range.start
out = {"schedule": a.schedule, "policy": a.policy, "iteration_ms": 1e-3 * it_s, "kernels": len(win),
       "kernel_time_ms": busy / 1e3, "gap_total_ms": sum(g for g, *_ in gaps) / 1e3,
       "gaps_over_5us": sum(1 for g, *_ in gaps if g > 5), "median_gap_us": statistics.median([g for g, *_ in gaps]) if gaps else 0,
       "top_gaps": [(round(g, 1), p, n) for g, p, n in sorted(gaps, reverse=True)[:15]],
       "families_ms": {k: (n, round(t / 1e3, 3)) for k, (n, t) in sorted(fam.items(), key=lambda kv: -kv[1][1])[:25]}}
print(json.dumps(out, indent=1))
if a.json:
    with open(a.json, "w") as f:
        json.dump(out, f, indent=1)
