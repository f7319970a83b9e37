"""Issue-path comparison on the C2 rank-0 program (emulated boundary): per-pass CUDA
graphs issued from the host vs one graph per iteration, with and without per-pass
timestamps inside it.  Prints ms/step per (schedule, plan, issue path)."""
import json
import statistics
import sys
import os
from fractions import Fraction

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2503_01328_b200 as po  # noqa: E402
from paper_2503_01328_b200.offload import plan_slots_duplex, select_offload_stages  # noqa: E402
from paper_2503_01328_b200.runtime.calibrate import calibrate_costs  # noqa: E402
from paper_2503_01328_b200.runtime.executor import execute  # noqa: E402
from paper_2503_01328_b200.runtime.model import ModelConfig  # noqa: E402

dev = torch.device("cuda:0")
torch.cuda.set_device(dev)
cfg = ModelConfig(n_layers=24, hidden=2048, heads=16, seq=4096, vocab=50304)
out = {}
for kind, v in (("1f1b", 1), ("gis-h", 3)):
    split = kind == "gis-h"
    n_stages = 8 * v
    units = 3 if kind == "1f1b" else 1
    costs, t_o, cal = calibrate_costs(cfg, n_stages, 32, dev, units=units, split=split)
    sched = po.build_1f1b(8, 3, 32, costs) if kind == "1f1b" else po.build_gis_h(8, 3, 32, costs)
    plans = {"none": None}
    if kind == "gis-h":
        st = select_offload_stages(po.po_block(8, 3, costs), 1)
        plans["n1_duplex"] = plan_slots_duplex(sched, st, Fraction(round(cal["t_duplex"] * 1e6), 10**6))
    for pname, plan in plans.items():
        sm = "dual" if plan is not None else "single"
        for path, kw in (("per_pass", {}), ("graph_timed", {"iteration_graph": True}),
                         ("graph_untimed", {"iteration_graph": True, "pass_timing": False})):
            res = execute(sched, plan, model=cfg, mode="emulate", rank=0, device=dev, iters=3, warmup=2,
                          stream_mode=sm, optimizer="sgd", **kw)
            ms = 1e3 * statistics.median(res.iteration_seconds)
            out[f"{kind}/{pname}/{path}"] = round(ms, 2)
            print(kind, pname, path, round(ms, 2), "ms", flush=True)
            res.close()
            del res
            torch.cuda.empty_cache()
print(json.dumps(out))
