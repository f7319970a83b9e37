"""C3: GPT 7B shape (h=4096, s=8192, 32 heads, 32 layers), interleaved 1F1B PP=8 with
selective offload -- rank 0 of the schedule on one B200 (emulated boundary).

Builds ``build_interleaved_1f1b(8, v, m, measured costs)`` and measures no offload,
the reference's selective plans (``select_offload_stages(po_block(8, v), n)`` for
n = 1..v) and the k-aware plan, each on one copy stream and on two.
One JSON line per policy to stdout and gpurun_out/c3_interleaved.jsonl.
"""
import argparse
import gc
import json
import os
import statistics
import sys
from fractions import Fraction

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2503_01328_b200.runtime.calibrate import calibrate  # noqa: E402
from paper_2503_01328_b200 import (BUILDERS, build_interleaved_1f1b, measured_pass_costs, plan_slots,  # noqa: E402
                                   po_block, select_offload_stages, simulate, peak_memory)
from paper_2503_01328_b200.policy import choose_offload  # noqa: E402
from paper_2503_01328_b200.runtime import native  # noqa: E402
from paper_2503_01328_b200.runtime.executor import execute  # noqa: E402
from paper_2503_01328_b200.runtime.model import ModelConfig, Stage  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--h", type=int, default=4096)
    ap.add_argument("--s", type=int, default=8192)
    ap.add_argument("--layers", type=int, default=32)
    ap.add_argument("--d", type=int, default=8)
    ap.add_argument("--v", type=int, default=4)
    ap.add_argument("--m", type=int, default=32)
    ap.add_argument("--iters", type=int, default=2)
    ap.add_argument("--warmup", type=int, default=1)
    ap.add_argument("--schedule", default="1f1b-i", choices=["1f1b-i", "gis-h", "po"],
                    help="interleaved 1F1B, or the split-backward GIS-H / PO (the paper's PipeOffload schedule)")
    ap.add_argument("--ns", default=None, help="offloaded local-stage counts to measure, e.g. 1,2 (default 1..v)")
    a = ap.parse_args()
    split = a.schedule != "1f1b-i"
    dev = torch.device("cuda:0")
    torch.cuda.set_device(dev)
    per_chunk = a.layers // (a.d * a.v)
    cfg = ModelConfig(n_layers=a.layers, hidden=a.h, heads=a.h // 128, seq=a.s, vocab=1024)
    st = Stage(cfg, 1, a.d * a.v, a.m, dev, layers=list(range(per_chunk)))
    cal = calibrate(st, split=split)
    del st
    torch.cuda.empty_cache()
    hop = (2 * a.s * a.h) / 770e9 + 10e-6
    costs = (measured_pass_costs(cal["t_f"], cal["t_b_split"], cal["t_w_split"], hop) if split
             else measured_pass_costs(cal["t_f"], cal["t_b"], 0.0, hop))
    t_o = Fraction(round((cal["t_d2h"] + cal["t_h2d"]) * 1e6), 1_000_000)
    sched = build_interleaved_1f1b(a.d, a.v, a.m, costs) if not split else BUILDERS[a.schedule](a.d, a.v, a.m, costs)
    head = {"schedule": sched.kind, "h": a.h, "s": a.s, "d": a.d, "v": a.v, "m": a.m, "layers_per_chunk": per_chunk,
            "k_measured": float(t_o / costs.total), "T_F_ms": cal["t_f"] * 1e3, "T_B_ms": cal["t_b"] * 1e3,
            "T_o_ms": float(t_o) * 1e3}
    block = po_block(a.d, a.v, sched.costs)
    plans = {"none": None}
    for n in (map(int, a.ns.split(",")) if a.ns else range(1, a.v + 1)):
        plans[f"selective_n{n}"] = plan_slots(sched, select_offload_stages(block, n), t_o)
    choice = choose_offload(sched, select_offload_stages(block, 1), t_o, tolerance=0.05, focus_rank=0)
    if choice.plan is not None:
        plans["auto_n1"] = choice.plan
    os.makedirs("gpurun_out", exist_ok=True)
    base = None
    with open("gpurun_out/c3_interleaved.jsonl", "a") as f:
        for name, plan in plans.items():
            for mode in (("single",) if plan is None else ("single", "dual")):
                model_peak = [u for u, _ in peak_memory(simulate(sched, plan, stream_mode=mode))["per_device"]]
                res = execute(sched, plan, model=cfg, mode="emulate", rank=0, device=dev, iters=a.iters,
                              warmup=a.warmup, optimizer="sgd", stream_mode=mode)
                it = statistics.median(res.iteration_seconds)
                prog = res.programs[0]
                row = dict(head, policy=name, stream_mode=mode, tokens_per_s=a.m * a.s / it, ms_per_step=it * 1e3,
                           peak_slabs=prog.n_slabs, peak_act_gb=prog.n_slabs * res.slab_bytes / 1e9,
                           offloaded=len(prog.offloaded), late=len(plan.late_list()) if plan is not None else 0,
                           model_rank0_peak=model_peak[0], stages=list(plan.stages) if plan is not None else [])
                if base is None:
                    base = row["tokens_per_s"]
                row["overhead_pct"] = 100 * (base / row["tokens_per_s"] - 1)
                res.close()
                del res
                gc.collect()
                torch.cuda.empty_cache()
                line = json.dumps(row)
                print(line, flush=True)
                f.write(line + "\n")


if __name__ == "__main__":
    main()
