"""C5: PP=8 sweep over (h, s) -- measured k = T_o / T_c vs offload overhead.

For each shape: a 1-layer stage (24->8 layers over PP=8 is C5's L=8), rank 0 of the
1F1B PP=8 schedule run alone (emulated boundary), m microbatches.  Calibrates T_F,
T_B and T_o on the GPU, builds the schedule from the measured costs, and measures
no offload, the reference's full-offload plan and the k-aware plan.  One JSON line
per shape to stdout and gpurun_out/k_sweep.jsonl.

usage: python tools/k_sweep.py [--hs 2048,4096,8192] [--ss 2048,4096,8192,16384,32768] [--m 16]
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
from paper_2503_01328_b200 import build_1f1b, measured_pass_costs, plan_slots  # noqa: E402
from paper_2503_01328_b200.policy import choose_offload, choose_offload_measured, choose_partial_offload  # noqa: E402
from paper_2503_01328_b200.runtime.layout import make_layout, offload_candidates  # noqa: E402
from paper_2503_01328_b200.runtime import native  # noqa: E402
from paper_2503_01328_b200.runtime.executor import execute  # noqa: E402
from paper_2503_01328_b200.runtime.model import ModelConfig, Stage  # noqa: E402


def run_point(h, s, m, d, iters, warmup, dev, args_measured=False):
    heads = h // 128
    cfg = ModelConfig(n_layers=d, hidden=h, heads=heads, seq=s, vocab=1024)
    st = Stage(cfg, 1, d, m, dev, layers=[0])  # a middle stage: no embedding / head
    cal = calibrate(st, split=False)
    del st
    torch.cuda.empty_cache()
    costs = measured_pass_costs(cal["t_f"], cal["t_b"], 0.0, (2 * s * h) / 770e9 + 10e-6)
    t_o = Fraction(round((cal["t_d2h"] + cal["t_h2d"]) * 1e6), 1_000_000)
    k = float(t_o / costs.total)
    sched = build_1f1b(d, 1, m, costs)
    out = {"h": h, "s": s, "m": m, "k_measured": k, "T_F_ms": cal["t_f"] * 1e3, "T_B_ms": cal["t_b"] * 1e3,
           "T_o_ms": float(t_o) * 1e3, "d2h_gbs": cal["d2h_gbs"], "h2d_gbs": cal["h2d_gbs"]}
    choice = choose_offload(sched, (0,), t_o, tolerance=0.05, focus_rank=0)
    order = offload_candidates(1)
    cands = []
    for j in range(1, len(order)):
        lay = make_layout(1, s, h, heads, offload=order[:j])
        cands.append(("+".join(f"{n}{l}" for l, n in order[:j]), tuple(order[:j]), lay.off_bytes, lay.res_bytes))
    part = choose_partial_offload(sched, (0,), t_o, cands, rank=0, tolerance=0.05, max_stride=2)
    plans = {"none": (None, "single", None), "full": (plan_slots(sched, (0,), t_o), "single", None),
             "auto": (choice.plan, "single", None)}
    if part:
        plans["partial"] = (part[0].plan, part[0].stream_mode, part[0].tensors)
        out["partial_tensors"] = part[0].label
    for name, (plan, sm, tensors) in plans.items():
        if plan is None and name != "none":
            out[name] = dict(out["none"], note="nothing offloadable within tolerance")
            continue
        res = execute(sched, plan, model=cfg, mode="emulate", rank=0, device=dev, iters=iters, warmup=warmup,
                      optimizer="sgd", stream_mode=sm, offload_tensors=tensors, iteration_graph=True)
        it = statistics.median(res.iteration_seconds)
        prog = res.programs[0]
        out[name] = {"tokens_per_s": m * s / it, "ms_per_step": it * 1e3, "peak_slabs": prog.n_slabs,
                     "peak_act_gb": res.act_bytes[0] / 1e9, "offloaded": len(prog.offloaded),
                     "late": len(plan.late_list()) if plan is not None else 0}
        res.close()
        del res
        gc.collect()
        torch.cuda.empty_cache()
    base = out["none"]["tokens_per_s"]
    for name in [n for n in ("full", "auto", "partial") if n in out]:
        out[name]["overhead_pct"] = 100 * (base / out[name]["tokens_per_s"] - 1)
    out["auto_stride"] = choice.stride
    if args_measured:
        # closed loop: stride plans least memory first, each measured, first within 5% kept
        runs = {}

        def measure(plan):
            res = execute(sched, plan, model=cfg, mode="emulate", rank=0, device=dev, iters=iters, warmup=warmup,
                          optimizer="sgd", stream_mode="single", iteration_graph=True)
            it = statistics.median(res.iteration_seconds)
            runs[id(plan)] = {"tokens_per_s": m * s / it, "ms_per_step": it * 1e3, "peak_slabs": res.programs[0].n_slabs,
                              "peak_act_gb": res.act_bytes[0] / 1e9}
            res.close()
            gc.collect()
            torch.cuda.empty_cache()
            return base / (m * s / it) - 1

        mc = choose_offload_measured(sched, (0,), t_o, measure, tolerance=0.05, focus_rank=0)
        out["auto_measured"] = dict(runs[id(mc.choice.plan)], overhead_pct=100 * mc.measured_overhead,
                                    stride=mc.choice.stride) if mc.choice else dict(out["none"], note="nothing within 5% measured")
        out["auto_measured"]["trials"] = [{"stride": q, "modelled_pct": 100 * a, "measured_pct": 100 * b}
                                          for q, a, b in mc.trials]
    from paper_2503_01328_b200.runtime import gemm_tune

    out["attn_backend"] = gemm_tune.attn_decisions()
    out["gemm_backend"] = gemm_tune.decisions()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--hs", default="2048,4096,8192")
    ap.add_argument("--ss", default="2048,4096,8192,16384,32768")
    ap.add_argument("--m", type=int, default=16)
    ap.add_argument("--d", type=int, default=8)
    ap.add_argument("--iters", type=int, default=2)
    ap.add_argument("--warmup", type=int, default=1)
    ap.add_argument("--measured", action="store_true", help="also run the closed-loop policy (choose_offload_measured)")
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    torch.cuda.set_device(dev)
    os.makedirs("gpurun_out", exist_ok=True)
    with open("gpurun_out/k_sweep.jsonl", "a") as f:
        for h in map(int, a.hs.split(",")):
            for s in map(int, a.ss.split(",")):
                try:
                    r = run_point(h, s, a.m, a.d, a.iters, a.warmup, dev, a.measured)
                except Exception as exc:  # keep sweeping; record the failure
                    r = {"h": h, "s": s, "error": repr(exc)[:300]}
                    torch.cuda.empty_cache()
                line = json.dumps(r)
                print(line, flush=True)
                f.write(line + "\n")
                f.flush()


if __name__ == "__main__":
    main()
