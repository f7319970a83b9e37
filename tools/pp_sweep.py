"""Peak activation GB per GPU and tokens/s vs pipeline depth (BASELINE metric:
"tokens/sec and peak activation GB/GPU at PP=1/2/4/8, offload overhead vs no-offload").

A fixed model (C2: 24 layers h=2048 s=4096; C4: 40 layers h=5120 s=16384) is cut
into d = 1, 2, 4, 8 stages of L/d layers.  For each d, rank 0 of the 1F1B schedule
-- the rank with the highest 1F1B peak -- runs alone on this GPU (emulated boundary,
`execute(mode="emulate")`) with costs calibrated on this GPU, under three plans:
no offload, the reference's full-offload plan (`plan_slots(sched, {0}, t_o)`), and
the k-aware plan (`choose_offload`, <= 5% modelled overhead).  Reported per (d,
plan): rank-0 activation arena (GB, = the measured per-GPU peak of activations),
tokens/s of the pipeline (m*s / step time), overhead vs no offload, and the
runner model's per-rank peaks for all d ranks.  One JSON line per (d, plan) to
stdout and gpurun_out/pp_sweep.jsonl.

usage: python tools/pp_sweep.py --config c2|c4 [--pps 1,2,4,8] [--m 8] [--iters 1] [--warmup 1]
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

from paper_2503_01328_b200 import build_1f1b, peak_memory, plan_slots, simulate  # noqa: E402
from paper_2503_01328_b200.policy import choose_offload  # noqa: E402
from paper_2503_01328_b200.runtime.calibrate import calibrate_costs  # noqa: E402
from paper_2503_01328_b200.runtime.executor import execute  # noqa: E402
from paper_2503_01328_b200.runtime.model import ModelConfig  # noqa: E402

CONFIGS = {"c2": (24, 2048, 16, 4096), "c4": (40, 5120, 40, 16384)}


def params_gb(L: int, h: int, vocab: int, layers: int) -> float:
    """bf16 weights + fp32 master + fp32 grads of `layers` blocks (+ embeddings)."""
    return (layers * 12 * h * h + 2 * vocab * h) * 10 / 1e9


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--pps", default="1,2,4,8")
    ap.add_argument("--m", type=int, default=8)
    ap.add_argument("--iters", type=int, default=1)
    ap.add_argument("--warmup", type=int, default=1)
    ap.add_argument("--vocab", type=int, default=1024)
    ap.add_argument("--plans", default="none,full,auto")
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    torch.cuda.set_device(dev)
    L, h, heads, s = CONFIGS[a.config]
    os.makedirs("gpurun_out", exist_ok=True)
    log = open("gpurun_out/pp_sweep.jsonl", "a")

    def emit(row):
        line = json.dumps(row)
        print(line, flush=True)
        log.write(line + "\n")
        log.flush()

    hbm = torch.cuda.get_device_properties(dev).total_memory / 1e9
    for d in map(int, a.pps.split(",")):
        lps = L // d
        head = {"config": a.config, "h": h, "s": s, "L": L, "d": d, "layers_per_stage": lps, "m": a.m}
        # a stage's weights + fp32 master + grads + one slab must fit next to the arena
        if params_gb(L, h, a.vocab, lps) > 0.6 * hbm:
            emit(dict(head, skipped=f"stage weights+master+grads {params_gb(L, h, a.vocab, lps):.0f} GB "
                                    f"do not fit next to activations in {hbm:.0f} GB"))
            continue
        cfg = ModelConfig(n_layers=L, hidden=h, heads=heads, seq=s, vocab=a.vocab)
        try:
            costs, t_o, cal = calibrate_costs(cfg, d, a.m, dev, units=lps)
        except (MemoryError, torch.cuda.OutOfMemoryError) as exc:
            emit(dict(head, skipped=f"calibration: {exc!r}"[:300]))
            gc.collect()
            torch.cuda.empty_cache()
            continue
        torch.cuda.empty_cache()
        sched = build_1f1b(d, lps, a.m, costs)
        k = float(t_o / (costs.total * lps))
        head.update(k_measured=k, T_F_ms=cal["t_f"] * 1e3, T_B_ms=cal["t_b"] * 1e3, T_o_ms=float(t_o) * 1e3)
        plans = {"none": None}
        if d > 1:
            plans["full"] = plan_slots(sched, (0,), t_o)
            plans["auto"] = choose_offload(sched, (0,), t_o, tolerance=0.05, focus_rank=0).plan
        base = None
        for name in a.plans.split(","):
            if name not in plans:
                emit(dict(head, plan=name, skipped="PP=1: the F->B window is zero, nothing can be offloaded "
                                                   "(reference builders.py:252-253)"))
                continue
            plan = plans[name]
            if name != "none" and plan is None:
                emit(dict(head, plan=name, skipped="k-aware policy keeps everything resident at this k"))
                continue
            model_peaks = [u for u, _ in peak_memory(simulate(sched, plan))["per_device"]]
            try:
                res = execute(sched, plan, model=cfg, mode="emulate", rank=0, device=dev, iters=a.iters,
                              warmup=a.warmup, optimizer="sgd")
            except (MemoryError, torch.cuda.OutOfMemoryError) as exc:
                emit(dict(head, plan=name, skipped=repr(exc)[:300]))
                gc.collect()
                torch.cuda.empty_cache()
                continue
            it = statistics.median(res.iteration_seconds)
            prog = res.programs[0]
            row = dict(head, plan=name, tokens_per_s=a.m * s / it, ms_per_step=it * 1e3,
                       peak_act_slabs=prog.n_slabs, slab_gb=res.slab_bytes / 1e9,
                       peak_act_gb=prog.n_slabs * res.slab_bytes / 1e9,
                       host_pinned_gb=prog.n_host_slots * res.slab_bytes / 1e9,
                       offloaded=len(prog.offloaded), late=len(plan.late_list()) if plan is not None else 0,
                       model_peak_layers_per_rank=[u for u in model_peaks],
                       max_mem_gb=torch.cuda.max_memory_allocated(dev) / 1e9)
            if base is None:
                base = row["tokens_per_s"]
            row["overhead_pct"] = 100 * (base / row["tokens_per_s"] - 1)
            emit(row)
            res.close()
            del res
            gc.collect()
            torch.cuda.empty_cache()
            torch.cuda.reset_peak_memory_stats(dev)


if __name__ == "__main__":
    main()
