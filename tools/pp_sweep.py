"""Peak activation GB per GPU and tokens/s vs pipeline depth (BASELINE metric:
"tokens/sec and peak activation GB/GPU at PP=1/2/4/8, offload overhead vs no-offload").

A fixed model (C2: 24 layers h=2048 s=4096; C4: 40 layers h=5120 s=16384) is cut
into d = 1, 2, 4, 8 stages of L/d layers.  For each d, rank 0 of the 1F1B schedule
-- the rank with the highest 1F1B peak -- runs alone on this GPU (emulated boundary,
`execute(mode="emulate")`) with costs calibrated on this GPU, under three plans:
no offload, the reference's full-offload plan (`plan_slots(sched, {0}, t_o)`), and
the k-aware plans (`choose_offload` stride search and `choose_partial_offload`
per-tensor partial offload, <= 5% modelled overhead), and the paper's GIS-H schedule
at v = L/d (1-layer chunks) without offload and with the reference's selective n=1
on duplex copy streams.  Reported per (d,
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

from paper_2503_01328_b200 import (build_1f1b, build_gis_h, peak_memory, plan_slots, po_block,  # noqa: E402
                                   select_offload_stages, simulate)
from paper_2503_01328_b200.offload import plan_slots_duplex  # noqa: E402
from paper_2503_01328_b200.policy import choose_offload, choose_partial_offload  # noqa: E402
from paper_2503_01328_b200.runtime.layout import make_layout, offload_candidates  # noqa: E402
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
    ap.add_argument("--plans", default="none,full,auto,partial,gis-h,gis-h_n1")
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
        plans = {"none": (sched, None, "single", None)}
        if d > 1:
            plans["full"] = (sched, plan_slots(sched, (0,), t_o), "single", None)
            auto = choose_offload(sched, (0,), t_o, tolerance=0.05, focus_rank=0).plan
            if auto is not None:
                plans["auto"] = (sched, auto, "single", None)
            order = offload_candidates(lps)
            cands = []
            for j in range(1, min(len(order), 4 * lps)):
                lay = make_layout(lps, s, h, heads, offload=order[:j])
                cands.append(("+".join(f"{n}{l}" for l, n in order[:j]), tuple(order[:j]), lay.off_bytes,
                              lay.res_bytes))
            best = choose_partial_offload(sched, (0,), t_o, cands, rank=0, tolerance=0.05, max_stride=2)
            if best:
                plans["partial"] = (sched, best[0].plan, best[0].stream_mode, best[0].tensors)
            if lps > 1 and "gis-h" in a.plans:
                c1, t1, cal1 = calibrate_costs(cfg, d * lps, a.m, dev, units=1, split=True)
                torch.cuda.empty_cache()
                sv = build_gis_h(d, lps, a.m, c1)
                w1 = Fraction(round(cal1["t_duplex"] * 1e6), 1_000_000)
                st = select_offload_stages(po_block(d, lps, c1), 1)
                plans["gis-h"] = (sv, None, "single", None)
                plans["gis-h_n1"] = (sv, plan_slots_duplex(sv, st, w1), "dual", None)
        base = None
        for name in a.plans.split(","):
            if name not in plans:
                why = ("PP=1: the F->B window is zero, nothing can be offloaded (reference builders.py:252-253)"
                       if d == 1 else "no plan within 5% at this k" if name in ("auto", "partial") else "n/a")
                emit(dict(head, plan=name, skipped=why))
                continue
            sv, plan, sm, tensors = plans[name]
            model_peaks = [u for u, _ in peak_memory(simulate(sv, plan))["per_device"]]
            try:
                res = execute(sv, plan, model=cfg, mode="emulate", rank=0, device=dev, iters=a.iters,
                              warmup=a.warmup, optimizer="sgd", stream_mode=sm, offload_tensors=tensors,
                              iteration_graph=True)
            except (MemoryError, torch.cuda.OutOfMemoryError) as exc:
                emit(dict(head, plan=name, skipped=repr(exc)[:300]))
                gc.collect()
                torch.cuda.empty_cache()
                continue
            it = statistics.median(res.iteration_seconds)
            prog = res.programs[0]
            row = dict(head, plan=name, schedule=sv.kind, stream_mode=sm, tensors=tensors and len(tensors),
                       tokens_per_s=a.m * s / it, ms_per_step=it * 1e3,
                       peak_act_gb=res.mem["alloc_peak_bytes"] / 1e9,  # measured: peak minus training state
                       device_act_gb=res.mem["device_bytes"] / 1e9, arena_gb=res.act_bytes[0] / 1e9,
                       wbuf_gb=res.mem["wbuf_bytes"] / 1e9, slab_gb=res.slab_bytes / 1e9,
                       offload_fraction=round(res.offload_fraction, 4),
                       host_pinned_gb=prog.n_host_slots * res.slab_bytes * res.offload_fraction / 1e9,
                       offloaded=len(prog.offloaded), late=len(plan.late_list()) if plan is not None else 0,
                       model_peak_units_per_rank=[u for u in model_peaks],
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
