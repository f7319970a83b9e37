"""Command line: ``python -m paper_2503_01328_b200 {plan,simulate,run} ...``

Flag names follow the reference CLI (``ppoff plan|simulate``, pkg/src/ppoff/cli.py:
328-367: --schedule --d --v --m --g --offload --costs --out) so existing scripts port
over; ``run`` is the B200 addition: it calibrates pass costs and
transfer times on the GPU, plans with them (offloaded stages chosen on ``po_block``
exactly like cli.py:159-160,201-203), executes the schedule, and writes the
reference's output files from the *measured* trace:

    <kind>.schedule        emit_schedule (planned, measured costs)
    <kind>.plan            OffloadPlan.emit
    <kind>-trace.csv       SimTrace.to_csv of the measured run (seconds)
    <kind>-summary.json    SimTrace.summary() + tokens/s, arena GB, k, predicted vs
                           measured makespan (the runner model fed the measured costs)
    <kind>.svg             timeline of the measured trace (render.render_svg)

Modes: ``emulate`` (rank 0 of the schedule alone on one GPU, loopback boundary),
``virtual`` (all ranks on one GPU), and torchrun with WORLD_SIZE > 1 (one rank per
GPU, NCCL stage boundary).
"""

from __future__ import annotations

import argparse
import json
import os
import sys
from fractions import Fraction

from . import (BUILDERS, PassCosts, build_gis_g, emit_schedule, peak_memory, plan_slots, po_block,
               select_offload_stages, simulate)
from .offload import plan_slots_duplex
from .policy import choose_offload
from .render import render_svg

SCHEDULES = ("1f1b", "1f1b-i", "gis", "gis-g", "gis-h", "po")


def _offload_count(spec, v: int) -> int | str:
    """none | half | full | N | auto (reference cli.py:133-143, plus the k-aware policy)."""
    if spec in (None, "none"):
        return 0
    if spec == "half":
        return (v + 1) // 2
    if spec == "full":
        return v
    if spec in ("auto", "auto-measured"):
        return spec
    n = int(spec)
    if not 0 <= n <= v:
        raise SystemExit(f"offload count {n} outside [0, {v}]")
    return n


def _build(kind, d, v, m, g, costs):
    if kind == "gis-g":
        if g is None:
            raise SystemExit("--schedule gis-g requires --g")
        return build_gis_g(d, v, m, g, costs)
    return BUILDERS[kind](d, v, m, costs)


def _write(out: str, name: str, text: str) -> None:
    os.makedirs(out, exist_ok=True)
    tmp = os.path.join(out, name + ".tmp")
    with open(tmp, "w") as f:
        f.write(text)
    os.replace(tmp, os.path.join(out, name))


def _plan(sched, d, v, costs, t_o, offload, planner="slots", t_duplex=None):
    """planner: "slots" = the reference's one-stream slot grid (offload.py:209-220);
    "duplex" = independent D2H / H2D grids (``plan_slots_duplex``) of one-way width
    ``t_duplex`` (measured with both directions in flight; default t_o / 2)."""
    n = _offload_count(offload, v)
    if not n:
        return None
    block = po_block(d, v, costs)
    if n == "auto":
        return choose_offload(sched, select_offload_stages(block, 1), t_o).plan
    if n == "auto-measured":  # resolved by cmd_run against the device (needs runs)
        return None
    stages = select_offload_stages(block, n)
    if planner == "duplex":
        return plan_slots_duplex(sched, stages, t_duplex if t_duplex is not None else t_o / 2)
    return plan_slots(sched, stages, t_o)


def cmd_plan(args) -> int:
    """Planner only, unit or given costs (the reference's ``plan`` + ``simulate``)."""
    tf, tb, tw, *rest = (Fraction(x) for x in args.costs.split(","))
    costs = PassCosts(tf, tb, tw, rest[0] if rest else 0)
    sched = _build(args.schedule, args.d, args.v, args.m, args.g, costs)
    plan = _plan(sched, args.d, args.v, costs, Fraction(args.t_o) * costs.total, args.offload)
    trace = simulate(sched, plan)
    _write(args.out, f"{sched.kind}.svg", render_svg(trace, title=f"{sched.kind} d={args.d} v={args.v} m={args.m}"))
    summary = dict(trace.summary(), schedule=sched.kind, d=args.d, v=args.v, m=args.m,
                   offloaded_stages=list(plan.stages) if plan else [],
                   skip_list=plan.skip_list() if plan else [], late_list=plan.late_list() if plan else [])
    _write(args.out, f"{sched.kind}.schedule", emit_schedule(sched))
    if plan:
        _write(args.out, f"{sched.kind}.plan", plan.emit())
    _write(args.out, f"{sched.kind}-summary.json", json.dumps(summary, indent=2, default=str))
    print(json.dumps(summary, indent=2, default=str))
    return 0


def cmd_run(args) -> int:
    import torch

    from .runtime.calibrate import calibrate_costs
    from .runtime.executor import execute
    from .runtime.model import ModelConfig

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    mode = args.mode
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)
        mode = "nccl"
        if args.d != world:
            raise SystemExit(f"--d {args.d} must equal WORLD_SIZE {world} under torchrun")
    n_stages = args.d * (args.v if args.schedule != "1f1b" else 1)
    if args.layers % n_stages:
        raise SystemExit(f"--layers {args.layers} must divide over {n_stages} stages")
    cfg = ModelConfig(n_layers=args.layers, hidden=args.hidden, heads=args.heads, seq=args.seq, vocab=args.vocab)
    units = args.v if args.schedule == "1f1b" else 1
    split = args.schedule in ("gis", "gis-g", "gis-h", "po")
    costs, t_o, cal = calibrate_costs(cfg, n_stages, args.m, dev, units=units, split=split)
    sched = _build(args.schedule, args.d, args.v, args.m, args.g, costs)
    t_dup = Fraction(round(cal["t_duplex"] * 1e6), 1_000_000) if cal.get("t_duplex") else None
    plan = _plan(sched, args.d, args.v, costs, t_o, args.offload, args.planner, t_dup)
    closed_loop = None
    if args.offload == "auto-measured":
        if world > 1:
            raise SystemExit("--offload auto-measured runs candidates on one process (--mode emulate|virtual)")
        from .policy import choose_offload_measured

        def _iter_s(p):
            r = execute(sched, p, model=cfg, mode=mode, rank=rank, device=dev, iters=args.iters,
                        warmup=args.warmup, stream_mode=args.stream_mode, optimizer=args.optimizer,
                        iteration_graph=args.iteration_graph)
            t = max(r.iteration_seconds)
            r.close()
            return t

        t_base = _iter_s(None)
        mc = choose_offload_measured(sched, select_offload_stages(po_block(args.d, args.v, costs), 1), t_o,
                                     lambda p: _iter_s(p) / t_base - 1, stream_mode=args.stream_mode,
                                     focus_rank=rank)
        plan = mc.choice.plan if mc.choice else None
        closed_loop = {"trials": [{"stride": q, "modelled_pct": 100 * a, "measured_pct": 100 * b} for q, a, b in mc.trials],
                       "chosen_stride": mc.choice.stride if mc.choice else None}
    res = execute(sched, plan, model=cfg, mode=mode, rank=rank, device=dev, iters=args.iters, warmup=args.warmup,
                  stream_mode=args.stream_mode, optimizer=args.optimizer, iteration_graph=args.iteration_graph,
                  spare_slabs=args.spare_slabs)
    trace = res.trace
    it = max(res.iteration_seconds)
    predicted = simulate(sched, plan, stream_mode=args.stream_mode)
    summary = dict(trace.summary(), schedule=sched.kind, mode=mode, d=args.d, v=args.v, m=args.m,
                   tokens_per_s=args.m * args.seq / it, ms_per_step=it * 1e3,
                   arena_slabs={str(k): v for k, v in res.peak_slabs.items()},
                   arena_gb={str(k): v / 1e9 for k, v in res.act_bytes.items()},
                   modelled_peak_units=[u for u, _ in peak_memory(simulate(sched, plan))["per_device"]],
                   k_measured=float(t_o / (costs.total * units)), calibration=cal,
                   predicted_makespan_s=float(predicted.makespan), measured_makespan_s=float(trace.makespan),
                   model_error_pct=100 * (float(trace.makespan) / float(predicted.makespan) - 1),
                   offloaded_stages=list(plan.stages) if plan else [], losses=res.losses,
                   closed_loop=closed_loop)
    if rank == 0:
        _write(args.out, f"{sched.kind}.schedule", emit_schedule(sched))
        if plan:
            _write(args.out, f"{sched.kind}.plan", plan.emit())
        _write(args.out, f"{sched.kind}-trace.csv", trace.to_csv())
        _write(args.out, f"{sched.kind}.svg", render_svg(trace, title=f"measured {sched.kind} ({mode}) d={args.d} m={args.m}"))
        _write(args.out, f"{sched.kind}-summary.json", json.dumps(summary, indent=2, default=str))
        print(json.dumps(summary, default=str))
    res.close()
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()
    return 0


def make_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="python -m paper_2503_01328_b200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    for name in ("plan", "run"):
        p = sub.add_parser(name)
        p.add_argument("--schedule", choices=SCHEDULES, default="1f1b")
        p.add_argument("--d", type=int, default=4)
        p.add_argument("--v", type=int, default=1)
        p.add_argument("--m", type=int, default=8)
        p.add_argument("--g", type=int, default=None)
        p.add_argument("--offload", default="none",
                       help="none | half | full | N | auto | auto-measured (run: closed-loop k-aware policy)")
        p.add_argument("--out", default="out")
    plan = sub.choices["plan"]
    plan.add_argument("--costs", default="1,1,1", help="tF,tB,tW[,comm]")
    plan.add_argument("--t-o", default="1/2", help="round trip as a multiple of the stage's compute time (k)")
    plan.set_defaults(func=cmd_plan)
    run = sub.choices["run"]
    run.add_argument("--layers", type=int, default=4)
    run.add_argument("--hidden", type=int, default=256)
    run.add_argument("--heads", type=int, default=4)
    run.add_argument("--seq", type=int, default=512)
    run.add_argument("--vocab", type=int, default=1024)
    run.add_argument("--mode", choices=("emulate", "virtual"), default="virtual")
    run.add_argument("--stream-mode", choices=("single", "dual"), default="single")
    run.add_argument("--iteration-graph", action="store_true",
                     help="capture each iteration as one CUDA graph (emulate / virtual modes)")
    run.add_argument("--planner", choices=("slots", "duplex"), default="slots",
                     help="slots: reference plan_slots; duplex: plan_slots_duplex (run with --stream-mode dual)")
    run.add_argument("--optimizer", choices=("none", "sgd", "adamw"), default="sgd")
    run.add_argument("--spare-slabs", type=int, default=0, help="offload-arena slabs beyond the modelled peak")
    run.add_argument("--iters", type=int, default=2)
    run.add_argument("--warmup", type=int, default=1)
    run.set_defaults(func=cmd_run)
    return ap


def main(argv=None) -> int:
    args = make_parser().parse_args(argv)
    return args.func(args)


if __name__ == "__main__":
    sys.exit(main())
