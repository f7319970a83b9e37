"""Measured pass costs and transfer times for planning (measured-cost feedback).

``calibrate`` times one microbatch's F and B of a stage with CUDA events and one
payload's D2H / H2D (alone and full-duplex) through the engine's own transfer path,
so ``measured_pass_costs`` + ``plan_slots`` plan on this machine's numbers instead of
the FLOP model of ``estimate_pass_costs`` (reference costs.py:139-161).
"""

from __future__ import annotations

import statistics

import torch

from . import native
from .model import SlabView


def calibrate(stage, reps: int = 3, split: bool = True) -> dict:
    """T_F, T_B (and, with ``split``, split T_B / T_W) of one microbatch of the stage,
    and the D2H / H2D time of its slab alone and under full-duplex load."""
    dev = stage.device
    slab_mem = torch.empty(stage.layout.slab_bytes, dtype=torch.uint8, device=dev)
    slab = SlabView(stage.layout, slab_mem)
    cfg = stage.cfg
    tok = torch.randint(0, cfg.vocab, (cfg.seq + 1,), device=dev)
    out = torch.empty(cfg.seq, cfg.hidden, dtype=torch.bfloat16, device=dev)
    dy = (torch.randn(cfg.seq, cfg.hidden, device=dev) * 1e-3).bfloat16()
    tf, tb = [], []
    for r in range(reps + 1):
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        e[0].record()
        if stage.first:
            stage.embed(slab, tok)
        else:
            slab.get(0, "x").copy_(dy)
        stage.forward(slab, 0, 0, out=None if stage.last else out, tokens=tok)
        e[1].record()
        stage.backward(slab, 0, 0, dy=None if stage.last else dy, dx_out=None if stage.first else out, tokens=tok)
        e[2].record()
        torch.cuda.synchronize()
        if r:
            tf.append(e[0].elapsed_time(e[1]) / 1e3)
            tb.append(e[1].elapsed_time(e[2]) / 1e3)
    # split backward (GIS / PO schedules): B = activation gradients, W = weight gradients
    tbs, tws = [float("nan")], [float("nan")]
    for r in range(reps + 1 if split else 0):
        if r == 0:
            wbuf = stage.new_wbuffer()
            tbs, tws = [], []
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        stage.set_pass_context(0, 0, tok)
        e[0].record()
        stage.backward_body(slab, None if stage.last else dy, None if stage.first else out, wbuf)
        e[1].record()
        stage.wgrad_body(slab, wbuf)
        e[2].record()
        torch.cuda.synchronize()
        if r:
            tbs.append(e[0].elapsed_time(e[1]) / 1e3)
            tws.append(e[1].elapsed_time(e[2]) / 1e3)
    wbuf = None
    lay = stage.layout
    from .executor import check_host_memory

    check_host_memory(2 * (lay.host_bytes + 4096))
    pool = native.PinnedPool(lay.host_bytes + 4096)
    bins, acc = [], pool.carve(lay.host_bytes)
    for b in lay.bins:
        bins.append(acc)
        acc += b
    segs = lay.segments(slab_mem.data_ptr(), tuple(bins))
    copy = torch.cuda.Stream()
    d2h, h2d = [], []
    for r in range(reps + 1):
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        e[0].record(copy)
        native.transfer(native.PPO_D2H, segs, copy.cuda_stream)
        e[1].record(copy)
        native.transfer(native.PPO_H2D, segs, copy.cuda_stream)
        e[2].record(copy)
        torch.cuda.synchronize()
        if r:
            d2h.append(e[0].elapsed_time(e[1]) / 1e3)
            h2d.append(e[1].elapsed_time(e[2]) / 1e3)
    # one-way time while the other direction is busy too (full duplex PCIe)
    slab2 = torch.empty_like(slab_mem)
    pool2 = native.PinnedPool(lay.host_bytes + 4096)
    bins2, acc2 = [], pool2.carve(lay.host_bytes)
    for b in lay.bins:
        bins2.append(acc2)
        acc2 += b
    segs2 = lay.segments(slab2.data_ptr(), tuple(bins2))
    copy2 = torch.cuda.Stream()
    dup = []
    for r in range(reps + 1):
        ea = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        eb = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        torch.cuda.synchronize()
        ea[0].record(copy)
        eb[0].record(copy2)
        native.transfer(native.PPO_D2H, segs, copy.cuda_stream)
        native.transfer(native.PPO_H2D, segs2, copy2.cuda_stream)
        ea[1].record(copy)
        eb[1].record(copy2)
        torch.cuda.synchronize()
        if r:
            dup.append(max(ea[0].elapsed_time(ea[1]), eb[0].elapsed_time(eb[1])) / 1e3)
    # compute slowdown under concurrent copy-engine traffic, per pass kind and direction
    # (copy-engine reads of HBM cost the SMs DRAM bandwidth: profiles/r1_dma_interference.txt);
    # the runner model prices link contention only (reference sim.py:274-304), policy.DmaSlowdown
    # adds this measured term
    slow = dma_slowdown(stage, slab, tok, out, dy, segs, segs2, copy, copy2, split=split)
    pool2.close()
    pool.close()
    nbytes = sum(lay.bin_used)
    return {
        "dma_slowdown": slow,
        "t_f": min(tf), "t_b": min(tb), "t_d2h": min(d2h), "t_h2d": min(h2d), "transfer_bytes": nbytes,
        "t_b_split": min(tbs), "t_w_split": min(tws),
        "t_duplex": statistics.median(dup), "duplex_gbs_per_direction": nbytes / statistics.median(dup) / 1e9,
        "d2h_gbs": nbytes / min(d2h) / 1e9, "h2d_gbs": nbytes / min(h2d) / 1e9,
    }


def dma_slowdown(stage, slab, tok, out, dy, segs, segs2, copy, copy2, split: bool = True, reps: int = 3,
                 passes: int = 4) -> dict:
    """Fractional slowdown of F, B (and split B / W) passes while D2H, H2D or both copy
    directions stream on the copy engines: t(with copies) / t(alone) - 1.  Each sample
    runs ``passes`` passes back to back under a chain of slab transfers long enough to
    cover them (eager issue, as ``calibrate`` times F and B); medians of ``reps``."""
    wbuf = stage.new_wbuffer() if split else None
    d2h, h2d = (segs, copy, native.PPO_D2H), (segs2, copy2, native.PPO_H2D)

    def run(kind):
        stage.set_pass_context(0, 0, tok)
        if kind == "F":
            stage.forward_body(slab, None if stage.last else out)
        elif kind == "B":
            stage.backward_body(slab, None if stage.last else dy, None if stage.first else out)
        elif kind == "Bs":
            stage.backward_body(slab, None if stage.last else dy, None if stage.first else out, wbuf)
        else:
            stage.wgrad_body(slab, wbuf)

    def sample(kind, copies):
        comp = torch.cuda.current_stream()
        torch.cuda.synchronize()
        for _ in range(2 if copies else 0):
            for seg_list, stream, direction in copies:
                native.transfer(direction, seg_list, stream.cuda_stream)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(comp)
        for _ in range(passes):
            run(kind)
        b.record(comp)
        torch.cuda.synchronize()
        return a.elapsed_time(b) / 1e3 / passes

    out_ = {}
    for kind in ["F", "B"] + (["Bs", "W"] if split else []):
        run(kind)  # warm
        t = {mode: statistics.median(sample(kind, copies) for _ in range(reps))
             for mode, copies in (("none", ()), ("d2h", (d2h,)), ("h2d", (h2d,)), ("duplex", (d2h, h2d)))}
        out_[kind] = {m: t[m] / t["none"] - 1 for m in ("d2h", "h2d", "duplex")}
        out_[kind]["t_alone"] = t["none"]
    return out_


def calibrate_costs(cfg, n_stages: int, microbatches: int, device, units: int = 1, split: bool = False):
    """(PassCosts per unit, T_o of one stage payload, raw calibration) for planning.

    ``units`` is the schedule's units per stage (1F1B's merged stage of v layer
    groups has v units; its pass durations are v x the per-unit costs).  The stage
    hop t_comm is the 2bsh message over NVLink at the measured 770 GB/s plus 10 us
    of launch latency (B200_PROFILING.md NVLink reference)."""
    from fractions import Fraction

    from ..costs import measured_pass_costs
    from .model import Stage, stage_layers

    middle = min(1, n_stages - 1)
    st = Stage(cfg, middle, n_stages, microbatches, device, layers=stage_layers(cfg, n_stages, middle))
    cal = calibrate(st, split=split)
    del st
    torch.cuda.empty_cache()
    hop = (2 * cfg.seq * cfg.hidden) / 770e9 + 10e-6
    if split:
        costs = measured_pass_costs(cal["t_f"] / units, cal["t_b_split"] / units, cal["t_w_split"] / units, hop)
    else:
        costs = measured_pass_costs(cal["t_f"] / units, cal["t_b"] / units, 0.0, hop)
    t_o = Fraction(round((cal["t_d2h"] + cal["t_h2d"]) * 1e6), 1_000_000)
    return costs, t_o, {k: v for k, v in cal.items()}
