"""LayerNorm-backward launch variants and the dual LayerNorm, timed at the
bench shapes (C2 4096x2048, C3 8192x4096, C4 16384x5120).

Each variant (PPO_LN_BWD=<id>, read once per process by the library) runs in its own
subprocess; one JSON line per (variant, shape, ln_out).  Timing: CUDA-graph replay of
16 launches over 4 rotating input sets (> L2), CUDA events on the replay stream.
usage: python tools/ln_bwd_sweep.py [--variants 0,1] > profiles/r2_ln_bwd_variants.jsonl
(variant 0: next-row prefetch, the default; 1: none)
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

SHAPES = [(4096, 2048), (8192, 4096), (16384, 5120)]


def graph_us(fns, torch, launches=16):
    stream = torch.cuda.Stream()
    with torch.cuda.stream(stream):
        for f in fns:
            f()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        for i in range(launches):
            fns[i % len(fns)]()
    best = None
    with torch.cuda.stream(stream):
        g.replay()
        torch.cuda.synchronize()
        for _ in range(5):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            g.replay()
            b.record(stream)
            b.synchronize()
            t = a.elapsed_time(b) * 1e3 / launches
            best = t if best is None else min(best, t)
    return best


def worker(variant):
    import torch

    from paper_2503_01328_b200.runtime import native

    dev = torch.device("cuda:0")
    bf = dict(device=dev, dtype=torch.bfloat16)
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("hbm_gbs", 6548.0) \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6548.0
    for s, h in SHAPES:
        E = 2 * s * h
        sets = [{k: torch.randn(s, h, **bf) for k in ("x", "dy", "r")} | {k: torch.empty(s, h, **bf) for k in ("dx", "do", "ln")}
                for _ in range(4)]
        gam, bet = torch.randn(h, device=dev) * 0.1 + 1, torch.randn(h, device=dev) * 0.1
        dg, db = torch.zeros(h, device=dev), torch.zeros(h, device=dev)
        for ln_out in (False, True):
            fns = [lambda t=t: native.layernorm_bwd(t["x"], gam, t["dy"], t["r"], t["dx"], dg, db, drop_out=t["do"],
                                                     p=0.1, drop_seed=3, drop_offset=7, beta=bet if ln_out else None,
                                                     ln_out=t["ln"] if ln_out else None) for t in sets]
            us = graph_us(fns, torch)
            nbytes = (6 if ln_out else 5) * E
            print(json.dumps({"kernel": "layernorm_bwd", "variant": variant, "s": s, "h": h, "ln_out": ln_out,
                              "us": round(us, 2), "gbs": round(nbytes / us / 1e3, 1),
                              "frac": round(nbytes / us / 1e3 / peak, 3)}), flush=True)
        if variant == 0:  # variant-independent kernels once
            dual = [lambda t=t: native.layernorm_fwd2(t["x"], gam, bet, t["ln"], t["r"], gam, bet, t["dx"]) for t in sets]
            us2 = graph_us(dual, torch)
            print(json.dumps({"kernel": "layernorm_fwd2 (LN1+LN2, one launch)", "s": s, "h": h, "us": round(us2, 2),
                              "gbs": round(4 * E / us2 / 1e3, 1), "frac": round(4 * E / us2 / 1e3 / peak, 3)}),
                  flush=True)
            ln = [lambda t=t: native.layernorm_fwd(t["x"], gam, bet, t["ln"]) for t in sets]
            us1 = graph_us(ln, torch)
            print(json.dumps({"kernel": "layernorm_fwd", "s": s, "h": h, "us": round(us1, 2),
                              "gbs": round(2 * E / us1 / 1e3, 1), "frac": round(2 * E / us1 / 1e3 / peak, 3)}), flush=True)
            cp = [lambda t=t: t["ln"].copy_(t["x"]) for t in sets]
            usc = graph_us(cp, torch)
            print(json.dumps({"kernel": "torch copy (same bytes as layernorm_fwd)", "s": s, "h": h, "us": round(usc, 2),
                              "gbs": round(2 * E / usc / 1e3, 1), "frac": round(2 * E / usc / 1e3 / peak, 3)}),
                  flush=True)
        del sets


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--variants", default="0,1")
    ap.add_argument("--worker", type=int, default=None)
    a = ap.parse_args()
    if a.worker is not None:
        worker(a.worker)
        return
    for v in a.variants.split(","):
        env = dict(os.environ, PPO_LN_BWD=v)
        r = subprocess.run([sys.executable, __file__, "--worker", v], env=env, capture_output=True, text=True)
        sys.stdout.write(r.stdout)
        if r.returncode:
            sys.stderr.write(r.stderr[-3000:])


if __name__ == "__main__":
    main()
