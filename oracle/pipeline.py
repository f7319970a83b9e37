"""CPU reference path of one pipeline stage, timed by bench.py (test infrastructure).

``stage_sample`` runs the serial fp32 restatement (oracle.gpt.run_layers) of one
stage's forward and backward for one microbatch on the host cores -- the
bounded sample behind ``cpu_baseline`` and ``bench.py --impl reference``.  The
reference package itself is a pure-Python planner/simulator with no tensor
code and cannot travel to the GPU box, so this port of the
path's arithmetic is the CPU implementation that is timed ("kind": "port").
"""

from __future__ import annotations

import os
import time

import torch

from .gpt import GPTConfig, init_params, run_layers


def stage_sample(hidden: int, heads: int, seq: int, layers: int, threads: int | None = None,
                 reps: int = 1, seed: int = 1234) -> dict:
    threads = threads or os.cpu_count() or 1
    torch.set_num_threads(threads)
    cfg = GPTConfig(n_layers=layers, hidden=hidden, heads=heads, seq=seq, vocab=8)
    params = {k: v for k, v in init_params(cfg, seed).items() if k.startswith("l")}
    leaf = {k: v.requires_grad_(True) for k, v in params.items()}
    gen = torch.Generator().manual_seed(7)
    x = (torch.randn(seq, hidden, generator=gen) * 0.5).requires_grad_(True)
    dy = torch.randn(seq, hidden, generator=gen) * 1e-3
    times = []
    for r in range(reps):
        t0 = time.perf_counter()
        y = run_layers(cfg, leaf, x, range(layers), r, reps)
        y.backward(dy)
        times.append(time.perf_counter() - t0)
    best = min(times)
    return {"seconds_per_microbatch": best, "tokens_per_s": seq / best, "threads": threads,
            "sample": f"1 microbatch F+B of a {layers}-layer stage (h={hidden}, s={seq}), fp32 torch CPU"}
