"""Per-shape GEMM backend choice, measured on the device (``gemm="auto"``).

Each layer GEMM of a stage has two implementations: libppo_b200's tcgen05 kernels
(CUTLASS sm100 2-SM UMMA collectives, TMA, TMEM accumulators, fused GeLU / dGeLU /
fp32-accumulate epilogues) and cuBLAS (nvjet) plus, where ours fuses an epilogue,
the separate libppo_b200 GeLU kernel.  Which is faster depends on the shape: ours
wins the wide-N forward and the fused epilogues at C2 (h=2048) and loses up to ~14%
on C4's h=5120, s=16384 shapes (profiles/r1_gemm_tuning.txt, bench C4 line).  The
first time a (kind, shape) is seen outside a CUDA-graph capture, both candidates run
on fresh operands of that shape (CUDA events on the current stream, median of 5
after 2 warm-ups) and the faster one is cached for the process.
"""

from __future__ import annotations

import statistics

import torch

_CHOICE: dict = {}
LOG: list = []  # (key, ours_us, cublas_us) of every decision, for reports


def _time_us(fn, reps: int = 5, warm: int = 2) -> float:
    for _ in range(warm):
        fn()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    return statistics.median(ts)


def prefer_ours(kind: str, shape: tuple, device, make, fallback: bool) -> bool:
    """True if libppo_b200's kernel is the faster one for (kind, shape).

    ``make()`` returns (run_ours, run_cublas) closures over fresh operands; it is
    only called on a cache miss.  Inside a stream capture (no synchronisation
    allowed) an unseen shape gets ``fallback``."""
    key = (torch.device(device).index, kind) + tuple(shape)
    hit = _CHOICE.get(key)
    if hit is not None:
        return hit
    if torch.cuda.is_current_stream_capturing():
        return fallback
    run_ours, run_cublas = make()
    t_ours, t_cublas = _time_us(run_ours), _time_us(run_cublas)
    _CHOICE[key] = t_ours <= t_cublas
    LOG.append((key, round(t_ours, 2), round(t_cublas, 2)))
    return _CHOICE[key]


def decisions() -> dict:
    """{"kind MxNxK": {"ours_us", "cublas_us", "choice"}} for every tuned shape."""
    out = {}
    for key, to, tc in LOG:
        out[f"{key[1]} {'x'.join(str(x) for x in key[2:])}"] = {
            "ours_us": to, "cublas_us": tc, "choice": "tcgen05" if to <= tc else "cublas"}
    return out
