"""Per-shape GEMM backend choice, measured on the device (``gemm="auto"``).

Each layer GEMM of a stage has two implementations: libppo_b200's tcgen05 kernels
(CUTLASS sm100 2-SM UMMA collectives, TMA, TMEM accumulators, fused GeLU / dGeLU /
fp32-accumulate epilogues) and cuBLAS (nvjet) plus, where ours fuses an epilogue,
the separate libppo_b200 GeLU kernel.  Which is faster depends on the shape: ours
wins the wide-N forward and the fused epilogues at C2 (h=2048) and loses up to ~14%
on C4's h=5120, s=16384 shapes (profiles/r1_gemm_tuning.txt, bench C4 line).  The
first time a (kind, shape) is seen outside a CUDA-graph capture, both candidates run
on fresh operands of that shape (CUDA events on the current stream; the two are
timed alternately, 4 rounds, medians, so clock and power-cap drift hits both alike)
and the faster one is cached for the process.  Our kernel is timed
at tile-scheduler swizzles 1, 2, 4 and 8 (``native.gemm_set_swizzle``: the raster band
width of the persistent CTAs, worth up to 20% on C4's h=5120 shapes through L2 reuse,
profiles/r1_gemm_swizzle.json) and keeps its best before facing cuBLAS.
"""

from __future__ import annotations

import statistics

import torch

SWIZZLES = (1, 2, 4, 8)
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


def _time_batch_us(fn, n: int) -> float:
    """Mean µs per launch of n back-to-back launches (one event pair around them)."""
    fn()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        fn()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) * 1e3 / n


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
    from . import native

    run_ours, run_cublas = make()
    # each sample spans >= ~10 ms of back-to-back launches, so it sees the clocks a
    # sustained (power-capped) step runs at, not a cold burst
    est = max(_time_us(run_ours, reps=1, warm=1), _time_us(run_cublas, reps=1, warm=1))
    n = int(min(50, max(3, 10_000 / max(est, 1.0))))
    per_sw = {}
    for _ in range(2):
        for sw in SWIZZLES:
            native.gemm_set_swizzle(kind, *shape, sw)
            t = _time_batch_us(run_ours, n)
            per_sw[sw] = min(per_sw.get(sw, t), t)
    best_sw = min(per_sw, key=per_sw.get)
    native.gemm_set_swizzle(kind, *shape, best_sw)
    # head to head, alternating so clock / power-cap drift hits both candidates alike
    t_o, t_c = [], []
    for _ in range(4):
        t_o.append(_time_batch_us(run_ours, n))
        t_c.append(_time_batch_us(run_cublas, n))
    t_ours, t_cublas = statistics.median(t_o), statistics.median(t_c)
    _CHOICE[key] = t_ours <= t_cublas
    LOG.append((key, round(t_ours, 2), round(t_cublas, 2), best_sw))
    return _CHOICE[key]


def decisions() -> dict:
    """{"kind MxNxK": {"ours_us", "cublas_us", "choice"}} for every tuned shape."""
    out = {}
    for key, to, tc, sw in LOG:
        out[f"{key[1]} {'x'.join(str(x) for x in key[2:])}"] = {
            "ours_us": to, "ours_swizzle": sw, "cublas_us": tc, "choice": "tcgen05" if to <= tc else "cublas"}
    return out


_ATTN_CHOICE: dict = {}
ATTN_LOG: list = []  # (key, ours_us, cudnn_us)


def prefer_ours_attn(shape: tuple, device, make) -> bool:
    """``attn="auto"``: True if libppo_b200's attention forward (writing o and lse into
    the slab) beats cuDNN's fused forward plus the K1 pack its separate outputs need,
    for shape = (seq, heads, head_dim).  Timed head to head like the GEMMs (alternating,
    >= ~10 ms per sample, medians); cached per process.  Must be called outside a
    stream capture (Stage construction)."""
    key = (torch.device(device).index,) + tuple(shape)
    hit = _ATTN_CHOICE.get(key)
    if hit is not None:
        return hit
    run_ours, run_cudnn = make()
    est = max(_time_us(run_ours, reps=1, warm=1), _time_us(run_cudnn, reps=1, warm=1))
    n = int(min(50, max(3, 10_000 / max(est, 1.0))))
    t_o, t_c = [], []
    for _ in range(4):
        t_o.append(_time_batch_us(run_ours, n))
        t_c.append(_time_batch_us(run_cudnn, n))
    t_ours, t_cudnn = statistics.median(t_o), statistics.median(t_c)
    _ATTN_CHOICE[key] = t_ours <= t_cudnn
    ATTN_LOG.append((key, round(t_ours, 2), round(t_cudnn, 2)))
    return _ATTN_CHOICE[key]


def attn_decisions() -> dict:
    """{"attn_fwd s x heads x head_dim": {"ours_us", "cudnn_pack_us", "choice"}}."""
    return {f"attn_fwd {'x'.join(str(x) for x in key[1:])}": {
        "ours_us": to, "cudnn_pack_us": tc, "choice": "tcgen05" if to <= tc else "cudnn"} for key, to, tc in ATTN_LOG}
