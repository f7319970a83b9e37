"""Per-shape GEMM / attention backend choice: a decision table, tuned once, never per pass.

Each layer GEMM of a stage has two implementations: libppo_b200's tcgen05 kernels
(CUTLASS sm100 2-SM UMMA collectives, TMA, TMEM accumulators, fused GeLU / dGeLU /
fp32-accumulate epilogues) and cuBLAS (nvjet) plus, where ours fuses an epilogue,
the separate libppo_b200 GeLU kernel.  Which is faster depends on the shape
(profiles/r1_gemm_tuning.txt).  The attention forward has libppo_b200's tcgen05
kernel (o and lse straight into the slab) and cuDNN's fused kernel + K1 pack; the
attention backward has libppo_b200's K7b (dqkv [s, 3h] directly) and cuDNN's fused
backward + the K1 gather into dqkv.

Numerics follow the backend, so the choice must be the same in every process that
is compared or pipelined together.  The contract:

* ``TABLE`` maps a shape key to a decision.  It is filled by ``ensure(cfg, device)``
  -- every layer shape of the model config, timed on a private stream outside any
  capture and before the first iteration (no copies in flight) -- or loaded from a
  JSON file (``load``; ``PPO_TUNE_TABLE`` names one that is loaded on first use).
* Under ``torch.distributed`` with world > 1, ``ensure`` is collective: rank 0 tunes
  and broadcasts its table; no other rank times anything.  ``execute`` and
  ``calibrate`` call it on every rank before constructing stages.
* Pass bodies only *look up* (``gemm_choice`` / ``attn_choice``).  A shape missing
  from the table gets the static rule of ``gemm="best"`` (deterministic) and is
  recorded in ``MISSES``.

Our kernel is timed at tile-scheduler swizzles 1, 2, 4 and 8 (``native.gemm_set_swizzle``:
the raster band width of the persistent CTAs, worth up to 20% on C4's h=5120 shapes
through L2 reuse, profiles/r1_gemm_swizzle.json) and keeps its best before facing
cuBLAS head to head (alternating, >= ~10 ms per sample, medians).
"""

from __future__ import annotations

import hashlib
import json
import os
import statistics

import torch

SWIZZLES = (1, 2, 4, 8)
TABLE: dict = {}  # key -> {"backend": "tcgen05"|"cublas"|"cudnn", "swizzle", "ours_us", "lib_us"}
MISSES: set = set()
_LOADED_ENV = False


# --------------------------------------------------------------------- keys


def gemm_key(kind: str, shape) -> str:
    return f"{kind} {'x'.join(str(int(x)) for x in shape)}"


def attn_key(seq: int, heads: int, head_dim: int) -> str:
    return f"attn_fwd {seq}x{heads}x{head_dim}"


def attn_bwd_key(seq: int, heads: int, head_dim: int) -> str:
    return f"attn_bwd {seq}x{heads}x{head_dim}"


def layer_gemm_shapes(seq: int, hidden: int) -> list[tuple]:
    """Every (kind, M, N, K) a transformer layer's F/B/W passes issue (model.Stage):
    forward QKV / proj / fc1+GeLU / fc2; backward dgrads (unsplit and split) and weight
    gradients (wgrad shape = (out, in, tokens))."""
    s, h = seq, hidden
    return [
        ("tn", s, 3 * h, h), ("tn", s, h, h), ("tn_gelu", s, 4 * h, h), ("tn", s, h, 4 * h),
        ("nn", s, 4 * h, h), ("nn_dgelu", s, 4 * h, h), ("nn", s, h, 4 * h), ("nn", s, h, h),
        ("nn_acc", s, h, h), ("nn", s, h, 3 * h),
        ("wgrad", h, 4 * h, s), ("wgrad", 4 * h, h, s), ("wgrad", h, h, s), ("wgrad", 3 * h, h, s),
    ]


def static_rule(kind: str, shape) -> bool:
    """``gemm="best"``: ours except narrow-N / deep-K plain GEMMs (N <= 2048, K >= 3N),
    where cuBLAS nvjet measured ~7% faster (profiles/r1_gemm_tuning.txt)."""
    if kind in ("tn", "nn", "nn_acc"):
        _, n, k = shape
        return not (n <= 2048 and k >= 3 * n)
    return True


# ------------------------------------------------------------------- lookups


def _env_table():
    global _LOADED_ENV
    if not _LOADED_ENV:
        _LOADED_ENV = True
        path = os.environ.get("PPO_TUNE_TABLE")
        if path and os.path.exists(path):
            load(path)


def gemm_choice(kind: str, shape) -> bool:
    """True if libppo_b200's kernel runs (kind, shape) under ``gemm="auto"``."""
    _env_table()
    d = TABLE.get(gemm_key(kind, shape))
    if d is None:
        MISSES.add(gemm_key(kind, shape))
        return static_rule(kind, shape)
    return d["backend"] == "tcgen05"


def attn_choice(seq: int, heads: int, head_dim: int) -> bool:
    """True if libppo_b200's attention forward runs this shape under ``attn="auto"``."""
    _env_table()
    d = TABLE.get(attn_key(seq, heads, head_dim))
    if d is None:
        MISSES.add(attn_key(seq, heads, head_dim))
        return False
    return d["backend"] == "tcgen05"


def attn_bwd_choice(seq: int, heads: int, head_dim: int) -> bool:
    """True if libppo_b200's attention backward (K7b) runs this shape under ``attn="auto"``."""
    _env_table()
    d = TABLE.get(attn_bwd_key(seq, heads, head_dim))
    if d is None:
        MISSES.add(attn_bwd_key(seq, heads, head_dim))
        return False
    return d["backend"] == "tcgen05"


# -------------------------------------------------------------------- timing


def _time_us(fn, stream, reps: int = 1, warm: int = 1) -> float:
    for _ in range(warm):
        fn()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        fn()
        b.record(stream)
        b.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    return statistics.median(ts)


def _time_batch_us(fn, n: int, stream) -> float:
    """Mean µs per launch of n back-to-back launches (one event pair around them)."""
    fn()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(n):
        fn()
    b.record(stream)
    b.synchronize()
    return a.elapsed_time(b) * 1e3 / n


def _rand(device, *shape, dtype=torch.bfloat16):
    return (torch.randn(*shape, device=device, dtype=torch.float32) * 0.1).to(dtype)


def gemm_candidates(kind: str, shape, device):
    """(run_ours, run_library) closures over fresh operands of (kind, shape); the
    library side includes the separate GeLU kernel where ours fuses it."""
    from . import native

    M, N, K = shape
    bf = dict(device=device, dtype=torch.bfloat16)
    if kind == "tn":
        a, w, o = _rand(device, M, K), _rand(device, N, K), torch.empty(M, N, **bf)
        return (lambda: native.gemm_tn(a, w, o)), (lambda: torch.mm(a, w.t(), out=o))
    if kind == "tn_gelu":
        a, w = _rand(device, M, K), _rand(device, N, K)
        f, g = torch.empty(M, N, **bf), torch.empty(M, N, **bf)
        zb = torch.zeros(N, device=device, dtype=torch.float32)
        return ((lambda: native.gemm_tn_gelu(a, w, g, f, zb)),
                (lambda: (torch.mm(a, w.t(), out=f), native.gelu_fwd(f, g))))
    if kind in ("nn", "nn_acc"):
        d, w, o = _rand(device, M, K), _rand(device, K, N), torch.zeros(M, N, **bf)
        if kind == "nn_acc":
            return (lambda: native.gemm_nn(d, w, o, 1.0)), (lambda: torch.addmm(o, d, w, out=o))
        return (lambda: native.gemm_nn(d, w, o, 0.0)), (lambda: torch.mm(d, w, out=o))
    if kind == "nn_dgelu":
        d, w, f = _rand(device, M, K), _rand(device, K, N), _rand(device, M, N)
        o = torch.empty(M, N, **bf)
        return ((lambda: native.gemm_nn_dgelu(d, w, f, o)),
                (lambda: (torch.mm(d, w, out=o), native.gelu_bwd(f, o, None, o))))
    if kind == "wgrad":  # acc [M=out, N=in] fp32 += dy[K, M]^T @ x[K, N]
        dy, x = _rand(device, K, M), _rand(device, K, N)
        acc = torch.zeros(M, N, device=device, dtype=torch.float32)
        return ((lambda: native.gemm_wgrad(dy, x, acc, 1.0)),
                (lambda: torch.addmm(acc, dy.t(), x, out_dtype=torch.float32, out=acc)))
    raise KeyError(kind)


def attn_candidates(seq: int, heads: int, head_dim: int, device):
    """(run_ours, run_cudnn_plus_pack) over fresh qkv of one layer."""
    from . import native

    h = heads * head_dim
    qkv = _rand(device, seq, 3 * h)
    o = torch.empty(seq, h, device=device, dtype=torch.bfloat16)
    lse = torch.empty(heads * seq, device=device, dtype=torch.float32)
    dst = torch.empty(2 * seq * h + 4 * heads * seq, device=device, dtype=torch.uint8)
    qv = qkv.view(1, seq, 3, heads, head_dim)
    q, k, v = (qv[:, :, i].transpose(1, 2) for i in range(3))

    def cudnn():
        r = torch.ops.aten._scaled_dot_product_cudnn_attention(q, k, v, None, True, 0.0, True, False)
        native.pack([(r[0], 0, 1, 2 * seq * h, 0), (r[1], 2 * seq * h, 1, 4 * heads * seq, 0)], dst)

    return (lambda: native.attn_fwd(qkv, o, lse, heads)), cudnn


def attn_bwd_candidates(seq: int, heads: int, head_dim: int, device):
    """(run_ours, run_cudnn_plus_gather): the backward of one layer's attention into the
    packed dqkv [s, 3h] both ways (cuDNN's three gradients gathered by one K1 launch, as
    the split backward does), from the same saved o / lse."""
    from . import native

    h = heads * head_dim
    qkv, do = _rand(device, seq, 3 * h), _rand(device, seq, h)
    qv = qkv.view(1, seq, 3, heads, head_dim)
    q, k, v = (qv[:, :, i].transpose(1, 2) for i in range(3))
    r = torch.ops.aten._scaled_dot_product_cudnn_attention(q, k, v, None, True, 0.0, True, False)
    o4, lse4 = r[0], r[1]
    o = o4.transpose(1, 2).reshape(seq, h).contiguous()
    lse = lse4.reshape(heads, seq).contiguous()
    do4 = do.view(1, seq, heads, head_dim).transpose(1, 2)
    dqkv = torch.empty_like(qkv)
    ws = torch.empty(native.attn_bwd_workspace_bytes(seq, heads, head_dim), device=device, dtype=torch.uint8)

    def cudnn():
        g = torch.ops.aten._scaled_dot_product_cudnn_attention_backward(
            do4, q, k, v, o4, lse4, r[6], r[7], None, r[2], r[3], r[4], r[5], 0.0, True)
        parts = [t.transpose(1, 2) for t in g]
        native.pack([(p_, 2 * h * j, seq, 2 * h, 2 * h, 6 * h) for j, p_ in enumerate(parts)], dqkv)

    return (lambda: native.attn_bwd(qkv, o, do, lse, dqkv, heads, ws)), cudnn


def _duel(ours, lib, stream) -> tuple[float, float]:
    est = max(_time_us(ours, stream), _time_us(lib, stream))
    n = int(min(50, max(3, 10_000 / max(est, 1.0))))
    t_o, t_l = [], []
    for _ in range(4):
        t_o.append(_time_batch_us(ours, n, stream))
        t_l.append(_time_batch_us(lib, n, stream))
    return statistics.median(t_o), statistics.median(t_l)


def tune_gemm(kind: str, shape, device, stream) -> dict:
    from . import native

    ours, lib = gemm_candidates(kind, shape, device)
    est = max(_time_us(ours, stream), _time_us(lib, stream))
    n = int(min(50, max(3, 10_000 / max(est, 1.0))))
    per_sw = {}
    for _ in range(2):
        for sw in SWIZZLES:
            native.gemm_set_swizzle(kind, *shape, sw)
            t = _time_batch_us(ours, n, stream)
            per_sw[sw] = min(per_sw.get(sw, t), t)
    best_sw = min(per_sw, key=per_sw.get)
    native.gemm_set_swizzle(kind, *shape, best_sw)
    t_ours, t_lib = _duel(ours, lib, stream)
    return {"backend": "tcgen05" if t_ours <= t_lib else "cublas", "swizzle": best_sw,
            "ours_us": round(t_ours, 2), "lib_us": round(t_lib, 2)}


def tune_attn(seq, heads, head_dim, device, stream, backward: bool = False) -> dict:
    ours, lib = (attn_bwd_candidates if backward else attn_candidates)(seq, heads, head_dim, device)
    t_ours, t_lib = _duel(ours, lib, stream)
    return {"backend": "tcgen05" if t_ours <= t_lib else "cudnn", "ours_us": round(t_ours, 2),
            "lib_us": round(t_lib, 2)}


# --------------------------------------------------------------- the table


def needed_keys(cfg, gemm: str = "auto", attn: str = "auto") -> list[tuple[str, tuple]]:
    """(key, spec) of every decision a stage of ``cfg`` looks up under these modes."""
    out = []
    if gemm == "auto":
        out += [(gemm_key(k, sh), ("gemm", k, sh)) for (k, *sh) in layer_gemm_shapes(cfg.seq, cfg.hidden)]
    if attn == "auto" and cfg.head_dim in (64, 128) and cfg.seq % 256 == 0:
        out.append((attn_key(cfg.seq, cfg.heads, cfg.head_dim), ("attn", cfg.seq, cfg.heads, cfg.head_dim)))
    if attn == "auto" and cfg.head_dim in (64, 128) and cfg.seq % 128 == 0:
        out.append((attn_bwd_key(cfg.seq, cfg.heads, cfg.head_dim), ("attn_bwd", cfg.seq, cfg.heads, cfg.head_dim)))
    return out


def install(entries: dict) -> None:
    """Merge decisions into TABLE and push the chosen swizzles into the library."""
    from . import native

    for key, d in entries.items():
        TABLE[key] = dict(d)
        kind, shape = key.split(" ", 1)
        if not kind.startswith("attn") and d.get("swizzle"):
            M, N, K = (int(x) for x in shape.split("x"))
            native.gemm_set_swizzle(kind, M, N, K, int(d["swizzle"]))


def _dist_world():
    try:
        import torch.distributed as dist

        if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
            return dist
    except Exception:
        pass
    return None


def ensure(cfg, device, gemm: str = "auto", attn: str = "auto") -> dict:
    """Make every decision a stage of ``cfg`` needs present in TABLE.

    Single process: tune the missing ones here.  Under torch.distributed (world > 1)
    this is a collective every rank must call with the same config: rank 0 tunes
    what it lacks and broadcasts its decisions for these keys; every rank installs
    them, so all ranks run identical kernels.  Returns the decisions for ``cfg``."""
    _env_table()
    keys = needed_keys(cfg, gemm, attn)
    dist = _dist_world()
    if dist is None or dist.get_rank() == 0:
        missing = [(k, spec) for k, spec in keys if k not in TABLE]
        if missing:
            if torch.cuda.is_current_stream_capturing():
                raise RuntimeError("gemm_tune.ensure inside a stream capture")
            dev = torch.device(device)
            stream = torch.cuda.Stream(dev)
            stream.wait_stream(torch.cuda.current_stream(dev))
            with torch.cuda.device(dev), torch.cuda.stream(stream):
                for k, spec in missing:
                    TABLE[k] = (tune_gemm(spec[1], spec[2], dev, stream) if spec[0] == "gemm"
                                else tune_attn(*spec[1:], dev, stream, backward=spec[0] == "attn_bwd"))
            stream.synchronize()
            torch.cuda.empty_cache()
    mine = {k: TABLE[k] for k, _ in keys if k in TABLE}
    if dist is not None:
        box = [mine]
        dist.broadcast_object_list(box, src=0)
        mine = box[0]
    install(mine)
    return mine


def decisions() -> dict:
    """Every decision in TABLE (GEMMs and attention), JSON-ready."""
    return {k: dict(v) for k, v in sorted(TABLE.items())}


def digest() -> str:
    """Short hash of the backend choices (not the timings): equal on ranks that run
    identical kernels."""
    body = json.dumps({k: [v["backend"], v.get("swizzle")] for k, v in sorted(TABLE.items())}, sort_keys=True)
    return hashlib.sha256(body.encode()).hexdigest()[:16]


def save(path: str) -> None:
    with open(path, "w") as f:
        json.dump(decisions(), f, indent=1, sort_keys=True)


def load(path: str) -> None:
    with open(path) as f:
        install(json.load(f))


def reset() -> None:
    TABLE.clear()
    MISSES.clear()


def require(cfg, device, gemm: str = "auto", attn: str = "auto") -> None:
    """Stage construction: single process -> ``ensure`` (tune what is missing here);
    under torch.distributed the table must already hold every key (``ensure`` was
    called collectively), otherwise ranks could tune different kernels."""
    _env_table()
    if _dist_world() is None:
        ensure(cfg, device, gemm, attn)
        return
    missing = [k for k, _ in needed_keys(cfg, gemm, attn) if k not in TABLE]
    if missing:
        raise RuntimeError(f"backend decisions missing under torch.distributed: {missing[:3]}...; call "
                           "gemm_tune.ensure(cfg, device) on every rank first")
