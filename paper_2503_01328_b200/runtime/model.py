"""One pipeline stage of the GPT model, with its saved set laid out in a slab.

Forward writes the 20bsh saved set of every layer straight into the
(stage, microbatch) slab (``layout.SlabLayout``): the QKV and fc1 GEMMs write
their outputs into slab views, the fused residual+dropout+LayerNorm kernel
writes h1 and the next layer's x, and the tcgen05 attention kernel writes the
attention output and its softmax statistics (the cuDNN baseline needs a K1 pack).  Backward reads the (possibly reloaded) slab, recomputes
LayerNorm, GeLU and both dropout masks (K3-K5, ``libppo_b200.so``) and never
needs anything that was not saved -- the recompute scheme of PAPER.md:439 that
turns the reference's 34bsh coefficient into 20bsh (costs.py:1-7,18-20).

Dense GEMMs run on libppo_b200's tcgen05 kernels or cuBLAS, per shape whichever the
decision table says (``gemm="auto"``, the default: tuned once before the first pass and
identical on every rank, runtime/gemm_tune.py);
``gemm="best"`` is the static round-1 rule (ours except narrow-N / deep-K shapes,
profiles/r1_gemm_tuning.txt).  fc1 fuses the GeLU into its epilogue (writes f into the slab and g for fc2), the
fc2 activation-gradient GEMM fuses the GeLU backward (df = (dm @ Wfc2) * gelu'(f)),
weight gradients accumulate in fp32 inside the GEMM epilogue.  ``gemm="cublas"``
keeps the library GEMMs as the comparison baseline.  Causal attention forward runs
on libppo_b200's tcgen05 kernel or cuDNN's fused kernel, per shape whichever the
device measured faster with cuDNN's output pack included (``attn="auto"``), its
backward on cuDNN's fused kernel; the embedding and loss head (first/last stage only) use
torch ops.
"""

from __future__ import annotations

import zlib
from dataclasses import dataclass

import torch

from . import native
from . import gemm_tune
from .layout import SlabLayout, make_layout


@dataclass(frozen=True)
class ModelConfig:
    n_layers: int = 4
    hidden: int = 256
    heads: int = 4
    seq: int = 512
    vocab: int = 1024
    p_drop: float = 0.1
    dropout_seed: int = 42
    eps: float = 1e-5

    @property
    def head_dim(self) -> int:
        return self.hidden // self.heads


def dropout_offset(cfg: ModelConfig, iteration: int, layer: int, mb: int, microbatches: int, branch: int) -> int:
    """Philox offset of one dropout site (branch 0: attention residual, 1: MLP residual)."""
    return (((iteration * cfg.n_layers + layer) * microbatches + mb) * 2) + branch


def init_params(cfg: ModelConfig, seed: int = 1234, names=None) -> dict[str, torch.Tensor]:
    """Deterministic N(0, 0.02) init on the CPU generator (bf16-representable values).

    Every matrix has its own generator seeded from (seed, crc32(name)), so each
    rank draws exactly the tensors it owns and all ranks agree without talking.
    """
    h, v, s = cfg.hidden, cfg.vocab, cfg.seq
    shapes = {"wte": (v, h), "wpe": (s, h)}
    for l in range(cfg.n_layers):
        shapes.update({
            f"l{l}.ln1_g": (h,), f"l{l}.ln1_b": (h,), f"l{l}.w_qkv": (3 * h, h), f"l{l}.w_proj": (h, h),
            f"l{l}.ln2_g": (h,), f"l{l}.ln2_b": (h,), f"l{l}.w_fc1": (4 * h, h), f"l{l}.w_fc2": (h, 4 * h),
        })
    shapes.update({"lnf_g": (h,), "lnf_b": (h,), "w_head": (v, h)})
    out = {}
    for name, shape in shapes.items():
        if names is not None and name not in names:
            continue
        if name.endswith("_g"):
            val = torch.ones(shape)
        elif name.endswith("_b"):
            val = torch.zeros(shape)
        else:
            gen = torch.Generator().manual_seed(seed * 1_000_003 + zlib.crc32(name.encode()))
            std = 0.02 / (2 * cfg.n_layers) ** 0.5 if name.endswith(("w_proj", "w_fc2")) else 0.02
            val = (torch.randn(shape, generator=gen) * std).bfloat16().float()
        out[name] = val
    return out


def stage_layers(cfg: ModelConfig, num_stages: int, stage: int) -> list[int]:
    """Global layer ids of a stage: contiguous, as even as possible."""
    base, extra = divmod(cfg.n_layers, num_stages)
    lo = stage * base + min(stage, extra)
    return list(range(lo, lo + base + (1 if stage < extra else 0)))


def _wgrad(acc: torch.Tensor, a_t: torch.Tensor, b: torch.Tensor) -> None:
    """acc(fp32) += a_t @ b with bf16 operands and fp32 accumulation in cuBLAS."""
    torch.addmm(acc, a_t, b, out_dtype=torch.float32, out=acc)


class SlabView:
    """Typed tensor views of one slab (device memory owned by the arena).

    ``base`` holds the offload part (the bytes that travel, layout.off_bytes); the
    resident part lives at ``res_base`` -- a separate arena slot under partial
    offload, or simply the rest of ``base`` when the slab is one contiguous buffer."""

    def __init__(self, layout: SlabLayout, base: torch.Tensor, res_base: torch.Tensor | None = None):
        self.layout = layout
        if res_base is None:  # one contiguous buffer of layout.slab_bytes
            res_base = base[layout.off_bytes: layout.slab_bytes]
            base = base[: layout.off_bytes]
        self.base = base  # uint8 tensor of layout.off_bytes
        self.res_base = res_base  # uint8 tensor of layout.res_bytes
        self._cache = {}

    def locate(self, layer: int, name: str) -> tuple[torch.Tensor, int]:
        """(part base tensor, byte offset inside it) of one saved tensor."""
        slot = self.layout.find(layer, name)
        if self.layout.travels(slot):
            return self.base, slot.dev_offset
        return self.res_base, slot.dev_offset - self.layout.off_bytes

    def get(self, layer: int, name: str) -> torch.Tensor:
        key = (layer, name)
        t = self._cache.get(key)
        if t is None:
            slot = self.layout.find(layer, name)
            part, off = self.locate(layer, name)
            raw = part[off: off + slot.nbytes]
            t = raw.view(torch.bfloat16 if slot.dtype == "bf16" else torch.float32).view(slot.shape)
            self._cache[key] = t
        return t


class Stage:
    """Parameters, gradients, workspace and the F/B passes of one pipeline stage."""

    def __init__(self, cfg: ModelConfig, stage: int, num_stages: int, microbatches: int, device, params=None,
                 layers: list[int] | None = None, seed: int = 1234, gemm: str = "auto", offload=None,
                 attn: str = "auto", workspace: dict | None = None):
        native.require_cuda()
        if gemm not in ("auto", "best", "tcgen05", "cublas"):
            raise ValueError(f"gemm backend {gemm!r}")
        if attn not in ("auto", "tcgen05", "cudnn"):
            raise ValueError(f"attention backend {attn!r}")
        # attention: "tcgen05" = libppo_b200's kernels -- the forward writing o and lse straight
        # into the slab (head_dim 64/128, seq % 256 == 0) and the backward (K7b) writing
        # dqkv [s, 3h] for one dgrad and one wgrad GEMM; "cudnn" = cuDNN's fused kernels + K1
        # pack / gather (the library baseline); "auto" = per direction, whichever measured
        # faster at this shape (gemm_tune decision table, looked up in _attn_init).  Both
        # backward kernels consume the same saved o and natural-log lse.
        self.attn_supported = cfg.head_dim in (64, 128) and cfg.seq % 256 == 0
        self.attn_bwd_supported = cfg.head_dim in (64, 128) and cfg.seq % 128 == 0
        if attn == "tcgen05" and not self.attn_supported:
            raise ValueError(f"tcgen05 attention needs head_dim 64/128 and seq % 256 == 0 (got {cfg.head_dim}, {cfg.seq})")
        self.attn_mode = attn
        self.attn_ours = attn == "tcgen05"
        self.attn_bwd_ours = attn == "tcgen05"
        # "tcgen05": every GEMM on libppo_b200's kernels (fused GeLU epilogues); "cublas": the
        # library baseline; "best": ours except narrow-N / deep-K shapes (N <= 2048, K >= 3N)
        # where cuBLAS nvjet measured ~7% faster (profiles/r1_gemm_tuning.txt).
        self.gemm = gemm
        self.cfg, self.stage, self.num_stages, self.m = cfg, stage, num_stages, microbatches
        self.first, self.last = stage == 0, stage == num_stages - 1
        self.layers = layers if layers is not None else stage_layers(cfg, num_stages, stage)
        self.device = torch.device(device)
        # offload: None = the whole saved set travels; else the (local layer, name)
        # tensors that do (partial offload, layout.make_layout)
        self.layout = make_layout(len(self.layers), cfg.seq, cfg.hidden, cfg.heads, head_grad=self.last,
                                  offload=offload)
        names = set()
        for l in self.layers:
            names |= {f"l{l}.{k}" for k in ("ln1_g", "ln1_b", "w_qkv", "w_proj", "ln2_g", "ln2_b", "w_fc1", "w_fc2")}
        if self.first:
            names |= {"wte", "wpe"}
        if self.last:
            names |= {"lnf_g", "lnf_b", "w_head"}
        src = params if params is not None else init_params(cfg, seed, names)
        self.w, self.g, self.master = {}, {}, {}
        for n in sorted(names):
            t = src[n].to(self.device, torch.float32)
            self.master[n] = t.clone()
            is_matrix = t.dim() == 2
            self.w[n] = t.to(torch.bfloat16) if is_matrix else t.contiguous()
            self.g[n] = torch.zeros_like(t, dtype=torch.float32)
        # persistent training state (bf16 weights, fp32 gradients, fp32 masters): what the
        # paper's "iteration-start memory" holds; everything else a run allocates is
        # activation memory (executor.RunResult.mem)
        self.state_bytes = sum(t.numel() * t.element_size() for d in (self.w, self.g, self.master) for t in d.values())
        s, h = cfg.seq, cfg.hidden
        bf = dict(device=self.device, dtype=torch.bfloat16)
        # recompute / GEMM workspace (18 s*h bf16): read and written only inside one pass, so
        # the stages of one rank share a single copy (``workspace=``; passes of a rank run
        # one at a time on its compute stream)
        self.ws = workspace if workspace is not None else self.new_workspace(cfg, self.device)
        self.zero_bias = torch.zeros(4 * h, device=self.device, dtype=torch.float32)
        self.loss_sum = torch.zeros((), device=self.device, dtype=torch.float32)
        # Per-pass context in device memory, so a captured pass (CUDA graph) serves every
        # microbatch: ctx[0] = Philox offset base of (iteration, mb); tok = token row.
        self.ctx = torch.zeros(1, device=self.device, dtype=torch.int64)
        # (iteration) part of ctx, device-resident so a captured whole-iteration graph
        # replays with the current iteration's Philox offsets (set_iteration, outside it)
        self.iter_base = torch.zeros(1, device=self.device, dtype=torch.int64)
        self.tok = torch.zeros(cfg.seq + 1, device=self.device, dtype=torch.int64)
        self._attn_meta = None
        if gemm == "auto" or attn == "auto":  # decisions tuned once, before any pass (gemm_tune)
            gemm_tune.require(cfg, self.device, gemm, attn)
        self._attn_init()
        self.probe = None  # kernel name -> [bytes_per_launch, [(start_event, end_event), ...]]

    @staticmethod
    def new_workspace(cfg: ModelConfig, device) -> dict:
        s, h = cfg.seq, cfg.hidden
        bf = dict(device=device, dtype=torch.bfloat16)
        return {
            "ln": torch.empty(s, h, **bf), "ln1": torch.empty(s, h, **bf), "a": torch.empty(s, h, **bf),
            "g": torch.empty(s, 4 * h, **bf),
            "big": torch.empty(s, 4 * h, **bf), "dm": torch.empty(s, h, **bf), "dh1": torch.empty(s, h, **bf),
            "da": torch.empty(s, h, **bf), "t": torch.empty(s, h, **bf), "dy": torch.empty(s, h, **bf),
            "dqkv": torch.empty(s, 3 * h, **bf),
        }

    def _attn_init(self):
        """One eager attention call on scratch buffers before any capture: records the
        cuDNN backward's metadata and statistics shape, and (tcgen05 path) lets the
        library create its per-seq device constants outside a stream capture."""
        cfg, ws = self.cfg, self.ws
        s, h = cfg.seq, cfg.hidden
        qkv = ws["big"].view(-1)[: s * 3 * h].view(s, 3 * h).zero_()
        q, k, v = self._qkv_views(qkv)
        res = torch.ops.aten._scaled_dot_product_cudnn_attention(q, k, v, None, True, 0.0, True, False)
        self._attn_meta = tuple(res[2:8])
        self._o_strides = res[0].stride()
        self._lse_shape = tuple(res[1].shape)
        if self.attn_mode != "cudnn" and self.attn_supported:
            lse = torch.empty(cfg.heads * s, device=self.device, dtype=torch.float32)
            native.attn_fwd(qkv, ws["a"], lse, cfg.heads)  # creates the library's per-seq constants
            if self.attn_mode == "auto":
                self.attn_ours = gemm_tune.attn_choice(s, cfg.heads, cfg.head_dim)
        if self.attn_mode == "auto" and self.attn_bwd_supported:
            self.attn_bwd_ours = gemm_tune.attn_bwd_choice(s, cfg.heads, cfg.head_dim)
        if self.attn_bwd_ours and "attn" not in ws:  # fp32 dq accumulator + row statistics
            ws["attn"] = torch.empty(native.attn_bwd_workspace_bytes(s, cfg.heads, cfg.head_dim), device=self.device,
                                     dtype=torch.uint8)
        del res

    def _k(self, name: str, nbytes: int, fn, *args, **kw):
        """Launch one native kernel; with probing on, bracket it with CUDA events."""
        if self.probe is None:
            return fn(*args, **kw)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn(*args, **kw)
        b.record()
        self.probe.setdefault(name, [nbytes, []])[1].append((a, b))

    # ------------------------------------------------------------------ utils
    def p(self, l: int, k: str) -> torch.Tensor:
        return self.w[f"l{l}.{k}"]

    def gp(self, l: int, k: str) -> torch.Tensor:
        return self.g[f"l{l}.{k}"]

    # ------------------------------------------------------------------ GEMMs
    def _tuned(self, kind: str, shape: tuple) -> bool:
        """True if libppo_b200's kernel runs (kind, shape): the decision table under
        gemm="auto" (tuned before the first pass, identical on every rank,
        runtime/gemm_tune.py), the static rule under "best", else the pinned backend."""
        if self.gemm == "auto":
            return gemm_tune.gemm_choice(kind, shape)
        if self.gemm == "best":
            return gemm_tune.static_rule(kind, shape)
        return self.gemm == "tcgen05"

    def mm_fwd(self, a, w, out):
        """out = a @ w^T (nn.Linear forward; w is [out, in])."""
        M, (N, K) = a.shape[0], w.shape
        if self._tuned("tn", (M, N, K)):
            native.gemm_tn(a, w, out)
        else:
            torch.mm(a, w.t(), out=out)

    def mm_fc1_gelu(self, a, w, f_out, g_out):
        """f = a @ w^T (saved GeLU input) and g = gelu(f) (fc2 operand)."""
        M, (N, K) = a.shape[0], w.shape
        if self._tuned("tn_gelu", (M, N, K)):
            native.gemm_tn_gelu(a, w, g_out, f_out, self.zero_bias[: w.shape[0]])
        else:
            torch.mm(a, w.t(), out=f_out)
            self._k("gelu_fwd", 4 * f_out.numel(), native.gelu_fwd, f_out, g_out)

    def mm_dgrad(self, dy, w, out, accumulate: bool = False):
        """out (+)= dy @ w (activation gradient of nn.Linear)."""
        M, (K, N) = dy.shape[0], w.shape
        if self._tuned("nn_acc" if accumulate else "nn", (M, N, K)):
            native.gemm_nn(dy, w, out, 1.0 if accumulate else 0.0)
        elif accumulate:
            torch.addmm(out, dy, w, out=out)
        else:
            torch.mm(dy, w, out=out)

    def mm_dgrad_dgelu(self, dm, w, f, df_out, g_out):
        """df = (dm @ w) * gelu'(f), plus g = gelu(f) for the fc2 weight gradient.

        When g is needed (unsplit backward) the plain dgrad GEMM + one gelu_bwd pass
        (reads f and dg once, writes df and g) is cheaper; when it is not (split
        backward: the W pass recomputes g) the GeLU backward rides in the GEMM
        epilogue (``gemm_nn_dgelu``) unless the table says GEMM + gelu_bwd is faster."""
        M, (K, N) = dm.shape[0], w.shape
        if g_out is None and self.gemm != "cublas" and self._tuned("nn_dgelu", (M, N, K)):
            native.gemm_nn_dgelu(dm, w, f, df_out)
            return
        self.mm_dgrad(dm, w, df_out)
        self._k("gelu_bwd", 8 * f.numel(), native.gelu_bwd, f, df_out, g_out, df_out)

    def wgrad(self, acc, dy, x):
        """acc (fp32, [out, in]) += dy^T @ x with dy [tokens, out], x [tokens, in]."""
        T, (O, I) = dy.shape[0], acc.shape
        if self._tuned("wgrad", (O, I, T)):
            native.gemm_wgrad(dy, x, acc, 1.0)
        else:
            _wgrad(acc, dy.t(), x)

    def _gather_dqkv(self, dq, dk, dv, out):
        """Concatenate the attention input gradients into out [s, 3h] (one K1 launch)."""
        s, h = self.cfg.seq, self.cfg.hidden
        parts = [t.transpose(1, 2) for t in (dq, dk, dv)]
        if all(p_.is_contiguous() for p_ in parts):
            native.pack([(p_, 2 * h * j, s, 2 * h, 2 * h, 6 * h) for j, p_ in enumerate(parts)], out)
        else:  # pragma: no cover - cuDNN layout other than [b, s, heads, d]
            for j, p_ in enumerate(parts):
                out[:, j * h:(j + 1) * h].copy_(p_.reshape(s, h))

    def _qkv_views(self, qkv: torch.Tensor):
        cfg = self.cfg
        v = qkv.view(1, cfg.seq, 3, cfg.heads, cfg.head_dim)
        return [v[:, :, i].transpose(1, 2) for i in range(3)]

    def _offsets(self, l_global: int):
        """Per-layer constant parts of the Philox offsets (attention branch, MLP branch);
        the (iteration, mb) part is ``self.ctx[0]`` (see dropout_offset)."""
        base = l_global * self.m * 2
        return base, base + 1

    def set_iteration(self, iteration: int):
        """Stream-ordered: the iteration part of every pass context (never captured)."""
        self.iter_base.fill_(iteration * self.cfg.n_layers * self.m * 2)

    def set_pass_context(self, mb: int, iteration: int | None = None, tokens: torch.Tensor | None = None):
        """Stream-ordered update of the per-pass device context: ctx = iter_base + 2 mb.
        Graph-safe (mb is static per pass; the iteration comes from ``iter_base``);
        passing ``iteration`` also sets ``iter_base`` (eager single-pass use)."""
        if iteration is not None:
            self.set_iteration(iteration)
        torch.add(self.iter_base, mb * 2, out=self.ctx)
        if tokens is not None:
            self.tok.copy_(tokens, non_blocking=True)

    def zero_grad(self):
        for t in self.g.values():
            t.zero_()
        self.loss_sum.zero_()

    # ---------------------------------------------------------------- forward
    def embed(self, slab: SlabView, tokens: torch.Tensor | None = None):
        """x0 = wte[tokens[:-1]] + wpe written into layer 0's x slot (first stage).
        ``tokens``: the microbatch's [s+1] token row (None: use the pass context)."""
        if tokens is not None:
            self.tok.copy_(tokens, non_blocking=True)
        native.embed_fwd(self.tok[:-1], self.w["wte"], self.w["wpe"], slab.get(0, "x"))

    def forward(self, slab: SlabView, mb: int, iteration: int, out: torch.Tensor | None = None,
                tokens: torch.Tensor | None = None):
        self.set_pass_context(mb, iteration, tokens)
        self.forward_body(slab, out)

    def forward_body(self, slab: SlabView, out: torch.Tensor | None = None):
        """Run the stage's layers on the activation already in slab x[0]; reads only
        fixed buffers and the pass context, so it can be captured in a CUDA graph.

        Non-last stages write the stage output into ``out`` (the send buffer);
        the last stage computes the loss and its output gradient (into the slab's
        head_dy slot) right away.
        """
        cfg, ws = self.cfg, self.ws
        p, seed, eps = cfg.p_drop, cfg.dropout_seed, cfg.eps
        s, h = cfg.seq, cfg.hidden
        n_local = len(self.layers)
        native.layernorm_fwd(slab.get(0, "x"), self.p(self.layers[0], "ln1_g"), self.p(self.layers[0], "ln1_b"), ws["ln"], eps)
        for i, l in enumerate(self.layers):
            off_a, off_m = self._offsets(l)
            x, qkv, h1, f = slab.get(i, "x"), slab.get(i, "qkv"), slab.get(i, "h1"), slab.get(i, "f")
            self.mm_fwd(ws["ln"], self.p(l, "w_qkv"), qkv)
            o = slab.get(i, "o")
            if self.attn_ours:  # K7 writes o and lse straight into the slab
                native.attn_fwd(qkv, o, slab.get(i, "lse"), cfg.heads)
            else:
                q, k, v = self._qkv_views(qkv)
                res = torch.ops.aten._scaled_dot_product_cudnn_attention(q, k, v, None, True, 0.0, True, False)
                self._pack_attention(slab, i, res[0], res[1])
            self.mm_fwd(o, self.p(l, "w_proj"), ws["a"])
            self._k("residual_dropout_ln_fwd", 8 * s * h, native.residual_dropout_ln_fwd, x, ws["a"], h1, self.p(l, "ln2_g"),
                    self.p(l, "ln2_b"), ws["ln"], p, seed, off_a, eps, offset_base=self.ctx)
            self.mm_fc1_gelu(ws["ln"], self.p(l, "w_fc1"), f, ws["g"])
            self.mm_fwd(ws["g"], self.p(l, "w_fc2"), ws["a"])
            if i + 1 < n_local:
                nxt = self.layers[i + 1]
                native.residual_dropout_ln_fwd(h1, ws["a"], slab.get(i + 1, "x"), self.p(nxt, "ln1_g"),
                                               self.p(nxt, "ln1_b"), ws["ln"], p, seed, off_m, eps, offset_base=self.ctx)
            elif self.last:
                native.residual_dropout_ln_fwd(h1, ws["a"], ws["dy"], self.w["lnf_g"], self.w["lnf_b"], ws["ln"],
                                               p, seed, off_m, eps, offset_base=self.ctx)
                self._head(slab, self.tok[1:])
            else:
                native.residual_dropout_ln_fwd(h1, ws["a"], out, None, None, None, p, seed, off_m, eps,
                                               offset_base=self.ctx)

    def _pack_attention(self, slab: SlabView, i: int, o_tmp: torch.Tensor, lse: torch.Tensor):
        s, h, H = self.cfg.seq, self.cfg.hidden, self.cfg.heads
        if not o_tmp.transpose(1, 2).is_contiguous() or not lse.is_contiguous():
            raise RuntimeError(f"unexpected cuDNN attention layout: o {o_tmp.stride()} lse {lse.stride()}")
        (o_base, o_off), (l_base, l_off) = slab.locate(i, "o"), slab.locate(i, "lse")
        items = [(o_tmp, o_off, 1, 2 * s * h, 0), (lse, l_off, 1, 4 * H * s, 0)]
        if o_base is l_base:
            self._k("pack", 2 * (2 * s * h + 4 * H * s), native.pack, items, o_base)
        else:  # partial offload: o and lse in different parts (lse travels with o; defensive)
            self._k("pack", 4 * s * h, native.pack, items[:1], o_base)
            self._k("pack", 8 * H * s, native.pack, items[1:], l_base)

    def _head(self, slab: SlabView, targets: torch.Tensor):
        """Loss head of the last stage, forward and backward fused into F.

        ws["dy"] holds y (final layer output), ws["ln"] holds LNf(y).  Writes the
        gradient of (loss / m) w.r.t. y into the slab's head_dy slot.
        """
        ws, cfg = self.ws, self.cfg
        logits = torch.mm(ws["ln"], self.w["w_head"].t()).float()
        loss = torch.nn.functional.cross_entropy(logits, targets)
        self.loss_sum += loss.detach()
        dlogits = torch.softmax(logits, -1)
        dlogits[torch.arange(cfg.seq, device=self.device), targets] -= 1.0
        dlogits = (dlogits / (cfg.seq * self.m)).to(torch.bfloat16)
        _wgrad(self.g["w_head"], dlogits.t(), ws["ln"])
        torch.mm(dlogits, self.w["w_head"], out=ws["t"])
        native.layernorm_bwd(ws["dy"], self.w["lnf_g"], ws["t"], None, slab.get(-1, "head_dy"),
                             self.g["lnf_g"], self.g["lnf_b"], eps=cfg.eps)

    # --------------------------------------------------------------- backward
    def backward(self, slab: SlabView, mb: int, iteration: int, dy: torch.Tensor | None = None,
                 dx_out: torch.Tensor | None = None, tokens: torch.Tensor | None = None):
        self.set_pass_context(mb, iteration, tokens)
        self.backward_body(slab, dy, dx_out)

    def new_wbuffer(self) -> dict:
        """Gradient tensors a deferred W pass needs (split backward, GIS/PO schedules):
        per local layer dm [s,h], df [s,4h], da [s,h] and dqkv [s,3h] (18bsh bytes)."""
        s, h = self.cfg.seq, self.cfg.hidden
        bf = dict(device=self.device, dtype=torch.bfloat16)
        return {i: {"dm": torch.empty(s, h, **bf), "df": torch.empty(s, 4 * h, **bf), "da": torch.empty(s, h, **bf),
                    "dqkv": torch.empty(s, 3 * h, **bf)} for i in range(len(self.layers))}

    def backward_body(self, slab: SlabView, dy: torch.Tensor | None = None, dx_out: torch.Tensor | None = None,
                      wbuf: dict | None = None):
        """Backward of the stage from the output gradient ``dy`` (received) or,
        on the last stage, the head gradient saved in the slab.  Writes the input
        gradient into ``dx_out`` (send buffer); the first stage scatters it into
        the embedding gradients instead.

        With ``wbuf`` this is the B pass of a split backward (reference PassKind.B with
        ``split_backward``, ir.py:27-32): activation gradients only; the tensors the
        weight gradients need are left in ``wbuf`` for ``wgrad_body`` (the W pass), which
        also owns the LN1/LN2/GeLU recomputes that only weight gradients use."""
        cfg, ws = self.cfg, self.ws
        p, seed, eps = cfg.p_drop, cfg.dropout_seed, cfg.eps
        s, h = cfg.seq, cfg.hidden
        n_local = len(self.layers)
        split = wbuf is not None
        dm_of = (lambda i: wbuf[i]["dm"]) if split else (lambda i: ws["dm"])  # noqa: E731
        dy_cur = slab.get(-1, "head_dy") if self.last else dy
        top_off_m = self._offsets(self.layers[-1])[1]
        native.dropout(dy_cur, dm_of(n_local - 1), p, seed, top_off_m, offset_base=self.ctx)
        for i in range(n_local - 1, -1, -1):
            l = self.layers[i]
            off_a, _ = self._offsets(l)
            x, qkv, o, lse, h1, f = (slab.get(i, n) for n in ("x", "qkv", "o", "lse", "h1", "f"))
            dm = dm_of(i)
            df = wbuf[i]["df"] if split else ws["big"]
            da = wbuf[i]["da"] if split else ws["da"]
            dqkv = wbuf[i]["dqkv"] if split else ws["dqkv"]
            # MLP: df = (dm @ Wfc2) * gelu'(f) in the GEMM epilogue; g = gelu(f) recomputed for dWfc2
            self.mm_dgrad_dgelu(dm, self.p(l, "w_fc2"), f, df, None if split else ws["g"])
            if not split:
                self.wgrad(self.gp(l, "w_fc2"), dm, ws["g"])
            self.mm_dgrad(df, self.p(l, "w_fc1"), ws["t"])
            # dh1 = dy + LN2_bwd(dln2); da = dropout_bwd(dh1) (attention-branch mask replay);
            # unsplit: the same kernel emits the LN2 recompute ln = LN2(h1) for dWfc1
            self._k("layernorm_bwd", (12 if not split else 10) * s * h, native.layernorm_bwd, h1, self.p(l, "ln2_g"),
                    ws["t"], dy_cur, ws["dh1"], self.gp(l, "ln2_g"), self.gp(l, "ln2_b"), drop_out=da, p=p,
                    drop_seed=seed, drop_offset=off_a, eps=eps, offset_base=self.ctx,
                    beta=None if split else self.p(l, "ln2_b"), ln_out=None if split else ws["ln"])
            if not split:
                self.wgrad(self.gp(l, "w_fc1"), df, ws["ln"])
            # attention projection and core
            if not split:
                self.wgrad(self.gp(l, "w_proj"), da, o)
            self.mm_dgrad(da, self.p(l, "w_proj"), ws["t"])
            grads = None
            if self.attn_bwd_ours:  # K7b: dqkv [s, 3h] straight from the saved o and lse
                native.attn_bwd(qkv, o, ws["t"], lse, dqkv, cfg.heads, ws["attn"])
                self.mm_dgrad(dqkv, self.p(l, "w_qkv"), ws["t"])
                if not split:
                    grads = [dqkv]
            else:
                q, k, v = self._qkv_views(qkv)
                o4 = o.view(1, s, cfg.heads, cfg.head_dim).transpose(1, 2)
                do4 = ws["t"].view(1, s, cfg.heads, cfg.head_dim).transpose(1, 2)
                lse3 = lse.view(self._lse_shape)
                cq, ck, mq, mk, ps, po = self._attn_meta[0], self._attn_meta[1], self._attn_meta[2], self._attn_meta[3], self._attn_meta[4], self._attn_meta[5]
                dq, dk, dv = torch.ops.aten._scaled_dot_product_cudnn_attention_backward(
                    do4, q, k, v, o4, lse3, ps, po, None, cq, ck, mq, mk, 0.0, True)
                if split:
                    self._gather_dqkv(dq, dk, dv, dqkv)  # the W pass needs them after cuDNN's buffers are reused
                    self.mm_dgrad(dqkv, self.p(l, "w_qkv"), ws["t"])
                else:
                    grads = [t.transpose(1, 2).reshape(s, h) for t in (dq, dk, dv)]
                    w_qkv = self.p(l, "w_qkv")
                    for j, gj in enumerate(grads):
                        self.mm_dgrad(gj, w_qkv[j * h:(j + 1) * h], ws["t"], accumulate=j > 0)
            # dx = dh1 + LN1_bwd(dln1); also the next-lower layer's MLP-branch dropout replay;
            # unsplit: the same kernel emits the LN1 recompute ln = LN1(x) for dWqkv
            below = i > 0
            dx_target = ws["dy"] if (below or self.first or dx_out is None) else dx_out
            drop_below = dm_of(i - 1) if below else None
            off_below = self._offsets(self.layers[i - 1])[1] if below else 0
            native.layernorm_bwd(x, self.p(l, "ln1_g"), ws["t"], ws["dh1"], dx_target, self.gp(l, "ln1_g"),
                                 self.gp(l, "ln1_b"), drop_out=drop_below, p=p if below else 0.0,
                                 drop_seed=seed, drop_offset=off_below, eps=eps, offset_base=self.ctx,
                                 beta=None if split else self.p(l, "ln1_b"), ln_out=None if split else ws["ln"])
            if grads is not None:
                g_qkv = self.gp(l, "w_qkv")
                if len(grads) == 1:  # packed dqkv: one weight-gradient GEMM (3h x h)
                    self.wgrad(g_qkv, grads[0], ws["ln"])
                else:
                    for j, gj in enumerate(grads):
                        self.wgrad(g_qkv[j * h:(j + 1) * h], gj, ws["ln"])
            dy_cur = dx_target
        if self.first:
            native.embed_bwd(self.tok[:-1], dy_cur, self.g["wte"], self.g["wpe"])

    def wgrad_body(self, slab: SlabView, wbuf: dict):
        """W pass of a split backward: weight gradients from the slab (recomputing
        LN1, LN2 and GeLU) and the gradients the B pass left in ``wbuf``."""
        cfg, ws = self.cfg, self.ws
        s, h, eps = cfg.seq, cfg.hidden, cfg.eps
        for i, l in enumerate(self.layers):
            x, o, h1, f = (slab.get(i, n) for n in ("x", "o", "h1", "f"))
            b = wbuf[i]
            # GeLU recompute, then LN1 and LN2 recompute in one launch (4E bytes)
            self._k("gelu_fwd", 16 * s * h, native.gelu_fwd, f, ws["g"])
            self._k("layernorm_fwd2", 8 * s * h, native.layernorm_fwd2, x, self.p(l, "ln1_g"), self.p(l, "ln1_b"),
                    ws["ln1"], h1, self.p(l, "ln2_g"), self.p(l, "ln2_b"), ws["ln"], eps)
            self.wgrad(self.gp(l, "w_fc2"), b["dm"], ws["g"])
            self.wgrad(self.gp(l, "w_fc1"), b["df"], ws["ln"])
            self.wgrad(self.gp(l, "w_proj"), b["da"], o)
            self.wgrad(self.gp(l, "w_qkv"), b["dqkv"], ws["ln1"])

    # -------------------------------------------------------------- optimizer
    def sgd_step(self, lr: float = 1e-4):
        """Plain SGD on fp32 master weights, then refresh the bf16 copies."""
        names = sorted(self.master)
        torch._foreach_add_([self.master[n] for n in names], [self.g[n] for n in names], alpha=-lr)
        for n in names:
            self.w[n].copy_(self.master[n])
