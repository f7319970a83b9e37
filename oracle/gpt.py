"""Serial fp32 CPU oracle of the pipelined transformer (test infrastructure).

The B200 runtime runs this model pipelined over stages with activation offload
and LN/GeLU/dropout recompute; pipelining and recompute are exact
transformations, so loss and gradients must match
this serial fp32 run up to bf16 storage/accumulation error (tolerances are in
the tests).

Model (GPT block, pre-LN, MHA, no linear biases, hidden dropout p on both
residual branches, causal attention, tanh GeLU):

    x0 = wte[tokens] + wpe
    per layer:  h1 = x + drop(o @ Wproj^T)      o = attn(LN1(x) @ Wqkv^T)
                y  = h1 + drop(gelu(LN2(h1) @ Wfc1^T) @ Wfc2^T)
    loss = mean CE(LNf(y_L) @ Whead^T, next-token targets)

Dropout element masks come from oracle.philox with offset
``dropout_offset(iteration, layer, mb, branch)``, identical to the runtime.
Each weight matrix is drawn from its own ``torch.Generator`` seeded with
(seed, crc32(name)) and rounded to bf16 so the oracle and the runtime start from identical values.
"""

from __future__ import annotations

import zlib
from dataclasses import dataclass

import numpy as np
import torch

from .philox import keep_mask


@dataclass(frozen=True)
class GPTConfig:
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


def dropout_offset(cfg: GPTConfig, iteration: int, layer: int, microbatch: int, microbatches: int, branch: int) -> int:
    """Philox offset of one dropout site; branch 0 = attention residual, 1 = MLP residual."""
    return (((iteration * cfg.n_layers + layer) * microbatches + microbatch) * 2) + branch


def param_shapes(cfg: GPTConfig):
    h, v, s = cfg.hidden, cfg.vocab, cfg.seq
    shapes = {"wte": (v, h), "wpe": (s, h)}
    for l in range(cfg.n_layers):
        shapes.update({
            f"l{l}.ln1_g": (h,), f"l{l}.ln1_b": (h,), f"l{l}.w_qkv": (3 * h, h), f"l{l}.w_proj": (h, h),
            f"l{l}.ln2_g": (h,), f"l{l}.ln2_b": (h,), f"l{l}.w_fc1": (4 * h, h), f"l{l}.w_fc2": (h, 4 * h),
        })
    shapes.update({"lnf_g": (h,), "lnf_b": (h,), "w_head": (v, h)})
    return shapes


def init_params(cfg: GPTConfig, seed: int = 1234) -> dict[str, torch.Tensor]:
    """N(0, 0.02) matrices (bf16-rounded, fp32 storage); LayerNorm gamma=1, beta=0."""
    out = {}
    for name, shape in param_shapes(cfg).items():
        if name.endswith("_g"):
            out[name] = torch.ones(shape)
        elif name.endswith("_b"):
            out[name] = torch.zeros(shape)
        else:
            gen = torch.Generator().manual_seed(seed * 1_000_003 + zlib.crc32(name.encode()))
            std = 0.02 / (2 * cfg.n_layers) ** 0.5 if name.endswith(("w_proj", "w_fc2")) else 0.02
            out[name] = (torch.randn(shape, generator=gen) * std).bfloat16().float()
    return out


def make_tokens(cfg: GPTConfig, microbatches: int, seed: int = 0) -> torch.Tensor:
    gen = torch.Generator().manual_seed(seed)
    return torch.randint(0, cfg.vocab, (microbatches, cfg.seq + 1), generator=gen)


class _Bf16(torch.autograd.Function):
    """Round to bf16 (nearest even) in the forward AND round the incoming gradient in
    the backward: marks a tensor the device path stores in bf16 (activations in the
    forward, activation gradients in the backward)."""

    @staticmethod
    def forward(ctx, x):
        return x.bfloat16().float()

    @staticmethod
    def backward(ctx, g):
        return g.bfloat16().float()


def _id(x):
    return x


def _mask(cfg, iteration, layer, mb, m, branch, shape):
    keep = keep_mask(int(np.prod(shape)), cfg.p_drop, cfg.dropout_seed, dropout_offset(cfg, iteration, layer, mb, m, branch))
    scale = np.float32(1.0) / np.float32(1.0 - cfg.p_drop)  # fp32 scale, as on device
    return torch.from_numpy(keep.reshape(shape)).float() * float(scale)


def _attention(cfg, qkv):
    s, h = qkv.shape[0], cfg.hidden
    q, k, v = qkv.view(s, 3, cfg.heads, cfg.head_dim).unbind(1)
    q, k, v = (t.transpose(0, 1) for t in (q, k, v))  # heads, s, d
    att = (q @ k.transpose(1, 2)) / cfg.head_dim ** 0.5
    causal = torch.ones(s, s, dtype=torch.bool).tril()
    att = att.masked_fill(~causal, float("-inf")).softmax(-1)
    return (att @ v).transpose(0, 1).reshape(s, h)


def _gelu(x):
    return 0.5 * x * (1.0 + torch.tanh(0.7978845608028654 * (x + 0.044715 * x ** 3)))


def run_layers(cfg, params, x, layers, mb, m, iteration=0, bf16=False):
    """The transformer layers ``layers`` (global ids) applied to x [s, h].

    ``bf16=True`` rounds every tensor the device path stores in bf16 (forward
    activations and their gradients, ``_Bf16``) and computes in fp32 in between --
    the device's storage precision with the oracle's exact arithmetic."""
    ln = torch.nn.functional.layer_norm
    r = _Bf16.apply if bf16 else _id
    for l in layers:
        p = lambda k: params[f"l{l}.{k}"]  # noqa: E731
        a = r(ln(x, (cfg.hidden,), p("ln1_g"), p("ln1_b"), cfg.eps))
        o = r(_attention(cfg, r(a @ p("w_qkv").t())))
        h1 = r(x + r(o @ p("w_proj").t()) * _mask(cfg, iteration, l, mb, m, 0, x.shape))
        f = r(r(ln(h1, (cfg.hidden,), p("ln2_g"), p("ln2_b"), cfg.eps)) @ p("w_fc1").t())
        x = r(h1 + r(r(_gelu(f)) @ p("w_fc2").t()) * _mask(cfg, iteration, l, mb, m, 1, x.shape))
    return x


def microbatch_loss(cfg, params, tokens_mb, mb, m, iteration=0, bf16=False):
    inp, tgt = tokens_mb[:-1], tokens_mb[1:]
    ln = torch.nn.functional.layer_norm
    r = _Bf16.apply if bf16 else _id
    x = run_layers(cfg, params, r(params["wte"][inp] + params["wpe"]), range(cfg.n_layers), mb, m, iteration, bf16)
    logits = r(r(ln(x, (cfg.hidden,), params["lnf_g"], params["lnf_b"], cfg.eps)) @ params["w_head"].t())
    return torch.nn.functional.cross_entropy(logits, tgt)


def forward_backward(cfg: GPTConfig, params: dict, tokens: torch.Tensor, iteration: int = 0, bf16: bool = False):
    """Mean loss over microbatches and gradients of that mean (serial fp32; ``bf16``:
    bf16 storage of activations and activation gradients, see ``run_layers``)."""
    leaf = {k: v.clone().requires_grad_(True) for k, v in params.items()}
    m = tokens.shape[0]
    losses = []
    for mb in range(m):
        loss = microbatch_loss(cfg, leaf, tokens[mb], mb, m, iteration, bf16)
        (loss / m).backward()
        losses.append(float(loss.detach()))
    return float(np.mean(losses)), losses, {k: v.grad.detach() for k, v in leaf.items()}
