"""numpy fp32 restatements of the recompute kernels (test infrastructure).

Each function states the math the CUDA kernel in
paper_2503_01328_b200/csrc/ppo_kernels.cu must reproduce; tolerances live in
the tests.  bf16 rounding is emulated with round-to-nearest-even on the fp32
bit pattern, the same rounding __float2bfloat16_rn performs.
"""

import numpy as np

from .philox import keep_mask

GELU_K0 = 0.7978845608028654
GELU_K1 = 0.044715


def bf16_round(x: np.ndarray) -> np.ndarray:
    """fp32 -> nearest-even bf16 -> fp32 (NaN-free inputs)."""
    b = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    rounded = (b + np.uint64(0x7FFF) + ((b >> np.uint64(16)) & np.uint64(1))) >> np.uint64(16) << np.uint64(16)
    return rounded.astype(np.uint32).view(np.float32).reshape(np.shape(x))


def layernorm(x, gamma, beta, eps=1e-5):
    x = x.astype(np.float32)
    mean = x.mean(-1, keepdims=True)
    var = ((x - mean) ** 2).mean(-1, keepdims=True)
    return (x - mean) / np.sqrt(var + eps) * gamma + beta


def layernorm_bwd(x, gamma, dy, eps=1e-5):
    """dx, dgamma, dbeta of y = LN(x)*gamma + beta (statistics recomputed from x)."""
    x = x.astype(np.float32)
    dy = dy.astype(np.float32)
    h = x.shape[-1]
    mean = x.mean(-1, keepdims=True)
    rstd = 1.0 / np.sqrt(((x - mean) ** 2).mean(-1, keepdims=True) + eps)
    xhat = (x - mean) * rstd
    g = dy * gamma
    dx = rstd * (g - g.mean(-1, keepdims=True) - xhat * (g * xhat).sum(-1, keepdims=True) / h)
    return dx, (dy * xhat).reshape(-1, h).sum(0), dy.reshape(-1, h).sum(0)


def gelu(x):
    x = x.astype(np.float32)
    return 0.5 * x * (1.0 + np.tanh(GELU_K0 * (x + GELU_K1 * x ** 3)))


def gelu_grad(x):
    x = x.astype(np.float32)
    th = np.tanh(GELU_K0 * (x + GELU_K1 * x ** 3))
    return 0.5 * (1.0 + th) + 0.5 * x * (1.0 - th * th) * GELU_K0 * (1.0 + 3.0 * GELU_K1 * x * x)


def dropout(x, p, seed, offset):
    keep = keep_mask(x.size, p, seed, offset).reshape(x.shape)
    scale = np.float32(1.0) / np.float32(1.0 - p)  # fp32 scale, applied by multiplication as on device
    return np.where(keep, x.astype(np.float32) * scale, np.float32(0.0)).astype(np.float32)


def bf16_ulp_diff(a, b) -> np.ndarray:
    """|a - b| in bf16 units in the last place (both already bf16-representable)."""
    ia = np.ascontiguousarray(a, np.float32).view(np.int32) >> 16
    ib = np.ascontiguousarray(b, np.float32).view(np.int32) >> 16
    # map sign-magnitude to a monotone integer line
    ia = np.where(ia < 0, -(ia & 0x7FFF), ia)
    ib = np.where(ib < 0, -(ib & 0x7FFF), ib)
    return np.abs(ia.astype(np.int64) - ib.astype(np.int64))


def residual_dropout(resid, branch, p, seed, offset):
    """out = resid + dropout(branch) rounded to bf16 (the stored h1 / y)."""
    return bf16_round(resid.astype(np.float32) + dropout(branch, p, seed, offset))


def pack(items, total_bytes, base=None):
    """Gather (src_bytes, dst_off, rows, row_bytes, src_pitch) byte ranges into one buffer
    (zeros, or a copy of ``base``: bytes outside the items keep their values)."""
    out = np.zeros(total_bytes, dtype=np.uint8) if base is None else np.array(base, dtype=np.uint8, copy=True)
    for src, off, rows, row_bytes, pitch in items:
        pitch = pitch or row_bytes
        for r in range(rows):
            out[off + r * row_bytes: off + (r + 1) * row_bytes] = src[r * pitch: r * pitch + row_bytes]
    return out
