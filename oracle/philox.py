"""Philox4x32-10 in numpy (test infrastructure; see oracle/__init__.py).

Matches ``philox4x32_10`` / ``keep_mask8`` in paper_2503_01328_b200/csrc/ppo_common.cuh:
element e of a tensor tagged (seed, offset) uses 16-bit half (e % 2) of word
(e % 8) // 2 of Philox(counter = (e//8 lo, e//8 hi, offset lo, offset hi),
key = (seed lo, seed hi)) and is kept iff that half >= floor(p * 2**16).
"""

import numpy as np

M0, M1 = np.uint64(0xD2511F53), np.uint64(0xCD9E8D57)
W0, W1 = 0x9E3779B9, 0xBB67AE85
MASK32 = np.uint64(0xFFFFFFFF)


def philox4x32_10(c0, c1, c2, c3, k0: int, k1: int):
    c0, c1, c2, c3 = (np.asarray(c, dtype=np.uint64) & MASK32 for c in (c0, c1, c2, c3))
    k0, k1 = k0 & 0xFFFFFFFF, k1 & 0xFFFFFFFF
    for _ in range(10):
        p0 = M0 * c0
        p1 = M1 * c2
        hi0, lo0 = p0 >> np.uint64(32), p0 & MASK32
        hi1, lo1 = p1 >> np.uint64(32), p1 & MASK32
        c0, c1, c2, c3 = hi1 ^ c1 ^ np.uint64(k0), lo1, hi0 ^ c3 ^ np.uint64(k1), lo0
        k0 = (k0 + W0) & 0xFFFFFFFF
        k1 = (k1 + W1) & 0xFFFFFFFF
    return [c.astype(np.uint32) for c in (c0, c1, c2, c3)]


def threshold(p: float) -> int:
    """floor(p * 2**16), clamped to [0, 65535]."""
    t = p * 65536.0
    if t <= 0:
        return 0
    if t >= 65535.0:
        return 65535
    return int(t)


def keep_mask(n: int, p: float, seed: int, offset: int) -> np.ndarray:
    """Boolean keep mask of the first n elements of tensor (seed, offset).

    One Philox block per 8 elements; element e uses the 16-bit half (e % 2) of
    word (e % 8) // 2 (low half first) and is kept iff it is >= threshold(p).
    """
    blocks = (n + 7) // 8
    ctr = np.arange(blocks, dtype=np.uint64)
    words = philox4x32_10(ctr & MASK32, ctr >> np.uint64(32), np.full(blocks, offset & 0xFFFFFFFF, np.uint64),
                          np.full(blocks, (offset >> 32) & 0xFFFFFFFF, np.uint64), seed & 0xFFFFFFFF, seed >> 32)
    w = np.stack(words, axis=1)  # blocks x 4
    halves = np.stack([w & np.uint32(0xFFFF), w >> np.uint32(16)], axis=2).reshape(-1)[:n]
    return halves >= np.uint32(threshold(p))
