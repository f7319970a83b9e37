"""Byte layout of one (stage, microbatch) saved set: device slab <-> host bins.

The saved set of one transformer layer is the 20bsh set the reference counts
(``activation_bytes_per_layer(recompute=True)``, pkg/src/ppoff/costs.py:99-105):

    x [s,h] (2bsh)  qkv [s,3h] (6bsh)  o [s,h] (2bsh)  h1 [s,h] (2bsh)  f [s,4h] (8bsh)

plus the flash-attention log-sum-exp (4 * heads * s bytes, reported as measured
overhead) and, on the last pipeline stage only, the loss
head's output gradient [s,h] (the head runs its backward inside F).

Host side, the tensors are packed into <= 3 power-of-two pinned bins with the
reference's own ``pack_host_bins`` (offload.py:305-340).  The
device slab lays the tensors out bin by bin, each bin's used bytes contiguous,
so one (stage, mb) transfer is one cudaMemcpyAsync per bin, and the reloaded
tensors are views into the slab -- no unpack kernel.
"""

from __future__ import annotations

from dataclasses import dataclass

from ..offload import pack_host_bins

ALIGN = 256  # every tensor starts 256-byte aligned (GEMM / TMA friendly)

# name, columns as a multiple of h (None = special), element bytes
LAYER_TENSORS = (("x", 1), ("qkv", 3), ("o", 1), ("lse", None), ("h1", 1), ("f", 4))


def _round_up(n: int, a: int = ALIGN) -> int:
    return (n + a - 1) // a * a


@dataclass(frozen=True)
class TensorSlot:
    layer: int  # local layer index; -1 = stage-level tensor
    name: str
    shape: tuple[int, ...]
    dtype: str  # "bf16" | "f32"
    nbytes: int
    bin: int
    bin_offset: int
    dev_offset: int


@dataclass(frozen=True)
class SlabLayout:
    seq: int
    hidden: int
    heads: int
    layers: int
    head_grad: bool
    tensors: tuple[TensorSlot, ...]
    bins: tuple[int, ...]  # host bin sizes (powers of two)
    bin_used: tuple[int, ...]  # bytes actually used in each bin
    bin_dev_base: tuple[int, ...]  # where each bin's bytes start in the device slab

    @property
    def slab_bytes(self) -> int:
        return self.bin_dev_base[-1] + _round_up(self.bin_used[-1])

    @property
    def host_bytes(self) -> int:
        return sum(self.bins)

    @property
    def payload_bytes(self) -> int:
        """The 20bsh saved set only (what activation_bytes_per_layer counts) x layers."""
        return sum(t.nbytes for t in self.tensors if t.name in ("x", "qkv", "o", "h1", "f"))

    @property
    def overhead_bytes(self) -> int:
        return self.slab_bytes - self.payload_bytes

    def find(self, layer: int, name: str) -> TensorSlot:
        for t in self.tensors:
            if t.layer == layer and t.name == name:
                return t
        raise KeyError((layer, name))

    def segments(self, dev_base: int, host_bins: tuple[int, ...]):
        """(device_ptr, host_ptr, bytes) per bin for ppo_transfer."""
        return [(dev_base + self.bin_dev_base[b], host_bins[b], self.bin_used[b]) for b in range(len(self.bins))]


def make_layout(layers: int, seq: int, hidden: int, heads: int, head_grad: bool = False) -> SlabLayout:
    specs = []
    for l in range(layers):
        for name, cols in LAYER_TENSORS:
            if name == "lse":
                specs.append((l, name, (heads, seq), "f32", 4 * heads * seq))
            else:
                specs.append((l, name, (seq, cols * hidden), "bf16", 2 * seq * cols * hidden))
    if head_grad:
        specs.append((-1, "head_dy", (seq, hidden), "bf16", 2 * seq * hidden))
    padded = [_round_up(s[4]) for s in specs]
    host = pack_host_bins(padded)
    used = [0] * len(host.bins)
    where = {}
    for idx, b, off in host.placements:
        where[idx] = (b, off)
        used[b] = max(used[b], off + padded[idx])
    base, acc = [], 0
    for b in range(len(host.bins)):
        base.append(acc)
        acc += _round_up(used[b])
    slots = []
    for idx, (l, name, shape, dtype, nbytes) in enumerate(specs):
        b, off = where[idx]
        slots.append(TensorSlot(l, name, shape, dtype, nbytes, b, off, base[b] + off))
    return SlabLayout(
        seq=seq, hidden=hidden, heads=heads, layers=layers, head_grad=head_grad,
        tensors=tuple(slots), bins=tuple(host.bins), bin_used=tuple(used), bin_dev_base=tuple(base),
    )
