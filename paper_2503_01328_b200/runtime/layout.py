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

Partial (per-tensor) offload: ``make_layout(..., offload=...)`` names the tensors
that travel.  Only those are binned; they form the slab's *offload part*
[0, off_bytes), the rest its *resident part* [off_bytes, slab_bytes).  The
executor gives the two parts separate arenas: an offloaded pair frees its offload
part at D2H end while the resident part stays until the pair's backward.  With
``offload=None`` every tensor travels and the resident part is empty.
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
    res_bytes: int = 0  # resident part (tensors that never travel), after the offload part

    @property
    def off_bytes(self) -> int:
        """Offload part: the binned tensors, [0, off_bytes) of the slab."""
        return (self.bin_dev_base[-1] + _round_up(self.bin_used[-1])) if self.bins else 0

    @property
    def slab_bytes(self) -> int:
        return self.off_bytes + self.res_bytes

    @property
    def offload_fraction(self) -> float:
        """Share of the slab that travels (1.0 = full offload of the saved set)."""
        return self.off_bytes / self.slab_bytes if self.slab_bytes else 0.0

    def travels(self, t: "TensorSlot") -> bool:
        return t.bin >= 0

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


def offload_candidates(layers: int) -> list[tuple[int, str]]:
    """Tensors in the order partial offload adds them: the largest first (f, then
    qkv), top layer first; then the [s,h] tensors.  Prefixes of this list are the
    per-tensor offload sets ``policy.choose_partial_offload`` searches."""
    out = []
    for name in ("f", "qkv", "h1", "o", "x"):
        for l in range(layers - 1, -1, -1):
            out.append((l, name))
    return out


def make_layout(layers: int, seq: int, hidden: int, heads: int, head_grad: bool = False,
                offload=None) -> SlabLayout:
    """``offload``: None (every tensor travels) or a collection of (layer, name) pairs;
    a layer's ``lse`` travels with its ``o`` and ``head_dy`` with the top layer's f."""
    specs = []
    for l in range(layers):
        for name, cols in LAYER_TENSORS:
            if name == "lse":
                specs.append((l, name, (heads, seq), "f32", 4 * heads * seq))
            else:
                specs.append((l, name, (seq, cols * hidden), "bf16", 2 * seq * cols * hidden))
    if head_grad:
        specs.append((-1, "head_dy", (seq, hidden), "bf16", 2 * seq * hidden))
    if offload is None:
        moving = list(range(len(specs)))
    else:
        chosen = set(offload)
        bad = chosen - {(l, n) for l in range(layers) for n, _ in LAYER_TENSORS if n != "lse"}
        if bad:
            raise ValueError(f"unknown offload tensors {sorted(bad)}")

        def travels(l, name):
            if name == "lse":
                return (l, "o") in chosen
            if name == "head_dy":
                return (layers - 1, "f") in chosen
            return (l, name) in chosen

        moving = [i for i, sp in enumerate(specs) if travels(sp[0], sp[1])]
    padded = [_round_up(s[4]) for s in specs]
    where = {}
    used, base = [], []
    host_bins: tuple = ()
    if moving:
        host = pack_host_bins([padded[i] for i in moving])
        host_bins = tuple(host.bins)
        used = [0] * len(host.bins)
        for j, b, off in host.placements:
            where[moving[j]] = (b, off)
            used[b] = max(used[b], off + padded[moving[j]])
        acc = 0
        for b in range(len(host.bins)):
            base.append(acc)
            acc += _round_up(used[b])
    off_bytes = (base[-1] + _round_up(used[-1])) if moving else 0
    res_acc = 0
    slots = []
    for idx, (l, name, shape, dtype, nbytes) in enumerate(specs):
        if idx in where:
            b, off = where[idx]
            slots.append(TensorSlot(l, name, shape, dtype, nbytes, b, off, base[b] + off))
        else:
            slots.append(TensorSlot(l, name, shape, dtype, nbytes, -1, -1, off_bytes + res_acc))
            res_acc += padded[idx]
    return SlabLayout(
        seq=seq, hidden=hidden, heads=heads, layers=layers, head_grad=head_grad,
        tensors=tuple(slots), bins=host_bins, bin_used=tuple(used), bin_dev_base=tuple(base),
        res_bytes=res_acc,
    )
