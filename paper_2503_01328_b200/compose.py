"""Op orders and dependency-tight timing (reference ``ir.py:176-469``).

* ``earliest_start``   -- start times of fixed per-device orders under the F/B/W
  chain dependencies plus the stage-hop lag (reference ``_earliest_start``,
  ir.py:176-249, and its wedge repair ``_escape_reorder``, ir.py:252-268).
* ``bi_level_orders``  -- the per-device op order of 1F1B / interleaved 1F1B /
  GIS (ir.py:408-429).
* ``interleave_compose`` / ``uniform_repeat`` -- the two composition rules
  (ir.py:357-469).

The start time of every pass under fixed orders is the longest path in a DAG,
so any correct sweep yields the same numbers; the only order-sensitive piece is
the wedge repair, which this module applies exactly at the maximal-progress
stuck state, the same point the reference does.
"""

from __future__ import annotations

from fractions import Fraction

from .costs import PassCosts
from .schedule_types import (
    KIND_RANK,
    BuildingBlock,
    InfeasibleIntervalError,
    Pass,
    PassKind,
    Schedule,
    ScheduleError,
)

F, B, W = PassKind.F, PassKind.B, PassKind.W


def _inputs(kind: PassKind, stage: int, mb: int, last_stage: int):
    """(producer key, needs stage hop) pairs a compute pass waits on."""
    if kind == F:
        return [((F, stage - 1, mb), True)] if stage > 0 else []
    if kind == B:
        deps = [((B, stage + 1, mb), True)] if stage < last_stage else []
        deps.append(((F, stage, mb), False))
        return deps
    return [((B, stage, mb), False)]


def _repair_wedge(orders, heads, finished) -> bool:
    """Move the first input-ready F of the lowest stuck device to its head."""
    for dev, order in enumerate(orders):
        head = heads[dev]
        if head >= len(order):
            continue
        for pos in range(head, len(order)):
            kind, stage, mb = order[pos]
            if kind != F:
                continue
            if stage != 0 and (F, stage - 1, mb) not in finished:
                continue
            if pos == head:
                break
            order.insert(head, order.pop(pos))
            return True
    return False


def repair_wedge_compat(orders, idx, end, num_stages) -> bool:
    """Signature-compatible alias of the reference's ``_escape_reorder``."""
    return _repair_wedge(orders, idx, end)


def earliest_start(
    orders,
    num_stages: int,
    durations,
    t_comm: Fraction,
    floors=None,
    reorder_escape: bool = False,
) -> dict:
    """Dependency-tight start time of every (kind, stage, mb) in ``orders``.

    ``orders`` is a list (per device) of mutable lists of keys; with
    ``reorder_escape`` a wedged state is repaired in place (see module doc).
    ``floors`` optionally maps keys to minimum start times.
    """
    last_stage = num_stages - 1
    floors = floors or {}
    start: dict = {}
    finish: dict = {}
    heads = [0] * len(orders)
    free_at = [Fraction(0)] * len(orders)
    remaining = sum(len(o) for o in orders)

    def place(dev: int) -> int:
        placed = 0
        order = orders[dev]
        while heads[dev] < len(order):
            key = order[heads[dev]]
            t = max(free_at[dev], floors.get(key, free_at[dev]))
            ready = True
            for dep, hop in _inputs(*key, last_stage):
                done = finish.get(dep)
                if done is None:
                    ready = False
                    break
                t = max(t, done + t_comm if hop else done)
            if not ready:
                break
            start[key] = t
            finish[key] = free_at[dev] = t + durations(key[0])
            heads[dev] += 1
            placed += 1
        return placed

    while remaining:
        moved = 0
        for dev in range(len(orders)):
            moved += place(dev)
        remaining -= moved
        if moved:
            continue
        if reorder_escape and _repair_wedge(orders, heads, finish):
            continue
        stuck = [o[h] for o, h in zip(orders, heads) if h < len(o)]
        raise ScheduleError(f"cyclic dependencies; next unschedulable passes: {stuck}")
    return start


def assemble(
    orders,
    start,
    *,
    devices: int,
    local_stages: int,
    num_stages: int,
    microbatches: int,
    units: int,
    split: bool,
    costs: PassCosts,
    kind: str,
    g: int | None = None,
    interval: Fraction | None = None,
) -> Schedule:
    """Freeze orders plus start times into a ``Schedule`` (ir.py:271-315)."""
    sched = Schedule(
        devices=devices,
        local_stages=local_stages,
        num_stages=num_stages,
        microbatches=microbatches,
        placement=tuple(s % devices for s in range(num_stages)),
        units_per_stage=units,
        split_backward=split,
        costs=costs,
        kind=kind,
        g=g,
        interval=interval,
    )
    lengths = {k: sched.duration(k) for k in (F, B, W)}
    per_device = tuple(
        tuple(Pass(k, dev, s, mb, start[(k, s, mb)], lengths[k]) for (k, s, mb) in order)
        for dev, order in enumerate(orders)
    )
    object.__setattr__(sched, "device_passes", per_device)
    return sched


def microbatch_groups(m: int, g: int) -> list[range]:
    """range(m) cut into consecutive groups of g; the last may be short."""
    return [range(lo, min(lo + g, m)) for lo in range(0, m, g)]


def bi_level_orders(d: int, v: int, g: int, m: int, warmups, split: bool):
    """Per-device op orders: ``warmups[i]`` forwards, then one B (+W) per F.

    Forwards walk groups of g microbatches through local chunks 0..v-1;
    backwards walk the same groups through the chunks in reverse.
    """
    groups = microbatch_groups(m, g)
    result = []
    for dev in range(d):
        fwd = [(c * d + dev, j) for grp in groups for c in range(v) for j in grp]
        bwd = [(c * d + dev, j) for grp in groups for c in range(v - 1, -1, -1) for j in grp]
        n_warm = min(warmups[dev], len(fwd))
        seq = [(F, s, j) for (s, j) in fwd[:n_warm]]
        pending_fwd = iter(fwd[n_warm:])
        for (s, j) in bwd:
            seq.append((B, s, j))
            if split:
                seq.append((W, s, j))
            nxt = next(pending_fwd, None)
            if nxt is not None:
                seq.append((F, nxt[0], nxt[1]))
        result.append(seq)
    return result


def interleave_compose(
    block: BuildingBlock,
    g: int,
    m: int,
    warmups=None,
    kind: str = "interleave",
) -> Schedule:
    """Two-level interleaving of ``block`` with inner group size g in [ceil(d/2), d]."""
    d, v = block.devices, block.local_stages
    lo = (d + 1) // 2
    if g < lo or g > d:
        raise ScheduleError(f"g={g} outside [{lo}, {d}]")
    if m < 1:
        raise ScheduleError("need at least one microbatch")
    if warmups is None:
        warmups = [g * (v - 1) + d - i for i in range(d)]
    orders = bi_level_orders(d, v, g, m, warmups, block.split_backward)
    start = earliest_start(
        orders,
        block.num_stages,
        block.duration,
        block.costs.t_comm,
        reorder_escape=(m % g != 0),
    )
    return assemble(
        orders,
        start,
        devices=d,
        local_stages=v,
        num_stages=block.num_stages,
        microbatches=m,
        units=block.units,
        split=block.split_backward,
        costs=block.costs,
        kind=kind,
        g=g,
    )


def shifted_block_orders(block: BuildingBlock, m: int, interval: Fraction):
    """Per-device orders of m copies of ``block`` shifted by ``interval``.

    Overlapping passes on a device are pushed right (minimal shift) in order of
    (start, microbatch, F<B<W, stage); the pushed start becomes a floor.
    Returns (orders, floors, largest push).
    """
    offsets = [(F, block.f_start), (B, block.b_start)]
    if block.w_start is not None:
        offsets.append((W, block.w_start))
    buckets = [[] for _ in range(block.devices)]
    for j in range(m):
        shift = j * interval
        for kind, table in offsets:
            for s in range(block.num_stages):
                buckets[block.device_of(s)].append((table[s] + shift, j, KIND_RANK[kind], kind, s))
    orders, floors = [], {}
    worst = Fraction(0)
    for bucket in buckets:
        bucket.sort()
        cursor = None
        seq = []
        for (t, j, _rank, kind, s) in bucket:
            if cursor is not None and t < cursor:
                worst = max(worst, cursor - t)
                t = cursor
            cursor = t + block.duration(kind)
            seq.append((kind, s, j))
            floors[(kind, s, j)] = t
        orders.append(seq)
    return orders, floors, worst


def uniform_repeat(block: BuildingBlock, m: int, interval: Fraction) -> Schedule:
    """Start microbatch j's copy of ``block`` at j*interval (reference ir.py:357-395)."""
    interval = Fraction(interval)
    if interval <= 0:
        raise ScheduleError("interval must be positive")
    if m < 1:
        raise ScheduleError("need at least one microbatch")
    kinds = [F, B] + ([W] if block.split_backward else [])
    load = [Fraction(0)] * block.devices
    for s in range(block.num_stages):
        load[block.device_of(s)] += sum((block.duration(k) for k in kinds), Fraction(0))
    if interval < max(load):
        raise InfeasibleIntervalError(
            f"interval {interval} below the per-microbatch device busy time {max(load)}"
        )
    orders, floors, _ = shifted_block_orders(block, m, interval)
    start = earliest_start(orders, block.num_stages, block.duration, block.costs.t_comm, floors=floors)
    return assemble(
        orders,
        start,
        devices=block.devices,
        local_stages=block.local_stages,
        num_stages=block.num_stages,
        microbatches=m,
        units=block.units,
        split=block.split_backward,
        costs=block.costs,
        kind="uniform-repeat",
        interval=interval,
    )
