"""Schedule IR facade: the names of ``ppoff.ir`` (reference ``pkg/src/ppoff/ir.py``).

Types live in ``schedule_types``, timing and composition in ``compose``; this
module adds validation (ir.py:477-547), activation-residency timelines
(ir.py:555-655), block extraction (ir.py:663-702) and the pass-line wire format
(ir.py:705-783) that the runtime's measured traces are also written in.
"""

from __future__ import annotations

from dataclasses import dataclass
from fractions import Fraction

from .compose import (
    assemble as _assemble,
    bi_level_orders,
    earliest_start as _earliest_start,
    interleave_compose,
    microbatch_groups as _grouped,
    repair_wedge_compat as _escape_reorder,
    shifted_block_orders as _block_shift_orders,
    uniform_repeat,
)
from .costs import ModelSpec, PassCosts, activation_bytes_per_layer
from .schedule_types import (
    KIND_RANK as _KIND_ORDER,
    BuildingBlock,
    InfeasibleIntervalError,
    Pass,
    PassKind,
    Schedule,
    ScheduleError,
    Violation,
    lifespan,
)

__all__ = [
    "PassKind", "Pass", "BuildingBlock", "Schedule", "Violation", "ScheduleError",
    "InfeasibleIntervalError", "MemoryTimeline", "lifespan", "uniform_repeat",
    "interleave_compose", "bi_level_orders", "validate", "memory_timeline",
    "stage_contribution_at_peak", "extract_block", "emit_schedule", "parse_schedule",
]


# ---------------------------------------------------------------------------
# validation
# ---------------------------------------------------------------------------


def validate(sched: Schedule, costs: PassCosts | None = None) -> list[Violation]:
    """Duplicate / missing / dependency / overlap violations as data (ir.py:477-547)."""
    costs = costs or sched.costs
    found: list[Violation] = []
    index: dict = {}
    for p in sched.all_passes():
        key = (p.kind, p.stage, p.microbatch)
        if key in index:
            found.append(Violation("duplicate", f"{key} appears more than once", (index[key], p)))
        index[key] = p

    kinds = [PassKind.F, PassKind.B] + ([PassKind.W] if sched.split_backward else [])
    for s in range(sched.num_stages):
        for j in range(sched.microbatches):
            for k in kinds:
                if (k, s, j) not in index:
                    found.append(Violation("missing", f"({k}, stage {s}, mb {j}) absent"))

    hop = costs.t_comm
    for s in range(sched.num_stages):
        for j in range(sched.microbatches):
            fwd = index.get((PassKind.F, s, j))
            bwd = index.get((PassKind.B, s, j))
            if s + 1 < sched.num_stages:
                fwd_next = index.get((PassKind.F, s + 1, j))
                if fwd and fwd_next and fwd_next.start < fwd.end + hop:
                    found.append(Violation(
                        "dependency",
                        f"F stage {s + 1} mb {j} starts before F stage {s} ends (+comm)",
                        (fwd, fwd_next),
                    ))
                bwd_next = index.get((PassKind.B, s + 1, j))
                if bwd and bwd_next and bwd.start < bwd_next.end + hop:
                    found.append(Violation(
                        "dependency",
                        f"B stage {s} mb {j} starts before B stage {s + 1} ends (+comm)",
                        (bwd_next, bwd),
                    ))
            if fwd and bwd and bwd.start < fwd.end:
                found.append(Violation(
                    "dependency", f"B stage {s} mb {j} starts before its F ends", (fwd, bwd)
                ))
            if sched.split_backward:
                wgt = index.get((PassKind.W, s, j))
                if bwd and wgt and wgt.start < bwd.end:
                    found.append(Violation(
                        "dependency", f"W stage {s} mb {j} starts before its B ends", (bwd, wgt)
                    ))

    for dev, passes in enumerate(sched.device_passes):
        holder = None
        for p in sorted(passes, key=lambda q: (q.start, q.microbatch, _KIND_ORDER[q.kind])):
            if p.duration == 0:
                continue
            if holder is not None and p.start < holder.end:
                found.append(Violation(
                    "overlap", f"device {dev}: {holder.kind} and {p.kind} overlap", (holder, p)
                ))
            if holder is None or p.end > holder.end:
                holder = p
    return found


# ---------------------------------------------------------------------------
# residency timelines
# ---------------------------------------------------------------------------


@dataclass(frozen=True)
class MemoryTimeline:
    """Per-device activation residency as sorted (time, stage, +/-units) events.

    Frees sort before allocations at equal times (half-open residency).
    """

    devices: int
    bytes_per_unit: int
    events: tuple[tuple[tuple[Fraction, int, int], ...], ...]
    base_units: int = 0

    def _walk(self, device: int, skip=()):
        level = self.base_units
        for (t, stage, delta) in self.events[device]:
            if stage in skip:
                continue
            level += delta
            yield t, stage, level

    def series(self, device: int):
        points = [(Fraction(0), self.base_units, self.base_units * self.bytes_per_unit)]
        for t, _stage, level in self._walk(device):
            entry = (t, level, level * self.bytes_per_unit)
            if points[-1][0] == t:
                points[-1] = entry
            else:
                points.append(entry)
        return points

    def peak(self, device: int, exclude_stages=()) -> int:
        return max([self.base_units] + [lv for _t, _s, lv in self._walk(device, exclude_stages)])

    def peak_bytes(self, device: int) -> int:
        return self.peak(device) * self.bytes_per_unit

    def peak_time(self, device: int) -> Fraction:
        best, when = self.base_units, Fraction(0)
        for t, _stage, level in self._walk(device):
            if level > best:
                best, when = level, t
        return when

    def attribution_at(self, device: int, time: Fraction) -> dict[int, int]:
        held: dict[int, int] = {}
        for (t, stage, delta) in self.events[device]:
            if t > time:
                break
            held[stage] = held.get(stage, 0) + delta
        return {s: u for s, u in held.items() if u}

    def integral(self, device: int) -> Fraction:
        area, level, last = Fraction(0), self.base_units, None
        for (t, _stage, delta) in self.events[device]:
            if last is not None:
                area += level * (t - last)
            level += delta
            last = t
        return area

    def global_peak(self) -> int:
        return max(self.peak(d) for d in range(self.devices))


def _event_order(ev):
    return (ev[0], ev[2])


def memory_timeline(
    sched: Schedule,
    model: ModelSpec | None = None,
    recompute: bool = True,
    wgrad_buffer_units: int = 0,
) -> MemoryTimeline:
    """No-offload residency: a unit lives from its F start to its B end."""
    per_unit = 0
    if model is not None:
        per_unit = activation_bytes_per_layer(model, recompute=recompute) * model.layers_per_stage
    units = sched.units_per_stage
    events = [[] for _ in range(sched.devices)]
    for p in sched.all_passes():
        if p.kind == PassKind.F:
            events[p.device].append((p.start, p.stage, units))
        elif p.kind == PassKind.B:
            events[p.device].append((p.end, p.stage, -units))
    return MemoryTimeline(
        devices=sched.devices,
        bytes_per_unit=per_unit,
        events=tuple(tuple(sorted(ev, key=_event_order)) for ev in events),
        base_units=wgrad_buffer_units,
    )


def stage_contribution_at_peak(tl: MemoryTimeline, device: int) -> dict[int, int]:
    return tl.attribution_at(device, tl.peak_time(device))


def extract_block(sched: Schedule, microbatch: int | None = None) -> BuildingBlock:
    """Relative offsets of one microbatch (default: the middle one)."""
    if microbatch is None:
        microbatch = sched.microbatches // 2
    n = sched.num_stages
    got = {PassKind.F: [None] * n, PassKind.B: [None] * n}
    if sched.split_backward:
        got[PassKind.W] = [None] * n
    for p in sched.all_passes():
        if p.microbatch == microbatch and p.kind in got:
            got[p.kind][p.stage] = p.start
    if None in got[PassKind.F] or None in got[PassKind.B]:
        raise ScheduleError(f"microbatch {microbatch} incomplete in schedule")
    origin = got[PassKind.F][0]

    def rel(xs):
        return tuple(x - origin for x in xs)

    return BuildingBlock(
        devices=sched.devices,
        local_stages=sched.local_stages,
        f_start=rel(got[PassKind.F]),
        b_start=rel(got[PassKind.B]),
        w_start=rel(got[PassKind.W]) if sched.split_backward else None,
        costs=sched.costs,
        units=sched.units_per_stage,
    )


# ---------------------------------------------------------------------------
# wire format: one pass per line, `device stage microbatch kind start duration`
# ---------------------------------------------------------------------------


def _frac_str(x: Fraction) -> str:
    x = Fraction(x)
    return f"{x.numerator}" if x.denominator == 1 else f"{x.numerator}/{x.denominator}"


def emit_schedule(sched: Schedule) -> str:
    header = (
        f"# schedule kind={sched.kind} d={sched.devices} v={sched.local_stages}"
        f" stages={sched.num_stages} m={sched.microbatches} units={sched.units_per_stage}"
        f" split={int(sched.split_backward)}"
    )
    if sched.g is not None:
        header += f" g={sched.g}"
    if sched.interval is not None:
        header += f" interval={_frac_str(sched.interval)}"
    c = sched.costs
    out = [
        header,
        f"# costs tF={_frac_str(c.t_f)} tB={_frac_str(c.t_b)} tW={_frac_str(c.t_w)}"
        f" comm={_frac_str(c.t_comm)}",
    ]
    out += [
        f"{p.device} {p.stage} {p.microbatch} {p.kind} {_frac_str(p.start)} {_frac_str(p.duration)}"
        for p in sched.all_passes()
    ]
    return "\n".join(out) + "\n"


def _kv(fields):
    return dict(f.split("=", 1) for f in fields)


def parse_schedule(text: str) -> Schedule:
    meta, cost_meta, passes = {}, {}, []
    for lineno, raw in enumerate(text.splitlines(), start=1):
        line = raw.strip()
        if not line:
            continue
        if line.startswith("#"):
            words = line[1:].split()
            if words[:1] == ["schedule"]:
                meta = _kv(words[1:])
            elif words[:1] == ["costs"]:
                cost_meta = _kv(words[1:])
            continue
        cols = line.split()
        if len(cols) != 6:
            raise ScheduleError(f"line {lineno}: expected 6 fields, got {len(cols)}")
        try:
            passes.append(Pass(
                PassKind(cols[3]), int(cols[0]), int(cols[1]), int(cols[2]),
                Fraction(cols[4]), Fraction(cols[5]),
            ))
        except ValueError as exc:
            raise ScheduleError(f"line {lineno}: {exc}") from exc
    if not meta:
        raise ScheduleError("missing '# schedule ...' header")
    costs = PassCosts(
        cost_meta.get("tF", 0), cost_meta.get("tB", 1), cost_meta.get("tW", 0), cost_meta.get("comm", 0)
    )
    d = int(meta["d"])
    stages = int(meta["stages"])
    per_dev = [[] for _ in range(d)]
    for p in passes:
        per_dev[p.device].append(p)
    for lst in per_dev:
        lst.sort(key=lambda p: (p.start, p.microbatch, _KIND_ORDER.get(p.kind, 3)))
    return Schedule(
        devices=d,
        local_stages=int(meta["v"]),
        num_stages=stages,
        microbatches=int(meta["m"]),
        placement=tuple(s % d for s in range(stages)),
        units_per_stage=int(meta["units"]),
        split_backward=bool(int(meta["split"])),
        costs=costs,
        kind=meta.get("kind", "custom"),
        g=int(meta["g"]) if "g" in meta else None,
        interval=Fraction(meta["interval"]) if "interval" in meta else None,
        device_passes=tuple(tuple(lst) for lst in per_dev),
    )
