"""Exact event-driven runner model (reference ``pkg/src/ppoff/sim.py``).

The B200 executor (``runtime.executor.execute``) is the measured replacement of
``simulate``; this module keeps the modelled runner so that

* plans can be judged before they are launched (k-aware selection),
* the executor's measured residency can be compared with the model's, and
* planner callers that import ``simulate`` keep working unchanged.

Semantics (reference sim.py:141-413), restated:

1. Compute passes run per device in ``device_passes`` order, each as soon as its
   inputs are done and the device is free.  F needs F(stage-1) + t_comm; B needs
   B(stage+1) + t_comm, its own F, and its own RELOAD when the pair was
   offloaded; W needs its B.
2. OFFLOAD needs its F to end; RELOAD needs its OFFLOAD to end and never starts
   before its slot (a synced plan pins every transfer to its slot); sync edges
   add cross-device precedence.
3. An idle copy stream takes its lowest-slot transfer whose inputs are already
   *scheduled* (a compute end is known once the pass starts, a transfer end once
   it finishes), waiting for that transfer's earliest start even if a later
   slot could go sooner.
4. Under shared-switch halving a transfer's rate halves while another transfer
   of the same direction is active on its switch and halves again while its own
   device moves the opposite direction (dual streams).
5. Device residency: +u at F start, -u at D2H end, +u at H2D start, -u at B end;
   host residency from D2H end to H2D end.
"""

from __future__ import annotations

import csv
import heapq
import io
import json
from dataclasses import dataclass
from fractions import Fraction

from .costs import ModelSpec, PassCosts, activation_bytes_per_layer
from .ir import MemoryTimeline, _frac_str
from .offload import NodeAssignment, OffloadPlan
from .schedule_types import Pass, PassKind, Schedule

__all__ = [
    "SimTrace", "ContentionModel", "DeadlockError", "simulate", "bubble_time",
    "peak_memory", "host_peak_memory",
]

F, B, W = PassKind.F, PassKind.B, PassKind.W
ZERO = Fraction(0)


class DeadlockError(Exception):
    def __init__(self, message: str, waiting=()):
        super().__init__(message)
        self.waiting = tuple(waiting)


@dataclass(frozen=True)
class ContentionModel:
    mode: str = "none"  # "none" | "shared-switch-halving"
    devices_per_switch: int = 2

    def __post_init__(self):
        if self.mode not in ("none", "shared-switch-halving"):
            raise ValueError(f"unknown contention mode {self.mode!r}")

    def switch_of(self, device: int) -> int:
        return device // self.devices_per_switch


@dataclass(frozen=True)
class SimTrace:
    schedule: Schedule
    passes: tuple[Pass, ...]
    makespan: Fraction
    device_busy: tuple[Fraction, ...]
    memory: MemoryTimeline
    host_events: tuple[tuple[Fraction, int, int], ...]
    contention_log: tuple[tuple[Fraction, Fraction, int, str, Fraction], ...]
    bytes_per_unit: int = 0

    def compute_passes(self):
        return [p for p in self.passes if p.kind in (F, B, W)]

    def transfer_passes(self):
        return [p for p in self.passes if p.kind in (PassKind.OFFLOAD, PassKind.RELOAD)]

    def last_transfer_end(self) -> Fraction:
        return max((p.end for p in self.transfer_passes()), default=ZERO)

    def pass_times(self) -> dict:
        return {(p.kind, p.stage, p.microbatch): (p.start, p.end) for p in self.passes}

    def to_csv(self) -> str:
        buf = io.StringIO()
        out = csv.writer(buf)
        out.writerow(["device", "stage", "microbatch", "kind", "start", "end", "duration"])
        for p in sorted(self.passes, key=lambda q: (q.start, q.device, str(q.kind))):
            out.writerow([p.device, p.stage, p.microbatch, str(p.kind), str(p.start), str(p.end), str(p.duration)])
        return buf.getvalue()

    def summary(self) -> dict:
        peaks = peak_memory(self)
        return {
            "makespan": float(self.makespan),
            "bubble": [float(x) for x in bubble_time(self)],
            "peak_units": [u for (u, _b) in peaks["per_device"]],
            "peak_bytes": [b for (_u, b) in peaks["per_device"]],
            "max_peak_units": peaks["max_units"],
            "contention_events": len(self.contention_log),
        }

    def to_json(self) -> str:
        return json.dumps(self.summary(), indent=2)

    def to_pass_lines(self) -> str:
        rows = [
            f"{p.device} {p.stage} {p.microbatch} {p.kind} {_frac_str(p.start)} {_frac_str(p.duration)}"
            for p in sorted(self.passes, key=lambda q: (q.device, q.start, str(q.kind)))
        ]
        return "\n".join(rows) + "\n"


class _CopyStream:
    """One serial transfer queue of a device, in slot order."""

    def __init__(self, device: int, transfers):
        self.device = device
        self.transfers = list(transfers)
        self.known: list = []  # heap of (slot, key, transfer) with scheduled inputs
        self.waiting = len(self.transfers)
        self.running = None
        self.free_at = ZERO


def _copy_streams(plan, mode):
    if plan is None:
        return []
    out = []
    for st in plan.streams:
        if mode == "single":
            groups = [st.transfers]
        elif mode == "dual":
            groups = [
                [t for t in st.transfers if t.direction == PassKind.OFFLOAD],
                [t for t in st.transfers if t.direction == PassKind.RELOAD],
            ]
        else:
            raise ValueError(f"unknown stream mode {mode!r}")
        out.extend(_CopyStream(st.device, g) for g in groups if g)
    return out


class _Runner:
    def __init__(self, sched, plan, t_comm, contention, stream_mode):
        self.sched = sched
        self.t_comm = t_comm
        self.halving = contention.mode == "shared-switch-halving"
        self.contention = contention
        self.orders = [list(d) for d in sched.device_passes]
        self.cursor = [0] * sched.devices
        self.dev_free = [ZERO] * sched.devices
        self.streams = _copy_streams(plan, stream_mode)
        self.start_at: dict = {}
        self.end_at: dict = {}
        self.events: list = []
        self.seq = 0
        self.flow: dict = {}  # key -> [remaining, since, rate, transfer]; insertion = start order
        self.realized: list[Pass] = []
        self.contention_log: list = []
        self.reload_of: dict = {}
        self.offload_of: dict = {}
        self.floor: dict = {}
        self.after: dict = {}
        if plan is not None:
            by_slot = {}
            for stm in self.streams:
                for t in stm.transfers:
                    key = ("T", t.device, t.slot)
                    by_slot[(t.device, t.slot)] = key
                    if t.direction == PassKind.RELOAD:
                        self.reload_of[(t.stage, t.microbatch)] = key
                        self.floor[key] = t.start
                    else:
                        self.offload_of[(t.stage, t.microbatch)] = key
                    if plan.pinned:
                        self.floor[key] = t.start
            for (a, b) in plan.sync_edges:
                ka, kb = by_slot.get(a), by_slot.get(b)
                if ka is not None and kb is not None:
                    self.after.setdefault(kb, []).append(ka)
        # incremental readiness of transfers
        self.t_inputs: dict = {}
        self.t_missing: dict = {}
        self.t_waiters: dict = {}
        self.t_home: dict = {}
        for stm in self.streams:
            for t in stm.transfers:
                key = ("T", t.device, t.slot)
                inputs = self._transfer_inputs(key, t)
                self.t_inputs[key] = inputs
                self.t_home[key] = stm
                missing = [k for k in inputs if k not in self.end_at]
                for k in missing:
                    self.t_waiters.setdefault(k, []).append((key, t))
                self.t_missing[key] = len(missing)
                if not missing:
                    heapq.heappush(stm.known, (t.slot, key, t))

    # -- dependency tables ------------------------------------------------
    def _compute_inputs(self, p: Pass):
        last = self.sched.num_stages - 1
        if p.kind == F:
            return [((F, p.stage - 1, p.microbatch), self.t_comm)] if p.stage > 0 else []
        if p.kind == B:
            deps = []
            if p.stage < last:
                deps.append(((B, p.stage + 1, p.microbatch), self.t_comm))
            deps.append(((F, p.stage, p.microbatch), ZERO))
            rk = self.reload_of.get((p.stage, p.microbatch))
            if rk is not None:
                deps.append((rk, ZERO))
            return deps
        return [((B, p.stage, p.microbatch), ZERO)]

    def _transfer_inputs(self, key, t):
        if t.direction == PassKind.OFFLOAD:
            inputs = [(F, t.stage, t.microbatch)]
        else:
            ok = self.offload_of.get((t.stage, t.microbatch))
            inputs = [ok] if ok is not None else []
        return inputs + list(self.after.get(key, ()))

    def _ready_time(self, deps):
        t = ZERO
        for key, lag in deps:
            e = self.end_at.get(key)
            if e is None:
                return None
            t = max(t, e + lag)
        return t

    # -- event plumbing ---------------------------------------------------
    def wake(self, t: Fraction):
        heapq.heappush(self.events, (t, self.seq))
        self.seq += 1

    def scheduled(self, key):
        for (tkey, t) in self.t_waiters.get(key, ()):
            self.t_missing[tkey] -= 1
            if self.t_missing[tkey] == 0:
                heapq.heappush(self.t_home[tkey].known, (t.slot, tkey, t))

    def rate_for(self, t, peers):
        if not self.halving:
            return Fraction(1)
        sw = self.contention.switch_of(t.device)
        shared = any(o is not t and o.direction == t.direction and self.contention.switch_of(o.device) == sw for o in peers)
        duplex = any(o is not t and o.device == t.device and o.direction != t.direction for o in peers)
        return Fraction(1, (2 if shared else 1) * (2 if duplex else 1))

    def retune(self, now):
        peers = [st[3] for st in self.flow.values()]
        for st in self.flow.values():
            left, since, rate, t = st
            new = self.rate_for(t, peers)
            if new != rate:
                if now > since:
                    if rate < 1:
                        self.contention_log.append((since, now, t.device, str(t.direction), rate))
                    left -= rate * (now - since)
                st[0], st[1], st[2] = left, now, new
                self.wake(now + left / new)
            elif since == now and left == t.duration:
                self.wake(now + left / new)

    def complete(self, now):
        done = [k for k, st in self.flow.items() if st[0] - st[2] * (now - st[1]) <= 0]
        for k in done:
            _left, since, rate, t = self.flow.pop(k)
            if rate < 1 and now > since:
                self.contention_log.append((since, now, t.device, str(t.direction), rate))
            self.end_at[k] = now
            self.scheduled(k)
            self.realized.append(Pass(t.direction, t.device, t.stage, t.microbatch, self.start_at[k], now - self.start_at[k]))

    # -- per-instant starts -------------------------------------------------
    def start_compute(self, now) -> bool:
        began = False
        for dev in range(self.sched.devices):
            order = self.orders[dev]
            while self.cursor[dev] < len(order):
                p = order[self.cursor[dev]]
                ready = self._ready_time(self._compute_inputs(p))
                if ready is None:
                    break
                when = max(ready, self.dev_free[dev])
                if when > now:
                    self.wake(when)
                    break
                key = (p.kind, p.stage, p.microbatch)
                self.start_at[key] = now
                self.end_at[key] = now + p.duration
                self.scheduled(key)
                self.dev_free[dev] = self.end_at[key]
                self.realized.append(Pass(p.kind, p.device, p.stage, p.microbatch, now, p.duration))
                self.wake(self.end_at[key])
                self.cursor[dev] += 1
                began = True
        return began

    def start_transfers(self, now) -> bool:
        began = False
        for stm in self.streams:
            if stm.running is not None or not stm.known:
                continue
            slot, key, t = stm.known[0]
            when = max(self._ready_time([(k, ZERO) for k in self.t_inputs[key]]), stm.free_at, self.floor.get(key, ZERO))
            if when > now:
                self.wake(when)
                continue
            heapq.heappop(stm.known)
            self.start_at[key] = now
            self.flow[key] = [t.duration, now, Fraction(1), t]
            stm.running = key
            stm.waiting -= 1
            began = True
        return began

    def run(self):
        total = sum(len(o) for o in self.orders) + sum(len(s.transfers) for s in self.streams)
        begun = 0
        now = ZERO
        while True:
            for stm in self.streams:
                if stm.running is not None and stm.running in self.end_at:
                    stm.free_at = self.end_at[stm.running]
                    stm.running = None
            moved_transfer = False
            while True:
                before = len(self.start_at)
                self.start_compute(now)
                if self.start_transfers(now):
                    moved_transfer = True
                if len(self.start_at) == before:
                    break
            begun = len(self.start_at)
            if moved_transfer and self.flow:
                self.retune(now)
            if begun >= total and not self.flow:
                break
            while self.events and self.events[0][0] <= now:
                heapq.heappop(self.events)
            if not self.events:
                raise self._deadlock()
            now = heapq.heappop(self.events)[0]
            self.complete(now)
            if self.flow:
                self.retune(now)

    # -- diagnostics --------------------------------------------------------
    def _deadlock(self) -> DeadlockError:
        heads = {}
        where = {}
        for dev, order in enumerate(self.orders):
            for p in order:
                where[(p.kind, p.stage, p.microbatch)] = dev
            if self.cursor[dev] < len(order):
                p = order[self.cursor[dev]]
                heads[dev] = p
        cycle = ()
        if heads:
            path, seen = [], {}
            p = next(iter(heads.values()))
            while p is not None:
                key = (p.kind, p.stage, p.microbatch)
                if key in seen:
                    cycle = tuple(path[seen[key]:])
                    break
                seen[key] = len(path)
                path.append(key)
                missing = [k for k, _lag in self._compute_inputs(p) if k not in self.end_at]
                if not missing or missing[0] not in where:
                    break
                p = heads.get(where[missing[0]])
        stuck = [(str(p.kind), p.stage, p.microbatch) for p in heads.values()]
        for stm in self.streams:
            if stm.waiting > 0 and stm.known:
                t = stm.known[0][2]
                stuck.append((str(t.direction), t.stage, t.microbatch))
            elif stm.waiting > 0:
                stuck.append((f"stream[{stm.device}]", stm.waiting, "unscheduled-inputs"))
        report = cycle or tuple(stuck)
        return DeadlockError(f"no runnable passes; wait cycle: {list(report)}", report)


def _residency(sched, starts, ends, reload_of, offload_of):
    units = sched.units_per_stage
    dev_events = [[] for _ in range(sched.devices)]
    host = []
    moved = set(reload_of) & set(offload_of)
    for dev in range(sched.devices):
        for p in sched.device_passes[dev]:
            pair = (p.stage, p.microbatch)
            if p.kind == F:
                dev_events[dev].append((starts[(F, p.stage, p.microbatch)], p.stage, units))
                if pair in moved:
                    out_end = ends[offload_of[pair]]
                    back_start = starts[reload_of[pair]]
                    dev_events[dev] += [(out_end, p.stage, -units), (back_start, p.stage, units)]
                    host += [(out_end, dev, units), (ends[reload_of[pair]], dev, -units)]
            elif p.kind == B:
                dev_events[dev].append((ends[(B, p.stage, p.microbatch)], p.stage, -units))
    order = lambda e: (e[0], e[2])  # noqa: E731 - frees before allocs at equal times
    return tuple(tuple(sorted(ev, key=order)) for ev in dev_events), sorted(host, key=order)


def simulate(
    sched: Schedule,
    plan: OffloadPlan | None = None,
    costs: PassCosts | None = None,
    hw=None,
    contention: ContentionModel | None = None,
    model: ModelSpec | None = None,
    stream_mode: str = "single",
) -> SimTrace:
    """Model one iteration of ``sched`` with ``plan`` (reference sim.py:141-413)."""
    costs = costs or sched.costs
    if contention is None:
        contention = ContentionModel("none", hw.devices_per_switch if hw is not None else 2)
    run = _Runner(sched, plan, costs.t_comm, contention, stream_mode)
    run.run()
    per_unit = 0
    if model is not None:
        per_unit = activation_bytes_per_layer(model, recompute=True) * model.layers_per_stage
    dev_events, host = _residency(sched, run.start_at, run.end_at, run.reload_of, run.offload_of)
    return SimTrace(
        schedule=sched,
        passes=tuple(sorted(run.realized, key=lambda p: (p.start, p.device, str(p.kind), p.stage, p.microbatch))),
        makespan=max(run.end_at.values(), default=ZERO),
        device_busy=tuple(sched.busy(i) for i in range(sched.devices)),
        memory=MemoryTimeline(devices=sched.devices, bytes_per_unit=per_unit, events=dev_events),
        host_events=tuple(host),
        contention_log=tuple(run.contention_log),
        bytes_per_unit=per_unit,
    )


def bubble_time(trace: SimTrace) -> tuple[Fraction, ...]:
    return tuple(trace.makespan - busy for busy in trace.device_busy)


def peak_memory(trace: SimTrace) -> dict:
    per_device = []
    for dev in range(trace.schedule.devices):
        u = trace.memory.peak(dev)
        per_device.append((u, u * trace.bytes_per_unit))
    top = max((u for u, _ in per_device), default=0)
    return {"per_device": per_device, "max_units": top, "max_bytes": top * trace.bytes_per_unit}


def host_peak_memory(trace: SimTrace, assignment: NodeAssignment | None = None) -> list:
    if assignment is None:
        assignment = NodeAssignment(1, tuple(0 for _ in range(trace.schedule.devices)))
    level = [0] * assignment.num_nodes
    peak = [0] * assignment.num_nodes
    for (_t, rank, delta) in sorted(trace.host_events, key=lambda e: (e[0], e[2])):
        node = assignment.node_of[rank]
        level[node] += delta
        peak[node] = max(peak[node], level[node])
    scale = trace.bytes_per_unit or 1
    return [p * scale for p in peak]
