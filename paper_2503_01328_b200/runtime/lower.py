"""Lower (Schedule, OffloadPlan, rank) into a static, event-anchored program.

The reference runner is a clock-driven simulation (pkg/src/ppoff/sim.py:141-413):
reloads are floored at absolute slot times (sim.py:177-181) and memory is freed
at D2H end (sim.py:477-479).  A GPU only knows streams and events, so lowering
turns every time relation into an event relation, using the runner model of
this package (``sim.simulate``, bit-exact with the reference) as the witness
timeline:

* compute stream  -- F/B passes in ``Schedule.device_passes`` order (op-order
  parity: the executed order IS the reference's order).
* copy stream(s)  -- OFFLOAD/RELOAD in the order the runner model realises them,
  which equals ``OffloadPlan.streams[d].transfers`` slot order whenever the plan
  has no late reloads; ``stream_mode="dual"`` splits D2H and H2D.
* reload anchors  -- a RELOAD waits for the start event of the compute pass that
  is running at its realised start (or the end event of the last pass that
  finished before it): the event form of the slot floor.
* device slabs    -- a fixed arena of K slabs, K = the realised peak residency;
  each (stage, mb) residency interval gets a slab by greedy interval colouring
  and waits for the release event (D2H done or B end) of the slab's previous
  occupant, so the arena can never exceed the planned peak.
* host slots      -- the same for pinned host bins over [D2H start, H2D end).
* stage boundary  -- RECV/SEND ops on per-edge channels (2-rank NCCL comms in
  the multi-process runtime); activations and gradients are staged through
  rings of R buffers so a send never waits on the consumer's compute.

Every wait points to an event whose witness time is <= the waiter's, so the
wait graph is acyclic; ``host_order`` topologically sorts all ops so every event
is recorded on the host before any stream is told to wait for it.
"""

from __future__ import annotations

import heapq
from dataclasses import dataclass, field
from fractions import Fraction

from ..offload import OffloadPlan
from ..schedule_types import PassKind, Schedule
from ..sim import simulate

F, B, W = PassKind.F, PassKind.B, PassKind.W
OFF, REL = PassKind.OFFLOAD, PassKind.RELOAD

RING = 2  # boundary buffers per channel direction


@dataclass
class Op:
    kind: str  # F B RECV_ACT SEND_ACT RECV_GRAD SEND_GRAD OFFLOAD RELOAD
    stage: int
    mb: int
    stream: str  # compute | copy | copy_h2d | recv_act | send_act | recv_grad | send_grad
    t: Fraction  # witness (modelled) issue time
    waits: list = field(default_factory=list)
    records: list = field(default_factory=list)
    slab: int | None = None
    res_slab: int | None = None  # resident-part slot (partial offload; = in-flight colouring)
    host_slot: int | None = None
    ring: int | None = None
    peer: int | None = None  # remote rank of a boundary op
    anchor: tuple | None = None  # reload anchor event
    send_ring: int | None = None  # ring slot of the boundary send this compute op feeds
    wbuf: int | None = None  # split backward: gradient buffer shared by a B and its W
    # topology-synchronised plans (OffloadPlan.sync_edges): flags this transfer waits for
    # before it starts / raises when it is done (index into the plan's sync_edges)
    flag_waits: list = field(default_factory=list)
    signals: list = field(default_factory=list)

    @property
    def key(self):
        return (self.kind, self.stage, self.mb)


@dataclass
class Program:
    rank: int
    devices: int
    ops: list  # host issue order
    n_slabs: int
    n_host_slots: int
    n_res_slabs: int
    n_wbufs: int
    offloaded: set
    witness_makespan: Fraction
    witness_peak_units: int
    compute_order: list  # [(kind, stage, mb)] == sched.device_passes[rank]
    copy_order: dict  # stream -> [(kind, stage, mb)]
    recv_orders: dict  # channel -> [(stage, mb)]
    send_orders: dict
    n_flags: int = 0  # len(plan.sync_edges): the flag board every rank of the run shares

    def ops_on(self, stream: str):
        return [op for op in self.ops if op.stream == stream]


def _colour(intervals, spare: int = 0):
    """Greedy interval colouring. intervals: list of (start, end, key).

    Frees sort before allocations at equal times (half-open residency, as in
    ir.py:649).  A new interval takes the colour that has been free the longest
    (LRU), so the release event it waits on is as old as possible: on the GPU the
    compute stream can run ahead of the witness timeline (an emulated rank has no
    pipeline bubbles) and a just-freed slab would stall it.  Greedy colouring uses
    max-overlap colours whatever free colour it picks.  ``spare`` extra colours widen
    the LRU choice (every acquirer then waits on a release at least one holder older):
    memory traded for slack against transfers that run slower than modelled.  Returns
    (assignment key -> (colour, previous occupant key or None), n_colours).
    """
    if spare:
        _, n0 = _colour(intervals)
        return _colour_fixed(intervals, n0 + spare), n0 + spare
    return _colour_fixed(intervals, None)


def _colour_fixed(intervals, n_fixed):
    """LRU greedy colouring; with ``n_fixed`` all colours exist up front (free, in
    index order), else they are created on demand.  Returns (assignment, n) or, with
    n_fixed, the assignment alone."""
    events = []
    for start, end, key in intervals:
        events.append((start, 1, key))
        events.append((end, 0, key))
    events.sort(key=lambda e: (e[0], e[1]))
    free: list = [(i - n_fixed, i) for i in range(n_fixed)] if n_fixed else []  # heap of (release order, colour)
    last_holder: dict = {}
    held: dict = {}
    assignment = {}
    n = n_fixed or 0
    order = 0
    for _t, is_alloc, key in events:
        if is_alloc:
            if free:
                _, c = heapq.heappop(free)
            else:
                assert n_fixed is None, "fixed colouring ran out of colours"
                c = n
                n += 1
            assignment[key] = (c, last_holder.get(c))
            held[key] = c
        else:
            c = held.pop(key)
            last_holder[c] = key
            heapq.heappush(free, (order, c))
            order += 1
    return assignment if n_fixed else (assignment, n)


def _anchor_for(t: Fraction, passes):
    """Event that marks witness time t on a device's compute stream."""
    before = None
    for p in passes:
        if p.start <= t < p.end:
            return ("start", p.kind, p.stage, p.microbatch)
        if p.end <= t:
            before = p
    if before is not None:
        return ("end", before.kind, before.stage, before.microbatch)
    return None


def lower(
    sched: Schedule,
    plan: OffloadPlan | None,
    rank: int,
    stream_mode: str = "single",
    emulate_neighbors: bool = False,
    spare_slabs: int = 0,
) -> Program:
    """Per-rank program.  ``emulate_neighbors`` drops cross-rank ops (the rank runs
    alone with a loopback stage boundary, e.g. the single-GPU bench of one rank
    of a PP=d schedule).  ``spare_slabs`` adds that many slabs to the offload arena
    beyond the modelled peak (see ``_colour``)."""
    trace = simulate(sched, plan, stream_mode=stream_mode)
    timed = {(p.kind, p.stage, p.microbatch): p for p in trace.passes}
    my_passes = [timed[(p.kind, p.stage, p.microbatch)] for p in sched.device_passes[rank]]
    split = sched.split_backward
    # with a split backward the W pass still reads the slab (and the B pass's gradient
    # buffer): residency ends at W end (the reference's model frees at B end, ir.py:630-655)
    last_use = W if split else B
    placement = sched.placement
    last_stage = sched.num_stages - 1
    ops: list[Op] = []

    transfers = sorted((p for p in trace.transfer_passes() if p.device == rank), key=lambda p: (p.start, p.kind != OFF))
    offloaded = {(p.stage, p.microbatch) for p in transfers if p.kind == REL}
    d2h = {(p.stage, p.microbatch): p for p in transfers if p.kind == OFF}
    h2d = {(p.stage, p.microbatch): p for p in transfers if p.kind == REL}
    # a pair offloaded but never reloaded (cannot happen with plan_slots) is not supported
    assert set(d2h) >= offloaded

    # ---------------------------------------------------------------- slabs
    intervals = []
    for p in my_passes:
        pair = (p.stage, p.microbatch)
        if p.kind == F:
            done = timed[(last_use, p.stage, p.microbatch)].end
            end = d2h[pair].end if pair in offloaded else done
            intervals.append((p.start, end, ("F",) + pair))
            if pair in offloaded:
                intervals.append((h2d[pair].start, done, ("R",) + pair))
    slab_of, n_slabs = _colour(intervals, spare=spare_slabs if offloaded else 0)
    # resident part of every slab (partial offload keeps it on the device from F start
    # to the pair's last use, offloaded or not): colours = the in-flight peak
    res_of, n_res = _colour([(p.start, timed[(last_use, p.stage, p.microbatch)].end, ("P", p.stage, p.microbatch))
                             for p in my_passes if p.kind == F])
    wbuf_of, n_wbufs = _colour([(timed[(B,) + pr].start, timed[(W,) + pr].end, ("G",) + pr)
                                for pr in ((p.stage, p.microbatch) for p in my_passes if p.kind == B)]) if split else ({}, 0)
    host_of, n_host = _colour([(d2h[pr].start, h2d[pr].end, ("H",) + pr) for pr in sorted(offloaded)])

    def release_event(holder):
        """Event that frees a slab held by ``holder`` (("F"|"R", stage, mb))."""
        if holder is None:
            return None
        tag, s, j = holder
        if tag == "F" and (s, j) in offloaded:
            return ("D2H", s, j)
        return (f"{last_use}_end", s, j)

    # --------------------------------------------------------- boundary rings
    recv_orders: dict = {}
    send_orders: dict = {}

    def consumer_of(channel, idx):
        """Event after which ring slot of the idx-th message on channel is free."""
        prev = idx - RING
        if prev < 0:
            return None
        s, j = recv_orders[channel][prev]
        return ("F_in", s, j) if channel[0] == "act" else ("B_end", s, j)

    compute_ops = []
    for p in my_passes:
        s, j = p.stage, p.microbatch
        pair = (s, j)
        if p.kind == F:
            op = Op("F", s, j, "compute", p.start)
            op.records = [("F_start", s, j), ("F_in", s, j), ("F_end", s, j)]
            op.slab, prev = slab_of[("F",) + pair]
            rel = release_event(prev)
            if rel:
                op.waits.append(rel)
            op.res_slab, prev_res = res_of[("P",) + pair]
            if prev_res is not None and (f"{last_use}_end",) + prev_res[1:] != rel:
                op.waits.append((f"{last_use}_end",) + prev_res[1:])
            if s > 0:
                src = placement[s - 1]
                # consecutive stages on one device (d=1, v>1) hand off through a local
                # channel of the same rank (peer == rank), not through the transport
                if not emulate_neighbors or src == rank:
                    ch = ("act", src, rank)
                    lst = recv_orders.setdefault(ch, [])
                    lst.append(pair)
                    idx = len(lst) - 1
                    r = Op("RECV_ACT", s, j, "recv_act", p.start, ring=idx % RING, peer=src)
                    cons = consumer_of(ch, idx)
                    if cons:
                        r.waits.append(cons)
                    r.records = [("RA", s, j)]
                    ops.append(r)
                    op.waits.append(("RA", s, j))
                    op.ring = r.ring
            compute_ops.append(op)
            if s < last_stage:
                dst = placement[s + 1]
                if not emulate_neighbors or dst == rank:
                    ch = ("act", rank, dst)
                    lst = send_orders.setdefault(ch, [])
                    lst.append(pair)
                    idx = len(lst) - 1
                    snd = Op("SEND_ACT", s, j, "send_act", p.end, ring=idx % RING, peer=dst)
                    snd.waits = [("F_end", s, j)]
                    snd.records = [("SA", s, j)]
                    if idx >= RING:
                        ps, pj = lst[idx - RING]
                        op.waits.append(("SA", ps, pj))  # F may overwrite this send buffer
                    op.send_ring = snd.ring
                    ops.append(snd)
        elif p.kind == W:
            op = Op("W", s, j, "compute", p.start)
            op.records = [("W_start", s, j), ("W_end", s, j)]
            op.slab = slab_of[(("R",) if pair in offloaded else ("F",)) + pair][0]
            op.res_slab = res_of[("P",) + pair][0]
            op.wbuf = wbuf_of[("G",) + pair][0]
            compute_ops.append(op)
            continue
        else:  # B
            op = Op("B", s, j, "compute", p.start)
            op.records = [("B_start", s, j), ("B_end", s, j)]
            if pair in offloaded:
                op.waits.append(("H2D", s, j))
                op.slab = slab_of[("R",) + pair][0]
            else:
                op.slab = slab_of[("F",) + pair][0]
            op.res_slab = res_of[("P",) + pair][0]
            if split:
                op.wbuf = wbuf_of[("G",) + pair][0]
            if s < last_stage:
                src = placement[s + 1]
                if not emulate_neighbors or src == rank:
                    ch = ("grad", src, rank)
                    lst = recv_orders.setdefault(ch, [])
                    lst.append(pair)
                    idx = len(lst) - 1
                    r = Op("RECV_GRAD", s, j, "recv_grad", p.start, ring=idx % RING, peer=src)
                    cons = consumer_of(ch, idx)
                    if cons:
                        r.waits.append(cons)
                    r.records = [("RG", s, j)]
                    ops.append(r)
                    op.waits.append(("RG", s, j))
                    op.ring = r.ring
            if s > 0:
                dst = placement[s - 1]
                if not emulate_neighbors or dst == rank:
                    ch = ("grad", rank, dst)
                    lst = send_orders.setdefault(ch, [])
                    lst.append(pair)
                    idx = len(lst) - 1
                    snd = Op("SEND_GRAD", s, j, "send_grad", p.end, ring=idx % RING, peer=dst)
                    snd.waits = [("B_end", s, j)]
                    snd.records = [("SG", s, j)]
                    if idx >= RING:
                        ps, pj = lst[idx - RING]
                        op.waits.append(("SG", ps, pj))
                    op.send_ring = snd.ring
                    ops.append(snd)
            compute_ops.append(op)
    ops.extend(compute_ops)

    # ------------------------------------------------------ sync edges / pinned
    # A topology-synchronised plan (offload.py:223-248) orders transfers of paired
    # devices: edge (a -> b) makes transfer b wait for the end of transfer a
    # (sim.py:186-189).  Same-rank edges are event waits; cross-rank edges are flags
    # (executor FlagBoard); with emulated neighbours the cross-rank ones are dropped.
    # A pinned plan also floors every transfer at its slot start (sim.py:184-185).
    flag_wait_of: dict = {}
    signal_of: dict = {}
    local_after: dict = {}
    if plan is not None and plan.sync_edges:
        by_slot = {(t.device, t.slot): t for stm in plan.streams for t in stm.transfers}
        tag = lambda t: ("OFFLOAD" if t.direction == OFF else "RELOAD", t.stage, t.microbatch)  # noqa: E731
        for idx, (a, b) in enumerate(plan.sync_edges):
            ta, tb = by_slot.get(a), by_slot.get(b)
            if ta is None or tb is None:
                continue
            if ta.device == rank and tb.device == rank:
                local_after.setdefault(tag(tb), []).append(tag(ta))
            elif emulate_neighbors:
                continue
            elif ta.device == rank:
                signal_of.setdefault(tag(ta), []).append(idx)
            elif tb.device == rank:
                flag_wait_of.setdefault(tag(tb), []).append(idx)
    pinned = plan is not None and plan.pinned

    # ------------------------------------------------------------- transfers
    copy_order: dict = {}
    for p in transfers:
        s, j = p.stage, p.microbatch
        pair = (s, j)
        if p.kind == OFF:
            stream = "copy"
            op = Op("OFFLOAD", s, j, stream, p.start)
            op.waits = [("F_end", s, j)]
            op.records = [("D2H", s, j)]
            op.slab = slab_of[("F",) + pair][0]
            op.host_slot, prev = host_of[("H",) + pair]
            if prev is not None:
                op.waits.append(("H2D", prev[1], prev[2]))
        else:
            stream = "copy" if stream_mode == "single" else "copy_h2d"
            op = Op("RELOAD", s, j, stream, p.start)
            op.slab, prev = slab_of[("R",) + pair]
            op.host_slot = host_of[("H",) + pair][0]
            op.waits = [("D2H", s, j)]
            rel = release_event(prev)
            if rel:
                op.waits.append(rel)
            anc = _anchor_for(p.start, my_passes)
            if anc is not None:
                which, kind, as_, aj = anc
                op.anchor = ((f"{kind}_start" if which == "start" else f"{kind}_end"), as_, aj)
                op.waits.append(op.anchor)
            op.records = [("H2D", s, j)]
        if pinned and op.kind == "OFFLOAD":  # floor at the slot start: anchor like a reload
            anc = _anchor_for(p.start, my_passes)
            if anc is not None:
                which, kind, as_, aj = anc
                op.anchor = ((f"{kind}_start" if which == "start" else f"{kind}_end"), as_, aj)
                if op.anchor != ("F_end", s, j):
                    op.waits.append(op.anchor)
        for k_, s_, j_ in local_after.get((op.kind, s, j), ()):
            op.waits.append(("D2H" if k_ == "OFFLOAD" else "H2D", s_, j_))
        op.flag_waits = list(flag_wait_of.get((op.kind, s, j), ()))
        op.signals = list(signal_of.get((op.kind, s, j), ()))
        copy_order.setdefault(stream, []).append((op.kind, s, j))
        ops.append(op)

    ordered = host_order(ops)
    # sanity: compute order is exactly the schedule's device order
    got = [(op.kind, op.stage, op.mb) for op in ordered if op.stream == "compute"]
    want = [(str(p.kind), p.stage, p.microbatch) for p in sched.device_passes[rank]]
    assert got == want, "lowering changed the per-device op order"
    peak = trace.memory.peak(rank)
    return Program(
        rank=rank, devices=sched.devices, ops=ordered, n_slabs=n_slabs, n_host_slots=n_host, n_res_slabs=n_res,
        n_wbufs=n_wbufs,
        offloaded=offloaded, witness_makespan=trace.makespan, witness_peak_units=peak,
        compute_order=want, copy_order=copy_order, recv_orders=recv_orders, send_orders=send_orders,
        n_flags=len(plan.sync_edges) if plan is not None else 0,
    )


_KIND_PRIORITY = {"OFFLOAD": 0, "RELOAD": 1, "SEND_ACT": 2, "SEND_GRAD": 2, "RECV_ACT": 3, "RECV_GRAD": 3, "F": 4, "B": 4, "W": 4}


def host_order(ops: list[Op]) -> list[Op]:
    """Topological order: stream FIFO order + record-before-wait, earliest witness time first."""
    producers = {}
    for i, op in enumerate(ops):
        for ev in op.records:
            producers[ev] = i
    succ = [[] for _ in ops]
    indeg = [0] * len(ops)
    last_on = {}
    order_in_stream = sorted(range(len(ops)), key=lambda i: (ops[i].stream, _stream_rank(ops, i)))
    for i in order_in_stream:
        st = ops[i].stream
        if st in last_on:
            succ[last_on[st]].append(i)
            indeg[i] += 1
        last_on[st] = i
    for i, op in enumerate(ops):
        for ev in op.waits:
            j = producers.get(ev)
            if j is None:
                raise ValueError(f"{op.key} waits on {ev} that no op records")
            if j != i:
                succ[j].append(i)
                indeg[i] += 1
    heap = [(ops[i].t, _KIND_PRIORITY[ops[i].kind], i) for i in range(len(ops)) if indeg[i] == 0]
    heapq.heapify(heap)
    out = []
    while heap:
        _t, _k, i = heapq.heappop(heap)
        out.append(ops[i])
        for k in succ[i]:
            indeg[k] -= 1
            if indeg[k] == 0:
                heapq.heappush(heap, (ops[k].t, _KIND_PRIORITY[ops[k].kind], k))
    if len(out) != len(ops):
        stuck = [ops[i].key for i in range(len(ops)) if indeg[i] > 0][:8]
        raise RuntimeError(f"lowered program has a wait cycle near {stuck}")
    return out


def _stream_rank(ops, i):
    """Position of op i within its stream: insertion order (already stream order)."""
    return i
