"""Lowered programs executed on CPU stand-ins: slab / host-slot reuse, boundary
matching and deadlock freedom of the per-rank programs (``runtime.lower``).

``CpuWalker`` executes one rank's ops strictly in host issue order, the order the
GPU runner enqueues them; because every wait in a program points to an event
recorded earlier in host order, this sequential walk is a valid linearisation of
the GPU run.  Activations are tagged integers: F writes its (stage, mb) tag into
its slab, OFFLOAD/RELOAD move it through the host slot, and B checks it finds its
own tag -- so any two live pairs sharing a slab or host slot, or any reload into
the wrong slab, fails.  Boundary messages carry values through the stages so the
final input gradient on stage 0 checks the routing end to end.

The world-size-2 test runs the same walker in two processes over gloo (N>1 host
path); the single-process tests drive all ranks through in-memory channels.
"""

from __future__ import annotations

import os
from collections import deque
from fractions import Fraction

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2503_01328_b200 as po
from paper_2503_01328_b200.runtime.lower import lower


class Blocked(Exception):
    pass


class CpuWalker:
    def __init__(self, sched, prog, channel):
        self.sched, self.prog, self.channel = sched, prog, channel
        self.slabs = [None] * max(1, prog.n_slabs)
        self.res = [None] * max(1, prog.n_res_slabs)  # resident parts (partial offload)
        self.host = [None] * max(1, prog.n_host_slots)
        self.rings = {k: [None] * 2 for k in ("recv_act", "send_act", "recv_grad", "send_grad")}
        self.cursor = 0
        self.grad_out = {}  # (stage, mb) -> input gradient produced by B
        self.live = set()
        self.wbufs = {}

    def done(self):
        return self.cursor >= len(self.prog.ops)

    board = None  # sync-edge flags shared by all walkers of a run (set by run_all_ranks)
    done_order = None  # global completion order of transfers: [(rank, kind, stage, mb)]

    def step(self):
        op = self.prog.ops[self.cursor]
        last = self.sched.num_stages - 1
        pair = (op.stage, op.mb)
        if op.flag_waits:
            if not all(self.board.get(f) for f in op.flag_waits):
                raise Blocked()
            for f in op.flag_waits:
                self.board[f] = False
        if op.kind in ("OFFLOAD", "RELOAD") and self.done_order is not None:
            self.done_order.append((self.prog.rank, op.kind, op.stage, op.mb))
        if op.kind == "F":
            x = float(op.mb) if op.stage == 0 else self.rings["recv_act"][op.ring]
            if x is None:
                raise AssertionError(f"F{pair} found no received activation")
            assert self.slabs[op.slab] is None or self.slabs[op.slab][0] not in self.live, "slab still live"
            self.slabs[op.slab] = (pair, x)
            self.live.add(pair)
            assert self.res[op.res_slab] is None, f"resident slot of F{pair} still held by {self.res[op.res_slab]}"
            self.res[op.res_slab] = pair
            y = x + 1.0
            if op.stage < last and op.send_ring is not None:
                self.rings["send_act"][op.send_ring] = y
        elif op.kind == "OFFLOAD":
            assert self.slabs[op.slab][0] == pair, f"D2H of {pair} found {self.slabs[op.slab][0]}"
            self.host[op.host_slot] = self.slabs[op.slab]
            self.live.discard(pair)
            self.slabs[op.slab] = None
        elif op.kind == "RELOAD":
            assert self.host[op.host_slot][0] == pair, f"H2D of {pair} found {self.host[op.host_slot][0]}"
            assert self.slabs[op.slab] is None or self.slabs[op.slab][0] not in self.live
            self.slabs[op.slab] = self.host[op.host_slot]
            self.live.add(pair)
        elif op.kind == "B":
            tag, x = self.slabs[op.slab]
            assert tag == pair, f"B{pair} found slab holding {tag}"
            assert self.res[op.res_slab] == pair, f"B{pair} found resident slot holding {self.res[op.res_slab]}"
            g = x + 1.0 if op.stage == last else self.rings["recv_grad"][op.ring]
            gx = 2.0 * g
            self.grad_out[pair] = gx
            if self.sched.split_backward:
                assert self.wbufs.get(op.wbuf) is None, "gradient buffer still in use"
                self.wbufs[op.wbuf] = pair
            else:
                self.live.discard(pair)
                self.slabs[op.slab] = None
                self.res[op.res_slab] = None
            if op.stage > 0 and op.send_ring is not None:
                self.rings["send_grad"][op.send_ring] = gx
        elif op.kind == "W":
            assert self.slabs[op.slab][0] == pair, f"W{pair} found slab holding {self.slabs[op.slab][0]}"
            assert self.wbufs.get(op.wbuf) == pair, f"W{pair} found gradient buffer of {self.wbufs.get(op.wbuf)}"
            assert self.res[op.res_slab] == pair, f"W{pair} found resident slot holding {self.res[op.res_slab]}"
            self.wbufs[op.wbuf] = None
            self.live.discard(pair)
            self.slabs[op.slab] = None
            self.res[op.res_slab] = None
        elif op.kind in ("SEND_ACT", "SEND_GRAD"):
            ring = "send_act" if op.kind == "SEND_ACT" else "send_grad"
            self.channel.send(op, self.rings[ring][op.ring])
        elif op.kind in ("RECV_ACT", "RECV_GRAD"):
            val = self.channel.recv(op)
            self.rings["recv_act" if op.kind == "RECV_ACT" else "recv_grad"][op.ring] = val
        else:  # pragma: no cover
            raise ValueError(op.kind)
        for f in op.signals:
            self.board[f] = True
        self.cursor += 1


class LocalChannels:
    def __init__(self):
        self.q = {}

    def bind(self, rank):
        outer = self

        class Bound:
            def send(self, op, val):
                outer.q.setdefault((op.kind[5:], rank, op.peer), deque()).append(((op.stage, op.mb), val))

            def recv(self, op):
                dq = outer.q.get((op.kind[5:], op.peer, rank))
                if not dq:
                    raise Blocked()
                (s, j), val = dq.popleft()
                want = (op.stage - 1, op.mb) if op.kind == "RECV_ACT" else (op.stage + 1, op.mb)
                assert (s, j) == want, f"{op.kind} {op.stage, op.mb} got message of {s, j}"
                return val

        return Bound()


def run_all_ranks(sched, plan, stream_mode="single", spare_slabs=0):
    chans = LocalChannels()
    walkers = [CpuWalker(sched, lower(sched, plan, r, stream_mode=stream_mode, spare_slabs=spare_slabs), chans.bind(r))
               for r in range(sched.devices)]
    board, order = {}, []
    for w in walkers:
        w.board, w.done_order = board, order
    while not all(w.done() for w in walkers):
        progressed = False
        for w in walkers:
            while not w.done():
                try:
                    w.step()
                    progressed = True
                except Blocked:
                    break
        assert progressed, "lowered programs deadlock"
    return walkers


def expected_input_grad(sched, mb):
    s = sched.num_stages
    return (mb + s) * 2.0 ** s


U = po.PassCosts.unit()
CASES = [
    ("1f1b d4 full k=1/2", lambda: po.build_1f1b_full_offload(4, 8, U, Fraction(3, 2))),
    ("1f1b d8 full k=1", lambda: po.build_1f1b_full_offload(8, 32, U, Fraction(3))),
    ("1f1b d8 full k=2 (late reloads)", lambda: po.build_1f1b_full_offload(8, 32, U, Fraction(6))),
    ("1f1b d8 v3 real costs", lambda: (lambda s: (s, po.plan_slots(s, (0,), Fraction(18000))))(po.build_1f1b(8, 3, 32, po.PassCosts(1650, 3350, 0, 40)))),
    ("1f1b-i d4 v2 n1", lambda: (lambda s: (s, po.plan_slots(s, po.select_offload_stages(po.po_block(4, 2, U), 1), Fraction(1))))(po.build_interleaved_1f1b(4, 2, 8, U))),
    ("1f1b-i d8 v4 n2", lambda: (lambda s: (s, po.plan_slots(s, po.select_offload_stages(po.po_block(8, 4, U), 2), Fraction(3, 2))))(po.build_interleaved_1f1b(8, 4, 16, U))),
    ("1f1b d4 no offload", lambda: (po.build_1f1b(4, 1, 8, U), None)),
    ("gis d4 v2 n1 (split W)", lambda: (lambda s: (s, po.plan_slots(s, po.select_offload_stages(po.po_block(4, 2, U), 1), Fraction(1))))(po.build_gis(4, 2, 8, U))),
    ("gis-h d8 v2 n1 (split W)", lambda: (lambda s: (s, po.plan_slots(s, po.select_offload_stages(po.po_block(8, 2, U), 1), Fraction(3, 2))))(po.build_gis_h(8, 2, 16, U))),
    ("po d8 v2 n2 (split W)", lambda: (lambda s: (s, po.plan_slots(s, po.select_offload_stages(po.po_block(8, 2, U), 2), Fraction(3))))(po.build_po(8, 2, 16, U))),
    # d = 1 with v > 1: consecutive stages on one device hand off through a local channel
    ("1f1b-i d1 v2 no offload", lambda: (po.build_interleaved_1f1b(1, 2, 4, U), None)),
    ("gis d1 v2 n1 (split W)", lambda: (lambda s: (s, po.plan_slots(s, po.select_offload_stages(po.po_block(1, 2, U), 1), Fraction(1))))(po.build_gis_h(1, 2, 4, U))),
    ("po d1 v3 (split W)", lambda: (po.build_po(1, 3, 4, U), None)),
]


@pytest.mark.parametrize("name,make", CASES, ids=[c[0] for c in CASES])
@pytest.mark.parametrize("stream_mode", ["single", "dual"])
def test_lowered_programs_execute_correctly(name, make, stream_mode):
    sched, plan = make()
    walkers = run_all_ranks(sched, plan, stream_mode)
    for j in range(sched.microbatches):
        assert walkers[0].grad_out[(0, j)] == expected_input_grad(sched, j)
    for r, w in enumerate(walkers):
        assert w.prog.compute_order == [(str(p.kind), p.stage, p.microbatch) for p in sched.device_passes[r]]
        # the arena holds exactly the runner model's peak (slabs are per pair; units = v per pair)
        assert w.prog.n_slabs * sched.units_per_stage == w.prog.witness_peak_units or plan is None


@pytest.mark.parametrize("name,make", [c for c in CASES if "no offload" not in c[0]], ids=lambda c: c if isinstance(c, str) else "")
def test_spare_slab_programs_execute_correctly(name, make):
    """One offload-arena slab beyond the modelled peak: same results and op order, one
    more slab on every rank that offloads, slab reuse still hazard-free (CpuWalker)."""
    sched, plan = make()
    walkers = run_all_ranks(sched, plan, "dual", spare_slabs=1)
    for j in range(sched.microbatches):
        assert walkers[0].grad_out[(0, j)] == expected_input_grad(sched, j)
    for r, w in enumerate(walkers):
        base = lower(sched, plan, r, stream_mode="dual")
        offloads = any(op.kind == "OFFLOAD" for op in base.ops)
        assert w.prog.n_slabs == base.n_slabs + (1 if offloads else 0)
        assert w.prog.compute_order == base.compute_order


def test_arena_matches_reference_peaks_c1():
    sched, plan = po.build_1f1b_full_offload(4, 8, U, Fraction(3, 2))
    progs = [lower(sched, plan, r) for r in range(4)]
    assert [p.n_slabs for p in progs] == [2, 2, 2, 1]  # peaks [2,2,2,1]
    assert [lower(sched, None, r).n_slabs for r in range(4)] == [4, 3, 2, 1]
    # resident parts (partial offload) are held F start .. B end: the no-offload peak
    assert [p.n_res_slabs for p in progs] == [4, 3, 2, 1]


def test_send_recv_orders_match_across_ranks():
    for _, make in CASES:
        sched, plan = make()
        progs = [lower(sched, plan, r) for r in range(sched.devices)]
        for p in progs:
            for ch, order in p.send_orders.items():
                kind, src, dst = ch
                assert progs[dst].recv_orders[ch] == [((s + 1, j) if kind == "act" else (s - 1, j)) for (s, j) in order]


# ----------------------------------------------------------------- gloo, 2 ranks


class GlooChannel:
    """Sends never block the walker (as NCCL sends on their own stream never block the
    compute stream); receives block, which is safe because every receive's matching
    send precedes it in the sender's host order."""

    def __init__(self):
        self.pending = []

    def send(self, op, val):
        t = torch.tensor([op.stage, op.mb, val], dtype=torch.float64)
        self.pending.append((dist.isend(t, dst=op.peer), t))

    def flush(self):
        for work, _t in self.pending:
            work.wait()
        self.pending.clear()

    def recv(self, op):
        buf = torch.empty(3, dtype=torch.float64)
        dist.recv(buf, src=op.peer)
        want = (op.stage - 1, op.mb) if op.kind == "RECV_ACT" else (op.stage + 1, op.mb)
        assert (int(buf[0]), int(buf[1])) == want, f"rank got {buf[:2].tolist()} want {want}"
        return float(buf[2])


def _worker(rank, world, port, result_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        for make in (lambda: po.build_1f1b_full_offload(2, 6, U, Fraction(1)),
                     lambda: (po.build_interleaved_1f1b(2, 2, 4, U), None)):
            sched, plan = make()
            chan = GlooChannel()
            w = CpuWalker(sched, lower(sched, plan, rank), chan)
            while not w.done():
                w.step()
            chan.flush()
            dist.barrier()
            if rank == 0:
                got = [w.grad_out[(0, j)] for j in range(sched.microbatches)]
                ok = got == [expected_input_grad(sched, j) for j in range(sched.microbatches)]
                if not ok:
                    result_q.put(("mismatch", got))
                    return
        result_q.put(("ok", True))
    except Exception as exc:  # pragma: no cover - reported to the parent
        result_q.put(("error", repr(exc)))
    finally:
        dist.destroy_process_group()


def test_two_ranks_over_gloo():
    import socket

    with socket.socket() as sock:
        sock.bind(("127.0.0.1", 0))
        port = sock.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    results = [q.get(timeout=5) for _ in range(2)]
    assert all(r == ("ok", True) for r in results), results


@pytest.mark.parametrize("stream_mode", ["single", "dual"])
def test_topology_synced_plans_lower_and_execute(stream_mode):
    """apply_topology_sync plans (reference offload.py:223-248): cross-rank sync edges
    become flags the consumer's copy stream waits on (executed here by the walker), the
    pinned floors become anchors on every transfer; the run completes with correct
    results and every edge's producer completes before its consumer starts."""
    sched, plan = po.build_1f1b_full_offload(4, 8, U, Fraction(3, 2))
    hw = po.HardwareSpec(compute_bandwidth=1.0, transfer_bandwidth=1.0, devices_per_switch=2)
    synced = po.apply_topology_sync(plan, hw)
    assert synced.sync_edges and synced.pinned
    walkers = run_all_ranks(sched, synced, stream_mode)
    for j in range(sched.microbatches):
        assert walkers[0].grad_out[(0, j)] == expected_input_grad(sched, j)
    progs = [w.prog for w in walkers]
    assert all(p.n_flags == len(synced.sync_edges) for p in progs)
    n_waits = sum(len(op.flag_waits) for p in progs for op in p.ops)
    n_sig = sum(len(op.signals) for p in progs for op in p.ops)
    assert n_waits == n_sig > 0
    # every cross-rank edge: the producer transfer is done before the consumer runs
    by_slot = {(t.device, t.slot): t for stm in synced.streams for t in stm.transfers}
    pos = {x: i for i, x in enumerate(walkers[0].done_order)}
    tag = lambda t: (t.device, "OFFLOAD" if t.direction == po.PassKind.OFFLOAD else "RELOAD", t.stage, t.microbatch)
    for a, b in synced.sync_edges:
        ta, tb = by_slot.get(a), by_slot.get(b)
        if ta is not None and tb is not None and ta.device != tb.device:
            assert pos[tag(ta)] < pos[tag(tb)]
    # emulated neighbours drop the cross-rank edges
    emu = lower(sched, synced, 0, emulate_neighbors=True)
    assert not any(op.flag_waits or op.signals for op in emu.ops)
