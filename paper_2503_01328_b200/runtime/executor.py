"""The measured pipeline runner: drop-in for the reference's ``simulate``.

``execute(sched, plan, ...)`` runs a lowered per-rank program (``lower.py``) on
the B200: compute on one stream, D2H/H2D on a dedicated copy stream (two in
``stream_mode="dual"``), stage-boundary sends/receives on per-edge streams, all
ordered by CUDA events -- no host synchronisation inside an iteration.  It
returns a ``SimTrace`` (reference pkg/src/ppoff/sim.py:44-102) whose times are
CUDA-event measurements in seconds, so ``peak_memory``, ``bubble_time``,
``summary()`` and the reference's analysis/render layers consume it unchanged.

Three ways to run a program:

* multi-process, one rank per GPU (``torchrun``), boundary over NCCL (K8)
  through ``libppo_b200.so`` with one 2-rank communicator per directed edge;
* ``virtual``: every rank of the schedule in one process on one GPU, boundary
  through a local channel (used by the single-GPU parity tests);
* ``emulate``: one rank alone with a loopback boundary (synthetic upstream
  activation / downstream gradient), the single-GPU benchmark of one rank of a
  PP=d schedule.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field
from fractions import Fraction

import torch

from ..costs import ModelSpec
from ..ir import MemoryTimeline
from ..offload import OffloadPlan
from ..schedule_types import Pass, PassKind, Schedule
from ..sim import SimTrace
from . import gemm_tune, native
from .lower import RING, Program, lower
from .model import ModelConfig, SlabView, Stage, stage_layers

STREAMS = ("compute", "copy", "copy_h2d", "recv_act", "send_act", "recv_grad", "send_grad")
TIMED = ("F_start", "F_end", "B_start", "B_end", "W_start", "W_end", "D2H", "H2D", "D2H_start", "H2D_start")


class DeadlockError(RuntimeError):
    pass


# --------------------------------------------------------------------- transports


class LocalTransport:
    """Boundary channel between virtual ranks living in one process (one GPU).

    A send snapshots the buffer into a fresh channel tensor on the sender's
    stream; the matching receive (same channel, same index) waits on that copy's
    event.  Receivers that run ahead of their sender report "not yet" and the
    cooperative driver switches rank.
    """

    def __init__(self):
        self.posted = {}
        self.sent = {}
        self.got = {}
        self.keep = []

    def send(self, rank, op, buf, stream) -> bool:
        ch = (op.kind[5:].lower(), rank, op.peer)
        idx = self.sent.get(ch, 0)
        with torch.cuda.stream(stream):
            snap = buf.clone()
        ev = torch.cuda.Event()
        ev.record(stream)
        self.posted[(ch, idx)] = (ev, snap)
        self.sent[ch] = idx + 1
        return True

    def recv(self, rank, op, buf, stream) -> bool:
        ch = (op.kind[5:].lower(), op.peer, rank)
        idx = self.got.get(ch, 0)
        item = self.posted.get((ch, idx))
        if item is None:
            return False
        ev, snap = item
        stream.wait_event(ev)
        with torch.cuda.stream(stream):
            buf.copy_(snap)
        self.keep.append(snap)
        self.got[ch] = idx + 1
        return True

    def end_iteration(self):
        self.posted.clear()
        self.sent.clear()
        self.got.clear()
        self.keep.clear()


class NcclTransport:
    """One 2-rank NCCL communicator per directed pipeline edge and direction.

    Each channel carries one kind of traffic one way (rank ``src`` sends, rank
    ``dst`` receives) in the same (stage, mb) order on both sides, so no send can
    wait behind an unrelated receive -- the ring deadlock of a shared
    communicator cannot form, also across the interleaved wrap d-1 -> 0.
    """

    _generation = 0  # bumped per transport, in the same sequence on every rank

    def __init__(self, rank: int, world: int, device: int, edges):
        import torch.distributed as dist

        self.rank = rank
        self.comms = {}
        NcclTransport._generation += 1
        gen = NcclTransport._generation
        for ch in sorted(set(edges)):  # identical global order on every rank
            kind, src, dst = ch
            if rank not in (src, dst):
                continue
            key = f"ppo_uid/{gen}/{kind}/{src}/{dst}"
            store = _store()
            if rank == src:
                uid = native.NcclComm.unique_id()
                store.set(key, uid.hex())
            else:
                uid = bytes.fromhex(store.get(key).decode())
            self.comms[ch] = native.NcclComm(uid, 2, 0 if rank == src else 1, device)
        if dist.is_initialized():
            dist.barrier()

    def send(self, rank, op, buf, stream) -> bool:
        comm = self.comms[(op.kind[5:].lower(), rank, op.peer)]
        comm.p2p([(True, 1, buf.data_ptr(), buf.numel() * buf.element_size())], stream.cuda_stream)
        return True

    def recv(self, rank, op, buf, stream) -> bool:
        comm = self.comms[(op.kind[5:].lower(), op.peer, rank)]
        comm.p2p([(False, 0, buf.data_ptr(), buf.numel() * buf.element_size())], stream.cuda_stream)
        return True

    def end_iteration(self):
        pass

    def close(self):
        for c in self.comms.values():
            c.close()
        self.comms.clear()


class HostTransport:
    """Boundary over ``torch.distributed`` point-to-point on host copies (gloo).

    A debugging/test transport for multi-process runs where NCCL cannot be used --
    e.g. several ranks sharing one GPU, which NCCL refuses ("duplicate GPU").  A
    send waits for the producing stream, copies the ring buffer to the host and
    posts a non-blocking ``isend``; a receive blocks the issuing host thread until
    the message is there, then copies it into the ring buffer on the receive
    stream.  Message order per channel is the program order on both sides (the
    same FIFO contract as the NCCL channels), so a program that runs over NCCL runs
    here; its timings include host round trips and mean nothing.
    """

    TAGS = {"act": 11, "grad": 12}

    def __init__(self, rank: int):
        self.rank = rank
        self.pending = []

    def send(self, rank, op, buf, stream) -> bool:
        import torch.distributed as dist

        stream.synchronize()
        host = buf.cpu()
        self.pending.append((dist.isend(host, op.peer, tag=self.TAGS[op.kind[5:].lower()]), host))
        return True

    def recv(self, rank, op, buf, stream) -> bool:
        import torch.distributed as dist

        host = torch.empty(buf.shape, dtype=buf.dtype)
        dist.recv(host, op.peer, tag=self.TAGS[op.kind[5:].lower()])
        with torch.cuda.stream(stream):
            buf.copy_(host)
        return True

    def end_iteration(self):
        for work, _ in self.pending:
            work.wait()
        self.pending.clear()

    def close(self):
        self.end_iteration()


class NcclLoopbackTransport:
    """``mode="nccl_loopback"``: one rank alone whose stage-boundary messages still go
    through NCCL -- a 1-rank communicator, each message a grouped self send/recv --
    with the neighbours emulated: a send's payload lands in a sink, a receive gets
    the runner's synthetic upstream activation / downstream gradient.  It exercises
    the NCCL path (incl. capture into the whole-iteration CUDA graph) on a one-GPU box
    with the same numerics as ``mode="emulate"``."""

    def __init__(self, device: int):
        self.comm = native.NcclComm(native.NcclComm.unique_id(), 1, 0, device)
        self.runner = None  # set by execute: the synthetic tensors live on the runner
        self.sink = None

    def send(self, rank, op, buf, stream) -> bool:
        if self.sink is None or self.sink.numel() < buf.numel():
            self.sink = torch.empty_like(buf)
        n = buf.numel() * buf.element_size()
        self.comm.p2p([(True, 0, buf.data_ptr(), n), (False, 0, self.sink.data_ptr(), n)], stream.cuda_stream)
        return True

    def recv(self, rank, op, buf, stream) -> bool:
        src = self.runner.synthetic_x if op.kind == "RECV_ACT" else self.runner.synthetic_dy
        n = buf.numel() * buf.element_size()
        self.comm.p2p([(True, 0, src.data_ptr(), n), (False, 0, buf.data_ptr(), n)], stream.cuda_stream)
        return True

    def end_iteration(self):
        pass

    def close(self):
        self.comm.close()


class FlagBoard:
    """The 32-bit flags of a topology-synchronised plan's cross-rank sync edges
    (``lower``: Op.flag_waits / Op.signals; reference offload.py:223-248).

    One process (virtual ranks): device memory.  Rank processes: one POSIX shared-memory
    page created by rank 0, attached by every rank and mapped into each GPU
    (``native.host_register``), so a copy stream on one GPU can wait for a flag another
    GPU's copy stream writes -- no host thread in the loop."""

    def __init__(self, n: int, device, dist_mode: bool):
        self.n = n
        self.shm = None
        self.tensor = None
        self.host_ptr = None
        if not dist_mode:
            self.tensor = torch.zeros(max(1, n), dtype=torch.int32, device=device)
            self.base = self.tensor.data_ptr()
            return
        import ctypes
        import uuid
        from multiprocessing import shared_memory

        dist = _dist()
        box = [f"ppo_flags_{uuid.uuid4().hex[:16]}" if dist.get_rank() == 0 else None]
        dist.broadcast_object_list(box, src=0)
        size = max(4096, (4 * n + 4095) // 4096 * 4096)
        if dist.get_rank() == 0:
            self.shm = shared_memory.SharedMemory(name=box[0], create=True, size=size)
            self.shm.buf[:size] = bytes(size)
        dist.barrier()
        if dist.get_rank() != 0:
            self.shm = shared_memory.SharedMemory(name=box[0], create=False)
        self.owner = dist.get_rank() == 0
        self.host_ptr = ctypes.addressof(ctypes.c_char.from_buffer(self.shm.buf))
        with torch.cuda.device(device):
            self.base = native.host_register(self.host_ptr, size)
        dist.barrier()

    def addr(self, idx: int) -> int:
        return self.base + 4 * idx

    def close(self):
        if self.shm is not None:
            native.host_unregister(self.host_ptr)
            self.host_ptr = None
            self.shm.close()
            if self.owner:
                self.shm.unlink()
            self.shm = None


_NCCL_TRANSPORTS = {}


def nccl_transport(rank: int, world: int, device: int, edges) -> NcclTransport:
    """The process's NCCL transport for this set of edges, created once and reused by
    later ``execute`` calls (communicator set-up is collective and costs seconds)."""
    key = (rank, world, device, tuple(sorted(set(edges))))
    t = _NCCL_TRANSPORTS.get(key)
    if t is None:
        t = _NCCL_TRANSPORTS[key] = NcclTransport(rank, world, device, edges)
    return t


def close_transports():
    for t in _NCCL_TRANSPORTS.values():
        t.close()
    _NCCL_TRANSPORTS.clear()


def _store():
    import torch.distributed as dist

    if not dist.is_initialized():
        raise RuntimeError("NCCL transport needs torch.distributed initialised (torchrun)")
    from torch.distributed.distributed_c10d import _get_default_store

    return _get_default_store()


def pipeline_edges(sched: Schedule):
    edges = []
    for s in range(sched.num_stages - 1):
        a, b = sched.placement[s], sched.placement[s + 1]
        if a != b:
            edges.append(("act", a, b))
            edges.append(("grad", b, a))
    return edges


# ---------------------------------------------------------------------- runner


@dataclass
class IterationStats:
    seconds: float
    events: dict = field(default_factory=dict)


class RankRunner:
    """Issues one rank's lowered program onto CUDA streams, iteration after iteration."""

    def __init__(self, program: Program, cfg: ModelConfig, sched: Schedule, microbatches: int, device,
                 transport=None, emulate: bool = False, params=None, seed: int = 1234, optimizer: str = "sgd",
                 lr: float = 1e-4, verify_roundtrip: bool = False, use_graphs: bool = True, gemm: str = "auto", attn: str = "auto",
                 offload_tensors=None):
        torch_ = native.require_cuda()
        self.torch = torch_
        self.prog, self.cfg, self.sched, self.m = program, cfg, sched, microbatches
        self.device = torch.device(device)
        self.rank = program.rank
        self.transport = transport
        self.flags = None  # FlagBoard of a topology-synchronised plan (set by execute)
        # consecutive stages on this device (d=1 with v>1): boundary messages stay local
        self.local = LocalTransport()
        self.emulate = emulate
        my_stages = [s for s in range(sched.num_stages) if sched.placement[s] == self.rank]
        with torch.cuda.device(self.device):
            ws = Stage.new_workspace(cfg, self.device)  # one workspace for all of this rank's stages
            self.stages = {
                s: Stage(cfg, s, sched.num_stages, microbatches, self.device, params=params,
                         layers=stage_layers(cfg, sched.num_stages, s), seed=seed, gemm=gemm, offload=offload_tensors,
                         attn=attn, workspace=ws)
                for s in my_stages
            }
            lays = [st.layout for st in self.stages.values()]
            self.slab_bytes = max(l.slab_bytes for l in lays)  # whole saved set of one pair
            self.off_bytes = max(l.off_bytes for l in lays)  # the part that travels
            self.res_bytes = max(l.res_bytes for l in lays)  # the part that never does
            self.host_bytes = max(l.host_bytes for l in lays)
            # two fixed arenas: offload parts coloured over their residency (freed at D2H end),
            # resident parts over F start .. last use (the in-flight peak)
            self.arena = torch.empty(max(1, program.n_slabs) * self.off_bytes, dtype=torch.uint8, device=self.device)
            self.res_arena = (torch.empty(max(1, program.n_res_slabs) * self.res_bytes, dtype=torch.uint8,
                                          device=self.device) if self.res_bytes else None)
            self.pool = None
            self.host_slot_base = []
            if program.n_host_slots:
                slot_bytes = (self.host_bytes + 4095) // 4096 * 4096
                check_host_memory(program.n_host_slots * slot_bytes)
                # NUMA-bound to this GPU's node before first touch (ppo_pool_create_numa)
                self.pool = native.PinnedPool(program.n_host_slots * slot_bytes, device=self.device.index)
                self.host_slot_base = [self.pool.carve(slot_bytes) for _ in range(program.n_host_slots)]
            s_, h = cfg.seq, cfg.hidden
            mk = lambda: torch.empty(s_, h, dtype=torch.bfloat16, device=self.device)  # noqa: E731
            self.rings = {k: [mk() for _ in range(RING)] for k in ("recv_act", "send_act", "recv_grad", "send_grad")}
            self.scratch_out = mk()
            gen = torch.Generator(device="cpu").manual_seed(7 + self.rank)
            self.synthetic_x = (torch.randn(s_, h, generator=gen) * 0.5).to(self.device, torch.bfloat16)
            self.synthetic_dy = (torch.randn(s_, h, generator=gen) * 1e-3).to(self.device, torch.bfloat16)
            self.streams = {name: torch.cuda.Stream(self.device) for name in STREAMS}
            self.events = {}
            self.views = {}
        self.optimizer = optimizer
        self.lr = lr
        self.verify_roundtrip = verify_roundtrip
        self.use_graphs = use_graphs
        self.graphs = {}
        # One memory pool for every pass graph of this rank: passes replay one at a
        # time on the compute stream and keep nothing in pool memory past their end
        # (outputs go to the slab arena, rings and workspaces), so their temporaries
        # (cuDNN attention outputs, dq/dk/dv) can share addresses instead of each graph
        # pinning a private copy -- at C4 shape that is tens of GB.
        self.graph_pool = None
        self.wbufs = {}
        self.graph_native_launches = {}  # libppo_b200 kernels inside each captured pass
        self.replayed_native_launches = 0  # ... executed through graph replays
        self.graph_calls = {}  # per captured pass: ABI calls (native.CALLS/SHAPES deltas) one replay runs
        self.digests = {}  # (stage, mb) -> [digest at F end, digest at B start]
        self._adam = None
        self.cursor = 0
        self.iteration = 0
        self.tokens = None
        self.t0 = None
        # whole-iteration CUDA graph (execute(iteration_graph=True)): while capturing,
        # pass bodies run inline (no per-pass graphs) and pass boundaries are timed by
        # stream-ordered global-timer writes (native.timestamp) into ``ts_buf`` instead of
        # event records, whose host-visible semaphore writes stall behind saturated PCIe
        self.capturing = False
        self.graph_timed = False  # measured_passes reads ts_buf
        self.pass_timing = True
        self.ts_index = {}
        self.ts_buf = None

    # -------------------------------------------------------------- plumbing
    def ev(self, key):
        e = self.events.get(key)
        if e is None:
            timed = key[0] in TIMED
            e = torch.cuda.Event(enable_timing=timed)
            self.events[key] = e
        return e

    def rec(self, key, stream):
        """Record event ``key`` on ``stream`` (sync), plus its timing twin in graph mode."""
        self.ev(key).record(stream)
        if self.capturing and self.pass_timing and key[0] in TIMED:
            self.timestamp(key, stream)

    def timestamp(self, key, stream):
        """Global-timer write for ``key`` into this runner's timestamp buffer."""
        if self.ts_buf is None:
            self.ts_buf = torch.zeros(2 * len(self.prog.ops) + 8, dtype=torch.int64, device=self.device)
        i = self.ts_index.setdefault(key, len(self.ts_index))
        native.timestamp(self.ts_buf.data_ptr() + 8 * i, stream)

    @property
    def act_bytes(self) -> int:
        """Device bytes held for activations: both arenas (the measured per-GPU peak)."""
        return self.prog.n_slabs * self.off_bytes + (self.prog.n_res_slabs * self.res_bytes if self.res_bytes else 0)

    @property
    def state_bytes(self) -> int:
        """Persistent training state of this rank's stages (weights, gradients, masters,
        AdamW moments once created): excluded from activation memory."""
        extra = 0
        if self.optimizer not in ("none", "sgd"):
            extra = 2 * sum(t.numel() * t.element_size() for st in self.stages.values() for t in st.master.values())
        return sum(st.state_bytes for st in self.stages.values()) + extra

    @property
    def wbuf_bytes(self) -> int:
        return sum(t.numel() * t.element_size() for b in self.wbufs.values() for per in b.values() for t in per.values())

    @property
    def ws_bytes(self) -> int:
        uniq = {t.data_ptr(): t for st in self.stages.values() for t in st.ws.values()}  # shared across stages
        return sum(t.numel() * t.element_size() for t in uniq.values())

    def _rkey(self, op):
        """Resident slot as part of a pass-graph key (None when there is no resident part)."""
        return op.res_slab if self.res_bytes else None

    def slab(self, op, stage: int) -> SlabView:
        idx, ridx = op.slab, (op.res_slab if self.res_bytes else 0)
        key = (idx, ridx, stage)
        v = self.views.get(key)
        if v is None:
            lay = self.stages[stage].layout
            base = self.arena[idx * self.off_bytes: idx * self.off_bytes + lay.off_bytes]
            res = (self.res_arena[ridx * self.res_bytes: ridx * self.res_bytes + lay.res_bytes]
                   if self.res_bytes else base[lay.off_bytes:])
            v = SlabView(lay, base, res)
            self.views[key] = v
        return v

    def host_bins(self, slot: int, stage: int):
        lay = self.stages[stage].layout
        base, acc, out = self.host_slot_base[slot], 0, []
        for b in lay.bins:
            out.append(base + acc)
            acc += b
        return tuple(out)

    # ------------------------------------------------------------ iteration
    def pre_iteration(self, stream):
        """Per-iteration device state a captured iteration graph reads (on ``stream``,
        outside any capture): the iteration part of the Philox offsets."""
        with torch.cuda.stream(stream):
            for st in self.stages.values():
                st.set_iteration(self.iteration)

    def begin_iteration(self, tokens_dev: torch.Tensor | None, timed: bool = True):
        """tokens_dev: [m, s+1] int64 already on this device (first/last stages use it).
        ``timed=False``: the iteration start event is recorded by the caller (around a
        whole-iteration graph replay)."""
        self.cursor = 0
        self.tokens = tokens_dev
        comp = self.streams["compute"]
        if timed:
            self.pre_iteration(torch.cuda.current_stream(self.device))
        comp.wait_stream(torch.cuda.current_stream(self.device))
        for name, st in self.streams.items():
            if name != "compute":
                st.wait_stream(comp)
        for st in self.stages.values():
            with torch.cuda.stream(comp):
                st.zero_grad()
        if timed:
            self.t0 = torch.cuda.Event(enable_timing=True)
            self.t0.record(comp)

    def done(self) -> bool:
        return self.cursor >= len(self.prog.ops)

    def issue_next(self) -> bool:
        """Issue the next op; False when it must wait for another (virtual) rank."""
        op = self.prog.ops[self.cursor]
        stream = self.streams[op.stream]
        if op.kind in ("RECV_ACT", "RECV_GRAD"):
            for key in op.waits:
                stream.wait_event(self.ev(key))
            buf = self.rings["recv_act" if op.kind == "RECV_ACT" else "recv_grad"][op.ring]
            if not self._transport(op).recv(self.rank, op, buf, stream):
                return False
            self.rec(op.records[0], stream)
            self.cursor += 1
            return True
        for key in op.waits:
            stream.wait_event(self.ev(key))
        if op.kind == "F":
            self._forward(op, stream)
        elif op.kind == "B":
            self._backward(op, stream)
        elif op.kind == "W":
            self._wgrad(op, stream)
        elif op.kind in ("OFFLOAD", "RELOAD"):
            self._transfer(op, stream)
        elif op.kind in ("SEND_ACT", "SEND_GRAD"):
            buf = self.rings["send_act" if op.kind == "SEND_ACT" else "send_grad"][op.ring]
            self._transport(op).send(self.rank, op, buf, stream)
            self.rec(op.records[0], stream)
        else:  # pragma: no cover
            raise ValueError(op.kind)
        self.cursor += 1
        return True

    def _transport(self, op):
        return self.local if op.peer == self.rank else self.transport

    def _forward(self, op, stream):
        s, j = op.stage, op.mb
        st = self.stages[s]
        self.rec(("F_start", s, j), stream)
        with torch.cuda.stream(stream):
            slab = self.slab(op, s)
            st.set_pass_context(j, None, self.tokens[j])
            if st.first:
                st.embed(slab)
            elif op.ring is not None:
                slab.get(0, "x").copy_(self.rings["recv_act"][op.ring])
            else:  # emulated upstream stage
                slab.get(0, "x").copy_(self.synthetic_x)
            self.rec(("F_in", s, j), stream)
            out = None
            if not st.last:
                out = self.rings["send_act"][op.send_ring] if op.send_ring is not None else self.scratch_out
            key = ("F", s, op.slab, self._rkey(op), out.data_ptr() if out is not None else 0)
            self._run_body(key, lambda: st.forward_body(slab, out), stream)
            if self.verify_roundtrip and (s, j) in self.prog.offloaded:
                self.digests[(s, j)] = [_digest(slab.base), None]
        self.rec(("F_end", s, j), stream)

    def _backward(self, op, stream):
        s, j = op.stage, op.mb
        st = self.stages[s]
        self.rec(("B_start", s, j), stream)
        with torch.cuda.stream(stream):
            slab = self.slab(op, s)
            if self.verify_roundtrip and (s, j) in self.prog.offloaded:
                self.digests[(s, j)][1] = _digest(slab.base)
            st.set_pass_context(j, None, self.tokens[j] if st.first else None)
            dy = None
            if not st.last:
                dy = self.rings["recv_grad"][op.ring] if op.ring is not None else self.synthetic_dy
            dx_out = None
            if not st.first:
                dx_out = self.rings["send_grad"][op.send_ring] if op.send_ring is not None else self.scratch_out
            wbuf = self.wbuf(op.wbuf, s) if op.wbuf is not None else None
            key = ("B", s, op.slab, self._rkey(op), dy.data_ptr() if dy is not None else 0, dx_out.data_ptr() if dx_out is not None else 0,
                   op.wbuf)
            self._run_body(key, lambda: st.backward_body(slab, dy, dx_out, wbuf), stream)
        self.rec(("B_end", s, j), stream)

    def _wgrad(self, op, stream):
        s, j = op.stage, op.mb
        st = self.stages[s]
        self.rec(("W_start", s, j), stream)
        with torch.cuda.stream(stream):
            slab = self.slab(op, s)
            wbuf = self.wbuf(op.wbuf, s)
            self._run_body(("W", s, op.slab, self._rkey(op), op.wbuf), lambda: st.wgrad_body(slab, wbuf), stream)
        self.rec(("W_end", s, j), stream)

    def wbuf(self, idx: int, stage: int) -> dict:
        """Split-backward gradient buffers of colour ``idx`` (shared by the rank's stages
        of equal depth; allocated once, before the first use)."""
        st = self.stages[stage]
        key = (idx, len(st.layers))
        b = self.wbufs.get(key)
        if b is None:
            b = self.wbufs[key] = st.new_wbuffer()
        return b

    def _run_body(self, key, body, stream):
        """Run one F/B pass body; with graphs on, the first run of each (pass, slab,
        boundary buffer) key is eager and is then captured, later runs replay it.
        Capture uses the low-level begin/end API (no device synchronisation), so it is
        safe mid-iteration and across NCCL ranks."""
        if not self.use_graphs or self.capturing:
            body()
            return
        graph = self.graphs.get(key)
        if graph is not None:
            graph.replay()
            self.replayed_native_launches += self.graph_native_launches[key]
            native.credit(self.graph_calls[key])
            return
        body()
        graph = torch.cuda.CUDAGraph()
        before = native.kernel_launches()
        snap = native.call_counts()
        if self.graph_pool is None:
            self.graph_pool = torch.cuda.graph_pool_handle()
        graph.capture_begin(pool=self.graph_pool, capture_error_mode="thread_local")
        try:
            body()
        finally:
            graph.capture_end()
        self.graphs[key] = graph
        self.graph_native_launches[key] = native.kernel_launches() - before
        # the capture recorded these calls without running them: native.CALLS /
        # SHAPES count executed calls, so they move to the replays
        self.graph_calls[key] = native.since(snap)
        native.credit(self.graph_calls[key], -1)

    def _transfer(self, op, stream):
        s, j = op.stage, op.mb
        lay = self.stages[s].layout
        slab_ptr = self.arena.data_ptr() + op.slab * self.off_bytes
        segs = lay.segments(slab_ptr, self.host_bins(op.host_slot, s))
        tag = "D2H" if op.kind == "OFFLOAD" else "H2D"
        for f in op.flag_waits:  # cross-rank sync edge: the paired device's transfer is done
            native.stream_wait_u32(stream, self.flags.addr(f), 1)
            native.stream_write_u32(stream, self.flags.addr(f), 0)
        self.rec((tag + "_start", s, j), stream)
        native.transfer(native.PPO_D2H if op.kind == "OFFLOAD" else native.PPO_H2D, segs, stream.cuda_stream)
        self.rec((tag, s, j), stream)
        for f in op.signals:
            native.stream_write_u32(stream, self.flags.addr(f), 1)

    def end_iteration(self, timed: bool = True):
        comp = self.streams["compute"]
        for name, st in self.streams.items():
            if name != "compute":
                comp.wait_stream(st)
        with torch.cuda.stream(comp):
            self._optimizer_step()
        if timed:
            self.t_end = torch.cuda.Event(enable_timing=True)
            self.t_end.record(comp)
        torch.cuda.current_stream(self.device).wait_stream(comp)
        self.iteration += 1

    def _optimizer_step(self):
        if self.optimizer == "none":
            return
        if self.optimizer == "sgd":
            for st in self.stages.values():
                st.sgd_step(self.lr)
            return
        if self._adam is None:
            params = [t for st in self.stages.values() for t in st.master.values()]
            for p in params:
                p.requires_grad_(False)
            self._adam = torch.optim.AdamW(params, lr=self.lr, fused=True)
            self._adam_pairs = [(st, n) for st in self.stages.values() for n in st.master]
        for (st, n) in self._adam_pairs:
            st.master[n].grad = st.g[n]
        self._adam.step()
        for (st, n) in self._adam_pairs:
            st.w[n].copy_(st.master[n])

    def probe_summary(self) -> dict:
        """Per native kernel: launches, mean/total CUDA-event duration, bytes per launch."""
        out = {}
        for st in self.stages.values():
            for name, (nbytes, pairs) in (st.probe or {}).items():
                ms = [a.elapsed_time(b) for a, b in pairs]
                agg = out.setdefault(name, {"bytes_per_launch": nbytes, "launches": 0, "total_ms": 0.0})
                agg["launches"] += len(ms)
                agg["total_ms"] += sum(ms)
        for agg in out.values():
            agg["avg_ms"] = agg["total_ms"] / max(1, agg["launches"])
        return out

    def result_scalar(self) -> torch.Tensor:
        """The step's result read back by the e2e path: the loss on the last stage,
        otherwise a gradient checksum of the rank's first stage."""
        ls = self.loss_sum()
        if ls is not None:
            return ls
        st = self.stages[min(self.stages)]
        return st.g[sorted(st.g)[0]].sum()

    def loss_sum(self) -> torch.Tensor | None:
        for st in self.stages.values():
            if st.last:
                return st.loss_sum
        return None

    # -------------------------------------------------------- measured trace
    def measured_passes(self) -> list[Pass]:
        """CUDA-event times (seconds from iteration start) of this rank's passes."""
        if self.graph_timed:
            ts = self.ts_buf.cpu().tolist()
            base = ts[self.ts_index[("iter_start",)]]
            evs = {k: ts[i] for k, i in self.ts_index.items()}
            sec = lambda t: Fraction(t - base, 10**9)  # noqa: E731
        else:
            t0 = self.t0
            sec = lambda ev: Fraction(t0.elapsed_time(ev)) / 1000  # noqa: E731
            evs = self.events
        out = []
        for (kind, s, j) in self.prog.compute_order:
            a, b = evs[(f"{kind}_start", s, j)], evs[(f"{kind}_end", s, j)]  # F, B or W
            st = sec(a)
            out.append(Pass(PassKind(kind), self.rank, s, j, st, sec(b) - st))
        for op in self.prog.ops:
            if op.kind in ("OFFLOAD", "RELOAD"):
                tag = "D2H" if op.kind == "OFFLOAD" else "H2D"
                st = sec(evs[(tag + "_start", op.stage, op.mb)])
                en = sec(evs[(tag, op.stage, op.mb)])
                out.append(Pass(PassKind(op.kind), self.rank, op.stage, op.mb, st, en - st))
        return out

    def iteration_seconds(self) -> float:
        return self.t0.elapsed_time(self.t_end) / 1000.0

    def close(self):
        if self.pool is not None:
            self.pool.close()
            self.pool = None
        if isinstance(self.transport, NcclLoopbackTransport):
            self.transport.close()
            self.transport = None
        owned = getattr(self, "owned_flags", None)
        if owned is not None:
            torch.cuda.synchronize(self.device)
            owned.close()
            self.owned_flags = None


def host_memory_available() -> int:
    """Bytes of host memory this process may still pin: MemAvailable, capped by the
    cgroup (v2 or v1) limit minus current usage when one is set."""
    avail = None
    try:
        with open("/proc/meminfo") as f:
            for line in f:
                if line.startswith("MemAvailable:"):
                    avail = int(line.split()[1]) * 1024
    except OSError:
        pass
    for lim_p, use_p in (("/sys/fs/cgroup/memory.max", "/sys/fs/cgroup/memory.current"),
                         ("/sys/fs/cgroup/memory/memory.limit_in_bytes", "/sys/fs/cgroup/memory/memory.usage_in_bytes")):
        try:
            with open(lim_p) as f:
                lim = f.read().strip()
            with open(use_p) as f:
                use = int(f.read().strip())
            if lim != "max" and int(lim) < (1 << 60):
                room = int(lim) - use
                avail = room if avail is None else min(avail, room)
                break
        except (OSError, ValueError):
            continue
    return avail if avail is not None else (1 << 62)


def check_host_memory(nbytes: int, fraction: float = 0.8) -> None:
    """Refuse a pinned pool larger than ``fraction`` of the host memory left: pinning
    past that takes the box down instead of failing."""
    avail = host_memory_available()
    if nbytes > fraction * avail:
        raise MemoryError(f"pinned host pool of {nbytes / 1e9:.1f} GB exceeds {fraction:.0%} of the "
                          f"{avail / 1e9:.1f} GB host memory available")


def _digest(buf: torch.Tensor) -> torch.Tensor:
    """Order-independent integer digest of a byte buffer (exact, deterministic)."""
    words = buf.view(torch.int32).to(torch.int64)
    weights = torch.arange(words.numel(), device=buf.device, dtype=torch.int64) % 65521 + 1
    return torch.stack([words.sum(), (words * weights).sum()])


def roundtrip_mismatches(runners) -> list:
    """(rank, stage, mb) whose reloaded slab differs from what was offloaded."""
    bad = []
    for r in runners:
        for (s, j), (a, b) in r.digests.items():
            if b is None or not torch.equal(a, b):
                bad.append((r.rank, s, j))
    return bad


def drive(runners: list[RankRunner]):
    """Cooperatively issue every runner's program (virtual ranks share one host thread)."""
    while True:
        progressed = False
        pending = False
        for r in runners:
            while not r.done():
                if not r.issue_next():
                    break
                progressed = True
            pending |= not r.done()
        if not pending:
            return
        if not progressed:
            stuck = [(r.rank, r.prog.ops[r.cursor].key) for r in runners if not r.done()]
            raise DeadlockError(f"virtual pipeline cannot make progress: {stuck}")


def _capture_iteration(runners, tokens_dev, origin, dev, transport):
    """Capture one whole iteration of every runner into a single CUDA graph on
    ``origin``: each runner's streams fork from origin (begin_iteration) and join back
    (end_iteration), so the lowered program's event waits become graph edges.
    Returns (graph, native launches one replay runs, ABI call deltas)."""
    graph = torch.cuda.CUDAGraph()
    pool = torch.cuda.graph_pool_handle()
    origin.wait_stream(torch.cuda.current_stream(dev))
    before = native.kernel_launches()
    snap = native.call_counts()
    for r in runners:
        if r.pass_timing and r.ts_buf is None:  # allocated outside the capture
            r.ts_buf = torch.zeros(2 * len(r.prog.ops) + 8, dtype=torch.int64, device=r.device)
    with torch.cuda.stream(origin):
        for r in runners:
            r.capturing = True
        graph.capture_begin(pool=pool, capture_error_mode="thread_local")
        try:
            for r in runners:
                if r.pass_timing:
                    r.timestamp(("iter_start",), origin)
                r.begin_iteration(tokens_dev, timed=False)
            drive(runners)
            for r in runners:
                r.end_iteration(timed=False)
        finally:
            graph.capture_end()
            for r in runners:
                r.capturing = False
                r.graph_timed = r.pass_timing
    for r in runners:
        r.iteration -= 1  # the capture ran nothing
    if transport is not None:
        transport.end_iteration()
    for r in runners:
        r.local.end_iteration()
    launched = native.kernel_launches() - before
    calls = native.since(snap)
    native.credit(calls, -1)  # recorded, not executed: each replay credits them back
    runners[0].graph_native_launches["iteration"] = launched
    return graph, launched, calls


def _replay_iteration(runners, captured, origin, dev):
    graph, launched, calls = captured
    origin.wait_stream(torch.cuda.current_stream(dev))
    for r in runners:
        r.pre_iteration(origin)
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(origin):
        t0.record(origin)
        graph.replay()
        t1.record(origin)
    torch.cuda.current_stream(dev).wait_stream(origin)
    for r in runners:
        r.t0, r.t_end = t0, t1
        r.iteration += 1
    runners[0].replayed_native_launches += launched
    native.credit(calls)


def measured_trace(sched: Schedule, passes: list[Pass], model: ModelSpec | None = None,
                   units_bytes: int = 0) -> SimTrace:
    """Assemble a reference-compatible ``SimTrace`` from measured passes (all ranks)."""
    ends = {(p.kind, p.stage, p.microbatch): p.end for p in passes}
    starts = {(p.kind, p.stage, p.microbatch): p.start for p in passes}
    reload_of = {(p.stage, p.microbatch): (PassKind.RELOAD, p.stage, p.microbatch) for p in passes if p.kind == PassKind.RELOAD}
    offload_of = {(p.stage, p.microbatch): (PassKind.OFFLOAD, p.stage, p.microbatch) for p in passes if p.kind == PassKind.OFFLOAD}
    u = sched.units_per_stage
    dev_events = [[] for _ in range(sched.devices)]
    host = []
    present = {p.device for p in passes}
    for dev in range(sched.devices):
        if dev not in present:
            continue
        for p in sched.device_passes[dev]:
            pair = (p.stage, p.microbatch)
            if p.kind == PassKind.F:
                dev_events[dev].append((starts[(PassKind.F,) + pair], p.stage, u))
                if pair in reload_of and pair in offload_of:
                    dev_events[dev].append((ends[offload_of[pair]], p.stage, -u))
                    dev_events[dev].append((starts[reload_of[pair]], p.stage, u))
                    host.append((ends[offload_of[pair]], dev, u))
                    host.append((ends[reload_of[pair]], dev, -u))
            elif p.kind == PassKind.B:
                dev_events[dev].append((ends[(PassKind.B,) + pair], p.stage, -u))
    order = lambda e: (e[0], e[2])  # noqa: E731
    busy = tuple(sum((p.duration for p in passes if p.device == d and p.kind in (PassKind.F, PassKind.B, PassKind.W)), Fraction(0))
                 for d in range(sched.devices))
    return SimTrace(
        schedule=sched,
        passes=tuple(sorted(passes, key=lambda p: (p.start, p.device, str(p.kind), p.stage, p.microbatch))),
        makespan=max((p.end for p in passes), default=Fraction(0)),
        device_busy=busy,
        memory=MemoryTimeline(sched.devices, units_bytes, tuple(tuple(sorted(ev, key=order)) for ev in dev_events)),
        host_events=tuple(sorted(host, key=order)),
        contention_log=(),
        bytes_per_unit=units_bytes,
    )


def _dist():
    import torch.distributed as dist

    return dist


def _reduce_over_ranks(sec, wall, host_issue, loss, dev):
    """MAX of the times over ranks; the loss from the rank that holds the last stage."""
    dist = _dist()
    on = dev if dist.get_backend() == "nccl" else torch.device("cpu")
    t = torch.tensor([sec, wall, host_issue], dtype=torch.float64, device=on)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    lv = torch.tensor([loss if loss is not None else 0.0, 1.0 if loss is not None else 0.0], dtype=torch.float64,
                      device=on)
    dist.all_reduce(lv, op=dist.ReduceOp.SUM)
    sec, wall, host_issue = (float(x) for x in t.tolist())
    return sec, wall, host_issue, (float(lv[0]) if float(lv[1]) else None)


@dataclass
class RunResult:
    trace: SimTrace
    iteration_seconds: list
    losses: list
    programs: dict
    runners: list
    slab_bytes: int
    peak_slabs: dict  # rank -> arena slabs (= planned peak units)
    host_slots: dict
    wall_seconds: list  # e2e: host clock per step incl. input H2D and result D2H
    host_issue_seconds: list = field(default_factory=list)  # host time to enqueue one iteration
    act_bytes: dict = field(default_factory=dict)  # rank -> activation arena bytes (both parts)
    offload_fraction: float = 1.0  # share of a pair's saved set that travels when it is offloaded
    # activation memory MEASURED the paper's way (peak minus iteration-start
    # memory) for the ranks of this process: see ``execute``
    mem: dict = field(default_factory=dict)

    def close(self):
        """Release the pinned pools and drop the runners (their device arenas, weights
        and graphs go with the last reference)."""
        for r in self.runners:
            r.close()
        self.runners.clear()


def execute(sched: Schedule, plan: OffloadPlan | None = None, *, model: ModelConfig, microbatches: int | None = None,
            mode: str = "virtual", rank: int | None = None, device=None, iters: int = 1, warmup: int = 0,
            stream_mode: str = "single", tokens: torch.Tensor | None = None, params=None, optimizer: str = "sgd",
            lr: float = 1e-4, verify_roundtrip: bool = False, probe_kernels: bool = False,
            use_graphs: bool = True, gemm: str = "auto", offload_tensors=None, attn: str = "auto",
            iteration_graph: bool = False, pass_timing: bool = True, spare_slabs: int = 0,
            tune_table=None) -> RunResult:
    """Run ``sched`` (+ ``plan``) for ``warmup + iters`` iterations and measure the last.

    mode: "virtual" (all ranks, one GPU), "emulate" (``rank`` alone, loopback
    boundary) or "nccl" (this process is ``rank`` of a torchrun job; "gloo" is the
    same over host copies, for ranks that share a GPU in tests; "nccl_loopback" is
    ``rank`` alone with its boundary messages through a 1-rank NCCL communicator).
    ``tokens``: [m, s+1] int64 host tensor (pinned for the e2e path).
    ``offload_tensors``: None (an offloaded pair moves its whole saved set) or the
    (local layer, name) tensors that move (partial offload, ``layout.make_layout``).
    ``iteration_graph``: after one eager iteration, capture a whole iteration -- every
    stream, event edge, pass, D2H/H2D and the optimizer step -- into ONE CUDA graph and
    replay it (every mode but "gloo"; NCCL p2p kernels become graph nodes): no host issue and no per-launch command
    fetch over the host link the copy engines are saturating.
    ``pass_timing=False`` (graph mode): no per-pass timestamps inside the graph, only
    the iteration's start/end -- the returned trace then has no passes.
    ``spare_slabs``: offload-arena slabs beyond the modelled peak (``lower``): device
    memory traded for slack when transfers run slower than the plan modelled.
    ``attn``: attention forward backend of every stage ("auto" | "tcgen05" | "cudnn").
    ``tune_table``: backend decisions to install first (a ``gemm_tune.decisions()``
    dict or a JSON path); under "auto" the missing ones are tuned before any pass --
    in the multi-process modes by rank 0 alone and broadcast, so every rank runs the
    same kernels (``gemm_tune.ensure``).

    In the multi-process modes every iteration starts after a device synchronise
    and a barrier, and the returned iteration/wall times and losses are the same on
    every rank: times are the MAX over ranks, the loss is the last stage's.
    """
    native.require_cuda()
    m = microbatches or sched.microbatches
    dev = torch.device(device if device is not None else f"cuda:{torch.cuda.current_device()}")
    if mode == "virtual":
        ranks = list(range(sched.devices))
    else:
        ranks = [rank if rank is not None else 0]
    programs = {r: lower(sched, plan, r, stream_mode=stream_mode, emulate_neighbors=(mode == "emulate"),
                      spare_slabs=spare_slabs) for r in ranks}
    if mode == "nccl_loopback" and len(ranks) != 1:  # pragma: no cover
        raise ValueError("nccl_loopback runs one rank")
    transport = None
    if mode == "virtual":
        transport = LocalTransport()
    elif mode == "nccl":
        import torch.distributed as dist

        transport = nccl_transport(ranks[0], dist.get_world_size(), dev.index, pipeline_edges(sched))
    elif mode == "gloo":
        transport = HostTransport(ranks[0])
    elif mode == "nccl_loopback":
        transport = NcclLoopbackTransport(dev.index)
    elif mode != "emulate":
        raise ValueError(f"unknown mode {mode!r}")
    dist_mode = mode in ("nccl", "gloo")
    if tune_table is not None:
        gemm_tune.load(tune_table) if isinstance(tune_table, str) else gemm_tune.install(tune_table)
    if gemm == "auto" or attn == "auto":
        with torch.cuda.device(dev):
            gemm_tune.ensure(model, dev, gemm, attn)  # collective in the multi-process modes
    # activation memory, the paper's way: everything allocated from here on except the
    # persistent training state (weights / gradients / masters) counts -- slab arenas,
    # split-backward W buffers, recompute workspaces, boundary rings, graph pools and
    # library temporaries.  Torch's allocator peak gives the allocated view,
    # cudaMemGetInfo the device view (cached segments and library workspaces included).
    torch.cuda.synchronize(dev)
    torch.cuda.empty_cache()
    torch.cuda.reset_peak_memory_stats(dev)
    alloc0 = torch.cuda.memory_allocated(dev)
    free0, total0 = torch.cuda.mem_get_info(dev)
    runners = [RankRunner(programs[r], model, sched, m, dev, transport=transport, emulate=(mode == "emulate"),
                          params=params, optimizer=optimizer, lr=lr, verify_roundtrip=verify_roundtrip,
                          use_graphs=use_graphs, gemm=gemm, offload_tensors=offload_tensors, attn=attn) for r in ranks]
    if mode == "nccl_loopback":
        transport.runner = runners[0]
    n_flags = max(p.n_flags for p in programs.values())
    flags = None
    if n_flags and any(op.flag_waits or op.signals for p in programs.values() for op in p.ops) or \
            (n_flags and dist_mode):  # every rank joins the board's set-up collectives
        flags = FlagBoard(n_flags, dev, dist_mode)
        for r in runners:
            r.flags = flags
    if tokens is None:
        gen = torch.Generator().manual_seed(0)
        tokens = torch.randint(0, model.vocab, (m, model.seq + 1), generator=gen)
    tokens_dev = torch.empty(tokens.shape, dtype=torch.int64, device=dev)
    secs, losses, walls, host_secs = [], [], [], []
    # the host-copy transport (gloo) cannot be captured; NCCL p2p can (also across ranks:
    # every rank captures the same per-rank program and replays it after a barrier)
    whole = (iteration_graph and mode in ("emulate", "virtual", "nccl", "nccl_loopback") and not probe_kernels
             and optimizer in ("none", "sgd") and warmup + iters > 1)
    origin = torch.cuda.Stream(dev) if whole else None
    graph = None
    if whole:
        for r in runners:
            r.use_graphs = False  # iteration 0 runs eagerly; then the whole iteration is one graph
            r.pass_timing = pass_timing
    torch.cuda.synchronize(dev)
    for it in range(warmup + iters):
        if dist_mode:
            torch.cuda.synchronize(dev)
            _dist().barrier()
        if it == warmup and probe_kernels:
            for r in runners:
                for st in r.stages.values():
                    st.probe = {}
        wall0 = time.perf_counter()
        tokens_dev.copy_(tokens, non_blocking=True)  # H2D of the step's inputs (pinned host)
        if whole and it >= 1:
            if graph is None:
                graph = _capture_iteration(runners, tokens_dev, origin, dev, transport)
            host0 = time.perf_counter()
            _replay_iteration(runners, graph, origin, dev)
            host_issue = time.perf_counter() - host0
        else:
            for r in runners:
                r.begin_iteration(tokens_dev)
            host0 = time.perf_counter()
            drive(runners)
            host_issue = time.perf_counter() - host0
            for r in runners:
                r.end_iteration()
        result = [r.result_scalar() for r in runners]
        values = [float(x) for x in result]  # D2H read of the step's result (syncs)
        wall = time.perf_counter() - wall0
        torch.cuda.synchronize(dev)
        if transport is not None:
            transport.end_iteration()
        for r in runners:  # local same-device hand-offs: snapshots freed after the sync
            r.local.end_iteration()
        if it >= warmup:
            torch.cuda.synchronize(dev)
            sec = max(r.iteration_seconds() for r in runners)
            ls = [v for r, v in zip(runners, values) if r.loss_sum() is not None]
            loss = ls[0] / m if ls else None
            if dist_mode:
                sec, wall, host_issue, loss = _reduce_over_ranks(sec, wall, host_issue, loss, dev)
            walls.append(wall)
            host_secs.append(host_issue)
            secs.append(sec)
            losses.append(loss)
    torch.cuda.synchronize(dev)
    state = sum(r.state_bytes for r in runners)
    free1, _ = torch.cuda.mem_get_info(dev)
    mem = {
        "alloc_peak_bytes": torch.cuda.max_memory_allocated(dev) - alloc0 - state,
        "device_bytes": (free0 - free1) - state,
        "arena_bytes": sum(r.act_bytes for r in runners),
        "wbuf_bytes": sum(r.wbuf_bytes for r in runners),
        "workspace_bytes": sum(r.ws_bytes for r in runners),
        "state_bytes": state,
        "pool_numa_node": {r.rank: (r.pool.numa_node if r.pool is not None else None) for r in runners},
    }
    passes = [p for r in runners for p in r.measured_passes()] if (pass_timing or not whole) else []
    slab_bytes = max(r.slab_bytes for r in runners)
    trace = measured_trace(sched, passes, units_bytes=slab_bytes // sched.units_per_stage)
    if flags is not None:
        runners[0].owned_flags = flags
    return RunResult(trace, secs, losses, programs, runners, slab_bytes,
                     {r.rank: r.prog.n_slabs for r in runners}, {r.rank: r.prog.n_host_slots for r in runners},
                     walls, host_secs, {r.rank: r.act_bytes for r in runners},
                     max(r.off_bytes for r in runners) / max(1, slab_bytes), mem)
