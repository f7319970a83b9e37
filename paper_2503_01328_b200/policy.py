"""k-aware offload policy (B200 extension).

The reference plans every microbatch of the chosen stages (``plan_slots``,
offload.py:209-220) and reports late reloads when the host link cannot keep up
(k > 1).  Eq. (1) with measured B200 numbers gives k ~ 1.5-4 over PCIe Gen5 for
the BASELINE shapes, where full offload costs +34%..+158%.

``choose_offload`` keeps the reference planner and simulator as the judge and
searches the microbatch density instead: for stride q = 1, 2, ... it offloads
every q-th microbatch of the chosen stages, simulates the result with the
measured costs, and returns the plan with the lowest peak whose modelled
makespan stays within ``tolerance`` of no offload (and has no late reloads).

``choose_offload_measured`` closes the loop with the device: the runner model does
not price the compute slowdown under concurrent DMA nor the duplex link rate, and at
k ~ 1.1-2.7 the plan it accepts at 5% modelled overhead measures 5-8% (C5 sweep,
DESIGN.md section 9).  It walks the same candidates from the least memory up, measures
each (``measure(plan)`` -> overhead fraction), and keeps the first whose *measured*
overhead is within tolerance; candidates whose modelled overhead already exceeds the
measured-to-modelled gap seen so far are skipped without a run.
"""

from __future__ import annotations

from dataclasses import dataclass
from fractions import Fraction

from .offload import OffloadPlan, plan_slots
from .schedule_types import PassKind, Schedule
from .sim import peak_memory, simulate


@dataclass(frozen=True)
class DmaSlowdown:
    """Measured compute slowdown while the copy engines stream (``runtime.calibrate
    .dma_slowdown``): fractional extra time of F, B and W passes with D2H alone, H2D
    alone or both directions in flight.  The reference runner model prices link
    contention only (sim.py:274-304); copy-engine reads of HBM also cost the SMs DRAM
    bandwidth (profiles/r1_dma_interference.txt), so a plan the model schedules "for
    free" still slows the compute it overlaps."""

    f: tuple = (0.0, 0.0, 0.0)  # (d2h, h2d, duplex)
    b: tuple = (0.0, 0.0, 0.0)
    w: tuple = (0.0, 0.0, 0.0)

    @classmethod
    def from_calibration(cls, cal: dict, split: bool = False) -> "DmaSlowdown":
        d = cal["dma_slowdown"]
        pick = lambda k: tuple(max(0.0, float(d[k][m])) for m in ("d2h", "h2d", "duplex"))  # noqa: E731
        if split:
            return cls(pick("F"), pick("Bs"), pick("W"))
        return cls(pick("F"), pick("B"), pick("B"))

    def of(self, kind) -> tuple:
        return {PassKind.F: self.f, PassKind.B: self.b, PassKind.W: self.w}[kind]


def _overlaps(a: float, b: float, transfers) -> tuple[float, float, float]:
    """Seconds of [a, b) with D2H only, H2D only and both directions in flight."""
    cuts = {a, b}
    for s, e, _ in transfers:
        if e > a and s < b:
            cuts.update(x for x in (s, e) if a < x < b)
    cuts = sorted(cuts)
    d_only = h_only = both = 0.0
    for lo, hi in zip(cuts, cuts[1:]):
        mid = 0.5 * (lo + hi)
        d = any(s <= mid < e for s, e, k in transfers if k == PassKind.OFFLOAD)
        h = any(s <= mid < e for s, e, k in transfers if k == PassKind.RELOAD)
        if d and h:
            both += hi - lo
        elif d:
            d_only += hi - lo
        elif h:
            h_only += hi - lo
    return d_only, h_only, both


def fit_dma_slowdown(trace, device: int, base_seconds: dict, fallback: DmaSlowdown | None = None,
                     min_mass: float = 2.0) -> DmaSlowdown:
    """In-situ DMA slowdown from a MEASURED run: every compute pass of ``device`` gives
    duration / base - 1 = s_d2h * f_d2h + s_h2d * f_h2d + s_duplex * f_both, with f the
    fractions of the pass overlapping D2H only, H2D only and both directions
    (``_overlaps`` on the measured trace) and ``base_seconds[kind]`` the same pass kind's
    mean duration without offload.  Least squares per pass kind (F, B, W), clipped to
    [0, 1]; a direction whose overlap sums to fewer than ``min_mass`` whole passes (too
    little signal against run-to-run noise) keeps ``fallback``'s value."""
    import numpy as np

    xfer = [(float(p.start), float(p.end), p.kind) for p in trace.transfer_passes() if p.device == device]
    rows: dict = {}
    for p in trace.compute_passes():
        if p.device != device or str(p.kind) not in base_seconds:
            continue
        a, b = float(p.start), float(p.end)
        if b <= a:
            continue
        od, oh, ox = _overlaps(a, b, xfer)
        rows.setdefault(p.kind, []).append(((od / (b - a), oh / (b - a), ox / (b - a)),
                                            (b - a) / base_seconds[str(p.kind)] - 1))
    fb = fallback or DmaSlowdown()
    fitted = {}
    for kind in (PassKind.F, PassKind.B, PassKind.W):
        data = rows.get(kind, [])
        X = np.array([x for x, _ in data], dtype=float).reshape(-1, 3)
        y = np.array([v for _, v in data], dtype=float)
        if len(data) < 3 or X.sum() == 0:
            fitted[kind] = fb.of(kind)
            continue
        coef = []
        for j in range(3):  # a direction overlapped by < min_mass pass-equivalents keeps the fallback
            coef.append(None if X[:, j].sum() < min_mass else 0.0)
        cols = [j for j in range(3) if coef[j] is not None]
        if cols:
            sol, *_ = np.linalg.lstsq(X[:, cols], y, rcond=None)
            for j, v in zip(cols, sol):
                coef[j] = min(1.0, max(0.0, float(v)))
        fitted[kind] = tuple(fb.of(kind)[j] if coef[j] is None else coef[j] for j in range(3))
    return DmaSlowdown(fitted[PassKind.F], fitted[PassKind.B], fitted[PassKind.W])


def link_factors(trace, plan: OffloadPlan, device: int) -> tuple[float, float]:
    """Measured / planned duration of the D2H and H2D transfers of ``device`` in a
    measured run of ``plan`` (1.0 where the device moved nothing): how much slower the
    host link ran in situ -- under duplex load and beside compute -- than the calibrated
    copy the plan's slots were sized with."""
    planned = {(t.direction, t.stage, t.microbatch): float(t.duration)
               for stm in plan.streams for t in stm.transfers if t.device == device}
    out = []
    for kind in (PassKind.OFFLOAD, PassKind.RELOAD):
        got = [(float(p.duration), planned[(kind, p.stage, p.microbatch)]) for p in trace.transfer_passes()
               if p.device == device and p.kind == kind and (kind, p.stage, p.microbatch) in planned]
        out.append(sum(g for g, _ in got) / sum(w for _, w in got) if got else 1.0)
    return out[0], out[1]


def scale_transfers(plan: OffloadPlan, f_d2h: float, f_h2d: float) -> OffloadPlan:
    """The same plan (slots, order, floors) with every transfer's duration scaled by the
    measured link factor of its direction: what the runner model needs to price stalls
    when the link runs slower than planned."""
    from dataclasses import replace

    def scaled(t):
        f = f_d2h if t.direction == PassKind.OFFLOAD else f_h2d
        return replace(t, duration=Fraction(t.duration * Fraction(f).limit_denominator(10**6)))

    return replace(plan, streams=tuple(replace(stm, transfers=tuple(scaled(t) for t in stm.transfers))
                                       for stm in plan.streams))


def dma_adjusted_end(trace, device: int, dma: DmaSlowdown | None) -> float:
    """End of ``device``'s last compute pass with every pass stretched by the measured
    slowdown for the copy traffic it overlaps (first order: a device that computes
    back to back is delayed by the sum of its passes' stretches)."""
    comp = [p for p in trace.compute_passes() if p.device == device]
    if not comp:
        return 0.0
    end = float(max(p.end for p in comp))
    if dma is None:
        return end
    xfer = [(float(p.start), float(p.end), p.kind) for p in trace.transfer_passes() if p.device == device]
    extra = 0.0
    for p in comp:
        sd, sh, sx = dma.of(p.kind)
        od, oh, ox = _overlaps(float(p.start), float(p.end), xfer)
        extra += od * sd + oh * sh + ox * sx
    return end + extra


def modelled_overheads(sched: Schedule, plan, device: int, dma: DmaSlowdown | None = None,
                       stream_mode: str = "single", base=None, link: tuple | None = None) -> dict:
    """Modelled overhead of ``plan`` at ``device`` versus no offload: the reference runner
    model alone, and with the measured DMA slowdown (``dma_adjusted_end``); ``link`` =
    (D2H, H2D) measured link factors (``link_factors``) stretch the plan's transfers."""
    base = base or simulate(sched, stream_mode=stream_mode)
    if link is not None:
        plan = scale_transfers(plan, *link)
    tr = simulate(sched, plan, stream_mode=stream_mode)
    b = dma_adjusted_end(base, device, None)
    return {"model": dma_adjusted_end(tr, device, None) / b - 1,
            "model_dma": dma_adjusted_end(tr, device, dma) / b - 1 if dma is not None else None}


@dataclass(frozen=True)
class PolicyChoice:
    plan: OffloadPlan | None
    stride: int | None
    makespan: Fraction
    base_makespan: Fraction
    peak_units: tuple[int, ...]
    base_peak_units: tuple[int, ...]
    offloaded_pairs: int

    @property
    def overhead(self) -> float:
        return float(self.makespan / self.base_makespan - 1)


def _peaks(trace) -> tuple[int, ...]:
    return tuple(u for u, _ in peak_memory(trace)["per_device"])


def choose_offload(
    sched: Schedule,
    stages,
    t_o: Fraction,
    tolerance: float = 0.05,
    focus_rank: int | None = None,
    stream_mode: str = "single",
    max_stride: int | None = None,
    dma: DmaSlowdown | None = None,
) -> PolicyChoice:
    """Least-peak stride plan within ``tolerance`` of no offload.  With ``dma`` (and a
    ``focus_rank``) the overhead is the DMA-aware one of ``modelled_overheads``."""
    base = simulate(sched, stream_mode=stream_mode)
    base_peaks = _peaks(base)
    best = PolicyChoice(None, None, base.makespan, base.makespan, base_peaks, base_peaks, 0)

    def score(peaks):
        return peaks[focus_rank] if focus_rank is not None else max(peaks)

    limit = base.makespan * (1 + Fraction(tolerance).limit_denominator(10_000))
    for q in range(1, (max_stride or sched.microbatches) + 1):
        pairs = {(s, j) for s in range(sched.num_stages) for j in range(sched.microbatches) if j % q == 0}
        plan = plan_slots(sched, stages, t_o, pairs=pairs)
        if plan.late_list() or not plan.offloaded_pairs():
            continue
        tr = simulate(sched, plan, stream_mode=stream_mode)
        if tr.makespan > limit:
            continue
        if dma is not None and focus_rank is not None:
            over = dma_adjusted_end(tr, focus_rank, dma) / dma_adjusted_end(base, focus_rank, None) - 1
            if over > tolerance:
                continue
        peaks = _peaks(tr)
        if score(peaks) < score(best.peak_units):
            best = PolicyChoice(plan, q, tr.makespan, base.makespan, peaks, base_peaks, len(plan.offloaded_pairs()))
    return best


def offload_candidates_by_memory(sched: Schedule, stages, t_o: Fraction, focus_rank: int | None = None,
                                 stream_mode: str = "single", max_stride: int | None = None,
                                 planner=None) -> list[PolicyChoice]:
    """Every stride plan without late reloads that lowers the peak (at ``focus_rank``,
    else the max over ranks), least memory first, then least modelled time.
    ``planner(sched, stages, t_o, pairs)`` builds a plan (default ``plan_slots``; e.g.
    ``plan_slots_duplex`` with its one-way width for dual copy streams)."""
    planner = planner or (lambda sc, st, t, pairs: plan_slots(sc, st, t, pairs=pairs))
    base = simulate(sched, stream_mode=stream_mode)
    base_peaks = _peaks(base)

    def score(peaks):
        return peaks[focus_rank] if focus_rank is not None else max(peaks)

    out = []
    for q in range(1, (max_stride or sched.microbatches) + 1):
        pairs = {(s, j) for s in range(sched.num_stages) for j in range(sched.microbatches) if j % q == 0}
        plan = planner(sched, stages, t_o, pairs)
        if plan.late_list() or not plan.offloaded_pairs():
            continue
        tr = simulate(sched, plan, stream_mode=stream_mode)
        peaks = _peaks(tr)
        if score(peaks) < score(base_peaks):
            out.append(PolicyChoice(plan, q, tr.makespan, base.makespan, peaks, base_peaks,
                                    len(plan.offloaded_pairs())))
    return sorted(out, key=lambda c: (score(c.peak_units), c.makespan))


@dataclass(frozen=True)
class MeasuredChoice:
    choice: PolicyChoice | None  # None: nothing measured within tolerance (keep everything resident)
    measured_overhead: float | None
    trials: tuple  # (stride, modelled overhead, measured overhead) per run, in order


def choose_offload_measured(sched: Schedule, stages, t_o: Fraction, measure, tolerance: float = 0.05,
                            focus_rank: int | None = None, stream_mode: str = "single",
                            max_stride: int | None = None, max_trials: int = 4,
                            model_tolerance: float = 0.25, planner=None,
                            dma: DmaSlowdown | None = None, dma_slack: float = 0.02) -> MeasuredChoice:
    """Least-memory stride plan whose *measured* overhead is within ``tolerance``.

    ``measure(plan) -> float`` runs the plan on the device and returns its overhead
    versus no offload.  Candidates are tried least memory first, at most
    ``max_trials`` runs; one whose modelled overhead alone exceeds ``model_tolerance``
    is never run.  After each miss the unmodelled cost is taken as proportional to the
    traffic (measured-minus-modelled overhead per offloaded pair, the smallest seen so
    far), and candidates predicted above ``tolerance`` by it are skipped: the device
    pays for concurrent DMA even where the model schedules the copies for free.  With
    ``dma`` (measured slowdowns) candidates whose DMA-aware modelled overhead exceeds
    ``tolerance + dma_slack`` are not run at all."""
    cands = [c for c in offload_candidates_by_memory(sched, stages, t_o, focus_rank, stream_mode, max_stride, planner)
             if c.overhead <= model_tolerance]
    if dma is not None and focus_rank is not None:
        base = simulate(sched, stream_mode=stream_mode)
        b_end = dma_adjusted_end(base, focus_rank, None)
        cands = [c for c in cands
                 if dma_adjusted_end(simulate(sched, c.plan, stream_mode=stream_mode), focus_rank, dma) / b_end - 1
                 <= tolerance + dma_slack]
    trials = []
    per_pair = None  # unmodelled overhead per offloaded pair
    for c in cands:
        if len(trials) >= max_trials:
            break
        if per_pair is not None and c.overhead + per_pair * c.offloaded_pairs > tolerance:
            continue
        m = float(measure(c.plan))
        trials.append((c.stride, c.overhead, m))
        if m <= tolerance:
            return MeasuredChoice(c, m, tuple(trials))
        g = max(0.0, m - c.overhead) / c.offloaded_pairs
        per_pair = g if per_pair is None else min(per_pair, g)
    return MeasuredChoice(None, None, tuple(trials))


@dataclass(frozen=True)
class PartialChoice:
    """One partial-offload candidate: which tensors travel, the plan, and its modelled cost."""

    label: str
    tensors: tuple | None  # (local layer, name) that travel; None = the whole saved set
    off_bytes: int
    res_bytes: int
    plan: OffloadPlan | None
    stream_mode: str
    stride: int | None
    overhead: float
    off_peak: int  # arena slots of offload parts (modelled peak, pairs)
    res_peak: int  # arena slots of resident parts (= in-flight peak)

    @property
    def act_bytes(self) -> int:
        return self.off_peak * self.off_bytes + (self.res_peak * self.res_bytes if self.res_bytes else 0)


def choose_partial_offload(
    sched: Schedule,
    stages,
    t_o: Fraction,
    candidates,
    rank: int = 0,
    tolerance: float = 0.05,
    stream_modes=("single", "dual"),
    max_stride: int = 4,
    dma: DmaSlowdown | None = None,
) -> list[PartialChoice]:
    """Per-tensor partial offload (B200 extension).

    At k > 1 a pair's whole saved set cannot make the round trip inside its F->B
    window, but a fraction a of it can: its round trip is a * t_o.  Each candidate
    (label, tensors, off_bytes, res_bytes) names the tensors that travel (the
    offload part) and the bytes that stay (the resident part).  For every candidate,
    stream discipline (one copy stream with the reference's ``plan_slots`` grid, or
    duplex streams with ``plan_slots_duplex``) and microbatch stride q, the reference
    runner model prices the plan at t_o * a; the resident parts stay from F start to
    the pair's last use, so rank ``rank`` holds

        off_peak * off_bytes + res_peak * res_bytes

    with off_peak the modelled peak of the offload parts and res_peak the in-flight
    peak.  Returns every candidate within ``tolerance`` of no offload, least
    activation bytes first (the no-offload baseline last)."""
    from .offload import plan_slots_duplex

    base = simulate(sched)
    res_peak = base.memory.peak(rank) // sched.units_per_stage
    units = sched.units_per_stage
    limit = base.makespan * (1 + Fraction(tolerance).limit_denominator(10_000))
    out = []
    for label, tensors, off_b, res_b in candidates:
        slab = off_b + res_b
        t_a = Fraction(t_o) * Fraction(off_b, slab)
        t_a = Fraction(max(1, round(t_a * 10**6)), 10**6)  # integer microseconds (costs.measured_pass_costs)
        for mode in stream_modes:
            for q in range(1, max_stride + 1):
                pairs = {(s, j) for s in range(sched.num_stages) for j in range(sched.microbatches) if j % q == 0}
                if mode == "single":
                    plan = plan_slots(sched, stages, t_a, pairs=pairs)
                else:
                    plan = plan_slots_duplex(sched, stages, t_a / 2, pairs=pairs)
                if plan.late_list() or not plan.offloaded_pairs():
                    continue
                tr = simulate(sched, plan, stream_mode=mode)
                if tr.makespan > limit:
                    continue
                over = float(tr.makespan / base.makespan - 1)
                if dma is not None:  # the DMA-aware overhead at ``rank`` must fit too
                    over = max(over, dma_adjusted_end(tr, rank, dma) / dma_adjusted_end(base, rank, None) - 1)
                    if over > tolerance:
                        continue
                off_peak = tr.memory.peak(rank) // units
                out.append(PartialChoice(label, tensors, off_b, res_b, plan, mode, q, over, off_peak, res_peak))
    out.sort(key=lambda c: (c.act_bytes, c.overhead))
    return out
