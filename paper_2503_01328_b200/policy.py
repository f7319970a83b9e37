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
from .schedule_types import Schedule
from .sim import peak_memory, simulate


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
) -> PolicyChoice:
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
                            model_tolerance: float = 0.25, planner=None) -> MeasuredChoice:
    """Least-memory stride plan whose *measured* overhead is within ``tolerance``.

    ``measure(plan) -> float`` runs the plan on the device and returns its overhead
    versus no offload.  Candidates are tried least memory first, at most
    ``max_trials`` runs; one whose modelled overhead alone exceeds ``model_tolerance``
    is never run.  After each miss the unmodelled cost is taken as proportional to the
    traffic (measured-minus-modelled overhead per offloaded pair, the smallest seen so
    far), and candidates predicted above ``tolerance`` by it are skipped: the device
    pays for concurrent DMA even where the model schedules the copies for free."""
    cands = [c for c in offload_candidates_by_memory(sched, stages, t_o, focus_rank, stream_mode, max_stride, planner)
             if c.overhead <= model_tolerance]
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
                off_peak = tr.memory.peak(rank) // units
                out.append(PartialChoice(label, tensors, off_b, res_b, plan, mode, q,
                                         float(tr.makespan / base.makespan - 1), off_peak, res_peak))
    out.sort(key=lambda c: (c.act_bytes, c.overhead))
    return out
