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
