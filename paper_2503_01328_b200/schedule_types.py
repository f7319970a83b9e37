"""Value types of the schedule IR (reference ``pkg/src/ppoff/ir.py:19-169``).

Every object is a frozen dataclass with exact ``Fraction`` times, so two
schedules built from the same costs compare equal field by field -- the property
the B200 executor's op-order parity tests rely on.

One *unit* is the saved activation set of one (pipeline stage, microbatch); a
merged-stage schedule (1F1B holding v layer groups per device) carries
``units_per_stage`` units per pass.
"""

from __future__ import annotations

from dataclasses import dataclass
from enum import Enum
from fractions import Fraction

from .costs import PassCosts

__all__ = [
    "ScheduleError",
    "InfeasibleIntervalError",
    "PassKind",
    "KIND_RANK",
    "Pass",
    "BuildingBlock",
    "Schedule",
    "Violation",
    "lifespan",
]


class ScheduleError(Exception):
    """Malformed or unschedulable pass structure (reference ir.py:19-20)."""


class InfeasibleIntervalError(ScheduleError):
    """A uniform-repeat interval shorter than one microbatch's device work."""


class PassKind(str, Enum):
    F = "F"
    B = "B"
    W = "W"
    OFFLOAD = "OFFLOAD"
    RELOAD = "RELOAD"

    def __str__(self) -> str:
        return self.value


# Tie-break rank of compute kinds at equal start times.
KIND_RANK = {PassKind.F: 0, PassKind.B: 1, PassKind.W: 2}


@dataclass(frozen=True)
class Pass:
    kind: PassKind
    device: int
    stage: int
    microbatch: int
    start: Fraction
    duration: Fraction

    @property
    def end(self) -> Fraction:
        return self.start + self.duration

    @property
    def key(self) -> tuple:
        return (self.kind, self.stage, self.microbatch)


def _pass_length(costs: PassCosts, kind: PassKind, units: int, split: bool) -> Fraction:
    """Duration of one pass of ``kind``; an unsplit B also carries the W work."""
    if kind == PassKind.F:
        per_unit = costs.t_f
    elif kind == PassKind.W:
        per_unit = costs.t_w
    elif split:
        per_unit = costs.t_b
    else:
        per_unit = costs.t_b + costs.t_w
    return per_unit * units


@dataclass(frozen=True)
class BuildingBlock:
    """Start offsets of one microbatch's F/B(/W) passes on every stage.

    Stage ``s`` is hosted by device ``s % devices``; ``w_start`` is None when the
    backward pass is not split into B and W.
    """

    devices: int
    local_stages: int
    f_start: tuple[Fraction, ...]
    b_start: tuple[Fraction, ...]
    w_start: tuple[Fraction, ...] | None
    costs: PassCosts
    units: int = 1

    def __post_init__(self):
        n = self.num_stages
        if len(self.f_start) != n or len(self.b_start) != n:
            raise ScheduleError("offset arrays must cover devices*local_stages stages")
        if self.w_start is not None and len(self.w_start) != n:
            raise ScheduleError("w_start must cover all stages when present")
        f_len = self.duration(PassKind.F)
        b_len = self.duration(PassKind.B)
        for s in range(n):
            if self.b_start[s] < self.f_start[s] + f_len:
                raise ScheduleError(f"stage {s}: backward begins before its forward ends")
            if self.w_start is not None and self.w_start[s] < self.b_start[s] + b_len:
                raise ScheduleError(f"stage {s}: weight pass begins before its backward ends")
        for s in range(1, n):
            if self.f_start[s] < self.f_start[s - 1]:
                raise ScheduleError("forward offsets must be non-decreasing along the chain")
            if self.b_start[s] > self.b_start[s - 1]:
                raise ScheduleError("backward offsets must be non-increasing along the chain")

    @property
    def num_stages(self) -> int:
        return self.devices * self.local_stages

    @property
    def split_backward(self) -> bool:
        return self.w_start is not None

    def device_of(self, stage: int) -> int:
        return stage % self.devices

    def duration(self, kind: PassKind) -> Fraction:
        return _pass_length(self.costs, kind, self.units, self.split_backward)

    def span(self) -> Fraction:
        finish = max(self.b_start) + self.duration(PassKind.B)
        if self.w_start is not None:
            finish = max(finish, max(self.w_start) + self.duration(PassKind.W))
        return finish - min(self.f_start)


def lifespan(block: BuildingBlock, stage: int) -> Fraction:
    """Residency of one stage's activations inside the block: F start to B end."""
    if stage < 0 or stage >= block.num_stages:
        raise ScheduleError(f"stage {stage} out of range")
    return block.b_start[stage] + block.duration(PassKind.B) - block.f_start[stage]


@dataclass(frozen=True)
class Schedule:
    devices: int
    local_stages: int
    num_stages: int
    microbatches: int
    placement: tuple[int, ...]
    units_per_stage: int
    split_backward: bool
    costs: PassCosts
    kind: str = "custom"
    g: int | None = None
    interval: Fraction | None = None
    device_passes: tuple[tuple[Pass, ...], ...] = ()

    def all_passes(self):
        for per_device in self.device_passes:
            yield from per_device

    @property
    def makespan(self) -> Fraction:
        return max((p.end for p in self.all_passes()), default=Fraction(0))

    def busy(self, device: int) -> Fraction:
        return sum((p.duration for p in self.device_passes[device]), Fraction(0))

    def duration(self, kind: PassKind) -> Fraction:
        return _pass_length(self.costs, kind, self.units_per_stage, self.split_backward)

    def find(self, kind: PassKind, stage: int, microbatch: int) -> Pass:
        for p in self.device_passes[self.placement[stage]]:
            if (p.kind, p.stage, p.microbatch) == (kind, stage, microbatch):
                return p
        raise KeyError((kind, stage, microbatch))

    def local_stages_of(self, device: int) -> list[int]:
        """Global stage ids hosted by ``device`` in chunk order."""
        return [s for s, dev in enumerate(self.placement) if dev == device]


@dataclass(frozen=True)
class Violation:
    kind: str  # "dependency" | "overlap" | "missing" | "duplicate"
    message: str
    passes: tuple = ()
