"""Byte and time contract of the activation round trip (reference layer L0).

Mirrors the public surface of ``ppoff.costs`` (reference ``pkg/src/ppoff/costs.py``)
so planner callers can switch packages without edits:

* ``ModelSpec`` / ``HardwareSpec`` / ``PassCosts``      costs.py:34-96
* ``activation_bytes_per_layer``                          costs.py:99-105
* ``layer_output_ratio``                                  costs.py:108-113
* ``compute_k`` (Eq. (1) of the paper)                    costs.py:116-124
* ``offload_round_trip``                                  costs.py:127-136
* ``estimate_pass_costs``                                 costs.py:139-161
* ``PRESETS``                                             costs.py:165-172

The B200 runtime adds ``measured_pass_costs``: the same ``PassCosts`` object built
from CUDA-event timings instead of the FLOP model, so the planner runs on real
numbers.

Byte accounting (per layer, per microbatch, 2-byte elements): 34*b*s*h without
recompute, 20*b*s*h when LayerNorm, GeLU and the dropout masks are recomputed in
backward.  The saved set of the runtime's transformer layer is exactly the 20bsh
set: x, q, k, v, attention output, h1 (2bsh each) and fc1-out (8bsh).
"""

from __future__ import annotations

from dataclasses import dataclass
from fractions import Fraction

__all__ = [
    "ModelSpec",
    "HardwareSpec",
    "PassCosts",
    "activation_bytes_per_layer",
    "layer_output_ratio",
    "compute_k",
    "offload_round_trip",
    "estimate_pass_costs",
    "measured_pass_costs",
    "PRESETS",
]

# Per-element coefficients at the 2-byte baseline (kept rational).
COEFF_SAVED_ALL = Fraction(34)
COEFF_SAVED_RECOMPUTE = Fraction(20)
COEFF_LAYER_OUT = Fraction(2)


def as_fraction(value) -> Fraction:
    """Exact rational from an int, float (exact binary value), str or Fraction."""
    return value if isinstance(value, Fraction) else Fraction(value)


@dataclass(frozen=True)
class ModelSpec:
    """Shape of one pipeline stage: hidden h, sequence s, microbatch b, L layers."""

    hidden_size: int
    sequence_length: int
    microbatch_size: int = 1
    layers_per_stage: int = 1
    bytes_per_element: int = 2

    def __post_init__(self):
        checks = (
            ("hidden_size", self.hidden_size),
            ("sequence_length", self.sequence_length),
            ("microbatch_size", self.microbatch_size),
            ("layers_per_stage", self.layers_per_stage),
        )
        for label, val in checks:
            if val < 1:
                raise ValueError(f"{label} must be >= 1")
        if self.bytes_per_element not in (1, 2, 4):
            raise ValueError("bytes_per_element must be one of 1, 2, 4")

    @property
    def tokens(self) -> int:
        return self.microbatch_size * self.sequence_length


@dataclass(frozen=True)
class HardwareSpec:
    """Compute rate B_c (FLOP/s), one-direction host-link rate B_o (byte/s)."""

    compute_bandwidth: float
    transfer_bandwidth: float
    p2p_latency: float = 0.0
    devices_per_switch: int = 2
    host_memory_capacity: int | None = None

    def __post_init__(self):
        if not (self.compute_bandwidth > 0 and self.transfer_bandwidth > 0):
            raise ValueError("bandwidths must be positive")
        if self.p2p_latency < 0:
            raise ValueError("p2p_latency must be >= 0")
        if self.devices_per_switch < 1:
            raise ValueError("devices_per_switch must be >= 1")


@dataclass(frozen=True)
class PassCosts:
    """Exact per-stage, per-microbatch durations of F, B, W and the stage hop."""

    t_f: Fraction
    t_b: Fraction
    t_w: Fraction
    t_comm: Fraction = Fraction(0)

    def __post_init__(self):
        for name in ("t_f", "t_b", "t_w", "t_comm"):
            object.__setattr__(self, name, as_fraction(getattr(self, name)))
        if min(self.t_f, self.t_b, self.t_w, self.t_comm) < 0:
            raise ValueError("pass costs must be >= 0")
        if self.t_b + self.t_w <= 0:
            raise ValueError("backward cost must be positive")

    @property
    def total(self) -> Fraction:
        return self.t_f + self.t_b + self.t_w

    @staticmethod
    def unit() -> "PassCosts":
        return PassCosts(Fraction(1), Fraction(1), Fraction(1))


def _elements(model: ModelSpec) -> int:
    return model.microbatch_size * model.sequence_length * model.hidden_size


def activation_bytes_per_layer(model: ModelSpec, recompute: bool = False) -> int:
    """Saved-activation bytes of one layer for one microbatch (34bsh or 20bsh)."""
    coeff = COEFF_SAVED_RECOMPUTE if recompute else COEFF_SAVED_ALL
    nbytes = coeff * _elements(model) * Fraction(model.bytes_per_element, 2)
    if nbytes.denominator != 1:
        raise AssertionError("activation byte count must be integral")
    return int(nbytes)


def layer_output_ratio(model: ModelSpec) -> Fraction:
    """Offloaded payload over the stage-boundary message; 10 under this accounting."""
    boundary = COEFF_LAYER_OUT * _elements(model) * Fraction(model.bytes_per_element, 2)
    return Fraction(activation_bytes_per_layer(model, recompute=True)) / boundary


def compute_k(model: ModelSpec, hw: HardwareSpec) -> float:
    """Eq. (1): k = 10 / (3 (6h + s)) * B_c / B_o  (round trip over compute time)."""
    h, s = model.hidden_size, model.sequence_length
    return (10.0 / (3.0 * (6 * h + s))) * (hw.compute_bandwidth / hw.transfer_bandwidth)


def offload_round_trip(model: ModelSpec, hw: HardwareSpec) -> Fraction:
    """T_o: both directions of one stage payload, run back to back on the link."""
    payload = activation_bytes_per_layer(model, recompute=True) * model.layers_per_stage
    return 2 * Fraction(payload) / as_fraction(hw.transfer_bandwidth)


def estimate_pass_costs(
    model: ModelSpec,
    hw: HardwareSpec,
    ratios: tuple[float, float, float] = (1, 1, 1),
) -> PassCosts:
    """Split the FLOP model 12 b s h (6h + s) L / B_c into T_F : T_B : T_W."""
    if any(r < 0 for r in ratios) or sum(ratios) <= 0:
        raise ValueError("ratios must be non-negative with positive sum")
    b, s, h = model.microbatch_size, model.sequence_length, model.hidden_size
    flops = 12 * b * s * h * (6 * h + s) * model.layers_per_stage
    seconds = Fraction(flops) / as_fraction(hw.compute_bandwidth)
    weights = [as_fraction(r) for r in ratios]
    norm = sum(weights, Fraction(0))
    t_f, t_b, t_w = (seconds * w / norm for w in weights)
    return PassCosts(t_f=t_f, t_b=t_b, t_w=t_w, t_comm=as_fraction(hw.p2p_latency))


def measured_pass_costs(
    t_f_seconds: float,
    t_bw_seconds: float,
    t_w_seconds: float = 0.0,
    t_comm_seconds: float = 0.0,
    resolution: int = 1_000_000,
) -> PassCosts:
    """``PassCosts`` from measured CUDA-event times, quantised to 1/resolution s.

    Quantising to integer microseconds keeps the planner's ceil/floor slot
    arithmetic exact (reference offload.py:170,186) while staying within 1 us of
    the measurement.
    """

    def q(x: float) -> Fraction:
        return Fraction(max(0, round(x * resolution)), resolution)

    return PassCosts(q(t_f_seconds), q(t_bw_seconds), q(t_w_seconds), q(t_comm_seconds))


PRESETS = {
    name: ModelSpec(hidden_size=h, sequence_length=4096)
    for name, h in (
        ("5.8B", 4096),
        ("10.5B", 5120),
        ("18.1B", 6144),
        ("42.9B", 8192),
        ("66.6B", 10240),
        ("83.8B", 10240),  # reference keeps 83.8B identical to 66.6B (costs.py:170-171)
    )
}
