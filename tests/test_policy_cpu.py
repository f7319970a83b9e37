"""k-aware policy with measured feedback (policy.choose_offload_measured), against a
synthetic device whose measured overhead is the runner model's plus a fixed gap."""
from fractions import Fraction

import pytest

import paper_2503_01328_b200 as po
from paper_2503_01328_b200.policy import choose_offload, choose_offload_measured, offload_candidates_by_memory
from paper_2503_01328_b200.sim import simulate


def _setup():
    costs = po.measured_pass_costs(2.27e-3, 5.44e-3, 0.0, 50e-6)  # C5 h=8192 s=2048 per-layer costs
    sched = po.build_1f1b(8, 1, 16, costs)
    t_o = Fraction(12130, 1_000_000)  # k ~ 1.5
    return sched, t_o


def _modelled(sched, plan):
    base = simulate(sched).makespan
    return float(simulate(sched, plan).makespan / base - 1)


def test_candidates_sorted_by_memory_then_time():
    sched, t_o = _setup()
    cands = offload_candidates_by_memory(sched, (0,), t_o, focus_rank=0)
    assert cands
    keys = [(c.peak_units[0], c.makespan) for c in cands]
    assert keys == sorted(keys)
    assert all(not c.plan.late_list() and c.plan.offloaded_pairs() for c in cands)
    assert all(c.peak_units[0] < c.base_peak_units[0] for c in cands)  # every candidate saves memory


@pytest.mark.parametrize("gap", [0.02, 0.045, 0.06])
def test_measured_choice_meets_the_measured_budget(gap):
    sched, t_o = _setup()
    calls = []

    def measure(plan):  # the device pays `gap` per 8 offloaded pairs beyond the model
        calls.append(plan)
        return _modelled(sched, plan) + gap * len(plan.offloaded_pairs()) / 8

    got = choose_offload_measured(sched, (0,), t_o, measure, tolerance=0.05, focus_rank=0)
    assert len(calls) == len(got.trials) <= 4
    if got.choice is not None:
        assert got.measured_overhead <= 0.05
        # no candidate with less memory measures within budget
        for c in offload_candidates_by_memory(sched, (0,), t_o, focus_rank=0):
            if c.peak_units[0] < got.choice.peak_units[0]:
                assert _modelled(sched, c.plan) + gap * len(c.plan.offloaded_pairs()) / 8 > 0.05
    # the model-only policy may pick a plan the synthetic device measures above budget
    model_only = choose_offload(sched, (0,), t_o, tolerance=0.05, focus_rank=0)
    if model_only.plan is not None and got.choice is not None:
        assert got.choice.peak_units[0] >= model_only.peak_units[0]


def test_measured_choice_without_gap_equals_model_choice():
    sched, t_o = _setup()
    got = choose_offload_measured(sched, (0,), t_o, lambda plan: _modelled(sched, plan), tolerance=0.05,
                                  focus_rank=0, max_trials=100)
    want = choose_offload(sched, (0,), t_o, tolerance=0.05, focus_rank=0)
    assert (got.choice is None) == (want.plan is None)
    if want.plan is not None:
        assert got.choice.peak_units[0] == want.peak_units[0]


def test_dma_overlap_accounting():
    """policy._overlaps splits a pass into D2H-only / H2D-only / both seconds."""
    from paper_2503_01328_b200.policy import _overlaps
    from paper_2503_01328_b200.schedule_types import PassKind

    x = [(0.0, 4.0, PassKind.OFFLOAD), (2.0, 6.0, PassKind.RELOAD)]
    assert _overlaps(1.0, 5.0, x) == (1.0, 1.0, 2.0)
    assert _overlaps(6.0, 7.0, x) == (0.0, 0.0, 0.0)


def test_dma_adjusted_overhead_monotone():
    """Zero slowdown reproduces the runner model; a positive slowdown stretches exactly
    the compute that overlaps copies, and never makes a plan look cheaper."""
    from fractions import Fraction

    import paper_2503_01328_b200 as po
    from paper_2503_01328_b200.policy import DmaSlowdown, dma_adjusted_end, modelled_overheads

    U = po.PassCosts.unit()
    sched, plan = po.build_1f1b_full_offload(4, 8, U, Fraction(3, 2))
    tr = po.simulate(sched, plan)
    end = float(max(p.end for p in tr.compute_passes() if p.device == 0))
    assert dma_adjusted_end(tr, 0, None) == end
    assert dma_adjusted_end(tr, 0, DmaSlowdown()) == end
    slow = DmaSlowdown(f=(0.1, 0.1, 0.2), b=(0.3, 0.1, 0.4), w=(0.3, 0.1, 0.4))
    assert dma_adjusted_end(tr, 0, slow) > end
    m = modelled_overheads(sched, plan, 0, slow)
    assert m["model_dma"] > m["model"] >= 0
    # no transfers on the last rank (its window is zero): no stretch there
    tr3 = [p for p in tr.transfer_passes() if p.device == 3]
    assert not tr3 and dma_adjusted_end(tr, 3, slow) == dma_adjusted_end(tr, 3, None)


def test_choose_offload_respects_dma_model():
    """With a large measured slowdown the DMA-aware planner keeps fewer pairs (or none)."""
    from fractions import Fraction

    import paper_2503_01328_b200 as po
    from paper_2503_01328_b200.policy import DmaSlowdown, choose_offload

    U = po.PassCosts.unit()
    sched = po.build_1f1b(8, 1, 16, U)
    plain = choose_offload(sched, (0,), Fraction(3, 2), tolerance=0.05, focus_rank=0)
    heavy = choose_offload(sched, (0,), Fraction(3, 2), tolerance=0.05, focus_rank=0,
                           dma=DmaSlowdown(f=(0.5, 0.5, 0.9), b=(0.5, 0.5, 0.9), w=(0.5, 0.5, 0.9)))
    assert plain.plan is not None
    assert heavy.offloaded_pairs <= plain.offloaded_pairs


def test_fit_dma_slowdown_recovers_synthetic_stretch():
    """Passes that run entirely under D2H only / H2D only / both directions, stretched by
    known factors: the in-situ least-squares fit recovers the factors per pass kind."""
    from fractions import Fraction as Fr

    from paper_2503_01328_b200.policy import fit_dma_slowdown
    from paper_2503_01328_b200.schedule_types import Pass, PassKind

    OFF, REL = PassKind.OFFLOAD, PassKind.RELOAD
    xfers = [Pass(OFF, 0, 0, 0, Fr(0), Fr(100)), Pass(REL, 0, 0, 1, Fr(200), Fr(100)),
             Pass(OFF, 0, 0, 2, Fr(400), Fr(100)), Pass(REL, 0, 0, 3, Fr(400), Fr(100))]
    want = {PassKind.F: (0.2, 0.05, 0.3), PassKind.B: (0.25, 0.1, 0.4)}
    base = {"F": 1.0, "B": 2.0}
    comp = []
    for kind, factors in want.items():
        for region, f in zip((0, 200, 400), factors):
            for i in range(4):
                start = Fr(region + 10 + 20 * i + (5 if kind == PassKind.B else 0))
                comp.append(Pass(kind, 0, 0, i, start, Fr(base[str(kind)] * (1 + f)).limit_denominator(10**6)))
        comp.append(Pass(kind, 0, 0, 9, Fr(700), Fr(base[str(kind)])))  # no copies in flight
    trace = type("T", (), {"compute_passes": lambda self: comp, "transfer_passes": lambda self: xfers})()
    fit = fit_dma_slowdown(trace, 0, base)
    for kind, factors in want.items():
        for got, w in zip(fit.of(kind), factors):
            assert abs(got - w) < 1e-6, (kind, fit)
    assert fit.w == (0.0, 0.0, 0.0)  # no W passes: the fallback


def test_scaled_transfers_price_stalls():
    """A link running 4x slower than planned: the same plan, transfers stretched, makes
    the runner model predict the stall (reloads floor later, B waits)."""
    from fractions import Fraction

    import paper_2503_01328_b200 as po
    from paper_2503_01328_b200.policy import modelled_overheads, scale_transfers

    U = po.PassCosts.unit()
    sched, plan = po.build_1f1b_full_offload(4, 8, U, Fraction(3, 2))
    slow = scale_transfers(plan, 2.0, 2.0)
    assert [t.slot for s in slow.streams for t in s.transfers] == [t.slot for s in plan.streams for t in s.transfers]
    assert all(b.duration == 2 * a.duration for sa, sb in zip(plan.streams, slow.streams)
               for a, b in zip(sa.transfers, sb.transfers))
    m1 = modelled_overheads(sched, plan, 0)
    m2 = modelled_overheads(sched, plan, 0, link=(4.0, 4.0))  # k = 1/2: 2x still fits the window
    assert m2["model"] > m1["model"]
