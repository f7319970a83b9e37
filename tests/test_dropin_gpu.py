"""The drop-in runner: ``execute`` with ``simulate``'s signature (reference sim.py:141-149)
returning a SimTrace of measured times, and ``runner(...)`` bound into code written
against the reference runner (the call pattern of analysis.reduction_curve,
analysis.py:142-181: ``simulate(sched)``, ``simulate(sched, plan)``, then
``peak_memory(trace)["per_device"][0][0]``)."""

from fractions import Fraction

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2503_01328_b200 as po  # noqa: E402
from paper_2503_01328_b200.runtime.model import ModelConfig  # noqa: E402

CFG = ModelConfig(n_layers=4, hidden=256, heads=4, seq=512, vocab=1024)


def test_execute_has_simulate_signature_and_returns_simtrace():
    U = po.PassCosts.unit()
    sched, plan = po.build_1f1b_full_offload(4, 8, U, Fraction(3, 2))
    spec = po.ModelSpec(256, 512, 1, 1)
    tr = po.execute(sched, plan, U, None, None, spec, "single", iters=1, gemm="tcgen05", attn="tcgen05")
    assert isinstance(tr, po.SimTrace) and isinstance(tr, po.MeasuredTrace)
    # the measured trace feeds the reference's metrics; the planned peaks are realised
    assert [u for u, _ in po.peak_memory(tr)["per_device"]] == [2, 2, 2, 1]
    assert [u for u, _ in po.peak_memory(tr.predicted)["per_device"]] == [2, 2, 2, 1]
    assert len(tr.compute_passes()) == len(tr.predicted.compute_passes())
    assert all(p.duration > 0 for p in tr.passes)
    assert tr.run.losses and tr.run.mem["alloc_peak_bytes"] > 0
    summary = tr.summary()
    assert summary["makespan"] and tr.to_csv().startswith("device,stage")
    tr.run.close()
    with pytest.raises(ValueError):
        po.execute(sched, plan)  # no model: nothing to train


def test_runner_drives_reduction_curve_call_pattern():
    """Peak memory versus number of offloaded stages, n = 0..v (reduction_curve's loop),
    computed from MEASURED traces: the measured peaks equal the runner model's, and
    offloading more local stages never raises the rank-0 peak."""
    simulate = po.runner(config=CFG, iters=1, gemm="tcgen05", attn="tcgen05")
    U = po.PassCosts.unit()
    d, v, m = 2, 2, 8
    sched = po.build_po(d, v, m, U)
    block = po.po_block(d, v, U)
    peaks, model_peaks = [], []
    for n in range(v + 1):
        stages = po.select_offload_stages(block, n)
        if n == 0:
            trace, plan = simulate(sched), None
        else:
            plan = po.plan_slots(sched, stages, Fraction(1))
            trace = simulate(sched, plan)
        peaks.append(po.peak_memory(trace)["per_device"][0][0])
        model_peaks.append(po.peak_memory(po.simulate(sched, plan))["per_device"][0][0])
    assert peaks == model_peaks
    assert peaks[-1] <= peaks[0]


def test_d1_interleaved_runs_locally():
    """d = 1, v = 2 (consecutive stages on one device): boundary messages stay local."""
    U = po.PassCosts.unit()
    sched = po.build_interleaved_1f1b(1, 2, 4, U)
    cfg = ModelConfig(n_layers=2, hidden=256, heads=4, seq=512, vocab=1024)
    tokens = torch.randint(0, cfg.vocab, (4, cfg.seq + 1), generator=torch.Generator().manual_seed(0))
    tr = po.execute(sched, None, config=cfg, tokens=tokens, iters=1, gemm="tcgen05", attn="tcgen05")
    ref = po.execute(po.build_1f1b(1, 2, 4, U), None, config=cfg, tokens=tokens, iters=1, gemm="tcgen05",
                     attn="tcgen05")
    # the same model in two chunks or one merged stage: same first-step loss
    assert tr.run.losses[0] == pytest.approx(ref.run.losses[0], rel=1e-4)
    tr.run.close()
    ref.run.close()
