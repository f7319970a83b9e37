"""End-to-end pipelined runs on one B200 (all ranks of the schedule as virtual
ranks in one process, boundary through the local channel).

C1 (BASELINE.json configs[0]): tiny GPT, 4 layers, h=256, s=512, PP=4, 1F1B,
8 microbatches, full offload at k=1/2 (build_1f1b_full_offload(4, 8, unit, 3/2)).
Bars:
* op order executed on every rank == Schedule.device_passes (reference order);
* copy-stream order == OffloadPlan slot order (no late reloads at k=1/2);
* every offloaded slab reloads bit-exact (integer digests, in situ);
* loss and every gradient within the bars of tests/helpers/parity.py of the
  serial fp32 oracle (loss 2e-4 relative; gradients 1.2e-2 relative L2 per matrix,
  2e-2 per LayerNorm vector -- just above the bf16-storage noise floor);
* offload on vs off: same loss to 1e-3 relative (only nondeterministic atomics
  and cuDNN's dQ accumulation differ).
"""

from fractions import Fraction

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2503_01328_b200 as po  # noqa: E402
from helpers.parity import violations  # noqa: E402
from oracle import gpt as oracle_gpt  # noqa: E402
from paper_2503_01328_b200.runtime import executor as ex  # noqa: E402
from paper_2503_01328_b200.runtime.model import ModelConfig  # noqa: E402

CFG = ModelConfig(n_layers=4, hidden=256, heads=4, seq=512, vocab=1024)
OCFG = oracle_gpt.GPTConfig(n_layers=4, hidden=256, heads=4, seq=512, vocab=1024)


def rel(a, b):
    return float((a - b).norm() / (b.norm() + 1e-12))


@pytest.fixture(scope="module")
def oracle_result():
    tokens = oracle_gpt.make_tokens(OCFG, 8, seed=0)
    params = oracle_gpt.init_params(OCFG, seed=1234)
    loss, _, grads = oracle_gpt.forward_backward(OCFG, params, tokens)
    return tokens, loss, grads


def _grads(res):
    out = {}
    for r in res.runners:
        for st in r.stages.values():
            for k, g in st.g.items():
                out[k] = g.float().cpu()
    return out


def test_c1_full_offload_matches_oracle(oracle_result):
    tokens, want_loss, want_grads = oracle_result
    U = po.PassCosts.unit()
    sched, plan = po.build_1f1b_full_offload(4, 8, U, Fraction(3, 2))
    res = ex.execute(sched, plan, model=CFG, mode="virtual", tokens=tokens, optimizer="none", verify_roundtrip=True)
    # op-order parity with the reference schedule and plan
    for r, prog in res.programs.items():
        assert prog.compute_order == [(str(p.kind), p.stage, p.microbatch) for p in sched.device_passes[r]]
        want_copy = [(("OFFLOAD" if t.direction == po.PassKind.OFFLOAD else "RELOAD"), t.stage, t.microbatch)
                     for t in plan.streams[r].transfers]
        assert prog.copy_order.get("copy", []) == want_copy
    assert res.peak_slabs == {0: 2, 1: 2, 2: 2, 3: 1}
    assert ex.roundtrip_mismatches(res.runners) == []
    n_offloaded = sum(len(p.offloaded) for p in res.programs.values())
    assert n_offloaded == 24
    assert violations(res.losses[-1], want_loss, _grads(res), want_grads) == []
    # measured trace is a SimTrace: the reference's metrics apply
    pk = po.peak_memory(res.trace)
    assert [u for u, _ in pk["per_device"]] == [2, 2, 2, 1]


def test_c1_offload_equals_no_offload(oracle_result):
    tokens, _, _ = oracle_result
    U = po.PassCosts.unit()
    sched, plan = po.build_1f1b_full_offload(4, 8, U, Fraction(3, 2))
    on = ex.execute(sched, plan, model=CFG, mode="virtual", tokens=tokens, optimizer="none")
    off = ex.execute(sched, None, model=CFG, mode="virtual", tokens=tokens, optimizer="none")
    assert off.peak_slabs == {0: 4, 1: 3, 2: 2, 3: 1}
    assert abs(on.losses[-1] - off.losses[-1]) < 1e-3 * abs(off.losses[-1])
    g_on, g_off = _grads(on), _grads(off)
    for k in g_off:
        assert rel(g_on[k], g_off[k]) < 1e-3, k


def test_interleaved_selective_offload_runs():
    """1F1B-I d=2 v=2 m=4, first local stage offloaded (select_offload_stages on po_block)."""
    cfg = ModelConfig(n_layers=4, hidden=256, heads=4, seq=512, vocab=1024)
    U = po.PassCosts.unit()
    sched = po.build_interleaved_1f1b(2, 2, 4, U)
    stages = po.select_offload_stages(po.po_block(2, 2, U), 1)
    plan = po.plan_slots(sched, stages, Fraction(1, 2))
    res = ex.execute(sched, plan, model=cfg, mode="virtual", optimizer="none", verify_roundtrip=True)
    assert ex.roundtrip_mismatches(res.runners) == []
    assert sum(len(p.offloaded) for p in res.programs.values()) > 0
    off = ex.execute(sched, None, model=cfg, mode="virtual", optimizer="none")
    assert abs(res.losses[-1] - off.losses[-1]) < 1e-3 * abs(off.losses[-1])


def test_cuda_graph_replay_matches_eager(oracle_result):
    """Passes captured once per (pass, slab, boundary buffer) and replayed for later
    microbatches / iterations give the same training trajectory as eager issue."""
    tokens, _, _ = oracle_result
    U = po.PassCosts.unit()
    sched, plan = po.build_1f1b_full_offload(4, 8, U, Fraction(3, 2))
    kw = dict(model=CFG, mode="virtual", tokens=tokens, optimizer="sgd", lr=1e-2, iters=3, warmup=0)
    eager = ex.execute(sched, plan, use_graphs=False, **kw)
    graph = ex.execute(sched, plan, use_graphs=True, verify_roundtrip=True, **kw)
    assert sum(len(r.graphs) for r in graph.runners) > 0
    assert ex.roundtrip_mismatches(graph.runners) == []
    for a, b in zip(eager.losses, graph.losses):
        assert abs(a - b) < 1e-3 * abs(a), (eager.losses, graph.losses)
    assert graph.losses[-1] < graph.losses[0]  # SGD at lr 1e-2 makes progress


@pytest.mark.parametrize("kind", ["gis-h", "po"])
def test_split_backward_schedules_match_oracle(kind, oracle_result):
    """GIS-H and PO (the paper's own schedule family) run B and W as separate passes
    (dgrad now, weight gradients later); with first-local-stage offload they must still
    reproduce the serial oracle's loss and gradients."""
    tokens, want_loss, want_grads = oracle_result
    U = po.PassCosts.unit()
    sched = (po.build_gis_h if kind == "gis-h" else po.build_po)(2, 2, 8, U)
    assert sched.split_backward
    plan = po.plan_slots(sched, po.select_offload_stages(po.po_block(2, 2, U), 1), Fraction(1))
    res = ex.execute(sched, plan, model=CFG, mode="virtual", tokens=tokens, optimizer="none", verify_roundtrip=True)
    assert ex.roundtrip_mismatches(res.runners) == []
    assert sum(p.n_wbufs for p in res.programs.values()) > 0
    assert violations(res.losses[-1], want_loss, _grads(res), want_grads) == []


def _variant(name):
    """(schedule, plan, stream_mode) of the plan variants the engine must run exactly."""
    from paper_2503_01328_b200.offload import plan_slots_duplex
    from paper_2503_01328_b200.policy import choose_offload

    U = po.PassCosts.unit()
    if name == "late_reloads_k2":  # k = 2: reloads miss their slots (sim floors them later)
        sched = po.build_1f1b(4, 1, 8, U)
        plan = po.plan_slots(sched, (0,), Fraction(6))
        assert plan.late_list()
        return sched, plan, "single"
    if name == "dual_streams":
        sched, plan = po.build_1f1b_full_offload(4, 8, U, Fraction(3, 2))
        return sched, plan, "dual"
    if name == "duplex_plan":
        sched = po.build_1f1b(4, 1, 8, U)
        return sched, plan_slots_duplex(sched, (0,), Fraction(3, 2)), "dual"
    if name == "k_aware_stride":  # every 2nd microbatch offloaded (k = 4 / 3)
        sched = po.build_1f1b(8, 1, 16, U)
        choice = choose_offload(sched, (0,), Fraction(4), tolerance=0.05, focus_rank=0)
        assert choice.plan is not None and choice.stride > 1
        return sched, choice.plan, "single"
    if name == "pp1_all_skipped":  # d = 1: zero F->B window, every pair skips (builders.py:252-253)
        sched, plan = po.build_1f1b_full_offload(1, 4, U, Fraction(3, 2))
        assert not plan.offloaded_pairs()
        return sched, plan, "single"
    if name == "m_not_multiple_of_d":
        sched, plan = po.build_1f1b_full_offload(4, 6, U, Fraction(3, 2))
        return sched, plan, "single"
    if name == "topology_synced":  # paired devices' transfers ordered by cross-rank flags, pinned floors
        sched, plan = po.build_1f1b_full_offload(4, 8, U, Fraction(3, 2))
        hw = po.HardwareSpec(compute_bandwidth=1.0, transfer_bandwidth=1.0, devices_per_switch=2)
        plan = po.apply_topology_sync(plan, hw)
        assert plan.sync_edges and plan.pinned
        return sched, plan, "single"
    if name == "gis_g":
        sched = po.build_gis_g(4, 2, 8, 3, U)
        assert sched.kind == "gis-g"
        plan = po.plan_slots(sched, po.select_offload_stages(po.po_block(4, 2, U), 1), Fraction(2))
        return sched, plan, "single"
    raise KeyError(name)


@pytest.mark.parametrize("name", ["late_reloads_k2", "dual_streams", "duplex_plan", "k_aware_stride",
                                  "pp1_all_skipped", "m_not_multiple_of_d", "gis_g", "topology_synced"])
def test_plan_variants_exact(name, oracle_result):
    """Every plan shape the planner can emit runs with bit-exact round trips, and the
    first step's loss is bit-identical to the same schedule without offload (the
    forward is a pure function of weights, tokens and Philox seeds)."""
    sched, plan, mode = _variant(name)
    m = sched.microbatches
    cfg = CFG if sched.num_stages <= 4 else ModelConfig(n_layers=sched.num_stages, hidden=256, heads=4, seq=512,
                                                       vocab=1024)
    tokens = torch.randint(0, cfg.vocab, (m, cfg.seq + 1), generator=torch.Generator().manual_seed(m))
    kw = dict(model=cfg, mode="virtual", tokens=tokens, optimizer="none", iters=1, warmup=0)
    on = ex.execute(sched, plan, stream_mode=mode, verify_roundtrip=True, **kw)
    off = ex.execute(sched, None, **kw)
    assert ex.roundtrip_mismatches(on.runners) == []
    assert on.losses[0] == off.losses[0]
    g_on, g_off = _grads(on), _grads(off)
    for k in g_off:
        assert rel(g_on[k], g_off[k]) < 1e-3, k
    if plan.offloaded_pairs():
        assert sum(len(p.offloaded) for p in on.programs.values()) == len(plan.offloaded_pairs())


@pytest.mark.parametrize("tensors", [((0, "f"),), ((0, "f"), (0, "qkv"), (0, "o"))])
def test_c1_partial_offload_matches_oracle(oracle_result, tensors):
    """Per-tensor partial offload (layout.make_layout(offload=...)): only the named
    tensors travel (bit-exact round trip of the offload part), the resident part
    stays in its own arena; the run matches the oracle like full offload does."""
    tokens, want_loss, want_grads = oracle_result
    U = po.PassCosts.unit()
    sched, plan = po.build_1f1b_full_offload(4, 8, U, Fraction(3, 2))
    res = ex.execute(sched, plan, model=CFG, mode="virtual", tokens=tokens, optimizer="none", verify_roundtrip=True,
                     offload_tensors=tensors)
    assert ex.roundtrip_mismatches(res.runners) == []
    assert sum(len(p.offloaded) for p in res.programs.values()) == 24
    assert 0 < res.offload_fraction < 1
    for r in res.runners:
        lay = next(iter(r.stages.values())).layout
        assert r.act_bytes == r.prog.n_slabs * r.off_bytes + r.prog.n_res_slabs * r.res_bytes
        assert r.prog.n_res_slabs == [4, 3, 2, 1][r.rank]  # in-flight peak (no-offload arena)
        assert lay.host_bytes < lay.slab_bytes
    assert violations(res.losses[-1], want_loss, _grads(res), want_grads) == []


@pytest.mark.parametrize("mode,stream_mode", [("virtual", "single"), ("emulate", "dual")])
def test_whole_iteration_graph(oracle_result, mode, stream_mode):
    """execute(iteration_graph=True): one CUDA graph per iteration (every stream, event
    edge, pass, D2H/H2D and the SGD step) replays with the same results as the per-pass
    issue path: bit-exact round trips, same losses over 3 SGD steps (to the LN-bwd
    atomics' nondeterminism), every pass timed from inside the graph."""
    tokens, _, _ = oracle_result
    U = po.PassCosts.unit()
    sched, plan = po.build_1f1b_full_offload(4, 8, U, Fraction(3, 2))
    kw = dict(model=CFG, mode=mode, rank=0, tokens=tokens, optimizer="sgd", lr=1e-2, iters=3, warmup=1,
              stream_mode=stream_mode, verify_roundtrip=True)
    ref = ex.execute(sched, plan, **kw)
    got = ex.execute(sched, plan, iteration_graph=True, **kw)
    assert "iteration" in got.runners[0].graph_native_launches
    assert ex.roundtrip_mismatches(got.runners) == []
    if mode == "virtual":
        for a, b in zip(got.losses, ref.losses):
            assert abs(a - b) < 1e-3 * abs(b), (got.losses, ref.losses)
        assert got.losses[-1] < got.losses[0]  # SGD steps inside the graph take effect
    n_passes = sum(len(p.compute_order) for p in got.programs.values())
    assert len(got.trace.compute_passes()) == n_passes
    assert all(p.duration > 0 for p in got.trace.passes)
    assert 0 < got.iteration_seconds[-1] < 10
    got.close()
    ref.close()


def test_topology_synced_plan_in_iteration_graph(oracle_result):
    """Sync-edge flags (cuStreamWaitValue32 / WriteValue32 on the copy streams) inside
    the one-graph-per-iteration replay: same losses as the host-issued run over 3 SGD
    steps, bit-exact round trips, flags back to 0 after every iteration."""
    tokens, _, _ = oracle_result
    sched, plan, _m = _variant("topology_synced")
    kw = dict(model=CFG, mode="virtual", tokens=tokens, optimizer="sgd", lr=1e-2, iters=3, warmup=1,
              verify_roundtrip=True, gemm="tcgen05", attn="tcgen05")
    ref = ex.execute(sched, plan, **kw)
    got = ex.execute(sched, plan, iteration_graph=True, **kw)
    assert "iteration" in got.runners[0].graph_native_launches
    assert ex.roundtrip_mismatches(got.runners) == []
    for a, b in zip(got.losses, ref.losses):
        assert abs(a - b) < 1e-3 * abs(b), (got.losses, ref.losses)
    assert int(got.runners[0].flags.tensor.abs().sum()) == 0
    got.close()
    ref.close()
