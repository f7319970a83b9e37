"""Per-tensor partial offload, host side: slab layout split into offload / resident
parts, and the k-aware partial planner priced by the reference runner model."""

from fractions import Fraction

import pytest

import paper_2503_01328_b200 as po
from paper_2503_01328_b200.offload import pack_host_bins
from paper_2503_01328_b200.policy import choose_partial_offload
from paper_2503_01328_b200.runtime.layout import make_layout, offload_candidates
from paper_2503_01328_b200.sim import simulate


def test_full_layout_unchanged():
    lay = make_layout(3, 4096, 2048, 16)
    assert lay.res_bytes == 0 and lay.off_bytes == lay.slab_bytes == 504_102_912
    assert all(lay.travels(t) for t in lay.tensors)
    assert lay.payload_bytes == 20 * 4096 * 2048 * 3  # 20bsh x L, costs.py:99-105


@pytest.mark.parametrize("j", [1, 2, 3, 5, 9])
def test_partial_layout_parts(j):
    layers, s, h, heads = 3, 512, 256, 4
    order = offload_candidates(layers)
    lay = make_layout(layers, s, h, heads, head_grad=True, offload=order[:j])
    full = make_layout(layers, s, h, heads, head_grad=True)
    assert lay.slab_bytes <= full.slab_bytes + 3 * 256  # same tensors, at most bin-tail padding apart
    moving = [t for t in lay.tensors if lay.travels(t)]
    staying = [t for t in lay.tensors if not lay.travels(t)]
    names = {(t.layer, t.name) for t in moving}
    assert {(l, n) for l, n in order[:j]} <= names
    # lse travels with its o, head_dy with the top f
    assert all(((t.layer, "o") in names) == (t.name == "lse" and t in moving) for t in lay.tensors if t.name == "lse")
    assert (((-1, "head_dy") in names) == ((layers - 1, "f") in names))
    # offload part: only moving tensors, bin-packed by the reference's pack_host_bins
    assert lay.bins == tuple(pack_host_bins([(t.nbytes + 255) // 256 * 256 for t in moving]).bins)
    assert all(t.dev_offset + t.nbytes <= lay.off_bytes for t in moving)
    # resident part: after it, non-overlapping
    spans = sorted((t.dev_offset, t.dev_offset + t.nbytes) for t in staying)
    assert all(a >= lay.off_bytes for a, _ in spans)
    assert all(b <= c for (_, b), (c, _) in zip(spans, spans[1:]))
    assert spans[-1][1] <= lay.slab_bytes
    assert 0 < lay.offload_fraction < 1


def test_partial_fraction_grows_with_prefix():
    order = offload_candidates(3)
    fr = [make_layout(3, 4096, 2048, 16, offload=order[:j]).offload_fraction for j in range(1, len(order) + 1)]
    assert all(a < b for a, b in zip(fr, fr[1:]))
    assert fr[-1] == pytest.approx(1.0, abs=1e-3)


def test_unknown_tensor_rejected():
    with pytest.raises(ValueError):
        make_layout(2, 64, 64, 2, offload=[(5, "f")])


def test_partial_planner_c2_shape():
    """C2 rank 0 at the measured k ~ 4.5: whole-slab offload cannot stay within 5%,
    partial plans can and hold fewer activation bytes than no offload."""
    costs = po.measured_pass_costs(1.28e-3, 2.78e-3)
    sched = po.build_1f1b(8, 1, 32, costs)
    t_o = Fraction(18227, 10**6)
    order = offload_candidates(3)
    cands = []
    for j in (1, 2, 3):
        lay = make_layout(3, 4096, 2048, 16, offload=order[:j])
        cands.append((str(j), tuple(order[:j]), lay.off_bytes, lay.res_bytes))
    full = make_layout(3, 4096, 2048, 16)
    out = choose_partial_offload(sched, (0,), t_o, cands, tolerance=0.05, max_stride=2)
    assert out, "no partial plan within 5%"
    base_bytes = 8 * full.slab_bytes
    best = out[0]
    assert best.act_bytes < base_bytes
    assert best.overhead <= 0.05
    assert [c.act_bytes for c in out] == sorted(c.act_bytes for c in out)
    assert best.res_peak == 8  # rank 0 of PP=8 1F1B holds 8 microbatches
    tr = simulate(sched, best.plan, stream_mode=best.stream_mode)
    assert tr.memory.peak(0) == best.off_peak


def test_bench_partial_candidates_distinct():
    """bench.py measures at most `top` partial plans, one per tensor set, least memory first."""
    import bench

    costs = po.measured_pass_costs(1.28e-3, 2.78e-3)
    sched = po.build_1f1b(8, 3, 32, costs)
    out = bench.partial_candidates(sched, Fraction(18227, 10**6), 3, 4096, 2048, 16, top=3)
    assert 1 <= len(out) <= 3
    assert len({c.label for c in out}) == len(out)
    assert [c.act_bytes for c in out] == sorted(c.act_bytes for c in out)
    assert all(c.overhead <= 0.05 and not c.plan.late_list() for c in out)
