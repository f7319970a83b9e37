"""Planner parity: this package's schedules, plans and runner model against the
reference's recorded outputs (tests/golden/plans.json, made by
oracle/make_golden_plans.py from ppoff 0.1.0) -- bit-exact, rationals compared
as exact fractions."""

from fractions import Fraction

import pytest

import paper_2503_01328_b200 as po
from paper_2503_01328_b200 import costs, offload, sim


def _passes(seq):
    return [[str(p.kind), p.device, p.stage, p.microbatch, str(Fraction(p.start)), str(Fraction(p.duration))] for p in seq]


def _rebuild(case):
    sched = po.parse_schedule(case["schedule_text"])
    plan = None
    if "plan" in case:
        pl = case["plan"]
        streams = []
        for st in pl["streams"]:
            tr = tuple(
                offload.Transfer(po.PassKind(d), dev, s, j, slot, Fraction(a), Fraction(b))
                for (d, dev, s, j, slot, a, b) in st["transfers"]
            )
            streams.append(offload.DeviceStream(st["device"], Fraction(0), Fraction(0), tr, tuple(map(tuple, st["skips"])), tuple(map(tuple, st["late"])), ()))
        plan = offload.OffloadPlan(
            t_o=Fraction(pl["t_o"]), stages=tuple(pl["stages"]), streams=tuple(streams),
            sync_edges=tuple((tuple(a), tuple(b)) for a, b in pl["sync_edges"]), pinned=pl["pinned"],
        )
    return sched, plan


def _fresh(name):
    """Re-derive the named golden case from this package's own builders."""
    U = costs.PassCosts.unit()
    if name.startswith("C1_"):
        return po.build_1f1b_full_offload(4, 8, U, Fraction(3, 2))
    if name.startswith("1f1b_d8_m32_full_k"):
        k = Fraction(name.rsplit("k", 1)[1])
        return po.build_1f1b_full_offload(8, 32, U, k * 3)
    if name.startswith("C2_"):
        return po.build_1f1b_full_offload(8, 32, U, Fraction(9, 2), v=3)
    if name.startswith("pp_sweep_d"):
        d = int(name[len("pp_sweep_d"):])
        return po.build_1f1b_full_offload(d, 8 if d < 8 else 16, U, Fraction(3, 2))
    if name.startswith("1f1b-i_d8_v"):
        v = int(name.split("_v")[1].split("_")[0])
        n = int(name.rsplit("_n", 1)[1])
        sched = po.build_interleaved_1f1b(8, v, 32, U)
        st = po.select_offload_stages(po.po_block(8, v, U), n)
        return sched, (po.plan_slots(sched, st, Fraction(3, 2)) if n else None)
    if name.startswith("1f1b_d8_v3_real_to"):
        real = costs.PassCosts(1650, 3350, 0, 40)
        sched = po.build_1f1b(8, 3, 32, real)
        return sched, po.plan_slots(sched, (0,), Fraction(name.rsplit("to", 1)[1]))
    if name == "1f1b-i_d4_v3_odd_costs":
        sched = po.build_interleaved_1f1b(4, 3, 8, costs.PassCosts(3, 5, 1, Fraction(1, 3)))
        return sched, po.plan_slots(sched, (0, 2), Fraction(7))
    if name.startswith("1f1b_d8_full_k1"):
        s, p = po.build_1f1b_full_offload(8, 32, U, Fraction(3))
        if "synced" in name:
            p = po.apply_topology_sync(p, costs.HardwareSpec(1e15, 5e10))
        return s, p
    builder = {"gis_d4_v2_m8": lambda: po.build_gis(4, 2, 8, U), "gis-h_d8_v2_m16": lambda: po.build_gis_h(8, 2, 16, U), "po_d8_v2_m16": lambda: po.build_po(8, 2, 16, U)}[name]
    sched = builder()
    st = po.select_offload_stages(po.po_block(sched.devices, sched.local_stages, U), 1)
    return sched, po.plan_slots(sched, st, U.total)


def test_golden_cases_present(golden_plans):
    assert len(golden_plans["cases"]) >= 20


@pytest.mark.parametrize("idx", range(26))
def test_builder_and_planner_match_reference(golden_plans, idx):
    case = golden_plans["cases"][idx]
    sched, plan = _fresh(case["name"])
    assert [_passes(d) for d in sched.device_passes] == case["device_passes"], case["name"]
    assert po.emit_schedule(sched) == case["schedule_text"]
    if "plan" in case:
        gp = case["plan"]
        assert list(plan.stages) == gp["stages"]
        assert plan.pinned == gp["pinned"]
        assert [[list(a), list(b)] for a, b in plan.sync_edges] == gp["sync_edges"]
        for st, gst in zip(plan.streams, gp["streams"]):
            got = [[str(t.direction), t.device, t.stage, t.microbatch, t.slot, str(t.start), str(t.duration)] for t in st.transfers]
            assert got == gst["transfers"], (case["name"], st.device)
            assert [list(x) for x in st.skips] == gst["skips"]
            assert [list(x) for x in st.late] == gst["late"]
    else:
        assert plan is None


@pytest.mark.parametrize("idx", range(26))
def test_runner_model_matches_reference(golden_plans, idx):
    case = golden_plans["cases"][idx]
    sched, plan = _fresh(case["name"])
    g = case["sim"]
    model = costs.ModelSpec(*case["model"]) if "model" in case else None
    contention = sim.ContentionModel(g["contention"], 2) if g["contention"] else None
    tr = sim.simulate(sched, plan, model=model, stream_mode=g["stream_mode"], contention=contention)
    pk = sim.peak_memory(tr)
    assert str(tr.makespan) == g["makespan"]
    assert [u for u, _ in pk["per_device"]] == g["peak_units"]
    assert [b for _, b in pk["per_device"]] == g["peak_bytes"]
    assert sim.host_peak_memory(tr) == g["host_peak"]
    assert [str(b) for b in sim.bubble_time(tr)] == g["bubble"]
    assert _passes(tr.passes) == g["passes"]
    assert len(tr.contention_log) == g["contention_events"]


def test_parse_roundtrip_of_golden(golden_plans):
    for case in golden_plans["cases"]:
        sched, _ = _rebuild(case)
        assert po.emit_schedule(sched) == case["schedule_text"]


def test_host_bins_match_reference(golden_plans):
    for b in golden_plans["bins"]:
        lay = po.pack_host_bins(b["sizes"])
        assert list(lay.bins) == b["bins"]
        assert [list(x) for x in lay.placements] == b["placements"]


def test_c1_golden_from_survey():
    """per-device order, slot order, peaks [2,2,2,1], makespan 33."""
    U = costs.PassCosts.unit()
    s, p = po.build_1f1b_full_offload(4, 8, U, Fraction(3, 2))
    order0 = " ".join(f"{p_.kind}{p_.microbatch}" for p_ in s.device_passes[0])
    assert order0 == "F0 F1 F2 F3 B0 F4 B1 F5 B2 F6 B3 F7 B4 B5 B6 B7"
    slots0 = " ".join(f"{'O' if t.direction == po.PassKind.OFFLOAD else 'R'}{t.microbatch}@{t.slot}" for t in p.streams[0].transfers)
    assert slots0 == "O0@2 O1@4 O2@6 O3@8 R0@11 R1@15 O4@18 R2@19 O5@22 R3@23 O6@26 R4@27 O7@30 R5@31 R6@35 R7@39"
    assert p.streams[3].transfers == ()
    tr = po.simulate(s, p)
    assert tr.makespan == 33 == po.simulate(s).makespan
    assert [u for u, _ in po.peak_memory(tr)["per_device"]] == [2, 2, 2, 1]
    assert po.host_peak_memory(tr) == [8]
