"""Generate tests/golden/plans.json from the REFERENCE planner (test infrastructure).

Imports the read-only reference package (``/root/reference/pkg/src/ppoff``) in
this container and records, for every configuration below, the exact outputs of
the reference path the B200 executor consumes:

* ``Schedule.device_passes``      (builders.py:59-88,248-262; ir.py:176-469)
* ``OffloadPlan`` streams/skips/late (offload.py:133-220)
* ``simulate`` makespan, peaks, host peak, realized pass list (sim.py:141-520)

The fixture travels with the repo so parity tests run where the reference is
absent (the GPU box).  Regenerate with ``python oracle/make_golden_plans.py``.
"""

from __future__ import annotations

import json
import os
import sys
from fractions import Fraction

REF = os.environ.get("PPOFF_REFERENCE", "/root/reference/pkg/src")
sys.path.insert(0, REF)
sys.dont_write_bytecode = True

import ppoff  # noqa: E402  (the reference)
from ppoff import builders, costs, offload, sim  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden", "plans.json")


def fs(x) -> str:
    return str(Fraction(x))


def passes(seq):
    return [[str(p.kind), p.device, p.stage, p.microbatch, fs(p.start), fs(p.duration)] for p in seq]


def record(name, sched, plan, model=None, hw=None, stream_mode="single", contention=None):
    entry = {
        "name": name,
        "schedule_text": ppoff.emit_schedule(sched),
        "device_passes": [passes(d) for d in sched.device_passes],
    }
    if plan is not None:
        entry["plan"] = {
            "t_o": fs(plan.t_o),
            "stages": list(plan.stages),
            "pinned": plan.pinned,
            "sync_edges": [[list(a), list(b)] for a, b in plan.sync_edges],
            "streams": [
                {
                    "device": st.device,
                    "transfers": [[str(t.direction), t.device, t.stage, t.microbatch, t.slot, fs(t.start), fs(t.duration)] for t in st.transfers],
                    "skips": [list(x) for x in st.skips],
                    "late": [list(x) for x in st.late],
                }
                for st in plan.streams
            ],
        }
    tr = sim.simulate(sched, plan, model=model, hw=hw, stream_mode=stream_mode, contention=contention)
    pk = sim.peak_memory(tr)
    entry["sim"] = {
        "stream_mode": stream_mode,
        "contention": None if contention is None else contention.mode,
        "makespan": fs(tr.makespan),
        "peak_units": [u for u, _ in pk["per_device"]],
        "peak_bytes": [b for _, b in pk["per_device"]],
        "host_peak": sim.host_peak_memory(tr),
        "bubble": [fs(b) for b in sim.bubble_time(tr)],
        "passes": passes(tr.passes),
        "contention_events": len(tr.contention_log),
    }
    if model is not None:
        entry["model"] = [model.hidden_size, model.sequence_length, model.microbatch_size, model.layers_per_stage, model.bytes_per_element]
    return entry


def main():
    U = costs.PassCosts.unit()
    cases = []
    # C1 golden: tiny PP=4 1F1B m=8 full offload k=1/2
    s, p = builders.build_1f1b_full_offload(4, 8, U, Fraction(3, 2))
    cases.append(record("C1_1f1b_d4_m8_full_k0.5", s, p, model=costs.ModelSpec(256, 512, 1, 1, 4)))
    # 1F1B d=8 m=32 full offload at k in {1/2, 1, 3/2, 2}
    for k in (Fraction(1, 2), Fraction(1), Fraction(3, 2), Fraction(2)):
        s, p = builders.build_1f1b_full_offload(8, 32, U, k * 3)
        cases.append(record(f"1f1b_d8_m32_full_k{float(k)}", s, p))
    # 1F1B with merged stage v=3 (C2 shape: 3 layers per stage)
    s, p = builders.build_1f1b_full_offload(8, 32, U, Fraction(9, 2), v=3)
    cases.append(record("C2_1f1b_d8_v3_m32_full_k0.5", s, p, model=costs.ModelSpec(2048, 4096, 1, 3, 2)))
    # PP sweep 1/2/4/8
    for d in (1, 2, 4, 8):
        s, p = builders.build_1f1b_full_offload(d, 8 if d < 8 else 16, U, Fraction(3, 2))
        cases.append(record(f"pp_sweep_d{d}", s, p))
    # interleaved 1F1B d=8 v in {2,4}, selective n via po_block selection
    for v in (2, 4):
        sched = builders.build_interleaved_1f1b(8, v, 32, U)
        for n in range(0, v + 1):
            st = offload.select_offload_stages(builders.po_block(8, v, U), n)
            plan = offload.plan_slots(sched, st, Fraction(3, 2)) if n else None
            cases.append(record(f"1f1b-i_d8_v{v}_m32_n{n}", sched, plan, model=costs.ModelSpec(4096, 8192, 1, 32 // (8 * v), 2)))
    # non-unit measured-like costs (integer microseconds), B200 C2/C4 k
    real = costs.PassCosts(Fraction(1650), Fraction(3350), Fraction(0), Fraction(40))
    sched = builders.build_1f1b(8, 3, 32, real)
    for t_o in (Fraction(6000), Fraction(18000)):
        cases.append(record(f"1f1b_d8_v3_real_to{t_o}", sched, offload.plan_slots(sched, (0,), t_o)))
    sched = builders.build_interleaved_1f1b(4, 3, 8, costs.PassCosts(Fraction(3), Fraction(5), Fraction(1), Fraction(1, 3)))
    cases.append(record("1f1b-i_d4_v3_odd_costs", sched, offload.plan_slots(sched, (0, 2), Fraction(7))))
    # dual streams and contention + topology sync
    s, p = builders.build_1f1b_full_offload(8, 32, U, Fraction(3))
    cases.append(record("1f1b_d8_full_k1_dual", s, p, stream_mode="dual"))
    hw = costs.HardwareSpec(1e15, 5e10)
    synced = offload.apply_topology_sync(p, hw)
    cases.append(record("1f1b_d8_full_k1_synced_halving", s, synced, contention=sim.ContentionModel("shared-switch-halving", 2)))
    # split-backward family (next row, planner level)
    for name, sch in (("gis_d4_v2_m8", builders.build_gis(4, 2, 8, U)), ("gis-h_d8_v2_m16", builders.build_gis_h(8, 2, 16, U)), ("po_d8_v2_m16", builders.build_po(8, 2, 16, U))):
        st = offload.select_offload_stages(builders.po_block(sch.devices, sch.local_stages, U), 1)
        cases.append(record(name, sch, offload.plan_slots(sch, st, U.total)))
    # host bins
    bins = []
    for sizes in ([5, 3, 3, 1], [9, 9, 9], [262144] * 6 + [1048576], [167772160] * 6 + [671088640], [7, 100, 33, 1000, 5]):
        lay = offload.pack_host_bins(sizes)
        bins.append({"sizes": sizes, "bins": list(lay.bins), "placements": [list(x) for x in lay.placements]})
    doc = {"generator": "oracle/make_golden_plans.py", "reference": "ppoff 0.1.0 (" + REF + ")", "cases": cases, "bins": bins}
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    with open(OUT, "w") as f:
        json.dump(doc, f, separators=(",", ":"))
    print(f"wrote {len(cases)} cases, {len(bins)} bin layouts -> {OUT} ({os.path.getsize(OUT)} bytes)")


if __name__ == "__main__":
    main()
