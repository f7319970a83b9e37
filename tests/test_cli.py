"""CLI (reference flag names, cli.py:328-367): ``plan`` on CPU, ``run`` on the B200."""

import json
import subprocess
import sys

import pytest

from conftest import ROOT


def test_plan_writes_reference_files(tmp_path):
    out = tmp_path / "o"
    res = subprocess.run([sys.executable, "-m", "paper_2503_01328_b200", "plan", "--schedule", "1f1b", "--d", "4",
                          "--m", "8", "--offload", "full", "--t-o", "1/2", "--out", str(out)],
                         cwd=ROOT, capture_output=True, text=True, check=True)
    summary = json.loads(res.stdout)
    assert summary["peak_units"] == [2, 2, 2, 1]  # C1 golden: SURVEY App. A.3
    assert summary["makespan"] == 33.0
    text = (out / "1f1b.schedule").read_text()
    import paper_2503_01328_b200 as po

    assert po.emit_schedule(po.parse_schedule(text)) == text
    assert (out / "1f1b.plan").read_text().startswith("# plan t_o=")
    svg = (out / "1f1b.svg").read_text()
    assert svg.startswith("<svg") and svg.rstrip().endswith("</svg>")
    assert svg.count("<rect") >= 64 + 8  # 64 compute passes + lane backgrounds (+ transfers)


def test_render_svg_is_well_formed():
    import xml.dom.minidom
    from fractions import Fraction

    import paper_2503_01328_b200 as po
    from paper_2503_01328_b200.render import render_svg

    sched, plan = po.build_1f1b_full_offload(4, 8, po.PassCosts.unit(), Fraction(3, 2))
    trace = po.simulate(sched, plan)
    doc = xml.dom.minidom.parseString(render_svg(trace, title="c1 <golden>"))
    rects = doc.getElementsByTagName("rect")
    n_transfers = sum(1 for p in trace.passes if p.kind.value in ("OFFLOAD", "RELOAD"))
    assert len(rects) == 8 + len(trace.passes) and n_transfers > 0


@pytest.mark.gpu
def test_run_virtual_pipeline(tmp_path):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():  # pragma: no cover
        pytest.skip("needs a CUDA device")
    out = tmp_path / "r"
    res = subprocess.run([sys.executable, "-m", "paper_2503_01328_b200", "run", "--schedule", "gis-h", "--d", "2",
                          "--v", "2", "--m", "4", "--layers", "4", "--offload", "1", "--iters", "1", "--warmup", "1",
                          "--out", str(out)], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stderr[-3000:]
    summary = json.loads(res.stdout.strip().splitlines()[-1])
    assert summary["tokens_per_s"] > 0 and summary["schedule"] == "gis-h"
    assert (out / "gis-h-trace.csv").read_text().startswith("device,stage,microbatch,kind")
    assert (out / "gis-h.svg").read_text().startswith("<svg")
    assert summary["predicted_makespan_s"] > 0 and summary["measured_makespan_s"] > 0


@pytest.mark.gpu
def test_run_closed_loop_policy(tmp_path):
    """``run --offload auto-measured``: candidates measured on the device, the choice and
    every trial in the summary; a chosen plan measured within the 5% budget."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():  # pragma: no cover
        pytest.skip("needs a CUDA device")
    out = tmp_path / "c"
    res = subprocess.run([sys.executable, "-m", "paper_2503_01328_b200", "run", "--schedule", "1f1b", "--d", "4",
                          "--m", "8", "--layers", "4", "--mode", "emulate", "--offload", "auto-measured",
                          "--iters", "1", "--warmup", "1", "--out", str(out)], cwd=ROOT, capture_output=True,
                         text=True, timeout=900)
    assert res.returncode == 0, res.stderr[-3000:]
    summary = json.loads(res.stdout.strip().splitlines()[-1])
    cl = summary["closed_loop"]
    assert isinstance(cl["trials"], list) and len(cl["trials"]) <= 4
    if cl["chosen_stride"] is not None:
        assert cl["trials"][-1]["stride"] == cl["chosen_stride"] and cl["trials"][-1]["measured_pct"] <= 5.0
