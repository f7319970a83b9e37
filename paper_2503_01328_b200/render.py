"""SVG timeline of a ``SimTrace`` -- modelled (``simulate``) or measured (``execute``).

The reference draws its traces with ``render.py:59-118``; this is an independent,
dependency-free writer for the CLI ``run`` output: one compute
lane and one copy lane per device, passes as boxes coloured by kind and labelled
``stage.mb`` when they are wide enough, time axis in the trace's own unit
(seconds for measured traces, schedule units for modelled ones).
"""

from __future__ import annotations

from xml.sax.saxutils import escape

from .schedule_types import PassKind

COLOURS = {
    PassKind.F: "#4e79a7",
    PassKind.B: "#59a14f",
    PassKind.W: "#9c9c3a",
    PassKind.OFFLOAD: "#f28e2b",
    PassKind.RELOAD: "#b07aa1",
}
LANE_H, GAP, LEFT, TOP = 22, 6, 70, 28


def render_svg(trace, width: int = 1400, title: str = "") -> str:
    """SVG document (str) of every pass in ``trace``."""
    passes = list(trace.passes)
    devices = sorted({p.device for p in passes})
    span = float(trace.makespan) or 1.0
    scale = (width - LEFT - 10) / span
    lanes = {}
    for d in devices:
        lanes[(d, "compute")] = len(lanes)
        lanes[(d, "copy")] = len(lanes)
    height = TOP + len(lanes) * (LANE_H + GAP) + 30
    out = [f'<svg xmlns="http://www.w3.org/2000/svg" width="{width}" height="{height}" '
           f'font-family="monospace" font-size="10">',
           f'<text x="{LEFT}" y="16" font-size="12">{escape(title)} makespan={span:.6g}</text>']
    for (d, lane), i in lanes.items():
        y = TOP + i * (LANE_H + GAP)
        out.append(f'<text x="4" y="{y + 15}">d{d} {lane}</text>')
        out.append(f'<rect x="{LEFT}" y="{y}" width="{width - LEFT - 10}" height="{LANE_H}" fill="#f4f4f4"/>')
    for p in passes:
        lane = "copy" if p.kind in (PassKind.OFFLOAD, PassKind.RELOAD) else "compute"
        y = TOP + lanes[(p.device, lane)] * (LANE_H + GAP)
        x = LEFT + float(p.start) * scale
        w = max(0.5, float(p.duration) * scale)
        tip = f"{p.kind.value} stage={p.stage} mb={p.microbatch} start={float(p.start):.6g} dur={float(p.duration):.6g}"
        out.append(f'<rect x="{x:.2f}" y="{y}" width="{w:.2f}" height="{LANE_H}" fill="{COLOURS[p.kind]}" '
                   f'stroke="#ffffff" stroke-width="0.5"><title>{escape(tip)}</title></rect>')
        label = f"{p.stage}.{p.microbatch}"
        if w > 6 * len(label) + 2:
            out.append(f'<text x="{x + 2:.2f}" y="{y + 15}" fill="#ffffff">{label}</text>')
    ty = TOP + len(lanes) * (LANE_H + GAP) + 14
    for k in range(11):
        t = span * k / 10
        x = LEFT + t * scale
        out.append(f'<line x1="{x:.2f}" y1="{TOP - 4}" x2="{x:.2f}" y2="{ty - 10}" stroke="#cccccc" stroke-width="0.5"/>')
        out.append(f'<text x="{x:.2f}" y="{ty}">{t:.4g}</text>')
    out.append("</svg>")
    return "\n".join(out)
