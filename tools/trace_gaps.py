"""Where a measured run loses time: compute-stream idle gaps, attributed to the op
that ends them (a B waiting on its RELOAD, an F waiting on a free slab, ...).

usage: python tools/trace_gaps.py <trace.csv> [device]"""
import csv
import sys
from fractions import Fraction


def load(path, device=0):
    rows = []
    for r in csv.DictReader(open(path)):
        if int(r["device"]) != device:
            continue
        rows.append((r["kind"], int(r["stage"]), int(r["microbatch"]), Fraction(r["start"]), Fraction(r["end"])))
    return rows


def main():
    path = sys.argv[1]
    dev = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    rows = load(path, dev)
    comp = sorted((r for r in rows if r[0] in ("F", "B", "W")), key=lambda r: r[3])
    rel = {(r[1], r[2]): r for r in rows if r[0] == "RELOAD"}
    off = {(r[1], r[2]): r for r in rows if r[0] == "OFFLOAD"}
    t0, t1 = comp[0][3], max(r[4] for r in rows)
    busy = sum(r[4] - r[3] for r in comp)
    gaps = {"B waits RELOAD": 0, "other": 0}
    per = []
    for prev, cur in zip(comp, comp[1:]):
        g = cur[3] - prev[4]
        if g <= Fraction(1, 100000):  # < 10 us
            continue
        key = (cur[1], cur[2])
        why = "other"
        if cur[0] == "B" and key in rel and rel[key][4] >= cur[3] - Fraction(1, 100000):
            why = "B waits RELOAD"
        gaps[why] += g
        per.append((float(g) * 1e3, cur[0], key, why))
    span = t1 - t0
    print(f"span {float(span)*1e3:.1f} ms, compute busy {float(busy)*1e3:.1f} ms ({float(busy/span)*100:.1f}%)")
    for k, v in gaps.items():
        print(f"  idle before ops, {k}: {float(v)*1e3:.1f} ms")
    for g, kind, key, why in sorted(per, reverse=True)[:12]:
        print(f"  {g:7.2f} ms before {kind}{key} ({why})")
    if off:
        d2h = sum(r[4] - r[3] for r in off.values())
        h2d = sum(r[4] - r[3] for r in rel.values())
        print(f"transfers: {len(off)} D2H {float(d2h)*1e3:.1f} ms, {len(rel)} H2D {float(h2d)*1e3:.1f} ms")
    cs = sorted(comp, key=lambda r: r[3])
    durs = {}
    for r in cs:
        durs.setdefault(r[0], []).append(float(r[4] - r[3]) * 1e3)
    print("mean pass ms:", {k: round(sum(v) / len(v), 3) for k, v in durs.items()})


if __name__ == "__main__":
    main()
