"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list by kernel."""
import collections
import csv
import sys


def summarize(path, top=25):
    rows = list(csv.reader(open(path)))
    hdr_i = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr, data = rows[hdr_i], rows[hdr_i + 1:]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in data:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
        name = r[ki]
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(v[1] for v in agg.values())
    out = []
    for name, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        out.append(f"{100 * t / tot:6.2f}%  n={n:5d}  avg={t / n:9.2f} us  {name[:110]}")
    out.append(f"total device time {tot / 1e3:.2f} ms over {sum(v[0] for v in agg.values())} launches")
    return "\n".join(out)


if __name__ == "__main__":
    print(summarize(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25))
