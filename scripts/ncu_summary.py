"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel."""
import collections
import csv
import sys


def summarise(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, mi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[hi + 1:]:
        if len(r) <= mi:
            continue
        agg[r[ki]][0] += 1
        agg[r[ki]][1] += float(r[mi].replace(",", "")) * scale.get(r[ui], 1.0)
    tot = sum(v[1] for v in agg.values())
    out = [f"{'launches':>8} {'total_ms':>12} {'share':>7} {'avg_us':>12}  kernel"]
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"{v[0]:8d} {v[1] / 1e3:12.3f} {100 * v[1] / tot:6.2f}% {v[1] / v[0]:12.1f}  {k[:110]}")
    return "\n".join(out)


if __name__ == "__main__":
    print(summarise(sys.argv[1]))
