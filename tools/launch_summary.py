"""Aggregate an ncu --csv launch list (gpu__time_duration.sum) by kernel name."""
import collections
import csv
import sys


def main(path, top=25):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    scale = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0, "second": 1e3}
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        nm = r[ki].split("(")[0]
        v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1e-6)
        agg[nm][0] += 1
        agg[nm][1] += v
    tot = sum(v[1] for v in agg.values())
    print(f"{'ms':>10} {'share':>6} {'n':>5}  kernel")
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        print(f"{v[1]:10.3f} {100 * v[1] / tot:5.1f}% {v[0]:5d}  {k[:90]}")
    print(f"{tot:10.3f} total ms, {sum(v[0] for v in agg.values())} launches")


if __name__ == "__main__":
    main(sys.argv[1])
