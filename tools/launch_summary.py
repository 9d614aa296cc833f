"""Summarise an `ncu --metrics gpu__time_duration.sum --csv --log-file X` launch list per kernel."""
import collections
import csv
import sys

SCALE = {"ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0, "nsecond": 1e-6}


def main(path, steps=None):
    lines = [ln for ln in open(path) if not ln.startswith("==")]
    rows = list(csv.reader(lines))
    h = rows[0]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.OrderedDict()
    for r in rows[1:]:
        name = r[ki].split("(")[0][:64]
        ms = float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1.0)
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += ms
    tot = sum(a[1] for a in agg.values())
    print(f"{'kernel':64s} {'launches':>8s} {'total ms':>10s} {'share':>6s}")
    for name, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{name:64s} {c:8d} {t:10.3f} {100 * t / tot:5.1f}%")
    print(f"{len(rows) - 1} launches, {tot:.3f} ms total (cold-cache, serialised by ncu)")


if __name__ == "__main__":
    main(sys.argv[1])
