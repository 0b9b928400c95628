"""Per-kernel table of an ncu launch list (gpu__time_duration.sum CSV):
launches, mean and last duration. python tools/launch_table.py <csv>"""
import collections
import csv
import sys


def table(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = collections.defaultdict(list)
    for r in rows[hdr + 1:]:
        if len(r) > vi:
            try:
                agg[r[ki]].append(float(r[vi].replace(",", "")))
            except ValueError:
                pass
    return agg


if __name__ == "__main__":
    for k, v in sorted(table(sys.argv[1]).items(), key=lambda x: -sum(x[1])):
        print(f"{k[:64]:64s} n={len(v):3d} mean={sum(v) / len(v) / 1e3:8.1f}us "
              f"last={v[-1] / 1e3:8.1f}us")
