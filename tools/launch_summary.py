"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list:
per-kernel total time, share and count (optionally only launches [lo, hi))."""
from __future__ import annotations

import collections
import csv
import sys


def summary(path, lo=0, hi=None, width=90):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[h]
    ki, vi, ii = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("ID")
    agg = collections.defaultdict(lambda: [0.0, 0])
    for r in rows[h + 1:]:
        if len(r) <= vi:
            continue
        i = int(r[ii])
        if i < lo or (hi is not None and i >= hi):
            continue
        v = float(r[vi].replace(",", ""))
        a = agg[r[ki][:width]]
        a[0] += v
        a[1] += 1
    tot = sum(a[0] for a in agg.values())
    n = sum(a[1] for a in agg.values())
    lines = [f"total {tot / 1e3:.1f} us over {n} launches"]
    for k, (v, c) in sorted(agg.items(), key=lambda x: -x[1][0]):
        lines.append(f"{v / 1e3:10.1f} us {100 * v / tot:5.1f}% x{c:4d}  {k}")
    return "\n".join(lines)


if __name__ == "__main__":
    a = sys.argv[1:]
    print(summary(a[0], int(a[1]) if len(a) > 1 else 0, int(a[2]) if len(a) > 2 else None))
