"""One training epoch's kernels out of an ncu launch list (tools/ncu_target.py
run for several epochs): the launches between the last two loss kernels
(k_softmax_xent), i.e. backward + Adam + publish + forward, summarised with
tools/launch_summary.py."""
import csv
import sys

from launch_summary import summary


def window(path):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[h]
    ki, ii = hdr.index("Kernel Name"), hdr.index("ID")
    ids = [int(r[ii]) for r in rows[h + 1:] if len(r) > ki and "k_softmax_xent" in r[ki]]
    ids = sorted(set(ids))
    return ids[-2] + 1, ids[-1] + 1


if __name__ == "__main__":
    lo, hi = window(sys.argv[1])
    print(summary(sys.argv[1], lo, hi))
