"""Per-launch DRAM traffic of the dominant kernel from an ncu CSV taken with
--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum.
Merges one workload's entry into the JSON bench.py reads for roofline.traffic.

usage: traffic_summary.py CSV OUT.json WORKLOAD KERNELS CALLS [source words...]
(the last KERNELS launches matching k_spmm_fast -- unit, packed and follow-up
kernels -- summed and divided by the CALLS hg_spmm calls they belong to)."""
from __future__ import annotations

import collections
import csv
import json
import sys
from pathlib import Path


def main(path, out, workload, last, calls, pattern="k_spmm_fast", source=""):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[h]
    ki, mi, vi, ii = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
    per = collections.defaultdict(dict)
    names = {}
    for r in rows[h + 1:]:
        if len(r) <= vi:
            continue
        per[int(r[ii])][r[mi]] = float(r[vi].replace(",", ""))
        names[int(r[ii])] = r[ki]
    ids = [i for i in sorted(per) if pattern in names[i]][-last:]
    bytes_ = [per[i]["dram__bytes_read.sum"] + per[i]["dram__bytes_write.sum"] for i in ids]
    ns = [per[i]["gpu__time_duration.sum"] for i in ids]
    entry = {"bytes_per_launch": sum(bytes_) / calls, "calls": calls, "per_launch_bytes": bytes_,
             "per_launch_ns": ns, "kernels": [names[i][:80] for i in ids], "source": source}
    p = Path(out)
    d = json.loads(p.read_text()) if p.exists() else {}
    d[workload] = entry
    p.write_text(json.dumps(d, indent=1))
    print(json.dumps(entry))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3], int(sys.argv[4]), int(sys.argv[5]),
         source=" ".join(sys.argv[6:]))
