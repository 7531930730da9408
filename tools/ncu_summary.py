"""Markdown summary of an `ncu --set full` report (`ncu -i X --page raw --csv`):
key throughput metrics and the top stall reasons per profiled kernel."""
from __future__ import annotations

import csv
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_sector_hit_rate.pct", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "smsp__thread_inst_executed_per_inst_executed.ratio", "smsp__inst_executed.sum",
        "launch__grid_size", "launch__occupancy_limit_registers"]


def summarize(rep, title):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units = rows[0], rows[1]
    idx = {h: i for i, h in enumerate(hdr)}
    out = [f"## {title}"]
    for r in rows[2:]:
        out.append(f"- kernel `{r[idx['Kernel Name']][:90]}`")
        for k in KEYS:
            if k in idx:
                out.append(f"  - {k}: {r[idx[k]]} {units[idx[k]]}")
        stalls = []
        for h, i in idx.items():
            if (h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued")):
                try:
                    stalls.append((float(r[i].replace(",", "")), h.split("stalled_")[1]))
                except ValueError:
                    pass
        tot = sum(v for v, _ in stalls) or 1.0
        top = sorted(stalls, reverse=True)[:4]
        out.append(f"  - top stall samples (share): {[(n, round(v / tot, 3)) for v, n in top]}")
    return "\n".join(out)


if __name__ == "__main__":
    print(summarize(sys.argv[1], " ".join(sys.argv[2:])))
