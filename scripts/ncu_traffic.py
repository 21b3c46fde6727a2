#!/usr/bin/env python
"""Fold ncu --set full reports (.ncu-rep) of the traversal kernels into
profiles/traffic.json: per config/schedule and kernel, DRAM bytes read+write
per launch and ncu's duration, plus a text summary of the key metrics.

  python scripts/ncu_traffic.py CONFIG SCHEDULE OUT_SUMMARY.txt REPORT.ncu-rep [...]
"""
import csv
import io
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "smsp__thread_inst_executed_per_inst_executed.ratio",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "smsp__pcsamp_warps_issue_stalled_long_scoreboard",
        "smsp__pcsamp_warps_issue_stalled_short_scoreboard",
        "smsp__pcsamp_warps_issue_stalled_wait", "smsp__pcsamp_warps_issue_stalled_lg_throttle",
        "smsp__pcsamp_warps_issue_stalled_mio_throttle",
        "smsp__pcsamp_warps_issue_stalled_selected",
        "smsp__pcsamp_warps_issue_stalled_not_selected",
        "smsp__pcsamp_warps_issue_stalled_branch_resolving"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "s": 1.0,
         "second": 1.0, "nsecond": 1e-9}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {}
        for h, u, v in zip(hdr, units, r):
            d[h] = (v, u)
        res.append(d)
    return res


def val(d, k):
    v, u = d[k]
    x = float(v.replace(",", ""))
    return x * SCALE.get(u, 1.0)


def main():
    cfg, sched, summary = sys.argv[1], sys.argv[2], sys.argv[3]
    path = os.path.join(ROOT, "profiles", "traffic.json")
    tj = json.load(open(path)) if os.path.exists(path) else {}
    ent = tj.get(f"{cfg}/{sched}", {})
    if "kernels" not in ent:
        ent = {"kernels": {}}
    lines = []
    for rep in sys.argv[4:]:
        for d in raw(rep):
            name = re.sub(r"<[^<>]*>$", "", d["Kernel Name"][0].split("(")[0]).split("::")[-1]
            b = val(d, "dram__bytes_read.sum") + val(d, "dram__bytes_write.sum")
            t = val(d, "gpu__time_duration.sum")
            ent["kernels"][name] = {"dram_bytes": b, "duration_s": t}
            lines.append(f"== {name}  (ncu --set full --clock-control none; {os.path.basename(rep)})")
            for k in KEYS:
                if k in d:
                    lines.append(f"  {k:70s} {d[k][0]:>22s} {d[k][1]}")
            lines.append(f"  => DRAM {b / 1e9:.3f} GB in {t * 1e3:.3f} ms = {b / t / 1e9:.1f} GB/s")
    ent["source"] = os.path.relpath(summary, ROOT)
    tj[f"{cfg}/{sched}"] = ent
    json.dump(tj, open(path, "w"), indent=1)
    open(summary, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
