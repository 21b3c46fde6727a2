"""Summarise one scripts/measure.sh pass into profiles/r1/: the ncu launch list
(kernel shares), key metrics of the full captures of both traversal kernels,
the DRAM bytes per launch for bench.py's roofline.traffic
(profiles/traffic.json), and the bench JSON line.

usage: python scripts/profile_summary.py TAG [CONFIG]
"""
import csv
import io
import json
import os
import shutil
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1]
cfg = sys.argv[2] if len(sys.argv) > 2 else "C2"
src = os.path.join(ROOT, "gpurun_out")
dst = os.path.join(ROOT, "profiles", "r1")

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size"] + [
    "smsp__pcsamp_warps_issue_stalled_" + k for k in (
        "long_scoreboard", "short_scoreboard", "wait", "mio_throttle", "lg_throttle",
        "no_instructions", "selected", "not_selected", "branch_resolving")]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}

lines, traffic = [], {}
for k in ("solo_kernel", "stream_kernel"):
    rep = os.path.join(src, f"prof_{k}_{tag}_{cfg}.ncu-rep")
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    d, u = dict(zip(rows[0], rows[2])), dict(zip(rows[0], rows[1]))
    lines.append(f"== {k}  (ncu --set full --clock-control none, {cfg} via scripts/probe.py; "
                 "kernel run alone = serialized by ncu)")
    lines += [f"  {x:60s} {d[x]:>22s} {u.get(x, '')}" for x in KEYS if x in d]
    traffic[k] = sum(float(d[x].replace(",", "")) * SCALE.get(u[x], 1)
                     for x in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
full = f"ncu_full_{cfg}_{tag}_solo_stream.txt"
open(os.path.join(dst, full), "w").write("\n".join(lines) + "\n")

rows = list(csv.reader(open(os.path.join(src, f"launches_{tag}_{cfg}.csv"))))
start = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[start]
ik, iv = h.index("Kernel Name"), h.index("Metric Value")
agg = defaultdict(lambda: [0, 0.0])
for r in rows[start + 1:]:
    if len(r) > iv:
        agg[r[ik][:60]][0] += 1
        agg[r[ik][:60]][1] += float(r[iv].replace(",", ""))
tot = sum(v[1] for v in agg.values())
out = ["ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised) of",
       f"python bench.py --config {cfg} --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1   "
       "(7 factorizations)",
       f"{'kernel':62s} {'launches':>8s} {'total ms':>10s} {'share':>7s}"]
out += [f"{k:62s} {v[0]:8d} {v[1] / 1e6:10.2f} {v[1] / tot * 100:6.1f}%"
        for k, v in sorted(agg.items(), key=lambda x: -x[1][1])]
open(os.path.join(dst, f"launches_{cfg}_{tag}_summary.txt"), "w").write("\n".join(out) + "\n")
shutil.copy(os.path.join(src, f"launches_{tag}_{cfg}.csv"), os.path.join(dst, f"launches_{cfg}_{tag}.csv"))
shutil.copy(os.path.join(src, f"bench_{tag}_{cfg}.json"), os.path.join(dst, f"bench_{cfg}_{tag}.json"))
tpath = os.path.join(ROOT, "profiles", "traffic.json")
tj = json.load(open(tpath)) if os.path.exists(tpath) else {}
tj[f"{cfg}/threshold"] = {"kernel": "solo_kernel", "dram_bytes": traffic["solo_kernel"],
                          "stream_kernel_dram_bytes": traffic["stream_kernel"],
                          "source": f"profiles/r1/{full}"}
json.dump(tj, open(tpath, "w"), indent=1)
print("\n".join(out[:6]))
print(traffic)
