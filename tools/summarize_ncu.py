"""Summarise gpurun_out ncu artefacts into profiles/ (tracked)."""
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

OUT = sys.argv[1] if len(sys.argv) > 1 else "profiles"
TAG = sys.argv[2] if len(sys.argv) > 2 else "r01"
G = "gpurun_out"
os.makedirs(OUT, exist_ok=True)

# ---- launch list (gpu__time_duration per launch)
rows = list(csv.reader(open(os.path.join(G, "launches.csv"))))
start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
h = rows[start]
ix = {k: i for i, k in enumerate(h)}
agg = defaultdict(list)
for r in rows[start + 1:]:
    if len(r) < len(h) or r[ix["Metric Name"]] != "gpu__time_duration.sum":
        continue
    agg[r[ix["Kernel Name"]]].append(float(r[ix["Metric Value"]].replace(",", "")) / 1e3)
lines = ["# ncu launch list (gpu__time_duration.sum, --clock-control none; cold-cache, serialised)",
         "# command: ncu --metrics gpu__time_duration.sum --clock-control none python bench.py --steps 2 --warmup 3 "
         "--no-e2e --no-cpu-baseline", "# launches  mean_us  total_us  kernel"]
tot = sum(sum(v) for v in agg.values())
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    lines.append(f"{len(v):4d} {sum(v) / len(v):10.1f} {sum(v):10.1f}  ({100 * sum(v) / tot:4.1f}%)  {k}")
open(os.path.join(OUT, f"{TAG}_launches.txt"), "w").write("\n".join(lines) + "\n")

# ---- full capture: key metrics per kernel
raw = subprocess.run(["ncu", "-i", os.path.join(G, "full.ncu-rep"), "--page", "raw", "--csv"],
                     capture_output=True, text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
hdr = rr[0]
keys = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic", "launch__grid_size",
        "launch__block_size", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum", "smsp__inst_executed.sum",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"]
units = rr[1]
res = []
for r in rr[2:]:
    d = {}
    for k in keys:
        if k in hdr:
            i = hdr.index(k)
            d[k] = r[i] + ("" if units[i] in ("", "none") else " " + units[i])
    res.append(d)
with open(os.path.join(OUT, f"{TAG}_ncu_full.txt"), "w") as fh:
    fh.write("# ncu --set full --clock-control none --import-source on (tools/profile_step.py: cfg1 n=2^26 "
             "p=65536, second factor+solve)\n")
    for d in res:
        fh.write("\n")
        for k, v in d.items():
            fh.write(f"{k:75s} {v}\n")
# traffic of the dominant kernel for bench.py
for d in res:
    if "segment_solve" in d.get("Kernel Name", ""):
        def val(s):
            num, unit = s.split()[0].replace(",", ""), (s.split()[1] if len(s.split()) > 1 else "")
            mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
            return float(num) * mult
        t = val(d["dram__bytes_read.sum"]) + val(d["dram__bytes_write.sum"])
        json.dump({"kernel": d["Kernel Name"], "dram_bytes_per_launch": t,
                   "source": f"profiles/{TAG}_ncu_full.txt"}, open(os.path.join(OUT, "k3_traffic.json"), "w"),
                  indent=1)
print(open(os.path.join(OUT, f"{TAG}_launches.txt")).read())
