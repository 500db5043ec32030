"""Summarise gpurun_out ncu artefacts into profiles/ (tracked).

    python tools/summarize_ncu.py [OUT_DIR] [TAG]

Reads (whatever exists):
  gpurun_out/launches.csv            launch list of bench.py (cfg1 headline)
  gpurun_out/launches_cfg{0,2,3,4}.csv launch lists of tools/cfg_step.py
  gpurun_out/full.ncu-rep            --set full capture of the cfg1 kernels
  gpurun_out/full_cfg{2,3,4}.ncu-rep  --set full captures of the block / chain kernels
and writes {TAG}_launches[_cfgN].txt, {TAG}_ncu_full[_cfgN].txt and k3_traffic.json.
"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

OUT = sys.argv[1] if len(sys.argv) > 1 and __name__ == "__main__" else "profiles"
TAG = sys.argv[2] if len(sys.argv) > 2 and __name__ == "__main__" else "r01"
G = "gpurun_out"

CMD = {
    "": "ncu --metrics gpu__time_duration.sum --clock-control none python bench.py --steps 2 --warmup 3 "
        "--no-e2e --no-cpu-baseline --no-other-configs",
}


def launch_list(src, dst, cmd):
    rows = list(csv.reader(open(src)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[start]
    ix = {k: i for i, k in enumerate(h)}
    agg = defaultdict(list)
    for r in rows[start + 1:]:
        if len(r) < len(h) or r[ix["Metric Name"]] != "gpu__time_duration.sum":
            continue
        agg[r[ix["Kernel Name"]]].append(float(r[ix["Metric Value"]].replace(",", "")) / 1e3)
    lines = ["# ncu launch list (gpu__time_duration.sum, --clock-control none; cold-cache, serialised)",
             f"# command: {cmd}", "# launches  mean_us  total_us  share  kernel"]
    tot = sum(sum(v) for v in agg.values())
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        lines.append(f"{len(v):4d} {sum(v) / len(v):10.1f} {sum(v):10.1f}  ({100 * sum(v) / tot:4.1f}%)  {k}")
    open(dst, "w").write("\n".join(lines) + "\n")
    print(open(dst).read())


KEYS = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
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
        "smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"]


def full_capture(rep, dst, title):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    hdr, units = rr[0], rr[1]
    res = []
    for r in rr[2:]:
        d = {}
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                d[k] = r[i] + ("" if units[i] in ("", "none") else " " + units[i])
        res.append(d)
    with open(dst, "w") as fh:
        fh.write(f"# ncu --set full --clock-control none --import-source on ({title})\n")
        for d in res:
            fh.write("\n")
            for k, v in d.items():
                fh.write(f"{k:75s} {v}\n")
    return res


def val(s):
    num, unit = s.split()[0].replace(",", ""), (s.split()[1] if len(s.split()) > 1 else "")
    mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
    return float(num) * mult


def main():
    os.makedirs(OUT, exist_ok=True)
    if os.path.exists(os.path.join(G, "launches.csv")):
        launch_list(os.path.join(G, "launches.csv"), os.path.join(OUT, f"{TAG}_launches.txt"), CMD[""])
    for c in (0, 2, 3, 4):
        src = os.path.join(G, f"launches_cfg{c}.csv")
        if os.path.exists(src):
            launch_list(src, os.path.join(OUT, f"{TAG}_launches_cfg{c}.txt"),
                        f"ncu --metrics gpu__time_duration.sum --clock-control none python tools/cfg_step.py {c} 3")

    rep = os.path.join(G, "full.ncu-rep")
    if os.path.exists(rep):
        res = full_capture(rep, os.path.join(OUT, f"{TAG}_ncu_full.txt"),
                           "tools/profile_step.py: cfg1 n=2^26 p=65536, second factor+solve")
        for d in res:  # traffic of the dominant kernel for bench.py
            if "segment_solve" in d.get("Kernel Name", ""):
                t = val(d["dram__bytes_read.sum"]) + val(d["dram__bytes_write.sum"])
                json.dump({"kernel": d["Kernel Name"], "dram_bytes_per_launch": t,
                           "source": f"profiles/{TAG}_ncu_full.txt"}, open(os.path.join(OUT, "k3_traffic.json"), "w"),
                          indent=1)
    for c in (2, 3, 4):
        rep = os.path.join(G, f"full_cfg{c}.ncu-rep")
        if os.path.exists(rep):
            full_capture(rep, os.path.join(OUT, f"{TAG}_ncu_full_cfg{c}.txt"),
                         f"tools/cfg_step.py {c}: refactor + async solve, one launch per kernel")


if __name__ == "__main__":
    main()
