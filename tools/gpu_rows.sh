#!/bin/bash
# ncu evidence for the §8(f) rows (IVP trajectory, pivoting strategies,
# Parareal): each workload runs once plain (must exit 0), then under an ncu
# launch list and one --set full capture of its dominant kernel; summaries
# land in gpurun_out/prof (the .ncu-rep files stay on the box).
set -u
cd "$(dirname "$0")/.."
O=gpurun_out
TAG=${TAG:-r01}
mkdir -p $O/prof
make -C oracle ref > /dev/null 2>&1
declare -A CMD=(
  [ode]="tools/ode_bench.py --m 8 --p 4096 --N 64 --reps 1 --no-ref"
  [piv]="tools/piv_bench.py --kind 4 --n 1048576 --p 1024 --reps 1 --no-ref"
  [pr]="tools/pr_bench.py --m 64 --p 64 --N 1000 --reps 1 --no-ref"
)
declare -A KER=([ode]="ode_assemble|chain_tm" [piv]="piv_factor_kernel|piv_reduced_solve" [pr]="pr_fine_kernel|pr_sweep")
for w in ode piv pr; do
  python ${CMD[$w]} > $O/plain_$w.log 2>&1 || { echo "$w plain failed"; continue; }
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_$w.csv \
    python ${CMD[$w]} > /dev/null 2>&1; echo "$w list rc=$?"
  python tools/launches.py $O/launches_$w.csv > $O/prof/${TAG}_launches_$w.txt 2>&1
  ncu --set full --clock-control none --import-source on -k regex:"${KER[$w]}" -c 3 -o $O/full_$w \
    python ${CMD[$w]} > $O/ncu_full_$w.log 2>&1; echo "$w full rc=$?"
  ncu -i $O/full_$w.ncu-rep --page raw --csv > $O/raw_$w.csv 2>/dev/null
  python - "$O/raw_$w.csv" > $O/prof/${TAG}_ncu_full_$w.txt <<'PY'
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
h = rows[0]
want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "smsp__inst_executed.sum",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"]
idx = [h.index(w) for w in want if w in h]
print("# ncu --set full (clock-control none), first launches of the dominant kernels")
print(" | ".join(h[i] for i in idx))
for r in rows[2:]:
    print(" | ".join(r[i][:60] for i in idx))
PY
done
mv $O/*.ncu-rep /tmp/ 2>/dev/null
rm -f $O/raw_*.csv
du -sh $O
