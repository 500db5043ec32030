#!/bin/bash
# Per-config step timing (plain) and ncu launch lists; summaries in gpurun_out/.
#   tools/prof_cfgs.sh "0 2 3 4"
set -u
cd "$(dirname "$0")/.."
O=gpurun_out
mkdir -p $O
for c in ${1:-0 2 3 4}; do
  python tools/cfg_step.py $c 20 > $O/step_cfg$c.json 2>&1; echo "cfg$c rc=$? $(tail -1 $O/step_cfg$c.json)"
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/ll_cfg$c.csv \
    python tools/cfg_step.py $c 2 > /dev/null 2>&1
  python tools/launches.py $O/ll_cfg$c.csv > $O/ll_cfg$c.txt 2>&1; cat $O/ll_cfg$c.txt | head -25
done
