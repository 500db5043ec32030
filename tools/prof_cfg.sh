#!/bin/bash
# Profile one config step: launch list + full ncu capture of kernels matching REGEX.
#   tools/prof_cfg.sh CFG REGEX [COUNT] [TAG]
# Writes gpurun_out/<TAG>_launches_cfgN.txt and gpurun_out/<TAG>_digest_cfgN.txt
set -u
cd "$(dirname "$0")/.."
C=$1; K=$2; N=${3:-4}; TAG=${4:-r02}
O=gpurun_out; mkdir -p $O
python tools/cfg_step.py $C 20 > $O/${TAG}_cfg${C}_step.json 2>&1; cat $O/${TAG}_cfg${C}_step.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/_l.csv python tools/cfg_step.py $C 3 > /dev/null 2>&1
python - "$O/_l.csv" "$O/${TAG}_launches_cfg${C}.txt" "$C" <<'PY'
import sys
sys.path.insert(0, "tools")
from summarize_ncu import launch_list
launch_list(sys.argv[1], sys.argv[2], f"ncu --metrics gpu__time_duration.sum --clock-control none python tools/cfg_step.py {sys.argv[3]} 3")
PY
ncu --set full --clock-control none --import-source on -k regex:"$K" -c $N -o /tmp/prof_$C -f python tools/cfg_step.py $C 2 > /dev/null 2>&1
python tools/ncu_digest.py /tmp/prof_$C.ncu-rep "$K" --lines 30 > $O/${TAG}_digest_cfg${C}.txt 2>&1
head -40 $O/${TAG}_digest_cfg${C}.txt
