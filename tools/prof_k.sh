#!/bin/bash
# Full ncu capture of kernels matching REGEX in `tools/cfg_step.py CFG 2`: digest to gpurun_out/<TAG>_digest.txt
#   tools/prof_k.sh CFG REGEX COUNT TAG [SKIP]
set -u
cd "$(dirname "$0")/.."
C=$1; K=$2; N=${3:-1}; TAG=${4:-r02}; SK=${5:-0}
mkdir -p gpurun_out
python tools/cfg_step.py $C 2 > /dev/null 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:"$K" -s $SK -c $N -o /tmp/pk_$TAG -f python tools/cfg_step.py $C 2 > /dev/null 2>&1
python tools/ncu_digest.py /tmp/pk_$TAG.ncu-rep "$K" --lines 30 > gpurun_out/${TAG}_digest.txt 2>&1
head -30 gpurun_out/${TAG}_digest.txt
