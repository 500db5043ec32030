#!/bin/bash
# Compare library variants built into build/var/libpsg_<V>.so on one config:
#   tools/var_probe.sh <cfg> <kernel-regex> V1 V2 ...   ("base" = the in-tree libpsg.so)
cd "$(dirname "$0")/.."
CFG=$1; KER=$2; shift 2
cp paper_0912_3678_b200/libpsg.so build/var/libpsg_base.so
for v in "$@"; do
  cp build/var/libpsg_$v.so paper_0912_3678_b200/libpsg.so
  echo "=== variant $v"
  for r in 1 2; do python tools/cfg_step.py $CFG 20; done
  for r in 1 2; do ALONE=1 python tools/cfg_step.py $CFG 30; done
  for r in 1 2 3; do NOTIMING=1 python tools/cfg_step.py $CFG 50 | cut -c1-40; done
  ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"$KER" -s 5 -c 10 python tools/cfg_step.py $CFG 3 2>&1 | grep -E "^  [a-z_0-9]+.*\(|duration" | paste - - | awk '{print $1, $(NF)}'
done
cp build/var/libpsg_base.so paper_0912_3678_b200/libpsg.so
