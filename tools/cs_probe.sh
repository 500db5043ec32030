#!/bin/bash
# config-4 solve passes: tests, step time, per-kernel times
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_chain_gpu.py tests/test_ode_gpu.py -m gpu -q -x 2>&1 | tail -2
python tools/cfg_step.py 4 20
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:"chain_" -s 5 -c 5 python tools/cfg_step.py 4 2 2>&1 | grep -E "chain_|duration|dram__bytes|warps_active"
