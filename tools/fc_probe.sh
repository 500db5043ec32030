#!/bin/bash
# config-4 factor+condense kernel: tests, step time, kernel time and the shared-memory pipe counters
mkdir -p gpurun_out
python -m pytest tests/test_chain_gpu.py tests/test_ode_gpu.py -m gpu -q -x 2>&1 | tail -2
python tools/cfg_step.py 4 20
ncu --metrics gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active,sm__cycles_active.avg,sm__cycles_elapsed.max \
  --clock-control none -k regex:"chain_fc" -s 1 -c 1 python tools/cfg_step.py 4 2 2>&1 | grep -E "chain_fc|duration|wavefronts|conflicts|inst_executed|warps_active|cycles"
