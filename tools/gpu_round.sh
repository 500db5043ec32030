#!/bin/bash
# One GPU session: smoke, GPU tests, bench (both arms), launch list and a full
# ncu capture of the solver kernels.  Outputs land in gpurun_out/.
set -u
cd "$(dirname "$0")/.."
O=gpurun_out
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $O/gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_gpu.log
python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
python bench.py --impl reference --steps 5 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err; echo "ref rc=$?"
python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu_launches.log 2>&1; echo "ncu-list rc=$?"
python tools/profile_step.py > $O/pplain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"tri_spec_factor|tri_spec_sep|tri_segment_solve|tri_cert" \
  -s 4 -c 4 -o $O/full python tools/profile_step.py > $O/ncu_full.log 2>&1; echo "ncu-full rc=$?"
