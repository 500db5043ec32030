#!/bin/bash
# One GPU session: smoke, GPU tests, bench (both arms), launch lists and full
# ncu captures of the solver kernels of every path.  Outputs land in gpurun_out/.
#   tools/gpu_round.sh [--quick]   (--quick: skip pytest and the reference arm)
set -u
cd "$(dirname "$0")/.."
O=gpurun_out
TAG=${TAG:-r01}
mkdir -p $O
Q=${1:-}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $O/gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
if [ "$Q" != "--quick" ]; then
  timeout 900 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_gpu.log
fi
python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
if [ "$Q" != "--quick" ]; then
  python bench.py --impl reference --steps 5 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err; echo "ref rc=$?"
fi
B="bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-other-configs"
python $B > $O/plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
  python $B > $O/ncu_launches.log 2>&1; echo "ncu-list rc=$?"
python tools/profile_step.py > $O/pplain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"tri_spec_factor|tri_spec_sep|tri_segment_solve|tri_cert" \
  -s 4 -c 4 -o $O/full python tools/profile_step.py > $O/ncu_full.log 2>&1; echo "ncu-full rc=$?"
for c in 0 2 3 4; do
  python tools/cfg_step.py $c 3 > $O/cfg$c.log 2>&1 && \
    ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg$c.csv \
    python tools/cfg_step.py $c 3 > /dev/null 2>&1; echo "cfg$c list rc=$?"
done
python tools/cfg_step.py 2 3 > /dev/null 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"blk_spec_factor|blk_spec_sep|blk_segment|blk_body_narrow|blk_band_narrow|blk_cert" \
  -c 4 -o $O/full_cfg2 python tools/cfg_step.py 2 3 > $O/ncu_full2.log 2>&1; echo "ncu-full2 rc=$?"
python tools/cfg_step.py 3 3 > /dev/null 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"blk_spec_factor|blk_spec_sep|blk_segment|blk_body_narrow|blk_band_narrow|blk_cert" \
  -c 4 -o $O/full_cfg3 python tools/cfg_step.py 3 3 > $O/ncu_full3.log 2>&1; echo "ncu-full3 rc=$?"
python tools/cfg_step.py 4 3 > /dev/null 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"chain_" \
  -c 12 -o $O/full_cfg4 python tools/cfg_step.py 4 3 > $O/ncu_full4.log 2>&1; echo "ncu-full4 rc=$?"
# summarise on the box (the .ncu-rep files are too large to travel back)
python tools/summarize_ncu.py $O/prof ${TAG:-r01} > $O/summary.log 2>&1; echo "summary rc=$?"
for k in "tri_segment_solve" "tri_spec_factor" "tri_spec_sep"; do
  python tools/ncu_lines.py $O/full.ncu-rep "$k" --top 25 > $O/prof/lines_$k.txt 2>&1
done
python tools/ncu_lines.py $O/full_cfg2.ncu-rep "blk_segment|blk_body_narrow" --top 25 > $O/prof/lines_cfg2_blk_body.txt 2>&1
python tools/ncu_lines.py $O/full_cfg2.ncu-rep blk_spec_factor --top 25 > $O/prof/lines_cfg2_blk_spec_factor.txt 2>&1
python tools/ncu_lines.py $O/full_cfg3.ncu-rep "blk_segment|blk_band_narrow" --top 25 > $O/prof/lines_cfg3_blk_body.txt 2>&1
python tools/ncu_lines.py $O/full_cfg4.ncu-rep chain_tm --top 25 > $O/prof/lines_cfg4_chain_tm.txt 2>&1
python tools/ncu_lines.py $O/full_cfg4.ncu-rep chain_solve --skip 1 --top 25 > $O/prof/lines_cfg4_chain_final.txt 2>&1
mkdir -p /tmp/ncu_reps && mv $O/*.ncu-rep /tmp/ncu_reps/ 2>/dev/null
du -sh $O
