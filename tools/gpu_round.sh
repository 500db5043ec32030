#!/bin/bash
# One GPU evidence session: smoke, GPU tests, bench (both arms), then per
# config a launch list (ncu gpu__time_duration, cold-cache, serialised) and a
# full ncu capture of its dominant kernels digested to text (metrics + per-line
# stall hot spots).  Everything lands in gpurun_out/ (copy to profiles/).
#   tools/gpu_round.sh [--quick]      (--quick: no pytest, no reference arm)
set -u
cd "$(dirname "$0")/.."
O=gpurun_out
export TAG=${TAG:-r02}
mkdir -p $O
Q=${1:-}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $O/gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
if [ "$Q" != "--quick" ]; then
  timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_gpu.log
fi
python bench.py > $O/${TAG}_bench.json 2> $O/bench.err; echo "bench rc=$?"
if [ "$Q" != "--quick" ]; then
  python bench.py --impl reference --steps 3 --warmup 1 > $O/${TAG}_bench_ref.json 2> $O/bench_ref.err; echo "ref rc=$?"
fi
# headline launch list: the bench command itself (timed parts only)
B="bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-other-configs"
python $B > /dev/null 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/_l1.csv python $B > /dev/null 2>&1
python - <<'PY'
import sys
sys.path.insert(0, "tools")
from summarize_ncu import launch_list
launch_list("gpurun_out/_l1.csv", f"gpurun_out/{__import__('os').environ.get('TAG', 'r02')}_launches.txt",
            "ncu --metrics gpu__time_duration.sum --clock-control none python bench.py --steps 2 --warmup 3 "
            "--no-e2e --no-cpu-baseline --no-other-configs")
PY
declare -A KER=([0]="tri_spec_fused|tri_segment_solve|tri_cert" [1]="tri_spec_fused|tri_segment_solve|tri_cert"
                [2]="blktri_spec|blktri_body|blk_cert" [3]="band_spec|band_body|blk_cert"
                [4]="chain_")
declare -A CNT=([0]=3 [1]=3 [2]=3 [3]=3 [4]=5)
for c in 0 1 2 3 4; do
  python tools/cfg_step.py $c 20 > $O/${TAG}_cfg${c}_step.json 2>&1 || { echo "cfg$c plain failed"; continue; }
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/_l.csv \
    python tools/cfg_step.py $c 3 > /dev/null 2>&1
  python - "$c" <<'PY'
import sys
sys.path.insert(0, "tools")
from summarize_ncu import launch_list
c = sys.argv[1]
launch_list("gpurun_out/_l.csv", f"gpurun_out/{__import__('os').environ.get('TAG', 'r02')}_launches_cfg{c}.txt",
            f"ncu --metrics gpu__time_duration.sum --clock-control none python tools/cfg_step.py {c} 3")
PY
  # the second step's kernels (the first one builds plans and warms caches)
  ncu --set full --clock-control none --import-source on -k regex:"${KER[$c]}" -s ${CNT[$c]} -c ${CNT[$c]} \
    -o /tmp/full_cfg$c -f python tools/cfg_step.py $c 2 > $O/ncu_full_cfg$c.log 2>&1
  python tools/ncu_digest.py /tmp/full_cfg$c.ncu-rep "${KER[$c]}" --lines 30 > $O/${TAG}_ncu_full_cfg$c.txt 2>&1
  echo "cfg$c done"
done
du -sh $O
