"""Key metrics + per-line stall hot spots of the kernels in one ncu report.

    python tools/ncu_digest.py REPORT.ncu-rep [KERNEL_REGEX] [--lines N]
Used on the GPU box right after an `ncu --set full --import-source on` capture
(the .ncu-rep stays there; this text comes back in gpurun_out/).
"""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from summarize_ncu import full_capture  # noqa: E402

rep = sys.argv[1]
kre = sys.argv[2] if len(sys.argv) > 2 and not sys.argv[2].startswith("--") else None
nl = int(sys.argv[sys.argv.index("--lines") + 1]) if "--lines" in sys.argv else 25
tmp = "/tmp/_digest.txt"
full_capture(rep, tmp, rep)
print(open(tmp).read())
if kre:
    here = os.path.dirname(os.path.abspath(__file__))
    print(subprocess.run([sys.executable, os.path.join(here, "ncu_lines.py"), rep, kre, "--top", str(nl)],
                         capture_output=True, text=True).stdout)
