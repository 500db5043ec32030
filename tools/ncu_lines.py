"""Per-source-line warp-stall breakdown of one kernel in an ncu report
(needs a -lineinfo build and `ncu --import-source on`).

    python tools/ncu_lines.py REPORT.ncu-rep KERNEL_REGEX [--top N] [--skip K]
(KERNEL_REGEX matches the base name; --skip K selects the K-th matching launch)
"""
import csv
import io
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 30
skip = ["--launch-skip", sys.argv[sys.argv.index("--skip") + 1], "--launch-count", "1"] if "--skip" in sys.argv else []
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "--kernel-name", "regex:" + kre, *skip], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
fname, hdr, lines, func = None, None, [], None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        func = r[1]
        continue
    if r[0] == "Line No":
        hdr = {k: i for i, k in enumerate(r) if k not in ("Source",)}
        hdr["Source"] = 1
        ncol = len(r)
        continue
    if hdr and r[0] and len(r) == ncol and r[0].isdigit():
        num = lambda v: float(v) if v not in ("", "-") else 0.0
        lines.append((fname, int(r[0]), r[1], num(r[hdr["Warp Stall Sampling (All Samples)"]]),
                      num(r[hdr["Instructions Executed"]])))
if func is None:
    sys.exit(f"no kernel matching {kre!r} in {rep}")
tot = sum(x[3] for x in lines) or 1.0
print(func, "samples", tot)
for f, ln, src, v, ins in sorted(lines, key=lambda x: -x[3])[:top]:
    print(f"{v / tot * 100:5.1f}%  {f}:{ln:<5} inst {ins:11.0f}  {src.strip()[:85]}")
