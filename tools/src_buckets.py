"""Instruction / stall-sample share per source region of one kernel in an ncu
report (regions = the '// ----' section comments of the kernel's source file).

    python tools/src_buckets.py REPORT.ncu-rep KERNEL_REGEX SOURCE_FILE FIRST_LINE LAST_LINE
"""
import csv
import io
import subprocess
import sys

rep, kre, srcf, first, last = sys.argv[1], sys.argv[2], sys.argv[3], int(sys.argv[4]), int(sys.argv[5])
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "--kernel-name", "regex:" + kre], capture_output=True, text=True).stdout
base = srcf.split("/")[-1]
marks = [(i + 1, l.strip()[8:60]) for i, l in enumerate(open(srcf)) if l.strip().startswith("// ----")
         and first <= i + 1 <= last]
fname, hdr, ncol, data = None, None, 0, []
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
    elif r[0] == "Line No":
        hdr, ncol = {k: i for i, k in enumerate(r)}, len(r)
    elif hdr and r[0].isdigit() and len(r) == ncol:
        num = lambda v: float(v) if v not in ("", "-") else 0.0
        data.append((fname, int(r[0]), num(r[hdr["Instructions Executed"]]),
                     num(r[hdr["Warp Stall Sampling (All Samples)"]])))
ti = sum(d[2] for d in data) or 1.0
ts = sum(d[3] for d in data) or 1.0
acc = {}
for f, ln, i, s in data:
    name = "(other files / helpers)"
    if f == base and first <= ln <= last:
        name = "(kernel preamble)"
        for m, title in marks:
            if ln >= m:
                name = title
    a = acc.setdefault(name, [0.0, 0.0])
    a[0] += i
    a[1] += s
print(f"total instructions {ti:.0f}")
for k, (i, s) in sorted(acc.items(), key=lambda kv: -kv[1][1]):
    print(f"{i / ti * 100:5.1f}% inst  {s / ts * 100:5.1f}% samples  {k}")
