"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list: python tools/launches.py FILE"""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ik, iv = h.index("Kernel Name"), h.index("Metric Value")
agg = collections.defaultdict(list)
for r in rows[1:]:
    agg[r[ik][:80]].append(float(r[iv].replace(",", "")) / 1e3)
tot = sum(sum(v) for v in agg.values())
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print("%5d %10.1f us  %5.1f%%  %s" % (len(v), sum(v) / len(v), 100 * sum(v) / tot, k))
