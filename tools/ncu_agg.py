"""Aggregate an ncu --metrics gpu__time_duration.sum --csv launch list by kernel name."""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
agg = collections.defaultdict(list)
for r in rows[1:]:
    agg[r[ki][:60]].append(float(r[vi].replace(",", "")))
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"{k:60s} {len(v):4d} {sum(v) / 1e6:9.3f} ms  first: {[round(x / 1e3, 1) for x in v[:8]]}")
