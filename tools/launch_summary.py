"""Aggregate an ncu launch list (gpu__time_duration.sum CSV) by kernel."""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[1:]:
    k = r[ki].split("(")[0][-48:]
    agg[k][0] += 1
    agg[k][1] += float(r[vi].replace(",", ""))
tot = sum(t for _, t in agg.values())
print(f"total {tot / 1e6:.3f} ms over {sum(c for c, _ in agg.values())} launches")
for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{c:6d} {t / 1e6:9.3f} ms {100 * t / tot:5.1f}%  {k}")
