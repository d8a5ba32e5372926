"""Summarise an ncu --csv metrics log: per kernel name, launches and mean of each metric."""
import csv
import sys
from collections import defaultdict

rows = [r for r in csv.reader(l for l in open(sys.argv[1]) if l.startswith('"'))]
hdr = rows[0]
ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
acc = defaultdict(lambda: defaultdict(list))
for r in rows[1:]:
    try:
        acc[r[ki][:60]][r[mi]].append(float(r[vi].replace(",", "")))
    except ValueError:
        pass
for k, m in acc.items():
    print(k, {n: round(sum(v) / len(v), 1) for n, v in m.items()}, "n=%d" % len(next(iter(m.values()))))
