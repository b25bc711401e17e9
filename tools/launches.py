"""Summarise an ncu --csv launch list: one line per launch with its metrics."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
start = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h, rows = rows[start], [r for r in rows[start:] if len(r) == len(rows[start])]
ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
d = collections.defaultdict(dict)
for r in rows[1:]:
    d[(int(r[ii]), r[ki][:60])][r[mi]] = r[vi]
for (i, k), m in sorted(d.items()):
    print(i, k, {a.split("__")[1].split(".")[0] + "." + a.split(".")[-1][:3]: b for a, b in m.items()})
