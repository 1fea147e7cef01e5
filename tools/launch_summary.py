"""Summarise an ncu --metrics gpu__time_duration.sum launch list (dev tool).
usage: launch_summary.py CSV [skip_fraction]  (skip the first fraction of launches = warm-up)"""
import collections
import csv
import sys

lines = [l for l in open(sys.argv[1]) if l.startswith('"')]
rows = list(csv.reader(lines))
h = rows[0]
ik, iv, iid = h.index("Kernel Name"), h.index("Metric Value"), h.index("ID")
L = [(int(r[iid]), r[ik][:90], float(r[iv].replace(",", ""))) for r in rows[1:] if len(r) > iv and r[iv]]
skip = float(sys.argv[2]) if len(sys.argv) > 2 else 0.5
seq = L[int(len(L) * skip):]
tot = sum(x[2] for x in seq)
print(f"launches {len(seq)}  total {tot/1e6:.3f} ms")
agg = collections.OrderedDict()
for _, k, v in seq:
    agg.setdefault(k, [0, 0.0])
    agg[k][0] += 1
    agg[k][1] += v
for k, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1])[:25]:
    print(f"{v/1e6:8.3f} ms {100*v/tot:5.1f}% {c:5d}x  {k}")
