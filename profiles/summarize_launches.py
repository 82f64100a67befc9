"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list:
per-kernel share of the last training step (the last quarter of launches of a
`bench.py --steps 1 --warmup 3` run).  usage: python summarize_launches.py launches.csv"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h, data = rows[hi], rows[hi + 1:]
ki, vi, ii = h.index("Kernel Name"), h.index("Metric Value"), h.index("ID")
vals = []
for r in data:
    try:
        vals.append((int(r[ii]), r[ki][:100], float(r[vi].replace(",", ""))))
    except (ValueError, IndexError):
        pass
last = vals[int(len(vals) * 0.75):]
tot, cnt = collections.defaultdict(float), collections.Counter()
for _, k, v in last:
    tot[k] += v
    cnt[k] += 1
s = sum(tot.values())
print(f"launches captured: {len(vals)}; last-quarter kernel time: {s / 1e6:.2f} ms (ncu: serialised, cold cache)")
print(f"{'share':>7} {'us':>9} {'n':>4}  kernel")
for k, v in sorted(tot.items(), key=lambda x: -x[1])[:25]:
    print(f"{100 * v / s:6.2f}% {v / 1e3:9.0f} {cnt[k]:4d}  {k}")
