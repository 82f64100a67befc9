"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list of
`bench.py --eager --steps K --warmup W`: per-kernel share of ONE training
step: the launches between the last two Adam step-count ticks (one per
step; older captures without a tick kernel use the fused-Adam launch, which
then closed every step).  usage: python summarize_launches.py launches.csv"""
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
marks = [i for i, (_, k, _) in enumerate(vals) if "tick_kernel" in k]
if len(marks) < 2:
    marks = [i for i, (_, k, _) in enumerate(vals) if "adam_kernel" in k]
last = vals[marks[-2]:marks[-1]] if len(marks) >= 2 else vals[int(len(vals) * 0.75):]
tot, cnt = collections.defaultdict(float), collections.Counter()
for _, k, v in last:
    tot[k] += v
    cnt[k] += 1
s = sum(tot.values())
print(f"launches captured: {len(vals)}; one step: {len(last)} launches, {s / 1e6:.2f} ms kernel time "
      f"(ncu: serialised, cold cache)")
print(f"{'share':>7} {'us':>9} {'n':>4}  kernel")
for k, v in sorted(tot.items(), key=lambda x: -x[1])[:40]:
    print(f"{100 * v / s:6.2f}% {v / 1e3:9.0f} {cnt[k]:4d}  {k}")
