"""Top stall instructions of one kernel in an ncu report (source page, SASS)."""
import csv, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
ntop = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                      "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[1]
iS = h.index("Warp Stall Sampling (All Samples)")
data = [r for r in rows[2:] if len(r) > iS and r[iS].replace('.', '', 1).isdigit()]
n = len(data)
if n % 2 == 0 and n and data[0][0] == data[n // 2][0]:
    data = data[:n // 2]
tot = sum(float(r[iS]) for r in data)
cols = [c for c in h if c.startswith('stall_') and 'Not Issued' not in c]
agg = {c[6:]: sum(float(r[h.index(c)] or 0) for r in data) / tot * 100 for c in cols}
print("samples", tot, "instrs", len(data))
print("by reason:", ", ".join(f"{k}={v:.1f}" for k, v in sorted(agg.items(), key=lambda kv: -kv[1]) if v > 0.5))
top = sorted(range(len(data)), key=lambda i: -float(data[i][iS]))[:ntop]
for i in sorted(top):
    r = data[i]
    st = sorted(((c[6:], float(r[h.index(c)] or 0)) for c in cols), key=lambda kv: -kv[1])[:2]
    print(f"{i:5d} {float(r[iS]) / tot * 100:5.1f}% {r[1][:78]:78s} {st[0][0]}")
