"""Summarise `ncu --set full` reports (one launch each) into a table:
    python profiles/summarize_ncu.py gpurun_out/gdpa_fwd.ncu-rep ... [--grep REGEX]
Columns: duration, DRAM bytes (read + write), DRAM throughput %, tensor-pipe
activity %, issue-slot %, registers.  `--grep` lists every raw metric whose
name matches REGEX (to find the right counter names on a new ncu)."""
import csv
import io
import re
import subprocess
import sys

COLS = [
    ("us", "gpu__time_duration.sum", 1e-3),
    ("DRAM MB", ("dram__bytes_read.sum", "dram__bytes_write.sum"), 1e-6),
    ("DRAM %", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1),
    ("tensor %", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", 1),
    ("L2 hit %", "lts__t_sector_hit_rate.pct", 1),
    ("issue %", "sm__inst_issued.avg.pct_of_peak_sustained_active", 1),
    ("regs", "launch__registers_per_thread", 1),
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--print-units", "base"],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    return [dict(zip(hdr, r)) for r in rows[2:] if len(r) == len(hdr)]


def num(v):
    try:
        return float(v.replace(",", ""))
    except (ValueError, AttributeError):
        return float("nan")


def main(argv):
    grep = None
    if "--grep" in argv:
        i = argv.index("--grep")
        grep = re.compile(argv[i + 1])
        argv = argv[:i] + argv[i + 2:]
    print("%-28s " % "kernel" + " ".join("%9s" % c[0] for c in COLS))
    for rep in argv:
        for r in raw(rep):
            name = r.get("Kernel Name", "?").split("(")[0].split("<")[0].split("::")[-1]
            vals = []
            for _, key, scale in COLS:
                v = sum(num(r.get(k, "nan")) for k in key) if isinstance(key, tuple) else num(r.get(key, "nan"))
                vals.append("%9.1f" % (v * scale))
            print("%-28s " % name[:28] + " ".join(vals))
            if grep:
                for k, v in r.items():
                    if grep.search(k):
                        print("    %s = %s" % (k, v))


if __name__ == "__main__":
    main(sys.argv[1:])
