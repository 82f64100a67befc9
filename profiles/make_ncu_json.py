"""Per-family ncu --set full numbers for bench.py's roofline table:
    python profiles/make_ncu_json.py OUT.json REPORT.ncu-rep ...
Writes {"families": {family: {"dram_bytes_per_launch", "duration_us",
"tensor_pipe_pct", "dram_pct", "issue_pct", "kernels"}}}; a family that is
several kernels per call (swa_bwd = rowdot + dK/dV + dQ) sums them; for the
GEMM family the largest launch (the QKV projection) stands for the family."""
import json
import sys

sys.path.insert(0, __file__.rsplit("/", 1)[0])
from summarize_ncu import num, raw  # noqa: E402

FAM = [("gdpa_fwd", "gdpa_fwd"), ("gdpa_bwd", "gdpa_bwd"), ("hsp_fwd", "hsp_fwd"), ("hsp_bwd", "hsp_bwd"),
       ("swa_fwd", "swa_fwd_tc"), ("swa_bwd", "swa_bwd_"), ("swa_bwd", "swa_rowdot"), ("adam", "adam_kernel"),
       ("gemm", "gemm_tc_kernel")]


def main(out, reps):
    fams = {}
    for rep in reps:
        for r in raw(rep):
            name = r.get("Kernel Name", "")
            fam = next((f for f, sub in FAM if sub in name), None)
            if fam is None:
                continue
            e = {"dram_bytes_per_launch": num(r.get("dram__bytes_read.sum", "nan")) + num(r.get("dram__bytes_write.sum", "nan")),
                 "duration_us": num(r.get("gpu__time_duration.sum", "nan")) * 1e-3,
                 "tensor_pipe_pct": num(r.get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "nan")),
                 "dram_pct": num(r.get("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "nan")),
                 "issue_pct": num(r.get("sm__inst_issued.avg.pct_of_peak_sustained_active", "nan")),
                 "kernels": [name.split("(")[0][-60:]]}
            if fam == "gemm":
                if fam not in fams or e["duration_us"] > fams[fam]["duration_us"]:
                    fams[fam] = e
            elif fam == "swa_bwd":
                base = fams.setdefault(fam, {"dram_bytes_per_launch": 0.0, "duration_us": 0.0, "kernels": []})
                if e["kernels"][0] in base["kernels"]:
                    continue
                base["dram_bytes_per_launch"] += e["dram_bytes_per_launch"]
                base["duration_us"] += e["duration_us"]
                base["kernels"] += e["kernels"]
                for k in ("tensor_pipe_pct", "dram_pct", "issue_pct"):
                    base[k] = max(base.get(k, 0.0), e[k])
            elif fam not in fams:
                fams[fam] = e
    json.dump({"note": "ncu --set full --clock-control none, one launch each at the c4 bench shapes "
                       "(scripts/r2/prof_kernels.py); cold-cache, serialised", "families": fams},
              open(out, "w"), indent=1)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2:])
