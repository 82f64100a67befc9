timeout 1500 python -m pytest tests -q -m gpu -x 2>&1 | grep -E "^E  |passed|failed" | cut -c1-300 | head -20
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r2_c4.json 2> gpurun_out/r2_c4.err; echo rc $?
tail -3 gpurun_out/r2_c4.err
timeout 900 python bench.py --config c2 --steps 10 --warmup 3 --no-cpu > gpurun_out/r2_c2.json 2> gpurun_out/r2_c2.err; echo rc $?
python - <<'PY'
import json
for c in ("c4","c2"):
    d=json.load(open(f"gpurun_out/r2_{c}.json"))
    print(c, "value", round(d["value"],1), "ms", round(d["ms_per_step"],3), "mfu", round(d["mfu"]["value"],4), "e2e", round(d["e2e"]["value"],1), "cpu", d["cpu_baseline"])
    for k,v in sorted(d["roofline_table"].items(), key=lambda kv:-kv[1]["share_of_step"]):
        print(f"  {k:16s} {v['bound']:6s} n={v['launches']:4d} avg={v['avg_launch_ms']*1e3:8.1f}us share={v['share_of_step']:.3f} ach={v['achieved']:8.1f} {v['unit']} frac={v['frac']:.3f} gbs={v['achieved_gbs']:.0f} tfs={v['achieved_tflops']:.0f}")
    print("  roof", d["roofline"])
PY
