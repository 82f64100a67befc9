import json, sys
for f in sys.argv[1:]:
    d = json.load(open(f))
    print(f, "value", round(d["value"], 1), "ms", round(d["ms_per_step"], 3), "mfu", round(d["mfu"]["value"], 4),
          "e2e", round(d["e2e"]["value"], 1) if d.get("e2e") else None, "cpu", d.get("cpu_baseline"), "clk", d.get("clocks"))
    for k, v in sorted((d.get("roofline_table") or {}).items(), key=lambda kv: -kv[1]["share_of_step"]):
        if k.startswith("_"):
            print("  ", k, v); continue
        print(f"  {k:16s} {v['bound']:6s} n={v['launches']:4d} avg={v['avg_launch_ms']*1e3:8.1f}us share={v['share_of_step']:.3f} "
              f"ach={v['achieved']:8.1f} {v['unit']} frac={v['frac']:.3f} gbs={v['achieved_gbs']:.0f} tfs={v['achieved_tflops']:.0f}")
    print("  roof", d.get("roofline"))
