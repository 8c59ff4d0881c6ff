"""Print a compact summary of a bench.py JSON line: headline, roofline, per-layer ours vs cuDNN."""
import json
import sys

d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print("headline", d["metric"], round(d["value"], 1), d["unit"], "ms/step", round(d["ms_per_step"], 4), "vs_cudnn",
      round(d.get("vs_cudnn") or 0, 3), "clocks", d.get("clocks"))
print("e2e", {k: (round(v, 3) if isinstance(v, float) else v) for k, v in d["e2e"].items() if k != "ms_per_step_runs"})
r = d["roofline"]
print("roofline", {k: (round(v, 4) if isinstance(v, float) else v) for k, v in r.items() if k != "method"})
for rec in d["layers"]:
    print("  ", rec["layer"], rec["plan"][:50], "ours", round(rec["ours_us"], 1), "warm", round(rec["ours_warm_us"], 1),
          "cud", round(rec.get("cudnn_us", 0), 1), "cudw", round(rec.get("cudnn_warm_us", 0), 1))
for name, s in (d.get("suite") or {}).items():
    if "error" in s:
        print(name, s["error"])
        continue
    st = s["step"]
    print("==", name, s["dtype"], {k: round(v, 2) for k, v in st.items() if isinstance(v, float)})
    for rec in s["layers"]:
        print("    ", rec["layer"], rec["plan"][:44], "ours", round(rec["ours_us"], 1), "warm", round(rec["ours_warm_us"], 1),
              "cud", round(rec.get("cudnn_us", 0), 1), "cudw", round(rec.get("cudnn_warm_us", 0), 1),
              "frac", round(rec["frac"], 3), rec["bound"])
for k, v in (d.get("eops") or {}).items():
    print("eop", k, round(v["us"], 1) if isinstance(v, dict) else v, round(v.get("frac_of_hbm", 0), 3) if isinstance(v, dict) else "")
print("g2bmm", json.dumps(d.get("g2bmm"))[:300])
