"""Print the key fields of a bench.py JSON line: python scripts/bench_summary.py file [label]"""
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
lab = sys.argv[2] if len(sys.argv) > 2 else ""
r, s = d.get("roofline") or {}, d.get("scan") or {}
out = {"label": lab, "value": round(d["value"]), "ms_step": round(d["ms_per_step"], 3),
       "achieved": round(r.get("achieved", 0)), "frac": round(r.get("frac", 0), 3),
       "clock": (d.get("clocks") or {}).get("sm_mhz")}
if s:
    out.update({"scan_gbs": round(s["roofline"]["achieved"]), "scan_frac": round(s["roofline"]["frac"], 3),
                "scan_qps": round(s["value"])})
if d.get("latency_ms"):
    out.update({"p50": d["latency_ms"]["p50"], "p99": d["latency_ms"]["p99"]})
print(json.dumps(out))
