"""Print the key numbers of a bench.py JSON line: python tools/bench_summary.py FILE"""
import json
import sys

lines = [ln for ln in open(sys.argv[1]).read().splitlines() if ln.strip().startswith("{")]
if not lines:
    print("no json line in", sys.argv[1])
    sys.exit(0)
d = json.loads(lines[-1])
r = d.get("roofline") or {}
print("value %.4g %s | ms/step %.3f | stages %s" % (d["value"], d["unit"], d["ms_per_step"], d.get("stage_ms_per_step")))
print("roofline %s: %.4f ms/launch, achieved %.1f, frac %.3f (burst %.3f, probe %.3f) | clocks %s" % (
    r.get("kernel"), r.get("ms_per_launch", 0), r.get("achieved", 0), r.get("frac", 0), r.get("frac_burst", 0),
    r.get("frac_probe", 0), d.get("clocks")))
print("e2e", (d.get("e2e") or {}).get("value"), "parity", d.get("parity"))
