"""Prints value / frac / rot-per-pass / clocks of every bench JSON log in the given directory."""
import json, os, sys
d = sys.argv[1]
for f in sorted(os.listdir(d)):
    if not f.endswith(".log"):
        continue
    for line in open(os.path.join(d, f)):
        if line.startswith("{"):
            j = json.loads(line)
            r = j.get("roofline") or {}
            c = j.get("clocks") or {}
            print(f"{f:28s} {j['value']:9.1f} {j['unit']}  frac {r.get('frac', 0):.3f}  rpp {j.get('rotations_per_pass', 0):6.2f}  "
                  f"kern {r.get('kernel')} {r.get('avg_launch_ms', 0):.3f} ms  clk {c.get('sm_mhz')} {c.get('reasons')}")
