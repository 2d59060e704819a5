"""Prints one summary row per bench JSON log (tools/summarize.py gpurun_out/sweep_*.log)."""
import json
import sys

for path in sys.argv[1:]:
    try:
        d = json.loads(open(path).read().strip().splitlines()[-1])
    except Exception as e:  # noqa: BLE001
        print(path, "unparsable:", open(path).read()[-300:].replace("\n", " | "))
        continue
    r = d["roofline"]
    print(f"{path.split('/')[-1]:28s} {d['value']:9.1f} rot/s  {d['ms_per_step']:8.1f} ms/step  {r['kernel']:6s} "
          f"{r['achieved']:7.0f} GB/s frac {r['frac']:.3f}  rot/pass {d['rotations_per_pass']:6.2f} "
          f"passes {d['passes']}  clk {d['clocks']['sm_mhz'] if d.get('clocks') else None} "
          f"{d['clocks']['reasons'] if d.get('clocks') else ''}")
