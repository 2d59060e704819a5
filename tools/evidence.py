"""Writes the round's profile summaries from one gpurun evidence capture (development aid).

python tools/evidence.py LAUNCHES_CSV NCU_REP BENCH_LOG REF_LOG [OUT_DIR=profiles/r01]
  - OUT/launches.csv + launches_summary.txt  (ncu gpu__time_duration.sum launch list, shares)
  - OUT/ncu_coset_full.txt                     (key metrics of the --set full capture)
  - OUT/bench_default.jsonl, bench_reference.jsonl
  - profiles/traffic.json "coset"              (dram read + write bytes of that launch)
"""
import collections
import csv
import json
import os
import shutil
import subprocess
import sys

launches, rep, bench_log, ref_log = sys.argv[1:5]
out = sys.argv[5] if len(sys.argv) > 5 else "profiles/r01"
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

rows = list(csv.reader(l for l in open(launches) if not l.startswith("==")))
h = rows[0]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[1:]:
    if len(r) <= vi:
        continue
    v = float(r[vi].replace(",", ""))
    ms = {"ns": v / 1e6, "us": v / 1e3, "usecond": v / 1e3, "nsecond": v / 1e6, "ms": v, "msecond": v}.get(r[ui], v * 1e3)
    name = r[ki].split("(")[0]
    for pre in ("void (anonymous namespace)::", "void unnamed>::", "void "):
        name = name.replace(pre, "")
    agg[name][0] += 1
    agg[name][1] += ms
tot = sum(a[1] for a in agg.values())
lines = ["# ncu launch list (gpu__time_duration.sum, --clock-control none; cold-cache, serialised: compare SHARES)",
         "# command: python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu   (30q fp64, R10 layer of 1000 rotations, 2 calls)",
         f"{'kernel':60s} {'launches':>9s} {'total_ms':>10s} {'avg_ms':>9s} {'share':>7s}"]
for k, (c, ms) in sorted(agg.items(), key=lambda t: -t[1][1]):
    lines.append(f"{k[-60:]:60s} {c:9d} {ms:10.2f} {ms / c:9.3f} {ms / tot:7.3f}")
open(os.path.join(out, "launches_summary.txt"), "w").write("\n".join(lines) + "\n")
shutil.copy(launches, os.path.join(out, "launches.csv"))
print("\n".join(lines))

raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h, u, v = rows[0], rows[1], rows[2]
res = ["# ncu --set full --clock-control none --import-source on, the coset tile kernel (K7), 30q fp64 R10 layer, 4th launch",
       "# command: ncu ... -k regex:k_coset -s 3 -c 1 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu",
       f"{'Kernel Name':70s} {v[h.index('Kernel Name')].split('(')[0]}"]
for w in ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
          "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread", "launch__block_size",
          "launch__grid_size", "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
          "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
          "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
          "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__occupancy_limit_registers"]:
    if w in h:
        i = h.index(w)
        res.append(f"{w:70s} {v[i]} {u[i]}")
st = {}
for i, n in enumerate(h):
    if n.startswith("smsp__pcsamp_warps_issue_stalled_") and not n.endswith("_not_issued"):
        try:
            st[n.replace("smsp__pcsamp_warps_issue_stalled_", "")] = float(v[i].replace(",", ""))
        except ValueError:
            pass
res.append("stall samples (top): " + ", ".join(f"{k}={int(x)}" for k, x in sorted(st.items(), key=lambda t: -t[1])[:8]))
scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1}
rd = float(v[h.index("dram__bytes_read.sum")].replace(",", "")) * scale[u[h.index("dram__bytes_read.sum")]]
wr = float(v[h.index("dram__bytes_write.sum")].replace(",", "")) * scale[u[h.index("dram__bytes_write.sum")]]
alg = 2 * 2 ** 30 * 16
res.append(f"traffic per launch = {rd + wr:.0f} B vs algorithmic 2*2^30*16 = {alg} B  (ratio {(rd + wr) / alg:.4f})")
open(os.path.join(out, "ncu_coset_full.txt"), "w").write("\n".join(res) + "\n")
print("\n".join(res))
tp = os.path.join(root, "profiles", "traffic.json")
d = json.load(open(tp))
d["coset"] = rd + wr
json.dump(d, open(tp, "w"), indent=1)
for src, dst in ((bench_log, "bench_default.jsonl"), (ref_log, "bench_reference.jsonl")):
    open(os.path.join(out, dst), "w").write(open(src).read().strip().splitlines()[-1] + "\n")
