"""Summarises one ncu --set full capture (development aid; output is committed under profiles/).

python tools/ncu_summary.py REP [--algorithmic BYTES] [--title TEXT]

Prints, per captured kernel: duration, DRAM bytes (read + write) against the algorithmic bytes,
achieved DRAM GB/s, issue activity, fp64 pipe use, occupancy limits, warp-stall samples and -- from
the SASS source page -- the dynamic instruction mix by opcode.
"""
import argparse
import collections
import csv
import io
import subprocess

SCALE = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1, "Tbyte": 1e12}
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread", "launch__block_size",
        "launch__grid_size", "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "smsp__warps_issue_stalled_no_instruction_per_warp_active.pct"]


def num(s):
    try:
        return float(s.replace(",", ""))
    except ValueError:
        return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--algorithmic", type=float, default=0.0)
    ap.add_argument("--title", default="")
    a = ap.parse_args()
    raw = subprocess.run(["ncu", "-i", a.rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, u = rows[0], rows[1]
    if a.title:
        print("#", a.title)
    for v in rows[2:]:
        name = v[h.index("Kernel Name")].split("(")[0]
        print(f"{'Kernel Name':62s} {name}")
        for k in KEYS:
            if k in h:
                i = h.index(k)
                print(f"{k:62s} {v[i]} {u[i]}")
        t = num(v[h.index("gpu__time_duration.sum")])
        tu = u[h.index("gpu__time_duration.sum")]
        secs = t * {"nsecond": 1e-9, "ns": 1e-9, "usecond": 1e-6, "us": 1e-6, "msecond": 1e-3, "ms": 1e-3, "second": 1, "s": 1}.get(tu, 1e-9)
        rd = num(v[h.index("dram__bytes_read.sum")]) * SCALE.get(u[h.index("dram__bytes_read.sum")], 1)
        wr = num(v[h.index("dram__bytes_write.sum")]) * SCALE.get(u[h.index("dram__bytes_write.sum")], 1)
        print(f"{'dram traffic (read + write)':62s} {rd + wr:.0f} B  = {(rd + wr) / secs / 1e9:.1f} GB/s over the launch")
        if a.algorithmic:
            print(f"{'algorithmic bytes':62s} {a.algorithmic:.0f} B  (traffic / algorithmic = {(rd + wr) / a.algorithmic:.4f}; "
                  f"algorithmic GB/s = {a.algorithmic / secs / 1e9:.1f})")
        st = {}
        for i, n in enumerate(h):
            if n.startswith("smsp__pcsamp_warps_issue_stalled_") and not n.endswith("_not_issued"):
                x = num(v[i])
                if x is not None:
                    st[n.replace("smsp__pcsamp_warps_issue_stalled_", "")] = x
        tot = sum(st.values()) or 1
        print("warp-state samples:", ", ".join(f"{k} {x / tot * 100:.1f}%" for k, x in sorted(st.items(), key=lambda t: -t[1])[:10]))
    src = subprocess.run(["ncu", "-i", a.rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    srows = list(csv.reader(io.StringIO(src)))
    if len(srows) > 2:
        sh = srows[1]
        ix = {k: i for i, k in enumerate(sh)}
        mix = collections.Counter()
        tot = 0
        for r in srows[2:]:
            if len(r) < len(sh):
                continue
            n = num(r[ix["Instructions Executed"]] or "0") or 0
            s = r[ix["Source"]].strip().split()
            if not s:
                continue
            op = (s[1] if s[0].startswith("@") else s[0]).split(".")[0]
            mix[op] += n
            tot += n
        print(f"dynamic warp instructions {tot:.0f}; mix: " +
              ", ".join(f"{k} {x / tot * 100:.1f}%" for k, x in mix.most_common(14)))


if __name__ == "__main__":
    main()
