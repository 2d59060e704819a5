"""Per-source-line attribution of one ncu capture (development aid).

python tools/line_attrib.py LIB.so KERNEL_SUBSTRING SASS_CSV(.gz) [TOP]

Disassembles KERNEL from LIB.so with line info (cuobjdump -xelf + nvdisasm -g), joins the
instruction offsets with the per-instruction execution counts of the ncu source page (same
binary), and prints the source lines carrying the most dynamic warp instructions.
"""
import collections
import csv
import gzip
import io
import os
import re
import subprocess
import sys
import tempfile


def main():
    lib, kname, sass_csv = sys.argv[1:4]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=tmp, capture_output=True)
    cub = [f for f in os.listdir(tmp) if f.endswith(".cubin") and "kernels" in f and "api" not in f][0]
    dis = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(tmp, cub)], capture_output=True, text=True).stdout
    lines = dis.splitlines()
    start = None
    for i, l in enumerate(lines):
        if l.startswith(".text.") and kname in l:
            start = i
            break
    if start is None:
        raise SystemExit("kernel not found")
    off2line = {}
    cur = ("?", 0)
    for l in lines[start + 1:]:
        if l.startswith(".text.") or l.startswith("//----"):
            break
        m = re.search(r'//## File "([^"]+)", line (\d+)', l)
        if m:
            cur = (os.path.basename(m.group(1)), int(m.group(2)))
            continue
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*)", l)
        if m:
            off2line[int(m.group(1), 16)] = (cur, m.group(2).strip())
    op = gzip.open if sass_csv.endswith(".gz") else open
    rows = list(csv.reader(io.StringIO(op(sass_csv, "rt").read())))
    h = rows[1]
    ix = {k: i for i, k in enumerate(h)}
    recs = []
    for r in rows[2:]:
        try:
            recs.append((int(r[ix["Address"]], 16), float(r[ix["Instructions Executed"]] or 0),
                         float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)))
        except (ValueError, IndexError):
            continue
    base = min(a for a, _, _ in recs)
    agg = collections.defaultdict(lambda: [0.0, 0.0, collections.Counter()])
    tot = 0.0
    for a, n, smp in recs:
        ln, ins = off2line.get(a - base, (("?", 0), "?"))
        agg[ln][0] += n
        agg[ln][1] += smp
        agg[ln][2][ins.split()[0] if not ins.startswith("@") else ins.split()[1]] += n
        tot += n
    srcs = {}
    for (f, ln) in agg:
        for cand in ("paper_2504_17881_b200/csrc/" + f, f):
            if os.path.exists(cand):
                srcs.setdefault(f, open(cand).read().splitlines())
    stot = sum(v[1] for v in agg.values()) or 1
    print(f"total dynamic warp instructions {tot:.3e}")
    for (f, ln), (n, smp, ops) in sorted(agg.items(), key=lambda t: -t[1][0])[:top]:
        text = srcs.get(f, [""] * (ln + 1))[ln - 1].strip()[:70] if ln else ""
        print(f"{n / tot * 100:5.1f}% inst {smp / stot * 100:5.1f}% smp  {f}:{ln:<5d} {text:70s} "
              f"{', '.join(f'{k.split(chr(46))[0]}:{v / n * 100:.0f}' for k, v in ops.most_common(3))}")


if __name__ == "__main__":
    main()
