"""Static SASS statistics of one kernel in a built libps (development aid).

python tools/sass_stats.py LIB NAME_SUBSTRING  -> per-basic-block MOV / DFMA / other counts,
summed over blocks that contain DFMA (rotation cases) and blocks that do not (load/store/setup).
"""
import collections
import subprocess
import sys

lib, pat = sys.argv[1], sys.argv[2]
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
funcs = {}
cur = None
for line in out.splitlines():
    if "Function :" in line:
        cur = line.split("Function :")[1].strip()
        funcs[cur] = []
    elif cur and "/*" in line and ";" in line:
        ins = line.split("*/", 1)[1].split(";")[0].strip()
        if ins:
            funcs[cur].append(ins)
names = [f for f in funcs if pat in f]
for f in names:
    ins = funcs[f]
    blocks, b = [], []
    for i in ins:
        b.append(i)
        op = i.split()[1] if i.startswith("@") else i.split()[0]
        if op.startswith(("BRA", "BRX", "EXIT", "RET")):
            blocks.append(b)
            b = []
    blocks.append(b)
    agg = collections.Counter()
    for b in blocks:
        c = collections.Counter()
        for i in b:
            op = i.split()[1] if i.startswith("@") else i.split()[0]
            c["MOV" if "MOV" in op else "DFMA" if op == "DFMA" else "FFMA" if op == "FFMA" else "other"] += 1
        kind = "rot" if (c["DFMA"] or c["FFMA"]) else "misc"
        for k, v in c.items():
            agg[kind + "_" + k] += v
    print(f[:110], len(ins), dict(sorted(agg.items())))
