"""Collects the bench JSON line of every log in the given gpurun_out directories into one JSONL file,
each line tagged with its source ("src": "<dir>/<log>").  python tools/collect_jsonl.py OUT DIR..."""
import json
import os
import sys

out, dirs = sys.argv[1], sys.argv[2:]
with open(out, "w") as f:
    for d in dirs:
        for name in sorted(os.listdir(d)):
            if not name.endswith(".log"):
                continue
            for line in open(os.path.join(d, name)):
                if line.startswith("{"):
                    j = json.loads(line)
                    j["src"] = f"{os.path.basename(d.rstrip('/'))}/{name}"
                    f.write(json.dumps(j) + "\n")
