#!/bin/bash
# usage: scripts_bench_sweep.sh "<label>:<bench args>" ...   (runs each, writes gpurun_out/sweep_<label>.log)
for spec in "$@"; do
  label="${spec%%:*}"; args="${spec#*:}"
  timeout 300 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu $args > gpurun_out/sweep_$label.log 2>&1
  echo "$label rc=$?"
done
