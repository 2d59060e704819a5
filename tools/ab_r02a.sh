#!/bin/bash
# round 2 A/B: tile size 2^13 / 2^14 and 128-B chunks (30q R10), plus the large-n / big-tile parity tests
mkdir -p gpurun_out/r02a
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02a/gpu.txt 2>&1
nproc >> gpurun_out/r02a/gpu.txt
timeout 900 python -m pytest tests/test_gpu_large.py -x -q > gpurun_out/r02a/test_large.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02a/test_large.log
B="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu"
run() { label=$1; shift; timeout 300 $B "$@" > gpurun_out/r02a/$label.log 2>&1; echo "$label rc=$?"; }
run f64_tb12 --tile-bits 12
run f64_tb13 --tile-bits 13
run f64_tb12_c3 --tile-bits 12 --chunk-bits 3
run f64_tb13_c3 --tile-bits 13 --chunk-bits 3
run f64_tb12_again --tile-bits 12
run f32_tb11 --dtype c64 --tile-bits 11
run f32_tb12 --dtype c64 --tile-bits 12
run f32_tb13 --dtype c64 --tile-bits 13
run f32_tb14 --dtype c64 --tile-bits 14
run f32_tb13_c3 --dtype c64 --tile-bits 13 --chunk-bits 3
run f64_tb13_nopf --tile-bits 13 --tile-tune 1536
