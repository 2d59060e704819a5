#!/bin/bash
# minimum contiguous chunk of a coset tile: fp32 128 B (default 4 bits) vs 256 / 512 B; fp64 256 vs 512 B
D=gpurun_out/chunk; mkdir -p $D
B="python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu"
for rep in 1 2; do
  for cb in 4 5 6; do timeout 300 $B --dtype c64 --chunk-bits $cb > $D/c64_cb${cb}_$rep.log 2>&1; done
  for cb in 4 5; do timeout 300 $B --chunk-bits $cb > $D/R10_cb${cb}_$rep.log 2>&1; done
done
for cb in 4 5; do
  timeout 600 $B --kind JW --chunk-bits $cb > $D/JW_cb${cb}.log 2>&1
  timeout 600 $B --kind JW --dtype c64 --chunk-bits $cb > $D/JWc64_cb${cb}.log 2>&1
done
timeout 300 $B --dtype c64 --chunk-bits 5 --tile-bits 12 > $D/c64_cb5_t12.log 2>&1
python tools/summ.py $D
