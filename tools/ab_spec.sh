#!/bin/bash
# A/B: generic vs unit-dx specialised tile kernel (PS_OPT_SPECIALIZE 0 / 2 / 1) on shallow and deep passes
mkdir -p gpurun_out/spec
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "specialised or param_block or sizes_and_kinds" > gpurun_out/spec/tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/spec/tests.log
B="python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu"
for k in R10 JW GATES QAOA UCC; do
  for sp in 0 2 1; do
    extra=""
    [ $k = UCC ] && extra="--layer 3000"
    [ $k = GATES ] && extra="--layer 200"
    [ $k = QAOA ] && extra="--layer 100"
    timeout 600 $B --kind $k --specialize $sp $extra > gpurun_out/spec/${k}_sp${sp}.log 2>&1; echo "$k $sp rc=$?"
  done
done
for sp in 0 2; do timeout 300 $B --dtype c64 --specialize $sp > gpurun_out/spec/c64_R10_sp${sp}.log 2>&1; done
