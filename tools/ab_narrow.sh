#!/bin/bash
# A/B: 32-bit element indices in the default tile kernels (default build) vs 64-bit (libps_wide.so)
D=gpurun_out/narrow
mkdir -p $D
B="python bench.py --no-e2e --no-cpu"
for rep in 1 2; do
for lib in wide narrow; do
  if [ $lib = narrow ]; then unset PS_LIB_PATH; else export PS_LIB_PATH=$PWD/paper_2504_17881_b200/libps_$lib.so; fi
  timeout 300 $B > $D/R10_${lib}_$rep.log 2>&1
  timeout 300 $B --dtype c64 > $D/c64_${lib}_$rep.log 2>&1
  [ $rep = 1 ] && timeout 900 $B --kind JW --steps 2 --warmup 1 > $D/JW_${lib}.log 2>&1
done
done
unset PS_LIB_PATH
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_large.py -q -x > $D/tests.log 2>&1; echo "tests rc=$?" >> $D/tests.log
