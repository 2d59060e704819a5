#!/bin/bash
# A/B of the default fp64 tile kernel's launch knobs (30q R10) + the pre-XT build as a same-box reference
D=gpurun_out/tune
mkdir -p $D
B="python bench.py --no-e2e --no-cpu"
for rep in 1 2; do
  timeout 300 $B > $D/R10_default_$rep.log 2>&1
  timeout 300 $B --tile-tune $((3584 | (2 << 4))) > $D/R10_gm2_$rep.log 2>&1
  timeout 300 $B --tile-tune $((3584 | (8 << 4))) > $D/R10_gm8_$rep.log 2>&1
  timeout 300 $B --tile-tune 3072 > $D/R10_no256hint_$rep.log 2>&1
  PS_LIB_PATH=$PWD/paper_2504_17881_b200/libps_pretma.so timeout 300 $B > $D/R10_pretma_$rep.log 2>&1
done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_workloads.py -q -x > $D/tests.log 2>&1; echo "tests rc=$?" >> $D/tests.log
for rep in 1 2; do
  PS_LIB_PATH=$PWD/paper_2504_17881_b200/libps_d2.so timeout 300 $B > $D/R10_d2_$rep.log 2>&1
done
PS_LIB_PATH=$PWD/paper_2504_17881_b200/libps_d2.so timeout 900 $B --kind JW --steps 2 --warmup 1 > $D/JW_d2.log 2>&1
timeout 900 $B --kind JW --steps 2 --warmup 1 > $D/JW_default.log 2>&1
PS_LIB_PATH=$PWD/paper_2504_17881_b200/libps_d2.so timeout 300 $B --kind GATES --layer 200 > $D/GATES_d2.log 2>&1
timeout 300 $B --kind GATES --layer 200 > $D/GATES_default.log 2>&1
