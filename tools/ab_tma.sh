#!/bin/bash
# A/B: next-tile prefetch by LDGSTS (tune 3584, default) vs TMA bulk copies per chunk (tune 1536 | 4096)
D=gpurun_out/tma
mkdir -p $D
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "param_block or sizes_and_kinds or config1 or large" > $D/tests_default.log 2>&1
B="python bench.py --no-e2e --no-cpu"
for rep in 1 2; do
  timeout 300 $B --tile-tune 3584 > $D/R10_ldgsts_$rep.log 2>&1
  timeout 300 $B --tile-tune 5632 > $D/R10_tma_$rep.log 2>&1
  timeout 300 $B --dtype c64 --tile-tune 1536 > $D/c64_none_$rep.log 2>&1
  timeout 300 $B --dtype c64 --tile-tune 5632 > $D/c64_tma_$rep.log 2>&1
done
timeout 900 $B --kind JW --steps 2 --warmup 1 --tile-tune 5632 > $D/JW_tma.log 2>&1
timeout 900 $B --kind JW --steps 2 --warmup 1 --tile-tune 3584 > $D/JW_ldgsts.log 2>&1
export PS_LIB_PATH=$PWD/paper_2504_17881_b200/libps_pretma.so
for rep in 1 2; do timeout 300 $B > $D/R10_pretma_$rep.log 2>&1; done
timeout 900 $B --kind JW --steps 2 --warmup 1 > $D/JW_pretma.log 2>&1
unset PS_LIB_PATH
