#!/bin/bash
# fp32: 2^11 tiles (128 threads x 8 CTAs, default) vs 2^12 tiles on 256 threads x 4 CTAs (tune 1542)
D=gpurun_out/fp32; mkdir -p $D
B="python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu --dtype c64"
for rep in 1 2; do
  timeout 300 $B > $D/c64_def_$rep.log 2>&1
  timeout 300 $B --tile-bits 12 --tile-tune 1542 > $D/c64_t12o4_$rep.log 2>&1
  timeout 300 $B --tile-bits 12 --tile-tune 1542 --chunk-bits 5 > $D/c64_t12o4_cb5_$rep.log 2>&1
done
timeout 300 $B --tile-bits 12 > $D/c64_t12o2.log 2>&1
timeout 600 $B --kind JW > $D/JWc64_def.log 2>&1
timeout 600 $B --kind JW --tile-bits 12 --tile-tune 1542 > $D/JWc64_t12o4.log 2>&1
timeout 300 $B --kind GATES --layer 200 > $D/GATESc64_def.log 2>&1
timeout 300 $B --kind GATES --layer 200 --tile-bits 12 --tile-tune 1542 > $D/GATESc64_t12o4.log 2>&1
timeout 600 python -m pytest tests/test_gpu_large.py -q -x -k "c64" > $D/tests_def.log 2>&1; echo "tests rc=$?" >> $D/tests_def.log
python tools/summ.py $D
