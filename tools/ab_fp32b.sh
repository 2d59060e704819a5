#!/bin/bash
# fp32 default 2^12 tiles (256 x 4): parity suites, then with / without the LDGSTS next-tile prefetch
D=gpurun_out/fp32b; mkdir -p $D
timeout 1200 python -m pytest tests/test_gpu_large.py tests/test_gpu_parity.py tests/test_gpu_workloads.py tests/test_emulated.py -q -x > $D/tests.log 2>&1; echo "tests rc=$?" >> $D/tests.log; tail -2 $D/tests.log
B="python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu --dtype c64"
for rep in 1 2; do
  timeout 300 $B > $D/c64_def_$rep.log 2>&1
  timeout 300 $B --tile-tune 3584 > $D/c64_pf_$rep.log 2>&1
done
timeout 600 $B --kind JW > $D/JWc64_def.log 2>&1
timeout 600 $B --kind JW --tile-tune 3584 > $D/JWc64_pf.log 2>&1
timeout 300 $B --kind QAOA --layer 100 > $D/QAOAc64_def.log 2>&1
timeout 300 $B --kind QAOA --layer 100 --tile-bits 11 > $D/QAOAc64_t11.log 2>&1
python tools/summ.py $D
