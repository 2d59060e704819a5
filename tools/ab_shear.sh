#!/bin/bash
# A/B: unit-case rotations as three in-place shears (libps_shear.so, -DPS_SHEAR=1) vs the 4-FMA
# deferred-scale form (default build), same box
# build the A/B library first: python -m paper_2504_17881_b200.build --force -DPS_SHEAR=1 --out=paper_2504_17881_b200/libps_shear.so
D=gpurun_out/shear; mkdir -p $D
export PS_LIB_PATH=$PWD/paper_2504_17881_b200/libps_shear.so
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_workloads.py tests/test_emulated.py -q -x > $D/tests_shear.log 2>&1
echo "tests rc=$?" >> $D/tests_shear.log; tail -2 $D/tests_shear.log
B="python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu"
for rep in 1 2; do
for lib in def shear; do
  if [ $lib = shear ]; then export PS_LIB_PATH=$PWD/paper_2504_17881_b200/libps_shear.so; else unset PS_LIB_PATH; fi
  timeout 300 $B > $D/R10_${lib}_$rep.log 2>&1
  if [ $rep = 1 ]; then
    timeout 600 $B --kind JW > $D/JW_${lib}.log 2>&1
    timeout 300 $B --kind GATES --layer 200 > $D/GATES_${lib}.log 2>&1
    timeout 300 $B --kind QAOA --layer 100 > $D/QAOA_${lib}.log 2>&1
    timeout 300 $B --kind UCC --layer 3000 > $D/UCC_${lib}.log 2>&1
  fi
done
done
unset PS_LIB_PATH
python tools/summ.py $D
