#!/bin/bash
# A/B: old tile-kernel body (libps_old.so) vs the new one (tile at smem offset 0, xor-chain element
# offsets, 32 uint16 representative slots, unit-dx specialisation), same box
mkdir -p gpurun_out/body
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_large.py tests/test_gpu_workloads.py -q -x > gpurun_out/body/tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/body/tests.log
B="python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu"
for rep in 1 2; do
for lib in old new; do
  if [ $lib = old ]; then export PS_LIB_PATH=$PWD/paper_2504_17881_b200/libps_old.so; else unset PS_LIB_PATH; fi
  for sp in 0 2; do
    timeout 300 $B --specialize $sp > gpurun_out/body/R10_${lib}_sp${sp}_$rep.log 2>&1
    timeout 300 $B --dtype c64 --specialize $sp > gpurun_out/body/c64_${lib}_sp${sp}_$rep.log 2>&1
  done
done
done
for lib in old new; do
  if [ $lib = old ]; then export PS_LIB_PATH=$PWD/paper_2504_17881_b200/libps_old.so; else unset PS_LIB_PATH; fi
  for sp in 0 2; do
    timeout 900 $B --kind JW --specialize $sp > gpurun_out/body/JW_${lib}_sp${sp}.log 2>&1
    timeout 300 $B --kind GATES --layer 200 --specialize $sp > gpurun_out/body/GATES_${lib}_sp${sp}.log 2>&1
  done
done
unset PS_LIB_PATH
# deep-pass profile (JW Trotter step) with the new body and unit specialisation
B1="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --kind JW --specialize 2"
$B1 > gpurun_out/body/jw_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_coset -s 20 -c 1 -o gpurun_out/body/prof_jw $B1 > gpurun_out/body/ncu_jw.log 2>&1
echo "ncu jw rc=$?"
