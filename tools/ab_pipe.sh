#!/bin/bash
# A/B of the rotation loop: nopipe (decode after the previous rotation), pipe (software-pipelined
# decode; the default build), pp (pipe + ping-pong buffers for same-dx runs)
D=gpurun_out/pipe
mkdir -p $D
B="python bench.py --no-e2e --no-cpu"
for rep in 1 2; do
for lib in nopipe pipe pp; do
  if [ $lib = pipe ]; then unset PS_LIB_PATH; else export PS_LIB_PATH=$PWD/paper_2504_17881_b200/libps_$lib.so; fi
  timeout 300 $B > $D/R10_${lib}_$rep.log 2>&1
  [ $rep = 1 ] && timeout 900 $B --kind JW --steps 2 --warmup 1 > $D/JW_${lib}.log 2>&1
  [ $rep = 1 ] && timeout 300 $B --kind GATES --layer 200 > $D/GATES_${lib}.log 2>&1
  [ $rep = 1 ] && timeout 300 $B --kind QAOA --layer 100 > $D/QAOA_${lib}.log 2>&1
done
done
unset PS_LIB_PATH
export PS_LIB_PATH=$PWD/paper_2504_17881_b200/libps_pp.so
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_workloads.py -q -x > $D/tests_pp.log 2>&1; echo "pp tests rc=$?" >> $D/tests_pp.log
unset PS_LIB_PATH
