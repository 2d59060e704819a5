#!/bin/bash
# round 2: emulated-rank parity (new), then the whole GPU suite
mkdir -p gpurun_out/r02b
timeout 600 python -m pytest tests/test_emulated.py -q > gpurun_out/r02b/test_emulated.log 2>&1
echo "emulated rc=$?" >> gpurun_out/r02b/test_emulated.log
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/r02b/test_gpu.log 2>&1
echo "gpu rc=$?" >> gpurun_out/r02b/test_gpu.log
# instruction-level profile of the tile kernel on a shallow (R10) and a deep (JW) pass
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu"
$B > gpurun_out/r02b/bench_r10.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_coset -s 3 -c 1 -o gpurun_out/r02b/prof_r10 $B > gpurun_out/r02b/ncu_r10.log 2>&1
echo "ncu r10 rc=$?"
$B --kind JW > gpurun_out/r02b/bench_jw.log 2>&1
echo "bench jw rc=$?"
