#!/bin/bash
mkdir -p gpurun_out/tma
timeout 900 python -m pytest tests/test_emulated.py tests/test_gpu_large.py -q -x > gpurun_out/tma/tests_emu_large.log 2>&1
echo "tests rc=$?" >> gpurun_out/tma/tests_emu_large.log
bash tools/ab_tma.sh
timeout 300 python bench.py --emulate 2 --no-e2e --no-cpu --fused 1 > gpurun_out/tma/emu2_fused1.log 2>&1
timeout 300 python bench.py --emulate 2 --no-e2e --no-cpu --fused 0 > gpurun_out/tma/emu2_fused0.log 2>&1
