#!/bin/bash
# last check of the committed tree on a 2-GPU box: the full GPU suite (the multi-GPU tests run too),
# smoke, 1-GPU bench lines, launch list and ncu summary (tools/r02_final.sh), then the 2-GPU bench
FINAL_DIR=final3 SKIP_Z0=1 bash tools/r02_final.sh
D=gpurun_out/final3
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29718 \
  bench.py --gpus 2 --steps 3 --warmup 3 > $D/bench_2gpu.log 2>&1; echo "bench2gpu rc=$?"
grep -h "passed\|failed" $D/tests.log | tail -1
