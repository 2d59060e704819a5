#!/bin/bash
# slim overlap swap kernel (co-resides with the tile kernel) vs full-size swap CTAs, overlap modes
# 1 / 2, on N GPUs; then (1 GPU) the shear A/B
N=${NGPU:-2}
O=gpurun_out/${TAG:-swap}_$N; mkdir -p $O
timeout 900 python -m pytest tests/test_multigpu.py -q -k "sharded_state" > $O/tests.log 2>&1
echo "tests rc=$?" >> $O/tests.log; tail -2 $O/tests.log
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29713 bench.py --gpus $N --steps 3 --warmup 2 --no-e2e --no-cpu"
run() { label=$1; shift; timeout 600 $T "$@" > $O/$label.log 2>&1; echo "$label rc=$?"; grep '^{' $O/$label.log | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read() or '{}'); print(' ', d.get('value'), d.get('ms_per_step'), d.get('nvlink_gbs'))"; }
run R10_ovl1_slim --overlap 1
run R10_ovl2_slim_pb1 --overlap $(( (2 << 16) | 2 ))
run R10_ovl1_slim_pb3 --overlap $(( (4 << 16) | 1 ))
run R10_ovl2_slim --overlap 2
run R10_ovl1_full32 --overlap 1 --swap-ctas 32
run R10_ovl2_full32 --overlap 2 --swap-ctas 32

run R10_ovl2_slim296 --overlap 2 --swap-ctas -296
run R10_ovl0 --overlap 0
run R10_ovl1_slim296 --overlap 1 --swap-ctas -296
run JW_32_ovl1_slim --kind JW --qubits 32

