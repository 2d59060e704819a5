#!/bin/bash
# TMA swap kernel vs the slim register kernel (overlap mode 2), N GPUs; parity first
N=${NGPU:-2}
O=gpurun_out/${TAG:-tma}_$N; mkdir -p $O
timeout 900 python -m pytest tests/test_multigpu.py -q -x -k "sharded_state" > $O/tests.log 2>&1
echo "tests rc=$?" >> $O/tests.log; tail -2 $O/tests.log
grep -h "swap kernels\|FAIL\|False" $O/tests.log | head -5
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29715 bench.py --gpus $N --steps 3 --warmup 2 --no-e2e --no-cpu"
run() { label=$1; shift; timeout 600 $T "$@" > $O/$label.log 2>&1; echo "$label rc=$?"; grep '^{' $O/$label.log | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read() or '{}'); print(' ', d.get('value'), d.get('ms_per_step'), d.get('nvlink_gbs'))"; }
run R10_tma
run R10_reg --swap-tma 0
run R10_tma_c1 --swap-ctas -1
run R10_tma_ovl1 --overlap 1
run R10_reg_ovl1 --overlap 1 --swap-tma 0
run R10_tma_pb3 --overlap $(( (4 << 16) | 2 ))
run R10_tma_b
run R10_reg_b --swap-tma 0
