#!/bin/bash
# 4 GPUs: parity (sharded state incl. the 18-qubit swap-kernel block, 35q coset oracle), overlap
# variants of the 30q R10 layer, weak scaling (32q), JW 32q
N=${NGPU:-4}
O=gpurun_out/${TAG:-m4}_$N; mkdir -p $O
timeout 1500 python -m pytest tests/test_multigpu.py -q -x -k "sharded_state or (large and $N)" > $O/tests.log 2>&1
echo "tests rc=$?" >> $O/tests.log; tail -2 $O/tests.log
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29716 bench.py --gpus $N --steps 3 --warmup 2 --no-e2e --no-cpu"
run() { label=$1; shift; timeout 900 $T "$@" > $O/$label.log 2>&1; echo "$label rc=$?"; grep '^{' $O/$label.log | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read() or '{}'); print(' ', d.get('value'), d.get('ms_per_step'), d.get('exchanges'), d.get('nvlink_gbs'))"; }
run R10_default
run R10_ovl1_reg --overlap 1 --swap-tma 0 --swap-ctas -1
run R10_ovl2_reg --swap-tma 0
run R10_ovl0 --overlap 0
run R10_fused --fused 1
run R10_32_weak --qubits 32
run JW_32 --kind JW --qubits 32
