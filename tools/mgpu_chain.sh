#!/bin/bash
# overlap chains (pass, E, pass, E, ..., pass as one pipeline) on N GPUs: parity, then the 30q R10
# layer (default) twice, the 31q/32q weak point and JW 32q
N=${NGPU:-2}
O=gpurun_out/${TAG:-chain}_$N; mkdir -p $O
timeout 1500 python -m pytest tests/test_multigpu.py -q -x -k "sharded_state or (large and $N)" > $O/tests.log 2>&1
echo "tests rc=$?" >> $O/tests.log; tail -2 $O/tests.log
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29717 bench.py --gpus $N --steps 3 --warmup 2 --no-e2e --no-cpu"
run() { label=$1; shift; timeout 900 $T "$@" > $O/$label.log 2>&1; echo "$label rc=$?"; grep '^{' $O/$label.log | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read() or '{}'); print(' ', d.get('value'), d.get('ms_per_step'), d.get('exchanges'), d.get('nvlink_gbs'))"; }
run R10_chain
run R10_chain_b
run R10_chain_pb3 --overlap $(( (4 << 16) | 2 ))
nw=$((30 + $(python -c "print(($N).bit_length()-1)")))
run R10_${nw}_weak --qubits $nw
run JW_32 --kind JW --qubits 32
run R10_fused --fused 1
