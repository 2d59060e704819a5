#!/bin/bash
# overlap mode 2 on N GPUs: parity on real ranks (mp_worker ovl=2 configs), then the 30q R10 layer
# with overlap 1 vs 2, the JW 32q step and the L=1 suffix groups
N=${NGPU:-2}
O=gpurun_out/ovl2_$N; mkdir -p $O
timeout 900 python -m pytest tests/test_multigpu.py -q -k "sharded_state" > $O/tests.log 2>&1
echo "tests rc=$?" >> $O/tests.log
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29712 bench.py --gpus $N --steps 3 --warmup 2 --no-e2e --no-cpu"
run() { label=$1; shift; timeout 600 $T "$@" > $O/$label.log 2>&1; echo "$label rc=$?"; grep '^{' $O/$label.log | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read() or '{}'); print(' ', d.get('value'), d.get('ms_per_step'))"; }
run R10_30_ovl1 --overlap 1
run R10_30_ovl2 --overlap 2
run R10_30_ovl1b --overlap 1
run R10_30_ovl2b --overlap 2
run SUFFIX_L1_ovl1 --kind SUFFIX --group 1 --layer 1000 --qubits 30 --overlap 1
run SUFFIX_L1_ovl2 --kind SUFFIX --group 1 --layer 1000 --qubits 30 --overlap 2
run JW_32_ovl2 --kind JW --qubits 32 --overlap 2
