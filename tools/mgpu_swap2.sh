#!/bin/bash
# overlap mode 2: swap CTAs and piece count sweep on N GPUs
N=${NGPU:-2}
O=gpurun_out/${TAG:-swap2}_$N; mkdir -p $O
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29714 bench.py --gpus $N --steps 3 --warmup 2 --no-e2e --no-cpu"
run() { label=$1; shift; timeout 600 $T "$@" > $O/$label.log 2>&1; echo "$label rc=$?"; grep '^{' $O/$label.log | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read() or '{}'); print(' ', d.get('value'), d.get('ms_per_step'), d.get('nvlink_gbs'))"; }
for c in -296 -444 -592 -1184; do
  run R10_ovl2_c${c} --overlap 2 --swap-ctas $c
done
for c in -296 -592; do
  run R10_ovl2_pb3_c${c} --overlap $(( (4 << 16) | 2 )) --swap-ctas $c
  run R10_ovl1_pb3_c${c} --overlap $(( (4 << 16) | 1 )) --swap-ctas $c
done
run R10_ovl2_full148 --overlap 2 --swap-ctas 148
timeout 900 python -m pytest tests/test_multigpu.py -q -k "sharded_state" > $O/tests.log 2>&1
echo "tests rc=$?" >> $O/tests.log; tail -2 $O/tests.log
