#!/bin/bash
# the larger BASELINE.json configs on the 4 GPUs we can get: 34q QAOA / gate circuit (config 4 at
# half the GPUs: 64 GiB per GPU) and a 35q JW-shaped Trotter step (128 GiB per GPU, the per-GPU
# footprint of config 5's 36q on 8 GPUs; 4000 terms to bound the step time)
N=${NGPU:-4}
O=gpurun_out/big_$N; mkdir -p $O
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29721 bench.py --gpus $N --no-e2e --no-cpu"
run() { label=$1; shift; timeout 600 $T "$@" > $O/$label.log 2>&1; echo "$label rc=$?"; grep '^{' $O/$label.log | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read() or '{}'); print(' ', d.get('value'), d.get('ms_per_step'), d.get('exchanges'), (d.get('roofline') or {}).get('frac'))"; }
run QAOA_34 --kind QAOA --qubits 34 --layer 10 --steps 3 --warmup 3
run GATES_34 --kind GATES --qubits 34 --layer 20 --steps 3 --warmup 3
run JW_35 --kind JW --qubits 35 --terms 4000 --steps 2 --warmup 1
