#!/bin/bash
# multi-GPU round 2: parity (mp_worker: fused exchange over real NVLink peers), strong/weak scaling,
# fused vs swap, the NEXT-4 suffix-group A/B (L = 1/10/100; layouts 0/1/2)
N=${NGPU:-2}
mkdir -p gpurun_out/mgpu$N
timeout 1500 python -m pytest tests/test_multigpu.py -q -k "sharded_state or (large and $N)" > gpurun_out/mgpu$N/tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/mgpu$N/tests.log
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29711 bench.py --gpus $N --steps 3 --warmup 2 --no-e2e --no-cpu"
run() { label=$1; shift; timeout 900 $T "$@" > gpurun_out/mgpu$N/$label.log 2>&1; echo "$label rc=$?"; }
run R10_30_fused1 --fused 1
run R10_30_fused0 --fused 0
run R10_30_fused0_ovl0 --fused 0 --overlap 0
run R10_30_layout0 --layout 0
nw=$((30 + $(python -c "print(($N).bit_length()-1)")))
run R10_${nw}_weak --qubits $nw
for L in ${LS-1 10 100}; do
  for lay in 0 1 2; do
    run SUFFIX_L${L}_layout${lay} --kind SUFFIX --group $L --layout $lay --layer 1000 --qubits 30
  done
  run SUFFIX_L${L}_layout1_fused0 --kind SUFFIX --group $L --layout 1 --fused 0 --layer 1000 --qubits 30
done
run JW_32 --kind JW --qubits 32
run JW_32_fused1 --kind JW --qubits 32 --fused 1
