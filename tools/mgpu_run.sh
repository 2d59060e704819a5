# multi-GPU checks on one box: sharded parity tests, then the default bench at N = 2 (and 4)
mkdir -p gpurun_out
N=${1:-2}
timeout 900 python -m pytest tests/test_multigpu.py -m gpu -x -q > gpurun_out/mg_tests_g$N.log 2>&1; echo tests=$?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 \
  bench.py --gpus $N --steps 3 --warmup 3 > gpurun_out/mg_bench_g$N.log 2>&1; echo bench=$?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29512 \
  bench.py --gpus $N --steps 2 --warmup 3 --qubits 32 --kind JW --no-e2e > gpurun_out/mg_jw32_g$N.log 2>&1; echo jw32=$?
