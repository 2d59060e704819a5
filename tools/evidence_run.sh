# round-end evidence capture on one B200: GPU tests, smoke, default bench, reference arm,
# ncu launch list, one --set full capture of the tile kernel, fp32 line
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/ev_tests.log 2>&1; echo tests=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ev_smoke.log 2>&1; echo smoke=$?
timeout 600 python bench.py > gpurun_out/ev_bench.log 2>&1; echo bench=$?
timeout 600 python bench.py --impl reference --steps 1 --warmup 1 > gpurun_out/ev_ref.log 2>&1; echo ref=$?
timeout 300 python bench.py --dtype c64 --no-e2e --no-cpu > gpurun_out/ev_c64.log 2>&1; echo c64=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/ev_launches.csv \
  python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ev_ncu_launch.log 2>&1; echo launches=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_coset_p -s 3 -c 1 -f -o gpurun_out/ev_coset \
  python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ev_ncu_full.log 2>&1; echo full=$?
