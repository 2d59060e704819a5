#!/bin/bash
# round-2 end: the committed tree on one B200 -- GPU suite, smoke, default bench, reference arm,
# launch list and ncu --set full summary of the dominant kernel, fp32 and JW lines, Z_0 check
D=gpurun_out/${FINAL_DIR:-final}
mkdir -p $D
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv > $D/gpu.txt 2>&1
timeout 1500 python -m pytest tests -q -m gpu > $D/tests.log 2>&1; echo "tests rc=$?" >> $D/tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.log 2>&1; echo "smoke rc=$?" >> $D/smoke.log
timeout 600 python bench.py > $D/bench.log 2>&1; echo "bench rc=$?"
timeout 600 python bench.py > $D/bench2.log 2>&1; echo "bench2 rc=$?"
timeout 600 python bench.py --impl reference > $D/ref.log 2>&1; echo "ref rc=$?"
timeout 300 python bench.py --dtype c64 --no-cpu > $D/c64.log 2>&1
timeout 900 python bench.py --kind JW --steps 2 --warmup 1 --no-e2e --no-cpu > $D/jw.log 2>&1
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu"
$B > $D/plain.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
  --log-file $D/launches.csv $B > $D/ncu_launch.log 2>&1; echo "launches rc=$?"
$B > $D/plain2.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_coset_p -s 3 -c 1 \
  -o $D/coset_r10 $B > $D/ncu_coset.log 2>&1; echo "coset rc=$?"
python tools/ncu_summary.py $D/coset_r10.ncu-rep --algorithmic 34359738368 \
  --title "30q fp64 R10, k_coset_p 4th launch, round-2 final build; ncu --set full --clock-control none -k regex:k_coset_p -s 3 -c 1 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu" > $D/ncu_coset_r10.txt 2>&1
rm -f $D/coset_r10.ncu-rep
[ -z "$SKIP_Z0" ] && timeout 1200 python tools/z0_curve.py --qubits 30 --embedded --terms 4000 --ldet 600 --deltas 0.02,0.1,0.3 --out $D/z0_30_embedded.json > $D/z0_30e.log 2>&1; echo "z0e rc=$?"
du -sh gpurun_out
