#!/bin/bash
# round 2 evidence on one B200: the GPU suite, the default bench, launch list, ncu --set full of the
# tile kernel, K1, the reductions, the swap/permute/fused-exchange kernels, and the Z_0 curve
D=gpurun_out/prof
mkdir -p $D
timeout 1200 python -m pytest tests -q -m gpu > $D/tests.log 2>&1; echo "tests rc=$?" >> $D/tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.log 2>&1; echo "smoke rc=$?" >> $D/smoke.log
timeout 600 python bench.py > $D/bench.log 2>&1; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $D/ref.log 2>&1; echo "ref rc=$?"
timeout 300 python bench.py --dtype c64 --no-e2e --no-cpu > $D/c64.log 2>&1
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu"
$B > $D/plain.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
  --log-file $D/launches.csv $B > $D/ncu_launch.log 2>&1; echo "launches rc=$?"
$B > $D/plain2.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_coset_p -s 3 -c 1 \
  -o $D/coset_r10 $B > $D/ncu_coset.log 2>&1; echo "coset rc=$?"
summ() {  # text summary + gzipped SASS source table, then drop the (large) report
  python tools/ncu_summary.py $D/$1.ncu-rep --algorithmic ${2:-0} --title "$3" > $D/$1.txt 2>&1
  ncu -i $D/$1.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > $D/$1.sass.csv.gz
  rm -f $D/$1.ncu-rep
}
summ coset_r10 34359738368 "30q fp64 R10 layer, k_coset_p, 4th launch (round-2 default build)"
for w in stream reduce swap; do timeout 300 python tools/kernel_probe.py $w > $D/probe_$w.log 2>&1; echo "probe $w rc=$?"; done
python tools/kernel_probe.py stream > /dev/null 2>&1 && timeout 600 ncu --set full --clock-control none -k regex:k_stream -s 20 -c 1 \
  -o $D/stream python tools/kernel_probe.py stream > $D/ncu_stream.log 2>&1
python tools/kernel_probe.py reduce > /dev/null 2>&1 && timeout 600 ncu --set full --clock-control none -k regex:"k_norm|k_inner|k_expect" -s 3 -c 4 \
  -o $D/reduce python tools/kernel_probe.py reduce > $D/ncu_reduce.log 2>&1
python tools/kernel_probe.py swap > /dev/null 2>&1 && timeout 900 ncu --set full --clock-control none -k regex:"k_p2p_swap|k_permute|k_xtile" -s 2 -c 3 \
  -o $D/swap python tools/kernel_probe.py swap > $D/ncu_swap.log 2>&1
summ stream 34359738368 "30q fp64 K1 k_stream (fusion 0), 21st launch"
summ reduce 0 "30q fp64 reductions: k_norm / k_inner / k_expect (algorithmic bytes: norm 16 GiB read, inner 32 GiB, expect 16 GiB per x-group)"
summ swap 0 "30q fp64 on 2 virtual ranks: k_p2p_swap / k_xtile / k_permute (peer = the other slice on the same GPU)"
echo "ncu probes done"
timeout 1200 python tools/z0_curve.py --qubits 30 --embedded --terms 4000 --ldet 600 --out $D/z0_30_embedded.json > $D/z0_30e.log 2>&1; echo "z0e rc=$?"
timeout 1800 python tools/z0_curve.py --qubits 32 --terms 60000 --ldet 4000 --out $D/z0_32.json > $D/z0_32.log 2>&1; echo "z0 rc=$?"
# fp32 with the specialised cases at 6 CTAs per SM (occupancy select 2 = tune bits 1-3 -> 4)
for t in 1536 1540; do timeout 300 python bench.py --dtype c64 --specialize 2 --tile-tune $t --no-e2e --no-cpu > $D/c64_sp2_t$t.log 2>&1; done
timeout 300 python bench.py --dtype c64 --specialize 0 --no-e2e --no-cpu > $D/c64_sp0.log 2>&1
# A/B: 3-dimensional sub-groups (8 amplitudes per thread, 512-thread CTAs, 2 per SM = 32 warps)
for lib in sd3 default; do
  if [ $lib = sd3 ]; then export PS_LIB_PATH=$PWD/paper_2504_17881_b200/libps_sd3.so; else unset PS_LIB_PATH; fi
  timeout 300 python bench.py --no-e2e --no-cpu > $D/ab_${lib}_R10.log 2>&1
  timeout 900 python bench.py --kind JW --no-e2e --no-cpu --steps 2 --warmup 1 > $D/ab_${lib}_JW.log 2>&1
  timeout 300 python bench.py --kind GATES --layer 200 --no-e2e --no-cpu > $D/ab_${lib}_GATES.log 2>&1
done
unset PS_LIB_PATH
# config 3 on one GPU (strong-scaling base): 32q JW Trotter step (64 GiB)
timeout 1500 python bench.py --kind JW --qubits 32 --steps 1 --warmup 1 --no-e2e --no-cpu > $D/JW32_1gpu.log 2>&1; echo "jw32 rc=$?"
bash tools/ab_pipe.sh
du -sh gpurun_out; du -a gpurun_out | sort -n | tail -5
