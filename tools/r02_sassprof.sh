#!/bin/bash
# one ncu capture of the default tile kernel (R10 and JW) with per-instruction counts for the
# per-source-line attribution (tools/line_attrib.py); reports are reduced on the box
D=gpurun_out/sassprof
mkdir -p $D
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu"
$B > $D/plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_coset_p -s 3 -c 1 -o $D/r10 $B > $D/ncu_r10.log 2>&1
ncu -i $D/r10.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > $D/r10.sass.csv.gz
python tools/ncu_summary.py $D/r10.ncu-rep --algorithmic 34359738368 --title "30q fp64 R10 k_coset_p (final dispatch)" > $D/r10.txt 2>&1
rm -f $D/r10.ncu-rep
$B --kind JW > $D/plainjw.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_coset_p -s 20 -c 1 -o $D/jw $B --kind JW > $D/ncu_jw.log 2>&1
ncu -i $D/jw.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > $D/jw.sass.csv.gz
python tools/ncu_summary.py $D/jw.ncu-rep --algorithmic 34359738368 --title "30q fp64 JW k_coset_p (final dispatch)" > $D/jw.txt 2>&1
rm -f $D/jw.ncu-rep
