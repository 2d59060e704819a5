# A/B of the tile kernel's next-tile shared-memory prefetch (PS_OPT_TILE_TUNE bit 11) and tile size
mkdir -p gpurun_out
B="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu"
for rep in 1 2 3; do
 for tb in 11 12; do timeout 300 $B --tile-bits $tb --tile-tune 3584 > gpurun_out/pf2_R10_tb${tb}_$rep.log 2>&1; done
done
timeout 300 $B --dtype c64 --tile-bits 12 --tile-tune 3584 > gpurun_out/pf2_c64_tb12_3584.log 2>&1
timeout 300 $B --dtype c64 --tile-bits 12 --tile-tune 1536 > gpurun_out/pf2_c64_tb12_1536.log 2>&1
for k in JW QAOA LOW; do
 timeout 600 $B --kind $k --tile-bits 11 --tile-tune 1536 > gpurun_out/pf2_${k}_tb11_1536.log 2>&1
 timeout 600 $B --kind $k --tile-bits 11 --tile-tune 3584 > gpurun_out/pf2_${k}_tb11_3584.log 2>&1
 timeout 600 $B --kind $k --tile-bits 12 --tile-tune 3584 > gpurun_out/pf2_${k}_tb12_3584.log 2>&1
done
timeout 300 $B --kind GATES --tile-bits 12 --tile-tune 3584 > gpurun_out/pf2_GATES_tb12_3584.log 2>&1
timeout 300 $B --kind S8 --tile-bits 12 --tile-tune 3584 > gpurun_out/pf2_S8_tb12_3584.log 2>&1
echo done
