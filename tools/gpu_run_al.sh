#!/bin/bash
# grouped tile order for the 64x64 (3M) tile: time and DRAM bytes of the C4 level-15 product
cd "$(dirname "$0")/.."
O=gpurun_out/al
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
for gm in 8 1 16; do for c in 3 5; do
timeout 120 python tools/gemm_one.py 5376x10752x1792x2x1 cfg=$c gemm_group=$gm >> $O/tiles.txt 2>&1
timeout 120 python tools/gemm_one.py 7168x14336x3584x1x1 cfg=$c gemm_group=$gm >> $O/tiles.txt 2>&1
done; done
for gm in 8 1; do
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:zgemm_kernel --csv \
  python tools/gemm_one.py 5376x10752x1792x2x1 cfg=3 gemm_group=$gm > $O/ncu_g$gm.csv 2>&1
done
timeout 900 python tools/knob_sweep.py 4 gemm_group 8 1 > $O/sweep_c4.txt 2>&1
echo done
