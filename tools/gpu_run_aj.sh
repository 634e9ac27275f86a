#!/bin/bash
# 3M tile survey on the C4 top-level product shape, ncu of the 3M 64x32 tile
cd "$(dirname "$0")/.."
O=gpurun_out/aj
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
for m3 in 1 0; do for c in 5 3 4 6 7 8 2; do
timeout 120 python tools/gemm_one.py 5376x10752x1792x2x1 cfg=$c gemm_3m=$m3 >> $O/tiles.txt 2>&1
done; done
timeout 300 ncu --set full --clock-control none --import-source on -k regex:zgemm_kernel -c 1 -o $O/z3m python tools/gemm_one.py 5376x10752x1792x2x1 cfg=5 gemm_3m=1 > $O/ncu3m.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:zgemm_kernel -c 1 -o $O/z4m python tools/gemm_one.py 5376x10752x1792x2x1 cfg=5 gemm_3m=0 > $O/ncu4m.log 2>&1
for f in z3m z4m; do
ncu -i $O/$f.ncu-rep --page raw --csv > $O/${f}_raw.csv 2>/dev/null
ncu -i $O/$f.ncu-rep --page source --csv --print-source sass > $O/${f}_sass.csv 2>/dev/null
done
rm -f $O/*.ncu-rep
echo done
