#!/bin/bash
# 3M with the operand sums staged once per stage (gemm_3m = 2): tests, tile timings, C4/C3 sweeps
cd "$(dirname "$0")/.."
O=gpurun_out/ap
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "zgemm or product_forms" > $O/pytest.txt 2>&1
for m in 2 1 0; do for c in 5 3 2; do
timeout 120 python tools/gemm_one.py 5376x10752x1792x2x1 cfg=$c gemm_3m=$m >> $O/tiles.txt 2>&1
done; done
timeout 120 python tools/gemm_one.py 1344x2688x448x32x1 cfg=2 gemm_3m=2 >> $O/tiles.txt 2>&1
timeout 120 python tools/gemm_one.py 1344x2688x448x32x1 cfg=2 gemm_3m=1 >> $O/tiles.txt 2>&1
timeout 900 python tools/knob_sweep.py 4 gemm_3m 2 1 > $O/sweep_c4.txt 2>&1
timeout 600 python tools/knob_sweep.py 3 gemm_3m 2 1 > $O/sweep_c3.txt 2>&1
timeout 300 ncu --set full --clock-control none -k regex:zgemm_kernel -c 1 -o $O/z3s python tools/gemm_one.py 5376x10752x1792x2x1 cfg=5 gemm_3m=2 > $O/ncu.log 2>&1
ncu -i $O/z3s.ncu-rep --page raw --csv > $O/z3s_raw.csv 2>/dev/null
rm -f $O/*.ncu-rep
echo done
