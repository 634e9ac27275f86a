#!/bin/bash
# 3M ZGEMM: tile tests in both forms, error bound, whole-problem parity, C2/C3/C4 timing 3M vs 4M,
# polynomial errors both ways
cd "$(dirname "$0")/.."
O=gpurun_out/ah
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "zgemm" > $O/pytest_zgemm.txt 2>&1
timeout 600 python tools/knob_sweep.py 4 gemm_3m 1 0 > $O/sweep_c4.txt 2>&1
timeout 600 python tools/knob_sweep.py 3 gemm_3m 1 0 > $O/sweep_c3.txt 2>&1
timeout 300 python tools/knob_sweep.py 2 gemm_3m 1 0 > $O/sweep_c2.txt 2>&1
timeout 600 python tools/poly_errors.py gemm_3m=1 > $O/poly_3m.txt 2>&1
timeout 600 python tools/poly_errors.py gemm_3m=0 > $O/poly_4m.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -k "not zgemm" > $O/pytest_rest.txt 2>&1
echo done
