#!/bin/bash
# grouped GEMM tile order at 3 CTAs/SM (launch bounds): C4 and C3 merges for gemm_group 1, 4, 8, 16
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/m
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/m/build.txt 2>&1
timeout 900 python tools/knob_sweep.py 4 gemm_group 1 8 16 > gpurun_out/m/sweep_c4.txt 2>&1
timeout 600 python tools/knob_sweep.py 3 gemm_group 1 4 8 16 > gpurun_out/m/sweep_c3.txt 2>&1
timeout 300 python tools/gemm_one.py 7168x14336x3584x1x1 > gpurun_out/m/one_g1.txt 2>&1
echo done
