#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/g_smoke.txt 2>&1
timeout 900 python tools/knob_sweep.py 4 gemm_group 1 4 16 > gpurun_out/g_sweep_group_c4.txt 2>&1
timeout 900 python tools/knob_sweep.py 4 nat_bb_min 512 1024 > gpurun_out/g_sweep_bb_c4.txt 2>&1
timeout 300 python tools/knob_sweep.py 2 gemm_group 1 16 > gpurun_out/g_sweep_group_c2.txt 2>&1
echo done
