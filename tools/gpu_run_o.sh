#!/bin/bash
# leaf epilogue ILP; ncu of the new leaf kernel (DRAM per leaf, DMMA %)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/o
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/o/build.txt 2>&1
timeout 300 python tools/leaf_trace_c3.py 32 > gpurun_out/o/leaf_trace_c3.txt 2>&1
timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider -k "leaf_schur or leaf_parity" > gpurun_out/o/pytest.txt 2>&1
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:zgj_seq_kernel \
    -s 0 -c 1 -o gpurun_out/o/c4_leaf python tools/profile_step.py 4 > gpurun_out/o/ncu_full_leaf.log 2>&1
ncu -i gpurun_out/o/c4_leaf.ncu-rep --page raw --csv > gpurun_out/o/c4_leaf_raw.csv 2>/dev/null
ncu -i gpurun_out/o/c4_leaf.ncu-rep --page source --csv > gpurun_out/o/c4_leaf_source.csv 2>/dev/null
rm -f gpurun_out/o/*.ncu-rep
echo done
