#!/bin/bash
# fused S assembly in the complex leaf inverse; solve-only launch lists (C4, C2) for the HBM rates
cd "$(dirname "$0")/.."
O=gpurun_out/ac
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
timeout 300 python tools/leaf_trace_c3.py 32 > $O/leaf_trace.txt 2>&1
timeout 300 python tools/leaf_trace_c3.py 32 leaf_fuse_asm=0 > $O/leaf_trace_nofuse.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "leaf or every_R or config3_sampled or gl_edges" > $O/pytest.txt 2>&1
timeout 900 python tools/knob_sweep.py 4 leaf_fuse_asm 1 0 > $O/sweep_c4.txt 2>&1
for C in 4 2; do
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none --csv --log-file $O/c${C}_solve_launches.csv python tools/profile_solve.py $C > $O/c${C}_solve.log 2>&1
done
echo done
