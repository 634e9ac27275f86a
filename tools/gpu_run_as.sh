#!/bin/bash
# threshold sweeps with the round-2 kernels (3M, lookahead): nat_bb_min and nat_min at C4 and C3
cd "$(dirname "$0")/.."
O=gpurun_out/as
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
timeout 900 python tools/knob_sweep.py 4 nat_bb_min 512 400 200 > $O/sweep_c4_bb.txt 2>&1
timeout 900 python tools/knob_sweep.py 4 nat_min 200 100 > $O/sweep_c4_nm.txt 2>&1
timeout 600 python tools/knob_sweep.py 3 nat_bb_min 512 400 200 > $O/sweep_c3_bb.txt 2>&1
timeout 600 python tools/knob_sweep.py 3 nat_min 200 100 > $O/sweep_c3_nm.txt 2>&1
echo done
