#!/bin/bash
# 32-wide natural-order block steps with the one-warp D^-1: tests, C2/C3 sweeps
cd "$(dirname "$0")/.."
O=gpurun_out/aq
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "block32 or natural_order_merge or lookahead" > $O/pytest.txt 2>&1
timeout 600 python tools/knob_sweep.py 2 nat_b32 0 200 96 "nat_min=100,nat_b32=100" "nat_min=100,nat_b32=0" > $O/sweep_c2.txt 2>&1
timeout 900 python tools/knob_sweep.py 3 nat_b32 0 200 "nat_min=100,nat_b32=100" > $O/sweep_c3.txt 2>&1
echo done
