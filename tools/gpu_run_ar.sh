#!/bin/bash
# natural-order W^-1 in one cooperative persistent launch: tests, C2/C3 sweeps
cd "$(dirname "$0")/.."
O=gpurun_out/ar
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "block32 or natural_order_merge" > $O/pytest.txt 2>&1
timeout 600 python tools/knob_sweep.py 2 nat_persist 0 8 "nat_min=100,nat_persist=16" > $O/sweep_c2.txt 2>&1
timeout 900 python tools/knob_sweep.py 3 nat_persist 0 8 > $O/sweep_c3.txt 2>&1
echo done
