#!/bin/bash
# lookahead in the block-step natural-order W^-1: tests, C3/C4 sweeps
cd "$(dirname "$0")/.."
O=gpurun_out/ao
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "lookahead or natural or every_R or config3_sharded or virtual_ranks" > $O/pytest.txt 2>&1
timeout 600 python tools/knob_sweep.py 3 nat_lookahead 1 0 > $O/sweep_c3.txt 2>&1
timeout 900 python tools/knob_sweep.py 4 nat_lookahead 1 0 > $O/sweep_c4.txt 2>&1
echo done
