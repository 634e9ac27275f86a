#!/bin/bash
# fused solve levels (solve_fuse): parity tests, then the threshold sweep at C2 (1 RHS) and C4 (16 RHS)
cd "$(dirname "$0")/.."
O=gpurun_out/au
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "fused or solve or config2 or tree or sharded or virtual" > $O/pytest_sel.txt 2>&1
timeout 600 python tools/knob_sweep.py 2 solve_fuse 0 28 56 112 224 448 > $O/sweep_c2.txt 2>&1
timeout 900 python tools/knob_sweep.py 4 solve_fuse 0 56 112 224 > $O/sweep_c4.txt 2>&1
timeout 300 python tools/host_probe.py 2 1 > $O/host_c2.txt 2>&1
echo done
