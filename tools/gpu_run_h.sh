#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/h_smoke.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -s -k "leaf_schur or config3_sampled or natural" > gpurun_out/h_pytest.txt 2>&1
timeout 900 python tools/knob_sweep.py 3 leaf_panel 0 1 > gpurun_out/h_sweep_leaf_c3.txt 2>&1
timeout 900 python tools/knob_sweep.py 4 leaf_panel 0 1 > gpurun_out/h_sweep_leaf_c4.txt 2>&1
echo done
