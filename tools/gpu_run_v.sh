#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/v
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/v/build.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "natural or zinv or config2 or every_R or planned" > gpurun_out/v/pytest.txt 2>&1
timeout 600 python tools/knob_sweep.py 2 nat_bb_min 200 512 > gpurun_out/v/sweep_c2.txt 2>&1
timeout 600 python tools/knob_sweep.py 3 nat_bb_min 200 512 > gpurun_out/v/sweep_c3.txt 2>&1
timeout 900 python tools/knob_sweep.py 4 nat_bb_min 200 512 > gpurun_out/v/sweep_c4.txt 2>&1
echo done
