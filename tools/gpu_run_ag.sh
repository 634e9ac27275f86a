#!/bin/bash
cd "$(dirname "$0")/.."
O=gpurun_out/ag
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "merge_small or every_R or config2 or polynomial or natural or planned" > $O/pytest.txt 2>&1
timeout 600 python tools/knob_sweep.py 2 merge_small 1 0 > $O/sweep_c2.txt 2>&1
timeout 600 python tools/knob_sweep.py 3 merge_small 1 0 > $O/sweep_c3.txt 2>&1
timeout 900 python tools/knob_sweep.py 4 merge_small 1 0 > $O/sweep_c4.txt 2>&1
echo done
