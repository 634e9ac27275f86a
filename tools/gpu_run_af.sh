#!/bin/bash
cd "$(dirname "$0")/.."
O=gpurun_out/af
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "leaf_real or leaf_path or config2 or every_R" > $O/pytest.txt 2>&1
timeout 600 python tools/knob_sweep.py 2 dgj_nt 512 256 > $O/sweep_c2.txt 2>&1
echo done
