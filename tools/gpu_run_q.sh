#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/q
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/q/build.txt 2>&1
timeout 300 python tools/leaf_trace_c3.py 32 leaf_panel=2 > gpurun_out/q/leaf_trace_bp2.txt 2>&1
timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider -k "leaf_schur" > gpurun_out/q/pytest.txt 2>&1
echo done
