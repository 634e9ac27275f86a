#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/p
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/p/build.txt 2>&1
timeout 300 python tools/leaf_trace_c3.py 32 leaf_panel=1 > gpurun_out/p/leaf_trace_bp.txt 2>&1
timeout 300 python tools/leaf_trace_c3.py 32 > gpurun_out/p/leaf_trace.txt 2>&1
echo done
