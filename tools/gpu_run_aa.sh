#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/aa
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/aa/build.txt 2>&1
timeout 300 python tools/leaf_trace_c3.py 32 > gpurun_out/aa/leaf_trace.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "leaf or zinv or every_R or config2 or planned" > gpurun_out/aa/pytest.txt 2>&1
echo done
