#!/bin/bash
# GL-edge parity tests + the complex leaf kernel's CTA-0 timeline on C3-like leaves
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/k
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/k/build.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "gl_" > gpurun_out/k/pytest_gl.txt 2>&1
timeout 300 python tools/leaf_trace_c3.py 32 > gpurun_out/k/leaf_trace_c3.txt 2>&1

timeout 600 python tools/gemm_trace.py 4 > /dev/null 2> gpurun_out/k/trace_c4.txt
timeout 600 python tools/gemm_trace.py 3 > /dev/null 2> gpurun_out/k/trace_c3.txt
echo done2
