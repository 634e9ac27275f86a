#!/bin/bash
# planned GEMM traces at C3 and C4 (solve products), leaf-product tile survey at C3's shape
cd "$(dirname "$0")/.."
O=gpurun_out/am
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
timeout 600 python tools/gemm_trace.py 3 --plan > $O/trace_c3.out 2> $O/trace_c3.txt
timeout 600 python tools/gemm_trace.py 4 --plan > $O/trace_c4.out 2> $O/trace_c4.txt
echo done
