#!/bin/bash
# solve CUDA graph (solve_graph): its parity test, the whole GPU suite, host probe (repeated solves)
cd "$(dirname "$0")/.."
O=gpurun_out/av
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider -k "graph" > $O/pytest_graph.txt 2>&1
timeout 300 python tools/host_probe.py 2 1 > $O/host_c2.txt 2>&1
timeout 300 python tools/host_probe.py 2 16 > $O/host_c2_16.txt 2>&1
timeout 600 python tools/host_probe.py 3 > $O/host_c3.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -x > $O/pytest_gpu.txt 2>&1
echo done
