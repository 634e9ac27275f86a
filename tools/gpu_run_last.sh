#!/bin/bash
# last check of the round: smoke + full GPU suite on the final code
cd "$(dirname "$0")/.."
O=gpurun_out/last
mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rs > $O/pytest_gpu.txt 2>&1
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err
echo done
