#!/bin/bash
# closing check of round 2: smoke, full GPU suite, default bench (headline, knobs at their defaults),
# and the same bench with the opt-in integer-slice products (--gemm-slices 8)
cd "$(dirname "$0")/.."
O=gpurun_out/az
mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rs > $O/pytest_gpu.txt 2>&1
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err
timeout 900 python bench.py --gemm-slices 8 --no-cpu-baseline > $O/bench_slices8.json 2> $O/bench_slices8.err
echo done
