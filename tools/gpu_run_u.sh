#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/u
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/u/build.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "plan" > gpurun_out/u/pytest.txt 2>&1
timeout 1200 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/u/bench_c4.json 2> gpurun_out/u/bench_c4.err
timeout 900 python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/u/bench_c3.json 2> gpurun_out/u/bench_c3.err
timeout 600 python bench.py --config 2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/u/bench_c2.json 2> gpurun_out/u/bench_c2.err
python - > gpurun_out/u/plan_c4.txt 2>&1 <<'PY'
import sys; sys.path.insert(0, '.')
from paper_1812_07167_b200 import hps
g = hps.grid(0, 1, 0, 1, 256, 256)
for a in hps.plan_build(g, 16):
    print(a)
PY
echo done
