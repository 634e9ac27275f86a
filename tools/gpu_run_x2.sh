#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/x2
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/x2/build.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "plan or many_rhs or zgemm or torch_device" > gpurun_out/x2/pytest.txt 2>&1
timeout 1200 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/x2/bench_c4.json 2> gpurun_out/x2/bench_c4.err
timeout 900 python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/x2/bench_c3.json 2> gpurun_out/x2/bench_c3.err
python - > gpurun_out/x2/plan_solve_c4.txt 2>&1 <<'PY'
import sys; sys.path.insert(0, '.')
from paper_1812_07167_b200 import hps
for nx, nr in ((256, 16), (128, 64)):
    g = hps.grid(0, 1, 0, 1, nx, nx)
    for a in hps.plan_solve(g, 16, nr):
        if a["level"] < 0 or a["cfg"] >= 0:
            print(nx, a)
PY
echo done
