#!/bin/bash
# k-fastest B loader for the solve's column-major s; complex leaf kernel timeline with epilogue
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/l
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/l/build.txt 2>&1
timeout 300 python tools/leaf_trace_c3.py 32 > gpurun_out/l/leaf_trace_c3.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "many_rhs or gl_edges_poly or config2 or every_R or torch_device" > gpurun_out/l/pytest.txt 2>&1
timeout 600 python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/l/bench_c3.json 2> gpurun_out/l/bench_c3.err
python - > gpurun_out/l/bcol_ab.txt 2>&1 <<'PY'
import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_1812_07167_b200 import hps, inputs
import bench
for cfgi in (3, 4):
    cfg = inputs.CONFIGS[cfgi]
    g, c, s, t = bench.setup(cfg, hps)
    d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    cd, sd, td = d(c), d(s), d(t)
    S = hps.Solver(g, cfg.p, cfg.kappa, cfg.eta, cd)
    for bcol in (0, 1, 0, 1):
        with hps.debug_knobs(gemm_bcol=bcol):
            S.solve(sd, td)
            print(f"C{cfgi} bcol={bcol}: up {S.time_ms(4):.2f} ms down {S.time_ms(5):.2f} ms", flush=True)
    S.close()
    del cd, sd, td
    torch.cuda.empty_cache()
PY
echo done
