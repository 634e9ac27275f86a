#!/bin/bash
# integer-slice products: threshold sweep at C4 / C3 (gemm_slices x gemm_slices_min), full-step bench with the knob on
cd "$(dirname "$0")/.."
O=gpurun_out/ay
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
for C in 4 3; do
timeout 900 python - $C > $O/sweep_min_c$C.txt 2>&1 <<'PY'
import sys, numpy as np, torch
import bench
from paper_1812_07167_b200 import hps, inputs
cfg = inputs.CONFIGS[int(sys.argv[1])]
g, c, s, t = bench.setup(cfg, hps)
d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
cd, sd, td = d(c), d(s), d(t)
torch.cuda.synchronize()
hps.set_cache_limit(int(0.9 * torch.cuda.get_device_properties(0).total_memory))
hps.plan_problem(g, cfg.p)
kr = bench.root_R_default(int(sys.argv[1]))
for (ns, mn) in ((0, 896), (8, 1536), (8, 2500), (8, 1100), (7, 1536), (0, 896), (8, 1536)):
    with hps.debug_knobs(gemm_slices=ns, gemm_slices_min=mn):
        ts = []
        for _ in range(3):
            S = hps.Solver(g, cfg.p, cfg.kappa, cfg.eta, cd, keep_root_R=kr)
            S.solve(sd, td)
            ts.append((S.time_ms(0), S.time_ms(2), S.time_ms(3)))
            S.close()
    print(f"gemm_slices={ns} min={mn} keep_root_R={kr}: build {min(x[0] for x in ts):.2f} ms (merges {min(x[1] for x in ts):.2f}), "
          f"solve {min(x[2] for x in ts):.2f} ms", flush=True)
PY
done
echo done
