"""One planned build + solve of a config with only the last one captured by the profiler
(ncu --profile-from-start off): per-kernel launch lists of exactly one step."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1812_07167_b200 import hps, inputs
import bench
ci = int(sys.argv[1]) if len(sys.argv) > 1 else 2
cfg = inputs.CONFIGS[ci]
kr = bench.root_R_default(ci)     # as bench.py's headline step
g, c, s, t = bench.setup(cfg, hps)
d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
hps.plan_problem(g, cfg.p)          # as bench.py: the inverse regimes and the GEMM tile plans
hps.plan_build(g, cfg.p, keep_root_R=kr)
hps.plan_solve(g, cfg.p, s.shape[0])
cd, sd, td = d(c), d(s), d(t)
for it in range(2):
    if it == 1:
        torch.cuda.synchronize()
        torch.cuda.cudart().cudaProfilerStart()
    S = hps.Solver(g, cfg.p, cfg.kappa, cfg.eta, cd, keep_root_R=kr)
    S.solve(sd, td)
    torch.cuda.synchronize()
    if it == 1:
        torch.cuda.cudart().cudaProfilerStop()
    S.close()
print("ok")
