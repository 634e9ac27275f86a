"""One build + solve of a config (for ncu launch lists)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1812_07167_b200 import hps, inputs
import bench
cfg = inputs.CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 2]
g, c, s, t = bench.setup(cfg, hps)
d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
if os.environ.get("HPS_PLAN", "1") == "1":
    hps.plan_problem(g, cfg.p)   # as bench.py does
S = hps.Solver(g, cfg.p, cfg.kappa, cfg.eta, d(c))
S.solve(d(s), d(t))
S.close()
S = hps.Solver(g, cfg.p, cfg.kappa, cfg.eta, d(c))
S.solve(d(s), d(t))
torch.cuda.synchronize()
print("build ms", S.time_ms(0), "solve ms", S.time_ms(3))
S.close()
