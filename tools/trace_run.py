"""One build + solve of a config with HPS_TRACE=1 (per-launch shapes and times to stderr)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1812_07167_b200 import hps, inputs
import bench
cfg = inputs.CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 2]
g, c, s, t = bench.setup(cfg, hps)
d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
for rep in range(2):
    S = hps.Solver(g, cfg.p, cfg.kappa, cfg.eta, d(c))
    print("build ms", S.time_ms(0), "leaf", S.time_ms(1), "merge", S.time_ms(2), file=sys.stderr)
    S.solve(d(s), d(t))
    print("solve ms", S.time_ms(3), "up", S.time_ms(4), "down", S.time_ms(5), file=sys.stderr)
    S.close()
