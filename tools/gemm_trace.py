"""One build + solve of a config with the library's per-launch ZGEMM / inverse trace on
(hps_debug_set("trace", 1): every zgemm and batched inverse is timed with events and printed to
stderr with its shape and TFLOP/s).  usage: python tools/gemm_trace.py CONFIG 2> trace.txt"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench
from paper_1812_07167_b200 import hps, inputs

cfg = inputs.CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 2]
g, c, s, t = bench.setup(cfg, hps)
d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
cd, sd, td = d(c), d(s), d(t)
hps.plan_problem(g, cfg.p)
if "--plan" in sys.argv:    # as bench.py: the build and solve GEMM plans too
    hps.plan_build(g, cfg.p, keep_root_R=bench.root_R_default(int(sys.argv[1])))
    hps.plan_solve(g, cfg.p, s.shape[0])
print("nrhs", s.shape[0], file=sys.stderr, flush=True)
S = hps.Solver(g, cfg.p, cfg.kappa, cfg.eta, cd)   # warm-up
S.solve(sd, td)
S.close()
with hps.debug_knobs(trace=1):
    S = hps.Solver(g, cfg.p, cfg.kappa, cfg.eta, cd)
    print("build ms", S.time_ms(0), file=sys.stderr, flush=True)
    S.solve(sd, td)
    print("solve ms", S.time_ms(3), file=sys.stderr, flush=True)
    S.close()
