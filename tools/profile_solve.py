"""One planned solve of a config (the build before it is not captured: ncu --profile-from-start off):
the launch list of the solve sweeps alone (Algorithm 2), for their DRAM bytes and HBM rates."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1812_07167_b200 import hps, inputs
import bench
cfg = inputs.CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 2]
g, c, s, t = bench.setup(cfg, hps)
d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
hps.plan_problem(g, cfg.p)
hps.plan_build(g, cfg.p)
hps.plan_solve(g, cfg.p, s.shape[0])
cd, sd, td = d(c), d(s), d(t)
S = hps.Solver(g, cfg.p, cfg.kappa, cfg.eta, cd)
S.solve(sd, td)                      # warm-up solve
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
S.solve(sd, td)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("solve ms", S.time_ms(3), "up", S.time_ms(4), "down", S.time_ms(5))
S.close()
