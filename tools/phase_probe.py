import os, sys, time
sys.path.insert(0, "/root/repo")
import numpy as np, torch
from paper_1812_07167_b200 import hps, inputs
import bench
cfg = inputs.CONFIGS[int(sys.argv[1])]
g, c, s, t = bench.setup(cfg, hps)
dev = "cuda:0"
c_d = torch.from_numpy(c).to(dev); s_d = torch.from_numpy(np.ascontiguousarray(s)).to(dev); t_d = torch.from_numpy(np.ascontiguousarray(t)).to(dev)
u_d = torch.empty((s.shape[0], cfg.nleaf, cfg.p * cfg.p - 4), dtype=torch.complex128, device=dev)
for mode in ["dev", "dev_prof", "dev", "host"]:
    for k in range(3):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        if mode == "host":
            S = hps.Solver(g, cfg.p, cfg.kappa, cfg.eta, c); u = S.solve(s, t)
        else:
            S = hps.Solver(g, cfg.p, cfg.kappa, cfg.eta, c_d, profile=(1 if mode == "dev_prof" else 0)); S.solve(s_d, t_d, u_d)
        torch.cuda.synchronize(); t1 = time.perf_counter()
        print(mode, k, "wall %.1f ms" % (1e3 * (t1 - t0)), "build %.1f leaf %.1f merge %.1f solve %.1f" % (S.time_ms(0), S.time_ms(1), S.time_ms(2), S.time_ms(3)), flush=True)
        S.close()
