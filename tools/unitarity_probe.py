import sys, time
sys.path.insert(0, "/root/repo")
import numpy as np, torch
from paper_1812_07167_b200 import hps, inputs
import bench
for cfgno in (2, 3, 4):
    cfg = inputs.CONFIGS[cfgno]
    g, c, s, t = bench.setup(cfg, hps)
    t0 = time.time()
    S = hps.Solver(g, cfg.p, cfg.kappa, cfg.eta, torch.from_numpy(c).cuda())
    n = S.nb(1)
    R = torch.empty((n, n), dtype=torch.complex128, device="cuda")
    hps.lib().hps_export_R(S.h, 1, R.data_ptr())
    E = R @ R.conj() - torch.eye(n, dtype=torch.complex128, device="cuda")
    ev = torch.linalg.eigvals(R) if n <= 8000 else None
    print(cfgno, "n", n, "max|RRbar-I|", E.abs().max().item(), "max||lam|-1|", None if ev is None else (ev.abs() - 1).abs().max().item(), "t", time.time() - t0, flush=True)
    S.close()
