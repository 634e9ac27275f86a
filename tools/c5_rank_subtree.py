"""C5 per-rank workload on one B200 (C5 = [0,2]x[0,1], 1024x512 leaves, p = 16, 10 points
per wavelength, 128 RHS, 8 GPUs).  Rank r of 8 owns the depth-3 subtree (256x256 leaves on a 0.5 x 0.5
square); this builds that subtree with C5's kappa and c field (keep_root_R: the sharded top levels need
the subtree root R) and solves 128 right-hand sides through the library's RHS chunks (device-resident
s, t drawn with torch, CN(0,1)).  It times what one rank does before and after the top-level exchange;
the top three levels (group split) are not run here (one GPU).
usage: python tools/c5_rank_subtree.py [rank] [nrhs]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1812_07167_b200 import hps, inputs

rank = int(sys.argv[1]) if len(sys.argv) > 1 else 0
nrhs = int(sys.argv[2]) if len(sys.argv) > 2 else 128
cfg = inputs.CONFIGS[5]
g = hps.grid(cfg.x0, cfg.x1, cfg.y0, cfg.y1, cfg.nx, cfg.ny)
sub, i0, j0 = hps.subtree_grid(g, 3, rank)
X, Y = hps.leaf_nodes(sub, cfg.p)
c = inputs.c_at(cfg, X, Y)                       # C5's bump field at this rank's nodes
nleaf, ni, nt = sub.nx * sub.ny, (cfg.p - 2) ** 2, cfg.p * cfg.p - 4
nb = 2 * (sub.nx + sub.ny) * (cfg.p - 2)
torch.manual_seed(rank)
cd = torch.from_numpy(np.ascontiguousarray(c)).cuda()
# s (26 GB) and u (34 GB) in pinned host memory: the library stages them chunk by chunk, so the
# device holds the subtree's operators (~108 GB) and one chunk of vectors
s = torch.empty((nrhs, nleaf, ni), dtype=torch.complex128, pin_memory=True)
torch.view_as_real(s).normal_(0.0, float(np.sqrt(0.5)))
t = torch.complex(torch.randn(nrhs, nb, dtype=torch.float64, device="cuda"),
                  torch.randn(nrhs, nb, dtype=torch.float64, device="cuda")) / np.sqrt(2.0)
u = torch.empty((nrhs, nleaf, nt), dtype=torch.complex128, pin_memory=True)
torch.cuda.synchronize()
free0, total = torch.cuda.mem_get_info()
out = {"rank": rank, "subtree": f"{sub.nx}x{sub.ny} leaves on [{sub.x0},{sub.x1}]x[{sub.y0},{sub.y1}]",
       "kappa": cfg.kappa, "nrhs": nrhs, "device_free_gb_before_build": round(free0 / 1e9, 1)}
# as bench.py: the cross-handle cache of large blocks (re-mapping 117 GB per build would time the driver)
hps.set_cache_limit(int(0.95 * total))
res = []
for rep in range(3):
    t0 = time.perf_counter()
    S = hps.Solver(sub, cfg.p, cfg.kappa, cfg.eta, cd, keep_root_R=True)
    free1, _ = torch.cuda.mem_get_info()
    S.solve(s, t, u)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    res.append(dict(build_s=S.time_ms(0) / 1e3, leaf_s=S.time_ms(1) / 1e3, merge_s=S.time_ms(2) / 1e3,
                    solve_s=S.time_ms(3) / 1e3, up_s=S.time_ms(4) / 1e3, down_s=S.time_ms(5) / 1e3,
                    wall_s=wall, operators_gb=round((free0 - free1) / 1e9, 1),
                    build_tflops=S.flops(0) / max(S.time_ms(0), 1e-9) / 1e9))
    S.close()
hps.set_cache_limit(0)
out["runs"] = res
out["finite"] = bool(torch.isfinite(torch.view_as_real(u[:, :64])).all().item())
print(json.dumps(out))
