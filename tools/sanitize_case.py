"""Small cases through every kernel family for compute-sanitizer (memcheck / racecheck /
synccheck): C1 (complex leaf path, small merges), a real-interior-elimination leaf path, the
block-step natural-order inverse, and a 2-virtual-rank sharded build + solve."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import __graft_entry__
from paper_1812_07167_b200 import dist, hps, inputs

__graft_entry__.build()
rng = np.random.default_rng(0)


def case(nx, ny, p, kappa, eta, cimag=0.0, nrhs=2):
    g = hps.grid(0.0, 1.0, 0.0, ny / nx, nx, ny)
    X, Y = hps.leaf_nodes(g, p)
    c = (1 + 0.3 * np.exp(-((X - 0.4) ** 2 + (Y - 0.3) ** 2) / 0.05) + 1j * cimag).astype(complex)
    ni, nbr = (p - 2) ** 2, 2 * (nx + ny) * (p - 2)
    s = rng.standard_normal((nrhs, nx * ny, ni)) + 1j * rng.standard_normal((nrhs, nx * ny, ni))
    t = rng.standard_normal((nrhs, nbr)) + 1j * rng.standard_normal((nrhs, nbr))
    return g, c, s, t


cfg = inputs.CONFIGS[1]
g = hps.grid(cfg.x0, cfg.x1, cfg.y0, cfg.y1, cfg.nx, cfg.ny)
X, Y = hps.leaf_nodes(g, cfg.p)
c, s, t = inputs.make_inputs(cfg, X, Y, *hps.root_boundary_nodes(g, cfg.p))
u = hps.Solver(g, cfg.p, cfg.kappa, cfg.eta, c).solve(s + 1.0, t)
print("C1 ok", np.abs(u).max())
g, c, s, t = case(4, 2, 16, 4.0, 4.0)            # real interior elimination (below resonance)
print("real leaf ok", np.abs(hps.Solver(g, 16, 4.0, 4.0, c).solve(s, t)).max())
g, c, s, t = case(2, 2, 16, 30.0, 30.0, 0.05)    # complex Schur leaf, natural order
print("complex leaf ok", np.abs(hps.Solver(g, 16, 30.0, 30.0, c).solve(s, t)).max())
with hps.debug_knobs(nat_min=14, nat_bb_min=20):  # block-step natural-order W^-1
    g, c, s, t = case(8, 4, 8, 9.0, 9.0 + 1j)
    print("block-step W ok", np.abs(hps.Solver(g, 8, 9.0, 9.0 + 1j, c).solve(s, t)).max())
g, c, s, t = case(4, 4, 8, 9.0, 9.0)
d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()


def fn(comm):
    r, w = comm.info()
    sub, i0, j0 = dist.local_block(g, w, r)
    D = dist.DistributedHPS(comm, g, 8, 9.0, 9.0, d(dist.slice_leaves(c, g, sub, i0, j0)))
    u = D.solve(d(dist.slice_leaves(s, g, sub, i0, j0)), d(t)).cpu().numpy()
    D.close()
    return np.abs(u).max()


print("sharded ok", dist.run_virtual(2, fn))
