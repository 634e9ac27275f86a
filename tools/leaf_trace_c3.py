"""Timeline of CTA 0 of the complex leaf Schur kernel (zgj_seq_kernel + fused epilogue) on C3-like
leaves (h = 1/128, kappa = 1286.8: the C3-C5 per-leaf problem) -- per pass panel / staging /
update clocks, the epilogue and the assembly.
Usage: python tools/leaf_trace_c3.py [nleaf_side [knob=value ...]]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1812_07167_b200 import hps, inputs
cfg = inputs.CONFIGS[3]
n = int(sys.argv[1]) if len(sys.argv) > 1 else 32
knobs = {k: int(v) for k, v in (a.split("=") for a in sys.argv[2:])}
sub = inputs.Config(**{**cfg.__dict__, "nx": n, "ny": n, "x1": cfg.x0 + (cfg.x1 - cfg.x0) * n / cfg.nx,
                       "y1": cfg.y0 + (cfg.y1 - cfg.y0) * n / cfg.ny, "nrhs": 1})
g = hps.grid(sub.x0, sub.x1, sub.y0, sub.y1, n, n)
X, Y = hps.leaf_nodes(g, sub.p)
c, s, t = inputs.make_inputs(sub, X, Y, *hps.root_boundary_nodes(g, sub.p))
cd = torch.from_numpy(np.ascontiguousarray(c)).cuda()
S = hps.Solver(g, sub.p, sub.kappa, sub.eta, cd); S.close()
for rep in range(2):
  with hps.debug_knobs(**knobs):
    hps.lib().hps_debug_ws_trace((sub.p - 2) ** 2, None)   # trace the leaf launch only
    S = hps.Solver(g, sub.p, sub.kappa, sub.eta, cd, profile=1 << 7)
    buf = np.zeros(320, dtype=np.int64)
    hps.lib().hps_debug_ws_trace(0, buf.ctypes.data)
    ks = S.kernel_stats()
    path = S.leaf_path()
    S.close()
T = buf[:256].reshape(16, 16)
t0 = T[0, 0]
print(f"leaf path {path}, {n * n} leaves, knobs {knobs}; leaf class {ks.get('leaf_gj')}")
for p in range(7):
    extra = ""
    if T[p, 4] and T[p, 6]:   # block-form panel: stage / D^-1 / T product / write-back
        extra = (f"   [stage {(T[p,4]-T[p,0])/1e3:.1f}k, D^-1 {(T[p,5]-T[p,4])/1e3:.1f}k, T {(T[p,6]-T[p,5])/1e3:.1f}k, "
                 f"write {(T[p,1]-T[p,6])/1e3:.1f}k]")
    print(f"pass {p}: panel {(T[p,1]-T[p,0])/1e3:6.1f}k  staging {(T[p,2]-T[p,1])/1e3:5.1f}k  update {(T[p,3]-T[p,2])/1e3:6.1f}k clk{extra}")
print(f"GJ total {(T[6,3]-t0)/1e3:.1f}k clk, epilogue {(T[15,1]-T[15,0])/1e3:.1f}k clk, kernel start->GJ (assembly) {(t0 - T[15,2])/1e3 if T[15,2] else 0:.1f}k, kernel total {(T[15,1]-T[15,2])/1e3:.1f}k")
print("epilogue per phase (k clk, CTA 0, all chunks): wait %.1f | load+Y_i %.1f | Psi_i %.1f | Y_b+accY %.1f | Psi_b+accP %.1f"
      % tuple(T[15, 4:9] / 1e3))
