"""Timeline of CTA 0 of the C2 leaf kernel (zgj_seq_kernel with the fused epilogue): per pass
panel / staging / update clocks and the epilogue."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1812_07167_b200 import hps, inputs
import bench
cfg = inputs.CONFIGS[2]
g, c, s, t = bench.setup(cfg, hps)
cd = torch.from_numpy(np.ascontiguousarray(c)).cuda()
S = hps.Solver(g, cfg.p, cfg.kappa, cfg.eta, cd); S.close()
hps.lib().hps_debug_ws_trace((cfg.p - 2) ** 2, None)   # trace the leaf launch only
S = hps.Solver(g, cfg.p, cfg.kappa, cfg.eta, cd)
buf = np.zeros(320, dtype=np.int64)
hps.lib().hps_debug_ws_trace(0, buf.ctypes.data)
S.close()
T = buf[:256].reshape(16, 16)
t0 = T[0, 0]
for p in range(7):
    print(f"pass {p}: panel {(T[p,1]-T[p,0])/1e3:6.1f}k  staging {(T[p,2]-T[p,1])/1e3:5.1f}k  update {(T[p,3]-T[p,2])/1e3:6.1f}k clk")
print(f"GJ total {(T[6,3]-t0)/1e3:.1f}k clk, assembly+init {(t0 - T[15,2])/1e3 if T[15,2] else 0:.1f}k, epilogue {(T[15,1]-T[15,0])/1e3:.1f}k clk")
print("epilogue per phase (k clk, CTA 0, all chunks): wait %.1f | load+Y_i %.1f | Psi_i %.1f | Y_b+accY %.1f | Psi_b+accP %.1f"
      % tuple(T[15, 4:9] / 1e3))
