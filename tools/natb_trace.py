"""Timeline of the first blocked natural-order panel (CTA 0, k0 = 0) of the C2 top-level inverse."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1812_07167_b200 import hps, inputs
import bench
cfg = inputs.CONFIGS[2]
g, c, s, t = bench.setup(cfg, hps)
d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
S = hps.Solver(g, cfg.p, cfg.kappa, cfg.eta, d(c))
S.close()
hps.lib().hps_debug_ws_trace(7, None)
S = hps.Solver(g, cfg.p, cfg.kappa, cfg.eta, d(c))
torch.cuda.synchronize()
buf = np.zeros(320, dtype=np.int64)
hps.lib().hps_debug_ws_trace(0, buf.ctypes.data)
tr = buf[256:]
print("block load %d, block GJ %d, stage1 total %d clk, stage2 %d clk, store %d clk" % (tr[4] - tr[0], tr[5] - tr[4], tr[1] - tr[0], tr[2] - tr[1], tr[3] - tr[2]))
