"""Build + solve time of a config for settings of one library knob (hps_debug_set):
python tools/knob_sweep.py CONFIG KNOB v1 v2 ..."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench
from paper_1812_07167_b200 import hps, inputs

cfg = inputs.CONFIGS[int(sys.argv[1])]
knob = sys.argv[2]
vals = [int(v) for v in sys.argv[3:]]
g, c, s, t = bench.setup(cfg, hps)
d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
cd, sd, td = d(c), d(s), d(t)
hps.set_cache_limit(int(0.9 * torch.cuda.get_device_properties(0).total_memory))
hps.plan_problem(g, cfg.p)
for v in vals * 2:
    with hps.debug_knobs(**{knob: v}):
        ts = []
        for _ in range(3):
            S = hps.Solver(g, cfg.p, cfg.kappa, cfg.eta, cd)
            S.solve(sd, td)
            ts.append((S.time_ms(0), S.time_ms(2), S.time_ms(3)))
            S.close()
    b = min(x[0] for x in ts)
    print(f"{knob}={v}: build {b:.2f} ms (merges {min(x[1] for x in ts):.2f}), solve {min(x[2] for x in ts):.2f} ms",
          flush=True)
