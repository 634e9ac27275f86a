"""Step phases with individual plan entries forced (diagnoses regime side effects)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1812_07167_b200 import hps, inputs
import bench
cfg = inputs.CONFIGS[2]
g, c, s, t = bench.setup(cfg, hps)
d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
c_d, s_d, t_d = d(c), d(s), d(t)
def run(tag):
    for k in range(3):
        S = hps.Solver(g, cfg.p, cfg.kappa, cfg.eta, c_d); S.solve(s_d, t_d)
        if k == 2: print(f"{tag:40s} build {S.time_ms(0):.2f} merge {S.time_ms(2):.2f} up {S.time_ms(4):.3f} down {S.time_ms(5):.3f}", flush=True)
        S.close()
run("default")
for (n, nb) in []:
    for reg in (4, 6):
        hps._check(hps.lib().hps_plan_set(n, nb, reg))
        run(f"({n},{nb}) -> {hps.REGIMES[reg]}")
        hps.plan_clear()
rows = hps.plan_problem(g, cfg.p)
run("full plan_problem")
for lab, n, nb, reg, tab in rows:
    hps._check(hps.lib().hps_plan_set(n, nb, 0))
    run(f"  minus {lab} ({n},{nb}) [{hps.REGIMES[reg]}]")
hps.plan_clear()
run("cleared")
