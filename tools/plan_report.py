"""Per-level plan of the representative actions (PAPER.md:881-953 / Table 1) for a BASELINE
config: for every level, the measured representative time r and eps = ceil(N/theta_o) r of each
inverse regime and the chosen one (the GPU analogue of the paper's Figs. 3-4 thread choices)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1812_07167_b200 import hps, inputs
cfg = inputs.CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 2]
g = hps.grid(cfg.x0, cfg.x1, cfg.y0, cfg.y1, cfg.nx, cfg.ny)
print(f"{cfg.name}: representative action = leaf interior inverse, then merge interface inverses")
print(f"{'level':>9s} {'n':>5s} {'N_boxes':>8s}  " + "  ".join(f"{hps.REGIMES[k]:>22s}" for k in range(1, 8)) + "   chosen")
print(f"{'':>25s}" + "  ".join(f"{'eps ms (r ms, th_o)':>22s}" for _ in range(1, 8)))
for lab, n, nb, reg, tab in hps.plan_problem(g, cfg.p):
    cells = []
    for k in range(1, 8):
        if k in tab:
            e, r, th = tab[k]
            cells.append(f"{e:9.3f} ({r:6.3f},{th:5d})")
        else:
            cells.append(f"{'-':>22s}")
    print(f"{lab:>9s} {n:5d} {nb:8d}  " + "  ".join(cells) + f"   {hps.REGIMES[reg]}", flush=True)
