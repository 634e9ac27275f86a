"""Host enqueue time against device time of one build and one solve (is a step host-bound?).

python tools/host_probe.py CONFIG [NRHS]

The handle orders its work on a torch stream (hps_opts.stream), so hps_solve returns once every
launch is enqueued: wall time of the call = host enqueue cost; wall time to the following
synchronize = device completion.  If enqueue ~ device time, the GPU waits for the host and a CUDA
graph (or fewer launches) would pay; if enqueue << device time, it would not."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1812_07167_b200 import hps, inputs  # noqa: E402


def main():
    k = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    cfg = inputs.CONFIGS[k]
    nrhs = int(sys.argv[2]) if len(sys.argv) > 2 else cfg.nrhs
    g = hps.grid(cfg.x0, cfg.x1, cfg.y0, cfg.y1, cfg.nx, cfg.ny)
    X, Y = hps.leaf_nodes(g, cfg.p)
    Xb, Yb, NX, NY = hps.root_boundary_nodes(g, cfg.p)
    c, s, t = inputs.make_inputs(cfg, X, Y, Xb, Yb, NX, NY, nrhs=nrhs)
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    c, s, t = dev(c), dev(s), dev(t)
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        for it in range(4):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            S = hps.Solver(g, cfg.p, cfg.kappa, cfg.eta, c, keep_root_R=False, stream=st)
            t1 = time.perf_counter()
            torch.cuda.synchronize()
            t2 = time.perf_counter()
            uo = S.solve(s, t)  # warm (allocates u)
            torch.cuda.synchronize()
            e_solve, d_solve = [], []
            for _ in range(10):
                a0 = time.perf_counter()
                S.solve(s, t, uo)
                a1 = time.perf_counter()
                S.sync()
                torch.cuda.synchronize()
                a2 = time.perf_counter()
                e_solve.append(a1 - a0)
                d_solve.append(a2 - a0)
            print(f"C{k} it {it}: build enqueue {1e3 * (t1 - t0):.3f} ms, build wall {1e3 * (t2 - t0):.3f} ms "
                  f"(launches {S.launches(0)}); solve enqueue {1e3 * np.median(e_solve):.3f} ms, "
                  f"solve wall {1e3 * np.median(d_solve):.3f} ms (launches {S.launches(1)}, nrhs {s.shape[0]})",
                  flush=True)
            S.close()


if __name__ == "__main__":
    main()
