"""Why the bench's back-to-back steps gain less from gemm_slices than isolated builds: per-build times
and SM clock / power samples for runs of consecutive builds, with and without the build planner."""
import os, sys, threading, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, pynvml
import bench
from paper_1812_07167_b200 import hps, inputs

cfg = inputs.CONFIGS[4]
g, c, s, t = bench.setup(cfg, hps)
d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
cd, sd, td = d(c), d(s), d(t)
torch.cuda.synchronize()
hps.set_cache_limit(int(0.9 * torch.cuda.get_device_properties(0).total_memory))
hps.plan_problem(g, cfg.p)
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
samples, stop = [], False


def sampler():
    while not stop:
        samples.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM), pynvml.nvmlDeviceGetPowerUsage(h) / 1e3))
        time.sleep(0.02)


def run(label, ns, n=8, gap=0.0):
    global samples, stop
    samples, stop = [], False
    th = threading.Thread(target=sampler)
    th.start()
    ts = []
    with hps.debug_knobs(gemm_slices=ns):
        for _ in range(n):
            S = hps.Solver(g, cfg.p, cfg.kappa, cfg.eta, cd, keep_root_R=False)
            S.solve(sd, td)
            ts.append((S.time_ms(0), S.time_ms(2), S.time_ms(3)))
            S.close()
            if gap:
                time.sleep(gap)
    stop = True
    th.join()
    clk = sorted(x[0] for x in samples)
    pw = sorted(x[1] for x in samples)
    print(f"{label}: builds " + " ".join(f"{x[0]:.0f}" for x in ts) + " ms; merges " + " ".join(f"{x[1]:.0f}" for x in ts)
          + f"; solve {min(x[2] for x in ts):.1f}..{max(x[2] for x in ts):.1f} ms; SM MHz min/median {clk[0]}/{clk[len(clk) // 2]}, "
          f"power median/max {pw[len(pw) // 2]:.0f}/{pw[-1]:.0f} W", flush=True)


run("no build plan, slices 0", 0)
run("no build plan, slices 8", 8)
run("no build plan, slices 8, 0.5 s idle between builds", 8, gap=0.5)
hps.plan_build(g, cfg.p, keep_root_R=False)
hps.plan_solve(g, cfg.p, s.shape[0])
run("build plan, slices 0", 0)
run("build plan, slices 8", 8)
