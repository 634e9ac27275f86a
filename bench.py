#!/usr/bin/env python
"""Benchmark: one step = the whole HPS hot path on one batch of synthetic input —
precomputation (batched leaf build + merge tree, Algorithm 1) followed by the solve sweeps
(Algorithm 2) — through the C-ABI of libhps.so.

Default workload: BASELINE.json configs[3] (C4: unit square, 256x256 leaves = 16.7M Chebyshev
nodes, p = 16, kappa = eta at 10 points per wavelength, 16 RHS) -- the largest configuration that
fits one GPU (BASELINE.json names no config for the metric; C5 needs 8 GPUs).  `--config 2`
runs C2 (32x32 leaves, 1 RHS), `--config 3` C3 (128x128 leaves, 64 RHS).

Metric (BASELINE.json): "HPS precompute sec & DOF/s; solve ms per RHS; FP64-TC % of peak;
HBM GB/s".  `value` is DOF/s of one full step (DOF = unique discretisation nodes, reading
Q16; step time = device time of build + solve on the library stream), summed over ranks;
the extra keys carry the build seconds, build DOF/s and solve ms per RHS.

Usage: python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl hps|reference]
Under torchrun (N > 1) the workload is SHARDED by subtree inside libhps:
each rank builds and solves its 1/N of the leaves and its subtree with no communication; the top
log2(N) levels run with the group split (W, W^-1 replicated in a group, Phi and R^tau split by
columns) over NCCL.  Strong scaling of the same workload; device time (library events, including
the collectives) max over ranks.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from paper_1812_07167_b200 import inputs  # noqa: E402

HBM_CLASSES = {"zgemv", "layout", "zgj_aux", "leaf_assemble"}  # bound by HBM, not the tensor pipe
METRIC = "HPS precompute sec & DOF/s; solve ms per RHS; FP64-TC % of peak; HBM GB/s"


def load_json(path, default=None):
    try:
        with open(path) as f:
            return json.load(f)
    except Exception:
        return default


_LIVE_PEAK = None


def fp64_peak():
    """FP64 tensor (DMMA m8n8k4) peak: measured live in this run (hps_fp64_peak, same process and
    clocks) when available, else the builder's measurement of this pool (tools/fp64_peaks.cu)."""
    if _LIVE_PEAK:
        return _LIVE_PEAK, "measured live in this run (hps_fp64_peak: DMMA.8x8x4 chains on every SM)"
    pk = load_json(os.path.join(ROOT, "bench", "peaks_fp64.json"), {})
    return pk.get("dmma_m8n8k4_tflops", 37.16), "builder-measured, bench/peaks_fp64.json (tools/fp64_peaks.cu)"


def hbm_peak():
    mp = load_json(os.path.join(ROOT, "MEASURED_PEAKS.json"), {})
    if "hbm_gbs" in mp:
        return mp["hbm_gbs"], "MEASURED_PEAKS.json hbm_gbs"
    return 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu):
        self.gpu = gpu
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.p = None

    def __enter__(self):
        try:
            import shutil
            cmd = ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                   "-lms", "20"]
            if shutil.which("stdbuf"):   # line-buffered: samples reach the file as they are taken
                cmd = ["stdbuf", "-oL"] + cmd
            self.p = subprocess.Popen(cmd, stdout=self.f, stderr=subprocess.DEVNULL)
            # the timed region of a small config lasts tens of ms: wait until the sampler runs
            t0 = time.time()
            while time.time() - t0 < 3.0 and os.path.getsize(self.f.name) == 0:
                time.sleep(0.01)
        except Exception:
            self.p = None
        return self

    def __exit__(self, *a):
        if self.p:
            self.p.terminate()
            try:
                self.p.wait(timeout=5)
            except Exception:
                self.p.kill()

    def summary(self):
        self.f.flush()
        self.f.seek(0)
        rows = [r.split(",") for r in self.f.read().strip().splitlines() if r.strip()]
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            try:
                sm.append(float(r[1]))
                mx = float(r[2])
                for n, v in zip(names, r[5:9]):
                    if v.strip().lower() == "active":
                        reasons.add(n)
            except Exception:
                continue
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def root_R_default(config):
    """SURVEY.md hard part 8: the root operator R^1 is formed for the parity configs 1-3 and skipped
    for 4-5 (Algorithm 2 never reads it)."""
    return config <= 3


def cfg_dict(cfg, nrhs, world, keep_root_R):
    """The workload description -- identical in both arms (the driver compares them)."""
    return {"workload": cfg.name, "leaves": f"{cfg.nx}x{cfg.ny}", "p": cfg.p, "nrhs": nrhs, "dof": cfg.n_unique,
            "kappa": round(cfg.kappa, 4), "keep_root_R": keep_root_R,
            "l2": "256 MiB buffer written between steps; stored operators (> 1 GB) exceed L2",
            "parallelism": "single GPU" if world == 1 else f"subtree shards x{world}"}


def merge_levels(cfg):
    """(depth d, n3, n1, ntau) of every merge level (SURVEY 8(a) A1 split rule)."""
    q = cfg.p - 2
    a, b = cfg.nx, cfg.ny
    dims = [(a, b)]
    while (a, b) != (1, 1):
        if a >= b:
            a //= 2
        else:
            b //= 2
        dims.append((a, b))
    out = []
    for d in range(len(dims) - 1):
        pa, pb = dims[d]
        ca, cb = dims[d + 1]
        n3 = (cb if pa >= pb else ca) * q
        n1 = 2 * (ca + cb) * q - n3
        out.append((d, n3, n1, 2 * n1))
    return out


def solve_model(cfg, nrhs):
    """SURVEY 8(d) algorithmic solve work per RHS batch: (bytes, flops).  Bytes: every stored
    operator read once (leaf [Psi | Y], and per merge W^-1, R33a, R33b, R13a, R23b, Phi^a, Phi^b) +
    s read, u~ written and read back, u written; flops: 8 per complex multiply-add."""
    p, q = cfg.p, cfg.p - 2
    nt, ni, nb = p * p - 4, q * q, 4 * q
    by = 16.0 * cfg.nleaf * (nt * nt + (ni + 3 * nt) * nrhs)
    fl = 8.0 * cfg.nleaf * nt * (ni + nb) * nrhs
    for d, n3, n1, ntau in merge_levels(cfg):
        m = 2 ** d
        by += 16.0 * m * (3 * n3 * n3 + 2 * n1 * n3 + 2 * n3 * ntau)
        fl += 8.0 * m * (3 * n3 * n3 + 2 * n1 * n3 + 2 * n3 * ntau) * nrhs
    return by, fl


def setup(cfg, hps):
    g = hps.grid(cfg.x0, cfg.x1, cfg.y0, cfg.y1, cfg.nx, cfg.ny)
    X, Y = hps.leaf_nodes(g, cfg.p)
    c, s, t = inputs.make_inputs(cfg, X, Y, *hps.root_boundary_nodes(g, cfg.p))
    return g, np.ascontiguousarray(c), np.ascontiguousarray(s), np.ascontiguousarray(t)


def flush_l2(torch, buf):
    buf.add_(1.0)   # 256 MiB write > 126 MB L2


def run_hps(args, rank, world, dist):
    import torch
    from paper_1812_07167_b200 import hps
    import __graft_entry__
    if rank == 0:
        __graft_entry__.build()
    if world > 1:
        dist.barrier()
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    cfg = inputs.CONFIGS[args.config]
    nrhs = args.nrhs or cfg.nrhs
    root_R = args.keep_root_R
    if args.gemm_slices > 0:   # process-wide knobs, set once and kept (not the default path)
        kn = {"gemm_slices": args.gemm_slices}
        if args.gemm_slices_min > 0:
            kn["gemm_slices_min"] = args.gemm_slices_min
        hps.debug_knobs(**kn).__enter__()
    g, c, s, t = setup(cfg, hps)
    s, t = s[:nrhs], t[:nrhs]
    comm, g_plan, nleaf = None, g, cfg.nleaf
    if world > 1:
        # subtree sharding: this rank's rectangle of c, s, u; the exchange runs inside libhps over NCCL
        from paper_1812_07167_b200 import dist as hdist
        comm = hdist.init_nccl()
        sub, i0, j0 = hdist.local_block(g, world, rank)
        c = np.ascontiguousarray(hdist.slice_leaves(c, g, sub, i0, j0))
        s = np.ascontiguousarray(hdist.slice_leaves(s, g, sub, i0, j0))
        g_plan, nleaf = sub, sub.nx * sub.ny
    dev = f"cuda:{local}"
    c_d = torch.from_numpy(c).to(dev)
    s_d = torch.from_numpy(np.ascontiguousarray(s)).to(dev)
    t_d = torch.from_numpy(np.ascontiguousarray(t)).to(dev)
    u_d = torch.empty((nrhs, nleaf, cfg.p * cfg.p - 4), dtype=torch.complex128, device=dev)
    l2buf = torch.zeros(32 * 1024 * 1024, dtype=torch.float64, device=dev)
    # opt in to the library's cross-handle cache of large blocks: every step builds a fresh handle
    # of the same shapes, and re-mapping tens of GB per step would time the driver, not the method
    total_mem = torch.cuda.get_device_properties(local).total_memory
    hps.set_cache_limit(int(0.9 * total_mem))
    plan = None
    if not args.no_plan:
        # representative-action planner: measured once per machine/process,
        # outside the timed region, like the paper's representative times
        plan = {lab: hps.REGIMES[reg] for lab, n, nb, reg, tab in hps.plan_problem(g_plan, cfg.p)}
        # the solve's matvec actions (Table 1's upward / downward rows): GEMM tile configuration per shape
        ps = hps.plan_solve(g_plan, cfg.p, nrhs)
        plan["solve_actions"] = {"actions": len(ps), "planned": sum(a["cfg"] >= 0 for a in ps),
                                 "rule_ms": round(sum(a["rule_ms"] for a in ps), 3),
                                 "planned_ms": round(sum(a["best_ms"] for a in ps), 3)}
        # and the build's merge products (Algorithm 1 lines 7-12) the same way
        pb = hps.plan_build(g_plan, cfg.p, keep_root_R=root_R)
        plan["build_actions"] = {"actions": len(pb), "planned": sum(a["cfg"] >= 0 for a in pb),
                                 "rule_ms": round(sum(a["rule_ms"] for a in pb), 3),
                                 "planned_ms": round(sum(a["best_ms"] for a in pb), 3)}

    def step(profile=0, keep_root_R=root_R):
        S = hps.Solver(g, cfg.p, cfg.kappa, cfg.eta, c_d, keep_root_R=keep_root_R, device=local, profile=profile,
                       comm=comm)
        S.solve(s_d, t_d, u_d)
        rec = dict(build_ms=S.time_ms(0), leaf_ms=S.time_ms(1), merge_ms=S.time_ms(2), solve_ms=S.time_ms(3),
                   up_ms=S.time_ms(4), down_ms=S.time_ms(5), launches=S.launches(0) + S.launches(1),
                   build_flops=S.flops(0), solve_flops=S.flops(1), kstats=S.kernel_stats())
        S.close()
        return rec

    for _ in range(args.warmup):
        flush_l2(torch, l2buf)
        step()
    global _LIVE_PEAK
    _LIVE_PEAK = hps.fp64_peak()   # roofline denominator at this run's clocks (outside the timed region)
    # one profiled step (all classes) picks the dominant kernel class
    flush_l2(torch, l2buf)
    probe = step(profile=True)
    dom_cls = max(probe["kstats"], key=lambda k: probe["kstats"][k]["ms"])
    dom_mask = 1 << hps.KCLASSES.index(dom_cls)
    torch.cuda.synchronize()
    recs, krecs = [], []
    with ClockSampler(local) as clk:
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        w0 = time.perf_counter()
        for _ in range(args.steps):   # the timed steps: no per-launch events
            flush_l2(torch, l2buf)
            torch.cuda.synchronize()
            recs.append(step())
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        wall = time.perf_counter() - w0
        # the dominant class's launches timed with CUDA events on the library stream over a second
        # set of steps (events between hundreds of small launches would lengthen the step)
        kx = min(args.steps, 3)
        for _ in range(kx):
            flush_l2(torch, l2buf)
            torch.cuda.synchronize()
            krecs.append(step(profile=dom_mask))
        # the build the other way round (with R^1 where the headline skips it, and vice versa)
        nrecs = []
        for _ in range(kx):
            flush_l2(torch, l2buf)
            torch.cuda.synchronize()
            nrecs.append(step(keep_root_R=not root_R))
    clocks = clk.summary()
    step_ms = statistics.mean(r["build_ms"] + r["solve_ms"] for r in recs)
    build_ms = statistics.mean(r["build_ms"] for r in recs)
    solve_ms = statistics.mean(r["solve_ms"] for r in recs)
    if world > 1:
        tt = torch.tensor([step_ms, build_ms, solve_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        step_ms, build_ms, solve_ms = tt.tolist()

    # ---- end-to-end through the public API with pinned HOST buffers ----
    c_h = torch.from_numpy(c).pin_memory()
    s_h = torch.from_numpy(np.ascontiguousarray(s)).pin_memory()
    t_h = torch.from_numpy(np.ascontiguousarray(t)).pin_memory()
    u_h = torch.empty((nrhs, nleaf, cfg.p * cfg.p - 4), dtype=torch.complex128).pin_memory()
    e2e = []
    for k in range(args.warmup + args.steps):
        flush_l2(torch, l2buf)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0 = time.perf_counter()
        S = hps.Solver(g, cfg.p, cfg.kappa, cfg.eta, c_h, keep_root_R=root_R, device=local, comm=comm)
        S.solve(s_h, t_h, u_h)
        _ = complex(u_h[0, 0, 0])        # result read on the host
        e1 = time.perf_counter()
        S.close()
        if k >= args.warmup:
            e2e.append(e1 - e0)
    e2e_s = statistics.mean(e2e)
    if world > 1:
        tt = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_s = tt.item()

    hps.set_cache_limit(0)   # give the parked blocks back
    build_alt_ms = statistics.mean(r["build_ms"] for r in nrecs)
    if world > 1:
        tt = torch.tensor([build_alt_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        build_alt_ms = tt.item()
        comm.close()
    build_r_ms, build_nr_ms = (build_ms, build_alt_ms) if root_R else (build_alt_ms, build_ms)
    if rank != 0:
        return None
    dof = cfg.n_unique       # the whole job's unknowns (strong scaling: the same problem on N GPUs)
    m3 = hps.debug_get("gemm_3m") != 0
    value = dof / (step_ms / 1e3)
    peak64, peak64_src = fp64_peak()
    hbm, hbm_src = hbm_peak()
    fl_build_r = flop_model(cfg)
    fl_build_nr = flop_model(cfg, root_R=False)
    fl_build = fl_build_r if root_R else fl_build_nr
    fl_leaf = 8.0 * (cfg.p * cfg.p - 4) ** 3 * cfg.nleaf
    sb, sf = solve_model(cfg, nrhs)
    t_build_roof = fl_build / (world * peak64 * 1e12)          # N GPUs: N x the per-GPU peaks
    t_solve_roof = max(sb / (world * hbm * 1e9), sf / (world * peak64 * 1e12))
    roofs = {
        "model": "SURVEY 8(d): build = leaf 8 n_tau^3 + merges (8 flop per complex MAC) / FP64 DMMA peak; "
                 "solve = max(bytes / HBM, flop / DMMA) with every stored operator read once; build_frac_3m_roof: "
                 "the merges' share at 6 tensor flop per complex MAC (the 3M products' own roof)",
        "keep_root_R": root_R,
        "build_flop": fl_build, "build_roofline_s": round(t_build_roof, 6),
        "build_frac": round(t_build_roof / (build_ms / 1e3), 4),
        "build_flop_with_root_R": fl_build_r,
        "build_frac_with_root_R": round(fl_build_r / (world * peak64 * 1e12) / (build_r_ms / 1e3), 4),
        "build_frac_3m_roof": (round((fl_leaf + (fl_build - fl_leaf) * 6 / 8) / (world * peak64 * 1e12) / (build_ms / 1e3), 4)
                               if m3 else None),
        "build_flop_no_root_R": fl_build_nr,
        "build_frac_no_root_R": round(fl_build_nr / (world * peak64 * 1e12) / (build_nr_ms / 1e3), 4),
        "build_executed_tflops": round(statistics.mean(r["build_flops"] for r in recs) / (build_ms / 1e3) / 1e12, 3),
        "solve_bytes": sb, "solve_flop": sf, "solve_roofline_ms": round(1e3 * t_solve_roof, 3),
        "solve_bound": "hbm" if sb / hbm / 1e9 >= sf / peak64 / 1e12 else "fp64",
        "solve_frac": round(t_solve_roof / (solve_ms / 1e3), 4),
        "solve_hbm_gbs": round(sb / (solve_ms / 1e3) / 1e9, 1),
    }
    # ---- roofline of the dominant kernel class (device time from CUDA events) ----
    agg = {}
    for r in krecs:
        for k, v in r["kstats"].items():
            a = agg.setdefault(k, dict(launches=0, ms=0.0, flops=0.0, bytes=0.0))
            for f in a:
                a[f] += v[f]
    dom = dom_cls
    A = agg[dom]
    traffic_tab = load_json(os.path.join(ROOT, "profiles", "ncu_traffic.json"), {})
    traffic = traffic_tab.get(f"C{args.config}", {}).get(dom)
    if isinstance(traffic, dict):   # class average over every launch of one ncu-captured step
        traffic = traffic.get("avg_dram_bytes_per_launch")
    if A["flops"] > 0 and dom not in HBM_CLASSES:
        peak, src = fp64_peak()
        if dom == "zgemm_dmma" and m3:
            # the 3M form issues 6 tensor flop per complex multiply-add where the zgemm convention
            # (the achieved figure's algorithmic count) counts 8: its roof in those units is 8/6 x DMMA
            peak, src = round(peak * 8 / 6, 3), src + " x 8/6 (3M form: 3 real DMMA products per complex MAC)"
        achieved = A["flops"] / (A["ms"] / 1e3) / 1e12
        roof = dict(bound="tensor", achieved=round(achieved, 3), peak=peak, unit="TFLOP/s",
                    frac=round(achieved / peak, 4), traffic=traffic, kernel=dom, peak_source=src,
                    launches=A["launches"] // len(krecs), avg_launch_us=round(1e3 * A["ms"] / A["launches"], 2),
                    share_of_step=round(A["ms"] / len(krecs) / step_ms, 3),
                    timing="CUDA events around each launch of the class on the library stream, over K extra "
                           "steps after the timed ones")
    else:
        peak, src = hbm_peak()
        achieved = A["bytes"] / (A["ms"] / 1e3) / 1e9
        roof = dict(bound="hbm", achieved=round(achieved, 1), peak=peak, unit="GB/s",
                    frac=round(achieved / peak, 4), traffic=traffic, kernel=dom, peak_source=src,
                    launches=A["launches"] // len(krecs), share_of_step=round(A["ms"] / len(krecs) / step_ms, 3))
    per_class = {k: dict(launches=v["launches"], ms=round(v["ms"], 3),
                         tflops=round(v["flops"] / max(v["ms"], 1e-9) / 1e9, 3) if v["flops"] else None,
                         gbs=round(v["bytes"] / max(v["ms"], 1e-9) / 1e6, 1))
                 for k, v in probe["kstats"].items()}
    out = {
        "metric": METRIC, "value": round(value, 1), "unit": "DOF/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(step_ms, 3), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "c128", "data": "synthetic",
        "config": cfg_dict(cfg, nrhs, world, root_R),
        "build_s": round(build_ms / 1e3, 6), "build_dof_per_s": round(dof / (build_ms / 1e3), 1),
        "build_s_with_root_R": round(build_r_ms / 1e3, 6),
        "build_s_no_root_R": round(build_nr_ms / 1e3, 6),
        "solve_ms_per_rhs": round(solve_ms / nrhs, 4),
        "build_tflops": round(statistics.mean(r["build_flops"] for r in recs) / (build_ms / 1e3) / 1e12, 3),
        "phase_ms": {k: round(statistics.mean(r[k] for r in recs), 3)
                     for k in ["leaf_ms", "merge_ms", "up_ms", "down_ms"]},
        "roofline_phases": roofs,
        "kernel_classes_probe_step": per_class,
        "plan": plan,
        "roofline": roof,
        "clocks": clocks,
        "wall_s_timed_region": round(wall, 3),
        "gpu_launches": int(sum(r["launches"] for r in recs)),
        "e2e": {"value": round(dof / e2e_s, 1), "unit": "DOF/s",
                "h2d_bytes_per_step": int(world * (c.nbytes + s.nbytes + t.nbytes)),
                "d2h_bytes_per_step": int(world * nrhs * nleaf * (cfg.p * cfg.p - 4) * 16), "s_per_step": round(e2e_s, 4),
                "note": "per-rank host buffers summed over ranks; time = max over ranks"},
    }
    out["host"] = {"cpu_model": cpu_model(), "nproc": os.cpu_count()}
    out["fp64_tensor_peak_tflops"] = {"live": round(_LIVE_PEAK, 3) if _LIVE_PEAK else None,
                                      "builder": load_json(os.path.join(ROOT, "bench", "peaks_fp64.json"), {}).get(
                                          "dmma_m8n8k4_tflops")}
    if args.gemm_slices > 0:
        out["gemm_slices"] = {"s": args.gemm_slices, "min": hps.debug_get("gemm_slices_min"),
                              "note": "opt-in: products with M, N, K >= min run as integer-slice products on the INT8 "
                                      "tensor path (cuBLASLt s8 GEMM between this repo's slicing and folding kernels); "
                                      "the roofline object's DMMA peak does not bound them"}
    if world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(cfg, c, s, t, args)
    return out


def oracle_run(cfg, c, s, t):
    """The oracle as it stands (Algorithm 1 + 2 on host cores, OpenMP over boxes)."""
    import oracle
    t0 = time.perf_counter()
    O = oracle.Oracle(cfg.x0, cfg.x1, cfg.y0, cfg.y1, cfg.nx, cfg.ny, cfg.p, cfg.kappa, cfg.eta, c)
    t1 = time.perf_counter()
    O.solve(s, t)
    t2 = time.perf_counter()
    O.close()
    return t1 - t0, t2 - t1


def cpu_cores():
    return int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))


def cpu_baseline(cfg, c, s, t, args):
    nrhs = s.shape[0]
    if cfg.nleaf <= 32 * 32:
        tb, ts = oracle_run(cfg, c, s, t)
        return {"value": round(cfg.n_unique / (tb + ts), 1), "unit": "DOF/s", "cores": cpu_cores(), "kind": "oracle",
                "sample": f"full workload ({cfg.nx}x{cfg.ny} leaves, {nrhs} RHS): oracle build {tb:.2f} s + solve "
                          f"{ts:.2f} s on {cpu_cores()} threads",
                "build_s": round(tb, 3), "solve_ms_per_rhs": round(1e3 * ts / nrhs, 3)}
    # larger configs: a 32x32-leaf corner of the same problem, extrapolated by the method's flop count
    sub = inputs.Config(**{**cfg.__dict__, "nx": 32, "ny": 32, "x1": cfg.x0 + (cfg.x1 - cfg.x0) * 32 / cfg.nx,
                           "y1": cfg.y0 + (cfg.y1 - cfg.y0) * 32 / cfg.ny, "nrhs": 1})
    from paper_1812_07167_b200 import hps
    g, cs, ss, ts_ = setup(sub, hps)
    tb, tsv = oracle_run(sub, cs, ss[:1], ts_[:1])   # the oracle always forms the corner's R^1
    f_full, f_sub = flop_model(cfg, root_R=args.keep_root_R), flop_model(sub)
    est = tb * f_full / f_sub + tsv * nrhs * (cfg.nleaf / sub.nleaf)
    return {"value": round(cfg.n_unique / est, 1), "unit": "DOF/s", "cores": cpu_cores(), "kind": "oracle",
            "sample": f"32x32-leaf corner, 1 RHS, build {tb:.2f} s + solve {tsv:.2f} s; extrapolated by the "
                      f"method's flop count to {cfg.nx}x{cfg.ny} leaves, {nrhs} RHS"}


def flop_model(cfg, root_R=True):
    """SURVEY 8(d) algorithmic build flops: leaf LU + inverse of B (8 n_tau^3) + every merge's
    W, W^-1, Phi^a, Phi^b and R^tau (8 flop per complex multiply-add); root_R=False drops the root
    level's R^tau product (Algorithm 2 never reads R^1)."""
    q, p = cfg.p - 2, cfg.p
    nt = p * p - 4
    fl = 8.0 * nt ** 3 * cfg.nleaf
    a, b = cfg.nx, cfg.ny
    dims = [(a, b)]
    while (a, b) != (1, 1):
        if a >= b:
            a //= 2
        else:
            b //= 2
        dims.append((a, b))
    for d in range(len(dims) - 1):
        pa, pb = dims[d]
        ca, cb = dims[d + 1]
        n3 = (cb if pa >= pb else ca) * q
        nbc = 2 * (ca + cb) * q
        n1 = nbc - n3
        ntau = 2 * n1
        fl += 8.0 * 2 ** d * (2 * n3 ** 3 + n3 * n3 * n1 + 2 * n3 * n3 * ntau + (ntau * ntau * n3 if (d or root_R) else 0))
    return fl


def run_reference(args, rank, world):
    """--impl reference: the CPU oracle as it stands, on the host cores (rank 0 only)."""
    if rank != 0:
        return None
    import oracle
    oracle.build()
    from paper_1812_07167_b200 import hps
    cfg = inputs.CONFIGS[args.config]
    nrhs = args.nrhs or cfg.nrhs
    # geometry from the oracle itself (no CUDA needed on this arm)
    X, Y = oracle.leaf_nodes(cfg.x0, cfg.x1, cfg.y0, cfg.y1, cfg.nx, cfg.ny, cfg.p)
    Xb = oracle.root_boundary(cfg.x0, cfg.x1, cfg.y0, cfg.y1, cfg.nx, cfg.ny, cfg.p)
    c, s, t = inputs.make_inputs(cfg, X, Y, *Xb, nrhs=nrhs)
    del hps
    small = inputs.CONFIGS[1]
    Xs, Ys = oracle.leaf_nodes(small.x0, small.x1, small.y0, small.y1, small.nx, small.ny, small.p)
    cs, ss, tss = inputs.make_inputs(small, Xs, Ys, *oracle.root_boundary(small.x0, small.x1, small.y0, small.y1,
                                                                          small.nx, small.ny, small.p))
    for _ in range(args.warmup):      # warm-up on the small case (bounded run time)
        oracle_run(small, cs, ss, tss)
    times = []
    sample = "full workload"
    for _ in range(args.steps):
        if cfg.nleaf <= 32 * 32:
            tb, ts = oracle_run(cfg, c, s, t)
            times.append(tb + ts)
        else:
            cb = cpu_baseline(cfg, c, s, t, args)
            times.append(cfg.n_unique / cb["value"])
            sample = cb["sample"]
    step_s = statistics.mean(times)
    val = cfg.n_unique / step_s
    return {"metric": METRIC, "value": round(val, 1), "unit": "DOF/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(1e3 * step_s, 1), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "c128", "data": "synthetic", "impl": "reference",
            "config": cfg_dict(cfg, nrhs, world, args.keep_root_R),
            "cpu_baseline": {"value": round(val, 1), "unit": "DOF/s", "cores": cpu_cores(), "kind": "oracle",
                             "sample": sample, "cpu_model": cpu_model()},
            "e2e": {"value": round(val, 1), "unit": "DOF/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--nrhs", type=int, default=0)
    ap.add_argument("--impl", default="hps", choices=["hps", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-plan", action="store_true", help="skip the representative-action planner (default rules)")
    ap.add_argument("--gemm-slices", type=int, default=0,
                    help="opt-in: big merge products as S 7-bit integer slices on the INT8 tensor path "
                         "(library knob gemm_slices, DESIGN.md 3.17; 0 = off, the default and the headline)")
    ap.add_argument("--gemm-slices-min", type=int, default=0, help="smallest M, N, K of a sliced product (0: library default)")
    ap.add_argument("--keep-root-R", type=int, default=None, choices=[0, 1],
                    help="form the root operator R^1 (default: configs 1-3 yes, 4-5 no; SURVEY hard part 8)")
    args = ap.parse_args()
    args.keep_root_R = root_R_default(args.config) if args.keep_root_R is None else bool(args.keep_root_R)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    dist = None
    if args.impl == "reference":
        out = run_reference(args, rank, world)
    else:
        if world > 1:
            import torch
            import torch.distributed as dist
            torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
            dist.init_process_group("nccl")
            out = run_hps(args, rank, world, dist)
        else:
            out = run_hps(args, rank, world, dist)
        if dist is not None:
            dist.destroy_process_group()
    if out is not None and rank == 0:
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
