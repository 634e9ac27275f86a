"""Sweep the DMMA tile configurations on the shapes the HPS path launches."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1812_07167_b200 import hps

shapes = [  # (M, N, K, batch, has_cin) — from the C2/C3 traces
    (196, 168, 28, 1024, 1), (196, 168, 28, 128, 1), (252, 64, 196, 2048, 0), (252, 64, 56, 2048, 1),
    (448, 1792, 448, 1, 0), (896, 1792, 448, 1, 1), (1792, 7168, 1792, 1, 0), (3584, 7168, 1792, 1, 1),
    (112, 448, 112, 16, 0), (224, 448, 112, 16, 1), (56, 224, 56, 64, 0), (14, 84, 14, 512, 0),
    (42, 84, 14, 512, 1), (28, 112, 28, 256, 0), (448, 416, 32, 1, 1), (1792, 1764, 28, 1, 1),
    (252, 1, 196, 1024, 0), (448, 1, 1792, 1, 1),
]
cfgs = list(range(9))
if len(sys.argv) > 1:
    shapes = [tuple(int(v) for v in a.split('x')) for a in sys.argv[1:]]
torch.manual_seed(0)
for (M, N, K, batch, cin) in shapes:
    A = torch.randn(batch, M, K, dtype=torch.complex128, device="cuda")
    B = torch.randn(batch, K, N, dtype=torch.complex128, device="cuda")
    Ci = torch.randn(batch, M, N, dtype=torch.complex128, device="cuda") if cin else None
    res = []
    for c in cfgs:
        try:
            _, ms = hps.zgemm_batched(A, B, Ci, 1.0, 1.0 if cin else 0.0, cfg=c, reps=5)
            res.append((ms, c))
        except Exception as e:
            res.append((float("inf"), c))
    _, ms_auto = hps.zgemm_batched(A, B, Ci, 1.0, 1.0 if cin else 0.0, cfg=-1, reps=5)
    fl = 8.0 * M * N * K * batch
    best = min(res)
    print(f"M={M:5d} N={N:5d} K={K:5d} b={batch:5d} cin={cin} auto {ms_auto*1e3:9.1f}us {fl/ms_auto/1e9:6.2f}TF | best cfg {best[1]} "
          f"{best[0]*1e3:9.1f}us {fl/best[0]/1e9:6.2f}TF | " + " ".join(f"{c}:{fl/ms/1e9:5.1f}" for ms, c in res), flush=True)
