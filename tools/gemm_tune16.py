"""Tile configurations of the DMMA GEMM on the solve shapes at 16 right-hand sides (C4):
leaf u~ = Y s (252 x 16 x 196), leaf u = Psi t (252 x 16 x 56), merge-level products."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1812_07167_b200 import hps

shapes = [(252, 16, 196, 8192), (252, 16, 56, 8192), (28, 16, 112, 16384), (42, 16, 14, 32768), (56, 16, 224, 4096),
          (1792, 16, 1792, 4), (3584, 16, 14336, 1), (448, 16, 448, 256)]
for M, N, K, b in shapes:
    A = torch.randn(b, M, K, dtype=torch.complex128, device="cuda")
    B = torch.randn(b, K, N, dtype=torch.complex128, device="cuda")
    row = []
    for cfg in (-1, 1, 2, 10, 12, 13, 0):
        if cfg == 0 and N > 8:
            continue
        try:
            _, ms = hps.zgemm_batched(A, B, cfg=cfg, reps=5)
            row.append(f"cfg{cfg}: {ms:8.3f} ms {8.0 * M * N * K * b / ms / 1e9:6.2f} TF")
        except Exception as e:  # noqa: BLE001
            row.append(f"cfg{cfg}: {e}")
    print(f"M={M} N={N} K={K} batch={b}:  " + " | ".join(row), flush=True)
