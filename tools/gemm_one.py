"""One batched ZGEMM of a given shape through the library (for ncu captures).
usage: python tools/gemm_one.py MxNxKxBATCHxCIN [knob=value ...]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1812_07167_b200 import hps
M, N, K, batch, cin = (int(v) for v in sys.argv[1].split("x"))
knobs = {k: int(v) for k, v in (a.split("=") for a in sys.argv[2:])}
cfg = knobs.pop("cfg", -1)   # tile configuration (hps_zgemm_batched cfg), -1 = the library's rule
A = torch.randn(batch, M, K, dtype=torch.complex128, device="cuda")
B = torch.randn(batch, K, N, dtype=torch.complex128, device="cuda")
Ci = torch.randn(batch, M, N, dtype=torch.complex128, device="cuda") if cin else None
with hps.debug_knobs(**knobs):
    _, ms = hps.zgemm_batched(A, B, Ci, 1.0, 1.0 if cin else 0.0, cfg=cfg, reps=2)
print(f"{M}x{N}x{K} b{batch} cfg {cfg} {knobs}: {ms*1e3:.1f} us, {8.0*M*N*K*batch/ms/1e9:.2f} TF", flush=True)
