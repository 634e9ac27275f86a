import sys; sys.path.insert(0, "/root/repo")
import torch
from paper_1812_07167_b200 import hps
A = torch.randn(1, 448, 448, dtype=torch.complex128, device="cuda")
hps.zinv_timed(A, mode=6, reps=1)
