"""B200-native HPS / ItI direct solver for the variable-coefficient Helmholtz impedance
problem (arXiv:1812.07167): precomputation (leaf build + merge tree) and solve sweeps as
hand-written sm_100a CUDA behind the C-ABI in include/hps.h.

Modules:
  hps     — ctypes binding of libhps.so (no CPU fallback)
  inputs  — seeded synthetic problem data (no method arithmetic)
  dist    — multi-GPU subtree sharding over torch.distributed
"""
import os

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
REPO_DIR = os.path.dirname(PKG_DIR)
