"""CPU oracle for arXiv:1812.07167 (HPS with ItI operators) — TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and the ``cpu_baseline`` /
``--impl reference`` legs of ``bench.py`` may import this package.  The product
path (``paper_1812_07167_b200``) never imports it.

``liboracle.so`` is plain C++ (``hps_oracle.cpp``): naive LU with partial
pivoting, triple-loop products, the paper's Algorithms 1 and 2 with explicit
Upsilon and Gamma^tau, and a brute-force global collocation solver.  This file
is ctypes marshalling only.

Parity pins live in ``tests/test_oracle_*.py``.  Every oracle function is
pinned by at least one check that does not re-derive it from itself (see
DESIGN.md, "Oracle pins").
"""
from .oracle import *  # noqa: F401,F403
