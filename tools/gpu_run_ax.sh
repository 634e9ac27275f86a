#!/bin/bash
# integer-slice products (knob gemm_slices, zgemm_slices.cu): parity tests, product timings, C3/C4 sweeps,
# polynomial errors with the knob on
cd "$(dirname "$0")/.."
O=gpurun_out/${OUT:-ax}
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "integer_slices" > $O/pytest_slices.txt 2>&1
timeout 600 python - > $O/product_times.txt 2>&1 <<'PY'
import numpy as np, torch
from paper_1812_07167_b200 import hps
g = torch.Generator(device="cuda").manual_seed(1)
for (M, K, N) in ((3584, 3584, 10752), (1792, 1792, 5376), (896, 896, 2688), (5376, 1792, 10752)):
    A = torch.view_as_complex(torch.randn(1, M, K, 2, dtype=torch.float64, device="cuda", generator=g))
    B = torch.view_as_complex(torch.randn(1, K, N, 2, dtype=torch.float64, device="cuda", generator=g))
    torch.cuda.synchronize()   # the library runs on its own stream: inputs complete on entry
    ref = None
    for ns in (0, 6, 7, 8):
        with hps.debug_knobs(gemm_slices=ns):
            hps.zgemm_batched(A, B)
            C, ms = hps.zgemm_batched(A, B, reps=3)
        if ns == 0:
            ref = C
        err = ((C - ref).abs().max() / ref.abs().max()).item()
        print(f"{M}x{K}x{N} gemm_slices={ns}: {ms:.3f} ms = {8.0 * M * N * K / ms / 1e9:.1f} TF/s (8 flop per complex MAC), "
              f"max rel diff vs DMMA {err:.2e}", flush=True)
PY
timeout 900 python tools/knob_sweep.py 4 gemm_slices 0 8 7 > $O/sweep_c4.txt 2>&1
timeout 600 python tools/knob_sweep.py 3 gemm_slices 0 8 7 > $O/sweep_c3.txt 2>&1
timeout 900 python tools/poly_errors.py gemm_slices=8 > $O/poly_errors_s8.txt 2>&1
timeout 900 python tools/poly_errors.py gemm_slices=7 > $O/poly_errors_s7.txt 2>&1
echo done
