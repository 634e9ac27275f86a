"""Time the batched Gauss-Jordan inverse kernel families on the shapes the HPS path launches
(leaf S at n = 196 and the merge W at n = 14 * 2^k), with a residual check per shape."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1812_07167_b200 import hps

shapes = [(196, 1024), (196, 148), (36, 1024), (56, 64), (56, 32), (112, 16), (112, 8), (224, 4), (224, 2),
          (224, 64), (168, 256), (84, 512)]
if len(sys.argv) > 1:
    shapes = [tuple(int(v) for v in s.split("x")) for s in sys.argv[1:]]
g = torch.Generator(device="cuda").manual_seed(0)
for n, batch in shapes:
    A = torch.randn(batch, n, n, dtype=torch.complex128, device="cuda", generator=g)
    fl = 8.0 * n ** 3 * batch
    row = []
    for mode in [int(m) for m in os.environ.get("GJ_MODES", "0,3,4,6,7").split(",")]:
        try:
            X, ms = hps.zinv_timed(A, mode=mode, reps=3)
            idx = [0, batch // 2, batch - 1]
            Ah, Xh = A[idx].cpu().numpy(), X[idx].cpu().numpy()
            res = max(np.abs(Ah[i] @ Xh[i] - np.eye(n)).max() for i in range(len(idx)))
            row.append(f"m{mode} {ms * 1e3:9.1f}us {fl / ms / 1e9:6.2f}TF res {res:.1e}")
        except Exception as e:
            row.append(f"m{mode} ERR {str(e)[:60]}")
    print(f"n={n:4d} batch={batch:5d} | " + " | ".join(row), flush=True)

if os.environ.get("WS_TRACE"):
    # timeline of CTA 0 of the warp-specialised kernel (clock64 deltas from the first mark)
    n, batch = shapes[0]
    A = torch.randn(batch, n, n, dtype=torch.complex128, device="cuda", generator=g)
    hps.lib().hps_debug_ws_trace(1, None)
    hps.zinv_timed(A, mode=int(os.environ.get("WS_TRACE_MODE", "3")), reps=1)
    buf = np.zeros(320, dtype=np.int64)
    hps.lib().hps_debug_ws_trace(0, buf.ctypes.data)
    t = buf[:256].reshape(16, 16)
    t0 = t[0, 4]
    names = ["P:ready", "P:factored", "P:tfree", "P:tready", "U:tready", "U:z1", "U:ph1", "U:z2", "U:ph2", "-"]
    print("n", n, "batch", batch, "(kclk relative to pass 0 start)")
    print("  p " + " ".join(f"{x:>10s}" for x in names[:9]))
    for p in range(15):
        if t[p].any():
            print(f"{p:3d} " + " ".join(f"{(v - t0) / 1e3:10.1f}" if v else f"{'':>10s}" for v in t[p, :9]))
