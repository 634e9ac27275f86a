"""The paper's convergence experiment (Fig. 5) on the
CUDA path: e_inf = max_j |u(x_j) - u_j| against N for n_c in {6, 9, 16} (n_c = p)."""
import numpy as np

from . import hps, inputs


def paper_error(p, nleaf_side, kappa=inputs.PAPER_KAPPA):
    g = hps.grid(0.0, 1.0, 0.0, 1.0, nleaf_side, nleaf_side)
    X, Y = hps.leaf_nodes(g, p)
    Xb, Yb, NX, NY = hps.root_boundary_nodes(g, p)
    c = inputs.paper_c(X, Y)
    Xi, Yi = inputs.interior_of(p, X), inputs.interior_of(p, Y)
    s = inputs.paper_s(Xi, Yi, kappa)[None]
    t = inputs.paper_t(Xb, Yb, NX, NY, kappa, kappa)[None]
    S = hps.Solver(g, p, kappa, kappa, np.ascontiguousarray(c), keep_root_R=False)
    u = S.solve(np.ascontiguousarray(s), np.ascontiguousarray(t))[0]
    err_i = np.max(np.abs(u[:, 4 * (p - 2):] - inputs.paper_u(Xi, Yi, kappa)))
    q = p - 2
    N = q * (nleaf_side * nleaf_side * q + 2 * (nleaf_side + 1) * nleaf_side)
    S.close()
    return N, err_i


def convergence_table(ps=(6, 9, 16), sides=(8, 16, 32, 64)):
    return {p: [paper_error(p, m) for m in sides] for p in ps}


if __name__ == "__main__":
    for p, rows in convergence_table().items():
        for N, e in rows:
            print(f"n_c={p:2d}  N={N:9d}  e_inf={e:.3e}")
