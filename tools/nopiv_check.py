"""Stability of natural-order (pivot-free) elimination of the real interior leaf matrix
A_ii = -(D2x (+) D2y) - kappa^2 diag(c) below the first interior resonance:
relative error of the pivot-free Gauss-Jordan inverse and the smallest pivot / original diagonal."""
import numpy as np


def cheb(p):
    x = -np.cos(np.pi * np.arange(p) / (p - 1))
    c = np.ones(p)
    c[0] = c[-1] = 2
    c *= (-1) ** np.arange(p)
    X = np.tile(x, (p, 1)).T
    D = np.outer(c, 1 / c) / (X - X.T + np.eye(p))
    return D - np.diag(D.sum(1))


def check(p, hx, hy, kappa, cmin, cmax, seed=0):
    D = cheb(p)
    q = p - 2
    Dxx = ((D * 2 / hx) @ (D * 2 / hx))[1:-1, 1:-1]
    Dyy = ((D * 2 / hy) @ (D * 2 / hy))[1:-1, 1:-1]
    c = np.random.default_rng(seed).uniform(cmin, cmax, q * q)
    A = -(np.kron(np.eye(q), Dxx) + np.kron(Dyy, np.eye(q))) - kappa ** 2 * np.diag(c)
    M, ratio = A.copy(), np.inf
    for k in range(A.shape[0]):
        piv = M[k, k]
        ratio = min(ratio, abs(piv) / abs(A[k, k]))
        prn, pc = M[k] / piv, M[:, k].copy()
        M -= np.outer(pc, prn)
        M[k], M[:, k], M[k, k] = prn, -pc / piv, 1 / piv
    Ai = np.linalg.inv(A)
    lam1 = np.pi ** 2 * (1 / hx ** 2 + 1 / hy ** 2)
    return kappa ** 2 * cmax / lam1, np.abs(M - Ai).max() / np.abs(Ai).max(), ratio


if __name__ == "__main__":
    for p in (4, 6, 8, 12, 16):
        for r in (0.0, 0.5, 0.89):
            lam1 = np.pi ** 2 * (1 / 0.25 + 1)
            print(p, "%.2f rel err %.1e min pivot/diag %.2f" % check(p, 0.5, 1.0, np.sqrt(r * lam1 / 1.3), 1.0, 1.3))
    print("C2 leaf", "%.2f rel err %.1e min pivot/diag %.2f" % check(16, 1 / 32, 1 / 32, 40 * np.pi, 0.5, 1.0))
