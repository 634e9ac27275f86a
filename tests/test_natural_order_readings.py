"""Readings Q20-Q22: the matrices the CUDA path eliminates in natural
order keep every pivot well above the checks the kernels apply, in the configs' regimes.  Pure
numpy / oracle (no GPU): the matrices are built here or taken from the oracle's merges."""
import numpy as np

import oracle
from paper_1812_07167_b200 import inputs


def cheb(p):
    x = -np.cos(np.pi * np.arange(p) / (p - 1))
    c = np.ones(p)
    c[0] = c[-1] = 2
    c *= (-1) ** np.arange(p)
    X = np.tile(x, (p, 1)).T
    D = np.outer(c, 1 / c) / (X - X.T + np.eye(p))
    return D - np.diag(D.sum(1))


def gj_natural(A):
    """Gauss-Jordan without pivoting; returns (result, min |pivot| / |original diagonal|)."""
    M = A.astype(complex).copy()
    ratio = np.inf
    for k in range(len(M)):
        piv = M[k, k]
        ratio = min(ratio, abs(piv) / abs(A[k, k]))
        prn, pc = M[k] / piv, M[:, k].copy()
        M -= np.outer(pc, prn)
        M[k], M[:, k], M[k, k] = prn, -pc / piv, 1 / piv
    return M, ratio


def test_real_interior_block_c2_leaf():
    """Q20: A_ii = -(D2x (+) D2y) - kappa^2 diag(c) of a C2 leaf (h = 1/32, kappa = 40 pi, c in
    [0.5, 1]): natural-order inverse to 1e-12, pivots >= 0.3 of the diagonal (check: 0.05)."""
    p, h, kappa = 16, 1 / 32, 40 * np.pi
    D = cheb(p) * 2 / h
    D2 = (D @ D)[1:-1, 1:-1]
    q = p - 2
    c = np.random.default_rng(0).uniform(0.5, 1.0, q * q)
    A = -(np.kron(np.eye(q), D2) + np.kron(D2, np.eye(q))) - kappa ** 2 * np.diag(c)
    M, ratio = gj_natural(A)
    assert np.max(np.abs(M - np.linalg.inv(A))) / np.max(np.abs(np.linalg.inv(A))) < 1e-12
    assert ratio > 0.3


def test_complex_schur_c3_leaf():
    """Q22: the complex interior Schur complement S = Lx (+) Ly - kappa^2 diag(c) of a C3 leaf
    (h = 1/128, kappa at 10 points per wavelength, eta = kappa): pivots >= 0.3 of the diagonal."""
    p, h, kappa = 16, 1 / 128, inputs.CONFIGS[3].kappa
    D = cheb(p) * 2 / h
    D2 = D @ D
    q = p - 2
    G = np.array([[-D[0, 0] + 1j * kappa, -D[0, p - 1]], [D[p - 1, 0], D[p - 1, p - 1] + 1j * kappa]])
    FI = np.vstack([-D[0, 1:-1], D[p - 1, 1:-1]])
    Ub = np.column_stack([D2[1:-1, 0], D2[1:-1, p - 1]]) @ np.linalg.inv(G)
    L = -D2[1:-1, 1:-1] + Ub @ FI
    c = np.random.default_rng(1).uniform(1.0, 1.6, q * q)
    S = np.kron(np.eye(q), L) + np.kron(L, np.eye(q)) - kappa ** 2 * np.diag(c)
    M, ratio = gj_natural(S)
    Si = np.linalg.inv(S)
    assert np.max(np.abs(M - Si)) / np.max(np.abs(Si)) < 1e-12
    assert ratio > 0.3


def test_merge_W_top_levels_c2_leaves():
    """Q21: W = I - R33b R33a of the top merges of an 8x8-leaf square with C2's leaf size and
    kappa (eta = kappa): natural-order inverse to 1e-12, pivots >= 0.5 of the diagonal and
    |pivot|^2 far above the 1e-6 check.  (||I - W||_2 is NOT below 1 here: the ItI maps are
    contractions in the boundary energy norm, not in the Euclidean one.)"""
    nx = ny = 8
    p, kappa = 16, 40 * np.pi
    X, Y = oracle.leaf_nodes(0.0, 0.25, 0.0, 0.25, nx, ny, p)
    c = (1 - 0.5 * np.exp(-160 * ((X - 0.125) ** 2 + (Y - 0.125) ** 2))).astype(complex)
    O = oracle.Oracle(0.0, 0.25, 0.0, 0.25, nx, ny, p, kappa, kappa, c, keep_all_R=True)
    for box in (1, 2, 3):
        a, b = 2 * box, 2 * box + 1
        i0, i1, j0, j1, vert = oracle.box_rect(nx, ny, box)
        ai = oracle.box_rect(nx, ny, a)
        m = oracle.merge(p, ai[1] - ai[0], ai[3] - ai[2], bool(vert), O.R(a), O.R(b))
        W = np.linalg.inv(m["Winv"])
        Mn, ratio = gj_natural(W)
        assert np.max(np.abs(Mn - m["Winv"])) / np.max(np.abs(m["Winv"])) < 1e-12
        assert ratio > 0.5
        assert np.min(np.abs(np.diag(W))) ** 2 * ratio ** 2 > 1e-3
    O.close()
