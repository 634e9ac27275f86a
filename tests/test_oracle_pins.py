"""Pins for the CPU oracle (oracle/hps_oracle.cpp) against things OTHER than
itself: values printed in the paper / SPEC, closed forms, exactness on
polynomials, invariants, library routines and brute force on tiny inputs.

Each test names the oracle function(s) it pins and the passage it follows.
"""
import json
import math
import os

import numpy as np
import numpy.polynomial.chebyshev as npc
import pytest

from paper_1812_07167_b200 import inputs

GOLD = os.path.join(os.path.dirname(__file__), "golden", "paper_counts.json")


def rel(a, b):
    return np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300)


# ---------------------------------------------------------------------------
# Golden values printed in the paper / SPEC
# ---------------------------------------------------------------------------
def test_golden_counts(orc):
    """oracle_tree_info, leaf index sets, merge index sets vs printed counts."""
    g = json.load(open(GOLD))
    for e in g["n_boxes"]:
        assert orc.tree_info(e["nx"], e["ny"])[0] == e["N_boxes"], e["cite"]
    for e in g["leaf_sizes"]:
        p = e["n_c"]
        lf = orc.leaf(p, 1.0, 1.0, 1.0, 1.0, np.ones(p * p))
        assert lf["R"].shape == (e["n_b"], e["n_b"]), e["cite"]
        assert lf["Y"].shape == (e["n_tau"], e["n_i"]), e["cite"]
        assert lf["Psi"].shape == (e["n_tau"], e["n_b"]), e["cite"]
    for e in g["merge_sizes"]:
        p = e["n_c"]
        nb = 4 * p - 8
        m = orc.merge(p, 1, 1, 1, np.zeros((nb, nb)), np.zeros((nb, nb)))
        assert m["Winv"].shape == (e["I3"], e["I3"]), e["cite"]
        assert m["PhiA"].shape == (e["I3"], e["I1"] + e["I2"]), e["cite"]
    for e in g["cheb_nodes"]:
        x, _ = orc.cheb(e["n_c"])
        assert np.allclose(x, e["nodes"], atol=1e-15), e["cite"]


def test_tree_counts(orc):
    """Uniform tree: N_boxes = 2 nx ny - 1; depth log2(nx ny)."""
    for nx, ny in [(1, 1), (2, 1), (2, 2), (4, 2), (8, 8), (32, 16)]:
        nb, d = orc.tree_info(nx, ny)
        assert nb == 2 * nx * ny - 1
        assert d == int(round(math.log2(nx * ny)))


# ---------------------------------------------------------------------------
# Chebyshev machinery
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("p", [2, 3, 5, 8, 9, 16, 20])
def test_cheb_nodes_closed_form(orc, p):
    x, _ = orc.cheb(p)
    assert np.all(np.diff(x) > 0)
    assert x[0] == -1.0 and x[-1] == 1.0
    assert np.allclose(x, -x[::-1], atol=1e-15)
    # closed form via numpy: extrema of T_{p-1} are the roots of U_{p-2} plus +-1
    if p > 2:
        inner = np.sort(npc.chebroots(npc.chebder([0] * (p - 1) + [1])))
        assert np.allclose(x[1:-1], inner, atol=1e-13)


@pytest.mark.parametrize("p", [4, 8, 10, 16])
def test_cheb_diff_exact_on_polynomials(orc, p):
    """D differentiates every polynomial of degree <= p-1 exactly."""
    x, D = orc.cheb(p)
    assert np.max(np.abs(D @ np.ones(p))) < 1e-12
    for k in range(p):
        coef = np.zeros(p)
        coef[k] = 1.0   # T_k, exact derivative from numpy's chebder
        f = npc.chebval(x, coef)
        df = npc.chebval(x, npc.chebder(coef)) if k else np.zeros(p)
        assert np.max(np.abs(D @ f - df)) < 1e-11 * max(1, k * k)


# ---------------------------------------------------------------------------
# Naive linear algebra
# ---------------------------------------------------------------------------
def test_lu_inverse_residual_and_library(orc):
    rng = np.random.default_rng(1)
    A = rng.standard_normal((200, 200)) + 1j * rng.standard_normal((200, 200))
    Ai = orc.invert(A)
    assert np.max(np.abs(A @ Ai - np.eye(200))) < 1e-10
    assert rel(Ai, np.linalg.inv(A)) < 1e-10                     # library routine
    # partial pivoting: a zero leading entry must not break it
    P = np.array([[0, 1], [1, 0]], complex)
    assert np.allclose(orc.invert(P), P)


def test_matmul_library(orc):
    rng = np.random.default_rng(2)
    A = rng.standard_normal((17, 9)) + 1j * rng.standard_normal((17, 9))
    B = rng.standard_normal((9, 5)) + 1j * rng.standard_normal((9, 5))
    assert rel(orc.matmul(A, B), A @ B) < 1e-14


# ---------------------------------------------------------------------------
# Leaf: manufactured polynomial solution is reproduced exactly
# ---------------------------------------------------------------------------
class Poly2D:
    """P(x, y) = sum a_jk T_j(xs) T_k(ys), xs, ys affine maps of [x0,x1]x[y0,y1]
    onto [-1,1]; exact derivatives from numpy.polynomial (independent of D)."""

    def __init__(self, deg, box, seed):
        rng = np.random.default_rng(seed)
        self.a = (rng.standard_normal((deg + 1, deg + 1)) + 1j * rng.standard_normal((deg + 1, deg + 1)))
        self.a /= np.arange(1, deg + 2)[:, None] * np.arange(1, deg + 2)[None, :]
        self.x0, self.x1, self.y0, self.y1 = box
        self.sx, self.sy = 2 / (self.x1 - self.x0), 2 / (self.y1 - self.y0)

    def _m(self, X, Y):
        return self.sx * (X - self.x0) - 1, self.sy * (Y - self.y0) - 1

    def val(self, X, Y, dx=0, dy=0):
        xs, ys = self._m(X, Y)
        a = self.a
        if dx:
            a = npc.chebder(a, dx, axis=0) * self.sx ** dx
        if dy:
            a = npc.chebder(a, dy, axis=1) * self.sy ** dy
        return npc.chebval2d(xs, ys, a) if a.size else np.zeros_like(X, dtype=complex)


def leaf_boundary_geometry(p, x0, y0, hx, hy, orc):
    """Coordinates/normals of one leaf's [S,E,N,W] nodes via the oracle root
    boundary of a 1x1 grid, and interior coordinates via oracle_leaf_nodes."""
    Xb, Yb, NX, NY = orc.root_boundary(x0, x0 + hx, y0, y0 + hy, 1, 1, p)
    X, Y = orc.leaf_nodes(x0, x0 + hx, y0, y0 + hy, 1, 1, p)
    return Xb, Yb, NX, NY, inputs.interior_of(p, X[0]), inputs.interior_of(p, Y[0])


@pytest.mark.parametrize("hx,hy", [(0.25, 0.25), (0.25, 0.5), (0.4, 0.15)])
@pytest.mark.parametrize("p,kappa,eta", [(6, 3.0, 3.0), (10, 7.0, 2.0 - 1.0j), (16, 20.0, 20.0)])
def test_leaf_polynomial_exact(orc, p, kappa, eta, hx, hy):
    """u = Psi t + Y s reproduces a degree-(p-1) polynomial exactly for any
    kappa, c, eta (PAPER.md:433-445 Remark; collocation is exact on it) — on square AND
    rectangular leaves (h_x != h_y: a swapped 2/h_x, 2/h_y scaling of D_x, D_y fails here)."""
    x0, y0 = 0.3, -0.2
    P = Poly2D(p - 1, (x0, x0 + hx, y0, y0 + hy), seed=p)
    X, Y = orc.leaf_nodes(x0, x0 + hx, y0, y0 + hy, 1, 1, p)
    c = (1 + 0.3 * np.sin(3 * X[0]) * np.cos(2 * Y[0])).astype(complex)
    lf = orc.leaf(p, hx, hy, kappa, eta, c)
    Xb, Yb, NX, NY, Xi, Yi = leaf_boundary_geometry(p, x0, y0, hx, hy, orc)
    dn = NX * P.val(Xb, Yb, dx=1) + NY * P.val(Xb, Yb, dy=1)
    t = dn + 1j * eta * P.val(Xb, Yb)
    ci = inputs.interior_of(p, c)
    s = -(P.val(Xi, Yi, dx=2) + P.val(Xi, Yi, dy=2)) - kappa ** 2 * ci * P.val(Xi, Yi)
    u = lf["Psi"] @ t + lf["Y"] @ s
    exact = np.concatenate([P.val(Xb, Yb), P.val(Xi, Yi)])
    assert rel(u, exact) < 1e-10
    # outgoing data g = R t + Gamma s equals du/dn - i eta u
    g = lf["R"] @ t + lf["Gamma"] @ s
    assert rel(g, dn - 1j * eta * P.val(Xb, Yb)) < 1e-9


def test_leaf_disc_structure(orc):
    """Ahat, N, F, G of PAPER.md:328-367 (reading Q1: geometric normals)."""
    p, h, kappa, eta = 7, 0.5, 2.0, 1.5
    c = np.linspace(1, 2, p * p).astype(complex)
    d = orc.leaf_disc(p, h, h, kappa, eta, c)
    x, D = orc.cheb(p)
    D = D * (2 / h)
    # Ahat = -(D^2 (x) I) - (I (x) D^2) - kappa^2 diag(c)  with x fastest
    D2 = D @ D
    Ahat = -(np.kron(np.eye(p), D2) + np.kron(D2, np.eye(p))) - kappa ** 2 * np.diag(c)
    assert rel(d["Ahat"], Ahat) < 1e-13
    nb = 4 * p - 8
    E = np.zeros((nb, p * p - 4))
    E[:, :nb] = np.eye(nb)
    assert rel(d["F"] - d["N"], 1j * eta * E) < 1e-15
    assert rel(d["G"] - d["N"], -1j * eta * E) < 1e-15
    # S row 0 is node (ix=1, iy=0): N row = -dy at that node
    q = p - 2
    xs = np.linspace(0.1, 0.2, p)
    # N applied to nodal values of f(x,y)=y gives -1 (S), 0 (E), +1 (N), 0 (W)
    X, Y = orc.leaf_nodes(0, h, 0, h, 1, 1, p)
    f = inputs.interior_of(p, Y[0])
    Xb, Yb, *_ = orc.root_boundary(0, h, 0, h, 1, 1, p)
    vals = np.concatenate([Yb, f])
    Nf = d["N"] @ vals
    assert np.allclose(Nf[:q], -1) and np.allclose(Nf[q:2 * q], 0)
    assert np.allclose(Nf[2 * q:3 * q], 1) and np.allclose(Nf[3 * q:], 0)
    del xs


def test_leaf_identities(orc):
    """B Psi = [I;0], B Y = [0;I] (eqs 8, 10); R = I - 2 i eta Psi_b and
    Gamma = -2 i eta Y_b (follow from F Psi = I, F Y = 0, G = F - 2 i eta E)."""
    p, h, kappa, eta = 12, 0.1, 30.0, 30.0
    rng = np.random.default_rng(5)
    c = (1 + 0.2 * rng.random(p * p)).astype(complex)
    lf = orc.leaf(p, h, h, kappa, eta, c)
    nb, nt = 4 * p - 8, p * p - 4
    Binv = np.hstack([lf["Psi"], lf["Y"]])
    assert np.max(np.abs(lf["B"] @ Binv - np.eye(nt))) < 1e-10
    assert rel(lf["R"], np.eye(nb) - 2j * eta * lf["Psi"][:nb]) < 1e-11
    assert rel(lf["Gamma"], -2j * eta * lf["Y"][:nb]) < 1e-11


@pytest.mark.parametrize("p", [8, 12, 16])
def test_leaf_R_unitary_conj(orc, p):
    """Real kappa, c, eta: R conj(R) = I and |lambda(R)| = 1 (reading Q9)."""
    h = 2.5 / 10.0
    kappa = 10.0
    X, Y = orc.leaf_nodes(0, h, 0, h, 1, 1, p)
    c = (1 + 0.3 * np.exp(-((X[0] - 0.1) ** 2 + (Y[0] - 0.1) ** 2) / 0.01)).astype(complex)
    R = orc.leaf(p, h, h, kappa, kappa, c)["R"]
    assert np.max(np.abs(R @ R.conj() - np.eye(R.shape[0]))) < 1e-10
    lam = np.linalg.eigvals(R)
    assert np.max(np.abs(np.abs(lam) - 1)) < 1e-10


def harmonic(k, X, Y):
    z = (X + 1j * Y) ** k
    dzx = k * (X + 1j * Y) ** (k - 1) if k else 0 * X
    return z, dzx, 1j * dzx      # P, dP/dx, dP/dy for P = (x + i y)^k


@pytest.mark.parametrize("nx,ny", [(1, 1), (2, 1), (2, 2), (4, 2)])
def test_kappa0_harmonic_polynomials(orc, nx, ny):
    """kappa = 0: R maps f = dP/dn + i eta P to g = dP/dn - i eta P for harmonic
    polynomials of degree <= p-1 (exact at every box); R 1 = -1."""
    p, eta = 8, 1.3
    x0, x1, y0, y1 = 0.0, 0.5 * nx, 0.0, 0.5 * ny
    c = np.ones((nx * ny, p * p), complex)
    O = orc.Oracle(x0, x1, y0, y1, nx, ny, p, 0.0, eta, c)
    R = O.R(1)
    Xb, Yb, NX, NY = orc.root_boundary(x0, x1, y0, y1, nx, ny, p)
    for k in range(p):
        P, Px, Py = harmonic(k, Xb - 0.1, Yb + 0.2)
        dn = NX * Px + NY * Py
        assert rel(R @ (dn + 1j * eta * P), dn - 1j * eta * P) < 1e-10
    assert np.allclose(R @ np.ones(R.shape[0]), -np.ones(R.shape[0]), atol=1e-10)


# ---------------------------------------------------------------------------
# Merge: brute-force global collocation, decoupling, explicit vs action forms
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("nx,ny,p,kappa,ar", [(2, 1, 10, 7.0, 1.0), (1, 2, 8, 2.0, 1.0), (2, 2, 8, 9.0, 1.0),
                                             (4, 4, 6, 5.0, 1.0), (2, 1, 8, 6.0, 2.0), (2, 2, 6, 4.0, 0.5)])
def test_tree_vs_global_dense(orc, nx, ny, p, kappa, ar):
    """Merged root R and the solve u equal the dense global collocation system
     — independent elimination of the same equations; ar = h_y / h_x
    (rectangular leaves in the last two cases)."""
    x0, x1, y0, y1 = 0.0, 0.3 * nx, 0.0, 0.3 * ny * ar
    X, Y = orc.leaf_nodes(x0, x1, y0, y1, nx, ny, p)
    c = (1 - 0.4 * np.exp(-((X - 0.2) ** 2 + (Y - 0.25) ** 2) / 0.02)).astype(complex)
    eta = kappa * (1 + 0.5j)
    rng = np.random.default_rng(nx * 10 + ny)
    nrhs, ni = 2, (p - 2) ** 2
    nbr = 2 * (nx + ny) * (p - 2)
    s = rng.standard_normal((nrhs, nx * ny, ni)) + 1j * rng.standard_normal((nrhs, nx * ny, ni))
    t = rng.standard_normal((nrhs, nbr)) + 1j * rng.standard_normal((nrhs, nbr))
    O = orc.Oracle(x0, x1, y0, y1, nx, ny, p, kappa, eta, c)
    u = O.solve(s, t)
    ug, Rg = orc.global_dense(x0, x1, y0, y1, nx, ny, p, kappa, eta, c, s, t, want_R=True)
    assert rel(O.R(1), Rg) < 1e-9
    assert rel(u, ug) < 1e-9


def test_merge_decoupled(orc):
    """R33^a = R33^b = 0 => W = I, Phi^a = [0 | -R32b], Phi^b = [-R31a | 0]
    (SPEC.md:280); the diagonal blocks of R^tau are R11a, R22b and the coupling
    blocks are -R13a R32b and -R23b R31a."""
    p = 6
    q, nb = p - 2, 4 * p - 8
    rng = np.random.default_rng(3)
    Ra = rng.standard_normal((nb, nb)) + 1j * rng.standard_normal((nb, nb))
    Rb = rng.standard_normal((nb, nb)) + 1j * rng.standard_normal((nb, nb))
    # vertical merge: I3 = alpha E = [q, 2q), beta W = [3q, 4q)
    Ia3, Ib3 = np.arange(q, 2 * q), np.arange(3 * q, 4 * q)
    Ra[np.ix_(Ia3, Ia3)] = 0
    Rb[np.ix_(Ib3, Ib3)] = 0
    m = orc.merge(p, 1, 1, 1, Ra, Rb)
    assert np.allclose(m["Winv"], np.eye(q))
    I1 = np.r_[0:q, 2 * q:4 * q]
    I2 = np.arange(0, 3 * q)
    assert np.allclose(m["PhiA"][:, :3 * q], 0)
    assert np.allclose(m["PhiA"][:, 3 * q:], -Rb[np.ix_(Ib3, I2)])
    assert np.allclose(m["PhiB"][:, :3 * q], -Ra[np.ix_(Ia3, I1)])
    assert np.allclose(m["PhiB"][:, 3 * q:], 0)
    # R^tau canonical: parent = [aS, bS, bE, aN, bN, aW]
    aS, aN, aW = np.r_[0:q], np.r_[2 * q:3 * q], np.r_[3 * q:4 * q]
    bS, bE, bN = np.r_[0:q], np.r_[q:2 * q], np.r_[2 * q:3 * q]
    Rt = m["Rtau"]
    pa = np.r_[0:q, 3 * q:4 * q, 5 * q:6 * q]          # parent positions of aS, aN, aW
    pb = np.r_[q:2 * q, 2 * q:3 * q, 4 * q:5 * q]      # parent positions of bS, bE, bN
    assert np.allclose(Rt[np.ix_(pa, pa)], Ra[np.ix_(np.r_[aS, aN, aW], np.r_[aS, aN, aW])])
    assert np.allclose(Rt[np.ix_(pb, pb)], Rb[np.ix_(np.r_[bS, bE, bN], np.r_[bS, bE, bN])])
    # off-diagonal blocks carry the coupling through Phi: R13a (-R32b), R23b (-R31a)
    Ia1 = np.r_[aS, aN, aW]
    Ib2 = np.r_[bS, bE, bN]
    assert np.allclose(Rt[np.ix_(pa, pb)], -Ra[np.ix_(Ia1, Ia3)] @ Rb[np.ix_(Ib3, Ib2)])
    assert np.allclose(Rt[np.ix_(pb, pa)], -Rb[np.ix_(Ib2, Ib3)] @ Ra[np.ix_(Ia3, Ia1)])


@pytest.mark.parametrize("vertical", [1, 0])
def test_merge_explicit_vs_action(orc, vertical):
    """Upsilon / Gamma^tau explicit (Alg. 1 lines 9, 11, 13) equal their
    matvec actions, Phi^b long form equals
    -[R31a|0] - R33a Phi^a, and the interface equations (11)-(12) hold."""
    p = 8
    q, nb = p - 2, 4 * p - 8
    h = 0.2
    rng = np.random.default_rng(7 + vertical)
    Rs = []
    for k in range(2):
        X, Y = orc.leaf_nodes(0, h, 0, h, 1, 1, p)
        c = (1 + 0.3 * rng.random(p * p)).astype(complex)
        Rs.append(orc.leaf(p, h, h, 12.0, 12.0 + 3j, c)["R"])
    Ra, Rb = Rs
    m = orc.merge(p, 1, 1, vertical, Ra, Rb)
    if vertical:
        Ia3, Ib3 = np.arange(q, 2 * q), np.arange(3 * q, 4 * q)
        I1, I2 = np.r_[0:q, 2 * q:4 * q], np.arange(0, 3 * q)
    else:
        Ia3, Ib3 = np.arange(2 * q, 3 * q), np.arange(0, q)
        I1, I2 = np.r_[0:2 * q, 3 * q:4 * q], np.arange(q, 4 * q)
    R33a, R33b = Ra[np.ix_(Ia3, Ia3)], Rb[np.ix_(Ib3, Ib3)]
    R31a, R13a = Ra[np.ix_(Ia3, I1)], Ra[np.ix_(I1, Ia3)]
    R32b, R23b = Rb[np.ix_(Ib3, I2)], Rb[np.ix_(I2, Ib3)]
    R11a, R22b = Ra[np.ix_(I1, I1)], Rb[np.ix_(I2, I2)]
    Wi = m["Winv"]
    assert np.max(np.abs((np.eye(q) - R33b @ R33a) @ Wi - np.eye(q))) < 1e-10
    h3 = rng.standard_normal(2 * q) + 1j * rng.standard_normal(2 * q)
    ha3, hb3 = h3[:q], h3[q:]
    tta = Wi @ (R33b @ ha3 - hb3)
    ttb = -ha3 - R33a @ tta
    assert rel(m["UpsA"] @ h3, tta) < 1e-12
    assert rel(m["UpsB"] @ h3, ttb) < 1e-12
    assert rel(m["GammaT"] @ h3, np.concatenate([R13a @ tta, R23b @ ttb])) < 1e-12
    nbt = len(I1) + len(I2)
    PhiB_short = -np.hstack([R31a, np.zeros((q, len(I2)))]) - R33a @ m["PhiA"]
    assert rel(m["PhiB"], PhiB_short) < 1e-12
    # interface equations for random exterior data
    t12 = rng.standard_normal(nbt) + 1j * rng.standard_normal(nbt)
    t3a, t3b = m["PhiA"] @ t12, m["PhiB"] @ t12
    g3a = R31a @ t12[:len(I1)] + R33a @ t3a
    g3b = Rb[np.ix_(Ib3, I2)] @ t12[len(I1):] + R33b @ t3b
    assert rel(t3a, -g3b) < 1e-11 and rel(g3a, -t3b) < 1e-11
    del R11a, R22b, R32b


def test_merged_R_unitary_conj(orc):
    """Merged R of a real problem satisfies R conj(R) = I (reading Q9)."""
    p, nx, ny = 8, 2, 2
    X, Y = orc.leaf_nodes(0, 1, 0, 1, nx, ny, p)
    c = (1 + 0.5 * np.exp(-((X - 0.4) ** 2 + (Y - 0.6) ** 2) / 0.05)).astype(complex)
    O = orc.Oracle(0, 1, 0, 1, nx, ny, p, 5.0, 5.0, c, keep_all_R=True)
    for box in [1, 2, 3, 4]:
        R = O.R(box)
        assert np.max(np.abs(R @ R.conj() - np.eye(R.shape[0]))) < 1e-10


# ---------------------------------------------------------------------------
# Whole solver: zero data, polynomial exactness, plane-wave spectral decay
# ---------------------------------------------------------------------------
def test_zero_data_zero_solution(orc):
    p, nx, ny = 6, 2, 2
    c = np.ones((nx * ny, p * p), complex)
    O = orc.Oracle(0, 1, 0, 1, nx, ny, p, 4.0, 4.0, c)
    u = O.solve(np.zeros((1, 4, 16)), np.zeros((1, 2 * 4 * 4)))
    assert np.all(u == 0)


@pytest.mark.parametrize("nx,ny,p,y1", [(4, 4, 8, None), (2, 4, 6, None), (4, 2, 10, None),
                                         (2, 1, 8, 1.0), (4, 2, 6, 1.0), (1, 2, 10, 0.6)])
def test_tree_polynomial_exact(orc, nx, ny, p, y1):
    """Algorithm 2 reproduces a global polynomial of degree p-1 exactly,
    including the upward pass (Y, Gamma, Upsilon, Gamma^tau) — SURVEY §8(c).  The last three
    cases have rectangular leaves (2x1 grid on the unit square: 0.5 x 1 leaves; 4x2: 0.25 x 0.5;
    1x2 on [0,1]x[0,0.6]: 1 x 0.3), so a swapped h_x / h_y anywhere in the tree fails."""
    x0, x1, y0 = 0.0, 1.0, 0.0
    y1 = 1.0 * ny / nx if y1 is None else y1
    kappa, eta = 6.0, 6.0 + 2j
    P = Poly2D(p - 1, (x0, x1, y0, y1), seed=11)
    X, Y = orc.leaf_nodes(x0, x1, y0, y1, nx, ny, p)
    c = (1 + 0.25 * np.cos(3 * X) * np.sin(2 * Y)).astype(complex)
    Xi, Yi = inputs.interior_of(p, X), inputs.interior_of(p, Y)
    ci = inputs.interior_of(p, c)
    s = -(P.val(Xi, Yi, dx=2) + P.val(Xi, Yi, dy=2)) - kappa ** 2 * ci * P.val(Xi, Yi)
    Xb, Yb, NX, NY = orc.root_boundary(x0, x1, y0, y1, nx, ny, p)
    t = NX * P.val(Xb, Yb, dx=1) + NY * P.val(Xb, Yb, dy=1) + 1j * eta * P.val(Xb, Yb)
    O = orc.Oracle(x0, x1, y0, y1, nx, ny, p, kappa, eta, c)
    u = O.solve(s[None], t[None])[0]
    # exact values at every leaf's [Ib; Ii] nodes
    err = 0.0
    scale = np.max(np.abs(P.val(X, Y)))
    for l in range(nx * ny):
        lx, ly = l % nx, l // nx
        hx, hy = (x1 - x0) / nx, (y1 - y0) / ny
        bx, by, *_ = orc.root_boundary(x0 + lx * hx, x0 + (lx + 1) * hx, y0 + ly * hy, y0 + (ly + 1) * hy, 1,
                                       1, p)
        ex = np.concatenate([P.val(bx, by), P.val(Xi[l], Yi[l])])
        err = max(err, np.max(np.abs(u[l] - ex)) / scale)
    assert err < 1e-9


def test_plane_wave_spectral_decay(orc):
    """C1 geometry (4x4 leaves, kappa=10, c=1, s=0, plane wave): error decays
    spectrally in p (SURVEY §8(c) plane-wave pin; BASELINE config 1)."""
    cfg = inputs.CONFIGS[1]
    errs = []
    for p in [6, 8, 10, 12]:
        X, Y = orc.leaf_nodes(0, 1, 0, 1, 4, 4, p)
        Xb, Yb, NX, NY = orc.root_boundary(0, 1, 0, 1, 4, 4, p)
        t = inputs.plane_wave_robin(cfg.kappa, cfg.eta, cfg.theta, Xb, Yb, NX, NY)
        O = orc.Oracle(0, 1, 0, 1, 4, 4, p, cfg.kappa, cfg.eta, np.ones((16, p * p)))
        u = O.solve(np.zeros((1, 16, (p - 2) ** 2)), t[None])[0]
        err = 0.0
        for l in range(16):
            lx, ly = l % 4, l // 4
            bx, by, *_ = orc.root_boundary(lx / 4, (lx + 1) / 4, ly / 4, (ly + 1) / 4, 1, 1, p)
            ex = np.concatenate([inputs.plane_wave(cfg.kappa, cfg.theta, bx, by),
                                 inputs.plane_wave(cfg.kappa, cfg.theta, inputs.interior_of(p, X[l]),
                                                   inputs.interior_of(p, Y[l]))])
            err = max(err, np.max(np.abs(u[l] - ex)))
        errs.append(err)
    assert all(b < a / 10 for a, b in zip(errs, errs[1:])), errs
    assert errs[1] < 1e-4 and errs[-1] < 1e-8, errs


def test_shared_edge_duplicates_agree(orc):
    """Both copies of an interface node carry the same u (reading Q15)."""
    p, nx, ny = 8, 2, 1
    c = np.ones((2, p * p), complex)
    rng = np.random.default_rng(0)
    O = orc.Oracle(0, 2, 0, 1, nx, ny, p, 5.0, 5.0, c)
    t = rng.standard_normal((1, 2 * 3 * (p - 2))) + 0j
    s = rng.standard_normal((1, 2, (p - 2) ** 2)) + 0j
    u = O.solve(s, t)[0]
    q = p - 2
    # leaf 0 east edge = leaf 1 west edge
    assert rel(u[0][q:2 * q], u[1][3 * q:4 * q]) < 1e-10


def test_oracle_threading_bitwise(orc):
    """The oracle's row/column-parallel loops (matmul rows, LU row updates, LU-solve column
    blocks) keep every element's operation order: results are BITWISE equal for 1 and many
    threads, so parallelising the checker changes no expected value."""
    rng = np.random.default_rng(12)
    A = rng.standard_normal((300, 280)) + 1j * rng.standard_normal((300, 280))
    B = rng.standard_normal((280, 310)) + 1j * rng.standard_normal((280, 310))
    M = rng.standard_normal((420, 420)) + 1j * rng.standard_normal((420, 420))
    nthr = orc.set_threads(0)
    try:
        orc.set_threads(1)
        C1, I1 = orc.matmul(A, B), orc.invert(M)
        p, nb = 8, 4 * 8 - 8
        X, Y = orc.leaf_nodes(0, 4, 0, 2, 4, 2, p)
        Ra = orc.Oracle(0, 2, 0, 2, 2, 2, p, 5.0, 5.0 + 1j, np.ones((4, p * p), complex)).R(1)
        Rb = orc.Oracle(2, 4, 0, 2, 2, 2, p, 5.0, 5.0 + 1j, np.ones((4, p * p), complex)).R(1)
        m1 = orc.merge(p, 2, 2, 1, Ra, Rb)["Rtau"]
        orc.set_threads(max(nthr, 4))
        C2, I2 = orc.matmul(A, B), orc.invert(M)
        m2 = orc.merge(p, 2, 2, 1, Ra, Rb)["Rtau"]
    finally:
        orc.set_threads(nthr)
    assert np.array_equal(C1, C2) and np.array_equal(I1, I2) and np.array_equal(m1, m2)
    del X, Y, nb
