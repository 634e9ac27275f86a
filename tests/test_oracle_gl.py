"""Pins for oracle/gl.py (Gauss-Legendre boundary representation) against
closed forms and exactness on polynomials (not against itself)."""
import numpy as np
import pytest

from oracle import gl


@pytest.mark.parametrize("q", [2, 4, 6, 7, 14])
def test_gl_quadrature_exact_to_degree_2q_minus_1(q):
    """int_{-1}^{1} x^k dx = 2/(k+1) (k even), 0 (k odd), exact for k < 2q: pins nodes AND weights."""
    xi, w = gl.gl_nodes_weights(q)
    for k in range(2 * q):
        exact = 2.0 / (k + 1) if k % 2 == 0 else 0.0
        assert abs(np.sum(w * xi ** k) - exact) < 1e-13
    # not exact at degree 2q (the rule has exactly degree 2q - 1)
    assert abs(np.sum(w * xi ** (2 * q)) - 2.0 / (2 * q + 1)) > 1e-10
    assert np.all(np.diff(xi) > 0) and np.all(np.abs(xi) < 1)


@pytest.mark.parametrize("p", [4, 6, 8, 16])
def test_gl_to_cheb_exact_on_polynomials(p):
    """P f(xi) = f(x_cheb) for every polynomial of degree < q (and only those, up to rounding)."""
    q = p - 2
    rng = np.random.default_rng(p)
    xi, _ = gl.gl_nodes_weights(q)
    xc = gl.cheb_edge_nodes(p)
    assert np.allclose(xc, -np.cos(np.pi * np.arange(1, p - 1) / (p - 1)), atol=1e-15)
    P = gl.gl_to_cheb(p)
    coef = rng.standard_normal(q) + 1j * rng.standard_normal(q)
    f = lambda x: np.polyval(coef, x)
    assert np.max(np.abs(P @ f(xi) - f(xc))) < 1e-12
    hi = lambda x: x ** q
    assert np.max(np.abs(P @ hi(xi) - hi(xc))) > 1e-6
    # interpolation reproduces constants: rows sum to one
    assert np.allclose(P.sum(axis=1), 1.0, atol=1e-13)


def test_t_to_cheb_segments_and_root_nodes():
    """Per-segment transform; GL root nodes lie on the same segments as the Chebyshev ones."""
    p, nx, ny = 6, 2, 4
    q = p - 2
    X, Y, NX, NY = gl.root_boundary_gl(0.0, 1.0, 0.0, 2.0, nx, ny, p)
    Xc, Yc, NXc, NYc = gl.root_boundary(0.0, 1.0, 0.0, 2.0, nx, ny, p)
    assert X.shape == Xc.shape == (2 * (nx + ny) * q,)
    assert np.array_equal(NX, NXc) and np.array_equal(NY, NYc)
    for s in range(2 * (nx + ny)):   # same segment: same bounding interval, interior points
        sl = slice(s * q, (s + 1) * q)
        for A, B in ((X, Xc), (Y, Yc)):
            lo, hi = min(A[sl].min(), B[sl].min()), max(A[sl].max(), B[sl].max())
            assert hi - lo <= 0.5 + 1e-12
    # a function linear on the boundary is reproduced at the Chebyshev nodes
    t_gl = (2 + 1j) * X - 3 * Y + 0.5
    t_c = gl.t_to_cheb(p, t_gl[None, :])[0]
    assert np.max(np.abs(t_c - ((2 + 1j) * Xc - 3 * Yc + 0.5))) < 1e-12


# ---------------------------------------------------------------------------
# Gauss-Legendre EDGE representation (q independent of p): oracle.Oracle(..., qe=q)
# ---------------------------------------------------------------------------
import oracle as orc  # noqa: E402
from paper_1812_07167_b200 import inputs  # noqa: E402


@pytest.mark.parametrize("p,q", [(8, 3), (10, 5), (16, 9), (6, 4)])
def test_cheb_to_gl_exact_on_polynomials(p, q):
    """Q g(x_cheb) = g(xi) for polynomials of degree <= p - 3 (the Chebyshev interpolant is exact);
    P f(xi) = f(x_cheb) for degree < q; for q = p - 2, Q = P^{-1}."""
    rng = np.random.default_rng(p * 31 + q)
    xi, _ = gl.gl_nodes_weights(q)
    xc = gl.cheb_edge_nodes(p)
    Q, P = gl.cheb_to_gl(p, q), gl.gl_to_cheb(p, q)
    assert Q.shape == (q, p - 2) and P.shape == (p - 2, q)
    cg = rng.standard_normal(p - 2)
    assert np.max(np.abs(Q @ np.polyval(cg, xc) - np.polyval(cg, xi))) < 1e-11
    cf = rng.standard_normal(q)
    assert np.max(np.abs(P @ np.polyval(cf, xi) - np.polyval(cf, xc))) < 1e-11
    if q < p - 2:
        assert np.max(np.abs(P @ xi ** q - xc ** q)) > 1e-6   # degree q is NOT reproduced
    Qs, Ps = gl.cheb_to_gl(p), gl.gl_to_cheb(p)
    assert np.max(np.abs(Qs @ Ps - np.eye(p - 2))) < 1e-11


def _poly_case(nx, ny, p, qe, deg, kappa=6.0, eta=6.0 + 2j):
    """Relative max error of the GL-edge oracle solve against a global polynomial of degree deg
    (per variable) with its body load and GL-sampled Robin data (pins like test_tree_polynomial_exact)."""
    from test_oracle_pins import Poly2D
    x0, x1, y0, y1 = 0.0, 1.0, 0.0, 1.0 * ny / nx
    P = Poly2D(deg, (x0, x1, y0, y1), seed=11)
    X, Y = orc.leaf_nodes(x0, x1, y0, y1, nx, ny, p)
    c = (1 + 0.25 * np.cos(3 * X) * np.sin(2 * Y)).astype(complex)
    Xi, Yi = inputs.interior_of(p, X), inputs.interior_of(p, Y)
    s = -(P.val(Xi, Yi, dx=2) + P.val(Xi, Yi, dy=2)) - kappa ** 2 * inputs.interior_of(p, c) * P.val(Xi, Yi)
    Xb, Yb, NX, NY = gl.root_boundary_gl(x0, x1, y0, y1, nx, ny, p, q=qe)
    t = NX * P.val(Xb, Yb, dx=1) + NY * P.val(Xb, Yb, dy=1) + 1j * eta * P.val(Xb, Yb)
    O = orc.Oracle(x0, x1, y0, y1, nx, ny, p, kappa, eta, c, qe=qe)
    u = O.solve(s[None], t[None])[0]
    scale, err = np.max(np.abs(P.val(X, Y))), 0.0
    hx, hy = (x1 - x0) / nx, (y1 - y0) / ny
    for l in range(nx * ny):
        lx, ly = l % nx, l // nx
        bx, by, *_ = orc.root_boundary(x0 + lx * hx, x0 + (lx + 1) * hx, y0 + ly * hy, y0 + (ly + 1) * hy, 1, 1, p)
        ex = np.concatenate([P.val(bx, by), P.val(Xi[l], Yi[l])])
        err = max(err, np.max(np.abs(u[l] - ex)) / scale)
    return err


@pytest.mark.parametrize("nx,ny,p,qe", [(2, 2, 10, 5), (4, 2, 8, 4), (2, 1, 10, 3), (4, 4, 8, 6)])
def test_gl_edges_polynomial_exact_below_q(nx, ny, p, qe):
    """With q GL nodes per leaf edge the interface data of a polynomial of degree <= q - 1 is
    represented exactly, so the whole tree reproduces it to rounding; one degree more is NOT
    reproduced (the representation really truncates at q: a tree that ignored q, or mixed up
    P and Q, fails one of the two).  Rectangular leaves in the 4x2 and 2x1 cases."""
    assert _poly_case(nx, ny, p, qe, qe - 1) < 1e-11
    assert _poly_case(nx, ny, p, qe, qe) > 1e-7


@pytest.mark.parametrize("nx,ny,p", [(2, 2, 8), (4, 2, 6)])
def test_gl_edges_full_q_equals_chebyshev_change_of_basis(nx, ny, p):
    """q = p - 2: the GL-edge tree is the Chebyshev tree in another basis on every edge
    (R_gl = P^{-1} R P per leaf, and the merges commute with the block-diagonal change of basis),
    so u equals the Chebyshev oracle's u for t converted by P segment by segment (t_to_cheb), and
    the root R_gl = Pblk^{-1} R_cheb Pblk."""
    kappa, eta = 9.0, 9.0 - 1j
    x1, y1 = 1.0, 1.0 * ny / nx
    X, Y = orc.leaf_nodes(0, x1, 0, y1, nx, ny, p)
    c = (1 + 0.3 * np.sin(2 * X) * np.cos(3 * Y)).astype(complex)
    rng = np.random.default_rng(5)
    q = p - 2
    nb = 2 * (nx + ny) * q
    s = rng.standard_normal((2, nx * ny, q * q)) + 1j * rng.standard_normal((2, nx * ny, q * q))
    t = rng.standard_normal((2, nb)) + 1j * rng.standard_normal((2, nb))
    Og = orc.Oracle(0, x1, 0, y1, nx, ny, p, kappa, eta, c, qe=q)
    Oc = orc.Oracle(0, x1, 0, y1, nx, ny, p, kappa, eta, c)
    ug, uc = Og.solve(s, t), Oc.solve(s, gl.t_to_cheb(p, t))
    assert np.max(np.abs(ug - uc)) / np.max(np.abs(uc)) < 1e-11
    Pb = np.kron(np.eye(nb // q), gl.gl_to_cheb(p))
    Rg, Rc = Og.R(1), Oc.R(1)
    assert np.max(np.abs(Pb @ Rg - Rc @ Pb)) / np.max(np.abs(Rc)) < 1e-11


def test_gl_edges_plane_wave_converges_in_q():
    """C1 geometry at p = 12: the plane-wave error falls as q grows toward p - 2 and is
    spectrally small at q = p - 2 (same as the Chebyshev scheme)."""
    cfg = inputs.CONFIGS[1]
    p, errs = 12, []
    X, Y = orc.leaf_nodes(0, 1, 0, 1, 4, 4, p)
    for qe in (4, 6, 8, 10):
        Xb, Yb, NX, NY = gl.root_boundary_gl(0, 1, 0, 1, 4, 4, p, q=qe)
        t = inputs.plane_wave_robin(cfg.kappa, cfg.eta, cfg.theta, Xb, Yb, NX, NY)
        O = orc.Oracle(0, 1, 0, 1, 4, 4, p, cfg.kappa, cfg.eta, np.ones((16, p * p)), qe=qe)
        u = O.solve(np.zeros((1, 16, (p - 2) ** 2)), t[None])[0]
        ex = np.stack([inputs.plane_wave(cfg.kappa, cfg.theta, inputs.interior_of(p, X[l]),
                                         inputs.interior_of(p, Y[l])) for l in range(16)])
        errs.append(np.max(np.abs(u[:, 4 * (p - 2):] - ex)))
    assert all(b < a / 5 for a, b in zip(errs, errs[1:])), errs
    assert errs[-1] < 1e-6, errs
