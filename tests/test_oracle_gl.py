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
