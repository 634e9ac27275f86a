"""Gauss-Legendre boundary representation — TEST INFRASTRUCTURE.

Only tests/ may import this module (see oracle/__init__.py).  Plain numpy, fp64.

The paper's scheme (reading Q8) samples the boundary at the q = p - 2
corner-free Chebyshev-Lobatto nodes of each leaf edge.  The configs name q Gauss-Legendre nodes
per leaf edge instead; with q = p - 2 that is a change of basis on every leaf-edge segment: the
boundary data t given at the q Gauss-Legendre nodes of a segment determine the degree-(q-1)
polynomial through them, which is sampled at the segment's q Chebyshev nodes.  Beyond the paper
(it only cites the ItI representation): built from first principles.
"""
import numpy as np

from .oracle import cheb, root_boundary


def gl_nodes_weights(q):
    """Gauss-Legendre nodes (ascending) and weights on [-1, 1] by the Golub-Welsch eigenproblem of
    the Jacobi matrix of the Legendre recurrence, off-diagonal k / sqrt(4k^2 - 1)."""
    k = np.arange(1, q)
    J = np.diag(k / np.sqrt(4.0 * k * k - 1.0), 1)
    J = J + J.T
    lam, V = np.linalg.eigh(J)
    return lam, 2.0 * V[0, :] ** 2


def cheb_edge_nodes(p):
    """The q = p - 2 interior Chebyshev-Lobatto nodes of an edge (reference [-1, 1])."""
    x, _ = cheb(p)
    return x[1:-1]


def lagrange_matrix(src, dst):
    """L[j, g] = l_g(dst_j), l_g the Lagrange basis polynomial of the nodes src (product formula)."""
    L = np.ones((len(dst), len(src)))
    for g in range(len(src)):
        for m in range(len(src)):
            if m != g:
                L[:, g] *= (dst - src[m]) / (src[g] - src[m])
    return L


def gl_to_cheb(p, q=None):
    """(p - 2) x q matrix taking segment samples at the q Gauss-Legendre nodes (the degree-(q-1)
    polynomial through them) to the segment's p - 2 Chebyshev nodes; q defaults to p - 2."""
    xi, _ = gl_nodes_weights(p - 2 if q is None else q)
    return lagrange_matrix(xi, cheb_edge_nodes(p))


def cheb_to_gl(p, q=None):
    """q x (p - 2) matrix taking segment samples at the p - 2 Chebyshev nodes (the degree-(p-3)
    polynomial through them) to the segment's q Gauss-Legendre nodes (GL edge representation,
    the outgoing side).  For q = p - 2 it is the inverse of gl_to_cheb(p)."""
    xi, _ = gl_nodes_weights(p - 2 if q is None else q)
    return lagrange_matrix(cheb_edge_nodes(p), xi)


def t_to_cheb(p, t_gl):
    """Root boundary data [..., nseg * q] at Gauss-Legendre nodes -> at Chebyshev nodes (per
    segment of q nodes, canonical order)."""
    q = p - 2
    P = gl_to_cheb(p)
    t = np.asarray(t_gl)
    seg = t.reshape(t.shape[:-1] + (t.shape[-1] // q, q))
    return np.einsum("jg,...sg->...sj", P, seg).reshape(t.shape)


def root_boundary_gl(x0, x1, y0, y1, nx, ny, p, q=None):
    """Root boundary Gauss-Legendre node coordinates and outward normals, canonical order [S, E, N,
    W], each leaf-edge segment in increasing coordinate (the segment layout of root_boundary);
    q nodes per segment (default p - 2)."""
    q = p - 2 if q is None else q
    xi, _ = gl_nodes_weights(q)
    hx, hy = (x1 - x0) / nx, (y1 - y0) / ny
    X, Y, NX, NY = [], [], [], []
    for side in range(4):
        nseg = nx if side in (0, 2) else ny
        for l in range(nseg):
            for g in range(q):
                if side in (0, 2):
                    X.append(x0 + l * hx + (1 + xi[g]) * 0.5 * hx)
                    Y.append(y0 if side == 0 else y1)
                    NX.append(0.0)
                    NY.append(-1.0 if side == 0 else 1.0)
                else:
                    X.append(x1 if side == 1 else x0)
                    Y.append(y0 + l * hy + (1 + xi[g]) * 0.5 * hy)
                    NX.append(1.0 if side == 1 else -1.0)
                    NY.append(0.0)
    return np.array(X), np.array(Y), np.array(NX), np.array(NY)


__all__ = ["gl_nodes_weights", "cheb_edge_nodes", "lagrange_matrix", "gl_to_cheb", "cheb_to_gl", "t_to_cheb",
           "root_boundary_gl",
           "root_boundary"]
