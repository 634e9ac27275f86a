"""ctypes binding for liboracle.so (test infrastructure; see __init__.py)."""
import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "hps_oracle.cpp")
_lib = None

__all__ = [
    "build", "lib", "cheb", "leaf_nodes", "root_boundary", "leaf", "leaf_disc", "merge", "box_rect", "tree_info",
    "Oracle", "global_dense", "invert", "matmul", "set_threads",
]


def set_threads(n):
    """Set the OpenMP thread count of the oracle (0: query); returns the count in effect."""
    return lib().oracle_set_threads(int(n))


def build(force=False):
    """Compile liboracle.so with g++ (-O2, OpenMP, no BLAS)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        subprocess.check_call(
            ["g++", "-O2", "-fopenmp", "-fcx-limited-range", "-fPIC", "-shared", "-std=c++17",
             "-o", _SO, _SRC])
    return _SO


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_SO)
        vp, i32, i64, d, dp = C.c_void_p, C.c_int, C.c_int64, C.c_double, C.c_void_p
        L.oracle_cheb.argtypes = [i32, dp, dp]
        L.oracle_leaf_nodes.argtypes = [d, d, d, d, i32, i32, i32, dp, dp]
        L.oracle_root_boundary.argtypes = [d, d, d, d, i32, i32, i32, dp, dp, dp, dp]
        L.oracle_leaf.argtypes = [i32, d, d, d, d, d, dp, dp, dp, dp, dp, dp]
        L.oracle_leaf_disc.argtypes = [i32, d, d, d, d, d, dp, dp, dp, dp, dp]
        L.oracle_merge.argtypes = [i32, i32, i32, i32, dp, dp, dp, dp, dp, dp, dp, dp, dp]
        L.oracle_box_rect.argtypes = [i32, i32, i64] + [C.POINTER(C.c_int)] * 5
        L.oracle_tree_info.argtypes = [i32, i32, i32, C.POINTER(i64), C.POINTER(i32)]
        L.oracle_build.argtypes = [d, d, d, d, i32, i32, i32, d, d, d, dp, i32]
        L.oracle_build.restype = vp
        L.oracle_build_gl.argtypes = [d, d, d, d, i32, i32, i32, i32, dp, dp, d, d, d, dp, i32]
        L.oracle_build_gl.restype = vp
        L.oracle_solve.argtypes = [vp, i32, dp, dp, dp]
        L.oracle_box_nb.argtypes = [vp, i64]
        L.oracle_box_nb.restype = i64
        L.oracle_export_R.argtypes = [vp, i64, dp]
        L.oracle_export_leaf.argtypes = [vp, i64, dp, dp]
        L.oracle_leaf_box.argtypes = [vp, i32, i32]
        L.oracle_leaf_box.restype = i64
        L.oracle_free.argtypes = [vp]
        L.oracle_build_seconds.argtypes = [vp]
        L.oracle_build_seconds.restype = d
        L.oracle_solve_seconds.argtypes = [vp]
        L.oracle_solve_seconds.restype = d
        L.oracle_global_dense.argtypes = [d, d, d, d, i32, i32, i32, d, d, d, dp, i32, dp, dp, dp, dp]
        L.oracle_invert.argtypes = [i32, dp, dp]
        L.oracle_matmul.argtypes = [i32, i32, i32, dp, dp, dp]
        L.oracle_set_threads.argtypes = [i32]
        L.oracle_last_error.restype = C.c_char_p
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data


def _c(a):
    return np.ascontiguousarray(a, dtype=np.complex128)


def _check(rc, what):
    if rc != 0:
        raise RuntimeError(f"{what} failed rc={rc}: {lib().oracle_last_error().decode()}")


def cheb(p):
    x = np.zeros(p)
    D = np.zeros((p, p))
    _check(lib().oracle_cheb(p, _p(x), _p(D)), "oracle_cheb")
    return x, D


def leaf_nodes(x0, x1, y0, y1, nx, ny, p):
    """Node coordinates [nleaf natural][p*p] (x fastest)."""
    X = np.zeros((nx * ny, p * p))
    Y = np.zeros((nx * ny, p * p))
    _check(lib().oracle_leaf_nodes(x0, x1, y0, y1, nx, ny, p, _p(X), _p(Y)), "oracle_leaf_nodes")
    return X, Y


def root_boundary(x0, x1, y0, y1, nx, ny, p):
    """Root boundary node coordinates and outward normals, canonical order."""
    n = 2 * (nx + ny) * (p - 2)
    X, Y, NX, NY = (np.zeros(n) for _ in range(4))
    _check(lib().oracle_root_boundary(x0, x1, y0, y1, nx, ny, p, _p(X), _p(Y), _p(NX), _p(NY)),
           "oracle_root_boundary")
    return X, Y, NX, NY


def leaf(p, hx, hy, kappa, eta, c):
    """Leaf operators dict(Psi, Y, R, Gamma, B) for one leaf; c: (p*p,) complex."""
    nb, ni, nt = 4 * p - 8, (p - 2) ** 2, p * p - 4
    out = dict(Psi=np.zeros((nt, nb), complex), Y=np.zeros((nt, ni), complex),
               R=np.zeros((nb, nb), complex), Gamma=np.zeros((nb, ni), complex),
               B=np.zeros((nt, nt), complex))
    c = _c(c)
    eta = complex(eta)
    _check(lib().oracle_leaf(p, hx, hy, kappa, eta.real, eta.imag, _p(c), _p(out["Psi"]), _p(out["Y"]),
                             _p(out["R"]), _p(out["Gamma"]), _p(out["B"])), "oracle_leaf")
    return out


def leaf_disc(p, hx, hy, kappa, eta, c):
    nb, nt = 4 * p - 8, p * p - 4
    out = dict(Ahat=np.zeros((p * p, p * p), complex), N=np.zeros((nb, nt), complex),
               F=np.zeros((nb, nt), complex), G=np.zeros((nb, nt), complex))
    c = _c(c)
    eta = complex(eta)
    _check(lib().oracle_leaf_disc(p, hx, hy, kappa, eta.real, eta.imag, _p(c), _p(out["Ahat"]), _p(out["N"]),
                                  _p(out["F"]), _p(out["G"])), "oracle_leaf_disc")
    return out


def merge(p, cnx, cny, vertical, Ra, Rb, q=None):
    """Standalone merge of two congruent children (cnx x cny leaves each); q boundary nodes per
    leaf edge (default p - 2; the merge sees only the edge node count)."""
    q = p - 2 if q is None else q
    p = q + 2
    nba = 2 * (cnx + cny) * q
    n3 = (cny if vertical else cnx) * q
    ntau = 2 * (nba - n3)
    out = dict(Rtau=np.zeros((ntau, ntau), complex), PhiA=np.zeros((n3, ntau), complex),
               PhiB=np.zeros((n3, ntau), complex), Winv=np.zeros((n3, n3), complex),
               UpsA=np.zeros((n3, 2 * n3), complex), UpsB=np.zeros((n3, 2 * n3), complex),
               GammaT=np.zeros((ntau, 2 * n3), complex))
    Ra, Rb = _c(Ra), _c(Rb)
    _check(lib().oracle_merge(p, cnx, cny, int(vertical), _p(Ra), _p(Rb), _p(out["Rtau"]), _p(out["PhiA"]),
                              _p(out["PhiB"]), _p(out["Winv"]), _p(out["UpsA"]), _p(out["UpsB"]),
                              _p(out["GammaT"])), "oracle_merge")
    return out


def box_rect(nx, ny, box):
    """(i0, i1, j0, j1, vertical) of a heap box (vertical = -1 for a leaf)."""
    v = [C.c_int() for _ in range(5)]
    _check(lib().oracle_box_rect(nx, ny, box, *[C.byref(x) for x in v]), "oracle_box_rect")
    return tuple(x.value for x in v)


def tree_info(nx, ny, p=4):
    nb = C.c_int64()
    d = C.c_int()
    lib().oracle_tree_info(nx, ny, p, C.byref(nb), C.byref(d))
    return nb.value, d.value


class Oracle:
    """Algorithm 1 build + Algorithm 2 solve on host cores."""

    def __init__(self, x0, x1, y0, y1, nx, ny, p, kappa, eta, c, keep_all_R=False, qe=None):
        """qe: None for the paper's p - 2 Chebyshev nodes per leaf edge; an int for the
        Gauss-Legendre edge representation with qe nodes per edge (oracle/gl.py maps; t of solve()
        is then given at the root's GL nodes, gl.root_boundary_gl(..., q=qe))."""
        self.nx, self.ny, self.p = nx, ny, p
        self.ne = p - 2 if qe is None else qe
        c = _c(c).reshape(nx * ny, p * p)
        eta = complex(eta)
        if qe is None:
            self.h = lib().oracle_build(x0, x1, y0, y1, nx, ny, p, kappa, eta.real, eta.imag, _p(c),
                                        int(keep_all_R))
        else:
            from . import gl
            P = np.ascontiguousarray(gl.gl_to_cheb(p, qe), dtype=np.float64)
            Q = np.ascontiguousarray(gl.cheb_to_gl(p, qe), dtype=np.float64)
            self.h = lib().oracle_build_gl(x0, x1, y0, y1, nx, ny, p, int(qe), _p(P), _p(Q), kappa, eta.real,
                                           eta.imag, _p(c), int(keep_all_R))
        if not self.h:
            raise RuntimeError("oracle_build failed: " + lib().oracle_last_error().decode())

    @property
    def build_seconds(self):
        return lib().oracle_build_seconds(self.h)

    @property
    def solve_seconds(self):
        return lib().oracle_solve_seconds(self.h)

    def solve(self, s, t):
        p, nleaf = self.p, self.nx * self.ny
        s = _c(s)
        t = _c(t)
        nrhs = t.shape[0]
        u = np.zeros((nrhs, nleaf, p * p - 4), complex)
        _check(lib().oracle_solve(self.h, nrhs, _p(s), _p(t), _p(u)), "oracle_solve")
        return u

    def nb(self, box):
        return lib().oracle_box_nb(self.h, box)

    def R(self, box=1):
        n = self.nb(box)
        out = np.zeros((n, n), complex)
        _check(lib().oracle_export_R(self.h, box, _p(out)), "oracle_export_R")
        return out

    def leaf_box(self, ix, iy):
        return lib().oracle_leaf_box(self.h, ix, iy)

    def leaf_ops(self, box):
        p = self.p
        Psi = np.zeros((p * p - 4, 4 * self.ne), complex)
        Y = np.zeros((p * p - 4, (p - 2) ** 2), complex)
        _check(lib().oracle_export_leaf(self.h, box, _p(Psi), _p(Y)), "oracle_export_leaf")
        return Psi, Y

    def close(self):
        if self.h:
            lib().oracle_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def global_dense(x0, x1, y0, y1, nx, ny, p, kappa, eta, c, s=None, t=None, want_R=False):
    nleaf, nt, q = nx * ny, p * p - 4, p - 2
    nbr = 2 * (nx + ny) * q
    c = _c(c).reshape(nleaf, p * p)
    eta = complex(eta)
    nrhs = 0 if t is None else t.shape[0]
    u = np.zeros((nrhs, nleaf, nt), complex) if nrhs else None
    R = np.zeros((nbr, nbr), complex) if want_R else None
    s = None if s is None else _c(s)
    t = None if t is None else _c(t)
    _check(lib().oracle_global_dense(x0, x1, y0, y1, nx, ny, p, kappa, eta.real, eta.imag, _p(c), nrhs, _p(s),
                                     _p(t), _p(u), _p(R)), "oracle_global_dense")
    return u, R


def invert(A):
    A = _c(A)
    out = np.zeros_like(A)
    _check(lib().oracle_invert(A.shape[0], _p(A), _p(out)), "oracle_invert")
    return out


def matmul(A, B):
    A, B = _c(A), _c(B)
    out = np.zeros((A.shape[0], B.shape[1]), complex)
    lib().oracle_matmul(A.shape[0], A.shape[1], B.shape[1], _p(A), _p(B), _p(out))
    return out
