"""Host-side checks of the C-ABI (no GPU): the library loads, exports every symbol the
header declares, validates arguments, and its host geometry matches the oracle's."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import __graft_entry__
from paper_1812_07167_b200 import hps

HDR = os.path.join(os.path.dirname(os.path.dirname(__file__)), "include", "hps.h")


@pytest.fixture(scope="module")
def L():
    __graft_entry__.build()
    return hps.lib()


def test_exports_every_declared_symbol(L):
    decl = set(re.findall(r"\b(hps_[a-z_A-Z0-9]+)\s*\(", open(HDR).read()))
    assert decl, "no declarations parsed"
    for name in decl:
        assert hasattr(L, name), name
    assert set(hps.SYMBOLS) == decl


@pytest.mark.parametrize("nx,ny,p", [(1, 1, 4), (2, 4, 8), (4, 4, 16)])
def test_geometry_matches_oracle(L, orc, nx, ny, p):
    g = hps.grid(0.1, 0.9, -0.3, 0.5, nx, ny)
    X, Y = hps.leaf_nodes(g, p)
    Xo, Yo = orc.leaf_nodes(0.1, 0.9, -0.3, 0.5, nx, ny, p)
    assert np.max(np.abs(X - Xo)) < 1e-15 and np.max(np.abs(Y - Yo)) < 1e-15
    b = hps.root_boundary_nodes(g, p)
    bo = orc.root_boundary(0.1, 0.9, -0.3, 0.5, nx, ny, p)
    for u, v in zip(b, bo):
        assert np.max(np.abs(u - v)) < 1e-15


@pytest.mark.parametrize("nx,ny,p", [(1, 1, 4), (2, 4, 8), (4, 2, 16)])
def test_gl_boundary_nodes_match_oracle(L, orc, nx, ny, p):
    """hps_boundary_nodes_gl (Newton on P_q) vs oracle.gl (Golub-Welsch), boundary_basis 1."""
    from oracle import gl
    g = hps.grid(0.1, 0.9, -0.3, 0.5, nx, ny)
    b = hps.root_boundary_nodes(g, p, basis=1)
    bo = gl.root_boundary_gl(0.1, 0.9, -0.3, 0.5, nx, ny, p)
    for u, v in zip(b, bo):
        assert np.max(np.abs(u - v)) < 1e-14


@pytest.mark.parametrize("nx,ny,q", [(1, 1, 2), (2, 4, 5), (4, 2, 9)])
def test_glq_boundary_nodes_match_oracle(L, orc, nx, ny, q):
    """hps_boundary_nodes_glq (q nodes per segment, boundary_basis 2) vs oracle.gl at 1e-14."""
    from oracle import gl
    g = hps.grid(0.1, 0.9, -0.3, 0.5, nx, ny)
    b = hps.root_boundary_nodes(g, 16, basis=2, q=q)
    bo = gl.root_boundary_gl(0.1, 0.9, -0.3, 0.5, nx, ny, 16, q=q)
    assert b[0].shape == (2 * (nx + ny) * q,)
    for u, v in zip(b, bo):
        assert np.max(np.abs(u - v)) < 1e-14


def _build_rc(L, **kw):
    args = dict(g=hps.grid(0, 1, 0, 1, 2, 2), p=8, q=6, kappa=1.0, eta=hps.hps_c128(1.0, 0.0))
    args.update(kw)
    c = np.ones(4 * 64, complex)
    h = C.c_void_p()
    rc = L.hps_build(C.byref(args["g"]), args["p"], args["q"], args["kappa"], args["eta"], c.ctypes.data, None,
                     C.byref(h))
    return rc, h


def test_argument_validation(L):
    # all rejected before any device work
    assert _build_rc(L, q=5)[0] == -1
    assert _build_rc(L, p=3, q=1)[0] == -1
    assert _build_rc(L, g=hps.grid(0, 1, 0, 1, 3, 2))[0] == -1
    assert _build_rc(L, g=hps.grid(1, 0, 0, 1, 2, 2))[0] == -1
    assert _build_rc(L, kappa=-1.0)[0] == -1
    assert _build_rc(L, eta=hps.hps_c128(0.0, 1.0))[0] == -1
    rc, h = _build_rc(L, q=5)
    assert not h.value
    assert b"q must equal" in L.hps_last_error()
    L.hps_free(None)   # no-op


def test_option_validation_and_small_calls(L):
    """leaf_mode outside 0..3, boundary_basis outside 0..2 and a q outside [2, p - 2] for the
    Gauss-Legendre edge representation (q != p - 2 for the others) are rejected before any device
    work; hps_leaf_path(NULL) is HPS_EINVAL; hps_release_cache with nothing cached returns 0."""
    g = hps.grid(0, 1, 0, 1, 2, 2)
    c = np.ones(4 * 64, complex)
    for lm, bb, q, msg in ((4, 0, 6, b"leaf_mode"), (0, 3, 6, b"boundary_basis"), (-1, 0, 6, b"leaf_mode"),
                           (0, 2, 7, b"[2, p - 2]"), (0, 2, 1, b"[2, p - 2]"), (0, 0, 5, b"p - 2"),
                           (0, 1, 4, b"p - 2")):
        opts = hps.hps_opts(1, 0, -1, 0, 0, lm, bb)
        h = C.c_void_p()
        rc = L.hps_build(C.byref(g), 8, q, 1.0, hps.hps_c128(1.0, 0.0), c.ctypes.data, C.byref(opts), C.byref(h))
        assert rc == -1 and not h.value
        assert msg in L.hps_last_error()
    assert L.hps_leaf_path(None) == -1
    assert L.hps_release_cache() == 0


def test_rep_actions_match_survey_table():
    """Representative actions per level (Table 1): the leaf interior inverse and the
    merge interface inverses; sizes and box counts as SURVEY 8(a)'s per-level table (C3, C5)."""
    from paper_1812_07167_b200 import hps
    g = hps.grid(0.0, 1.0, 0.0, 1.0, 128, 128)
    ra = hps.rep_actions(g, 16)
    assert ra[0] == (196, 16384)
    assert [n for n, _ in ra[1:]] == [14, 28, 28, 56, 56, 112, 112, 224, 224, 448, 448, 896, 896, 1792]
    assert [b for _, b in ra[1:]] == [2 ** d for d in range(13, -1, -1)]
    g5 = hps.grid(0.0, 2.0, 0.0, 1.0, 1024, 512)
    ra5 = hps.rep_actions(g5, 16)
    assert len(ra5) == 20 and ra5[0] == (196, 524288)
    assert [n for n, _ in ra5[-5:]] == [1792, 3584, 3584, 7168, 7168]   # levels 15-19


def test_opts_layout_and_multi_gpu_validation(L):
    """hps_opts matches include/hps.h (7 int32 + n_gpus, then nccl_comm, stream, comm pointers);
    the multi-GPU fields are validated before any device work: n_gpus > 1 without a communicator,
    and a non-power-of-two virtual group, are HPS_EINVAL."""
    assert C.sizeof(hps.hps_opts) == 8 * 4 + 3 * C.sizeof(C.c_void_p)
    assert hps.hps_opts.nccl_comm.offset == 32 and hps.hps_opts.comm.offset == 48
    g = hps.grid(0, 1, 0, 1, 2, 2)
    c = np.ones(4 * 64, complex)
    opts = hps.hps_opts(1, 0, -1, 0, 0, 0, 0, 2, None, None, None)
    h = C.c_void_p()
    rc = L.hps_build(C.byref(g), 8, 6, 1.0, hps.hps_c128(1.0, 0.0), c.ctypes.data, C.byref(opts), C.byref(h))
    assert rc == -1 and not h.value and b"communicator" in L.hps_last_error()
    grp = C.c_void_p()
    assert L.hps_vcomm_create(3, C.byref(grp)) == -1
    assert L.hps_sync(None) == -1


def test_debug_knobs_roundtrip(L):
    """Knobs are set only through hps_debug_set (no environment); -1 restores the default;
    unknown names are HPS_EINVAL."""
    v = C.c_int()
    assert L.hps_debug_get(b"nat_min", C.byref(v)) == 0 and v.value == 200
    assert L.hps_debug_set(b"nat_min", 14) == 0
    assert L.hps_debug_get(b"nat_min", C.byref(v)) == 0 and v.value == 14
    assert L.hps_debug_set(b"nat_min", -1) == 0
    assert L.hps_debug_get(b"nat_min", C.byref(v)) == 0 and v.value == 200
    assert L.hps_debug_set(b"no_such_knob", 1) == -1
    src = open(os.path.join(os.path.dirname(hps.__file__), "csrc", "hps_api.cu")).read()
    for f in ("zgj.cu", "zgemm.cu", "leaf.cu", "leaf_real.cu", "comm.cu"):
        src += open(os.path.join(os.path.dirname(hps.__file__), "csrc", f)).read()
    assert "getenv" not in src


def test_solve_actions_small_tree(L):
    """Solve-stage representative actions (host only) for 4 x 2 leaves at p = 6, nrhs = 3: the
    leaf products and five products per merge level with n3, n1, n_tau of the split schedule
    (written out by hand: q = 4; d = 0 parent 4x2 -> 2x2 children, vertical, n3 = 8, n_b = 32;
    d = 1 parent 2x2 -> 1x2, vertical, n3 = 8, n_b = 24; d = 2 parent 1x2 -> 1x1, horizontal,
    n3 = 4, n_b = 16)."""
    g = hps.grid(0, 2, 0, 1, 4, 2)
    acts = hps.solve_actions(g, 6, 3)
    got = [(a["level"], a["kind"], a["M"], a["N"], a["K"], a["batch"], a["cin"]) for a in acts]
    exp = [(-1, 0, 32, 3, 16, 8, 0), (-1, 1, 32, 3, 16, 8, 1), (-1, 1, 32, 3, 16, 8, 0)]
    for d, n3, nbc in ((0, 8, 32), (1, 8, 24), (2, 4, 16)):
        n1 = nbc - n3
        exp += [(d, 2, n3, 3, n3, 2 ** d, 1), (d, 3, n3, 3, n3, 2 ** d, 0), (d, 4, n1, 3, n3, 2 ** d, 1),
                (d, 5, n3, 3, 2 * n1, 2 ** d, 1), (d, 5, n3, 3, 2 * n1, 2 ** d, 0)]
    assert got == exp
    # the W^{-1} actions are the merge levels' representative inverses of hps_rep_actions
    ra = hps.rep_actions(g, 6)
    w = [(a["M"], a["batch"]) for a in acts if a["kind"] == 3]
    assert sorted(w) == sorted((n, nb) for n, nb in ra[1:])
    assert L.hps_solve_actions(C.byref(g), 6, 3, 2, np.zeros(14, np.int32).ctypes.data) == -1   # maxn too small
    assert L.hps_build_actions(C.byref(g), 6, 1, 2, np.zeros(14, np.int32).ctypes.data) == -1


def test_build_actions_small_tree(L):
    """The build's batched products per merge level (host only) for the 4 x 2 tree at p = 6 (same
    hand-written n3 / n_b as test_solve_actions_small_tree); no R^tau product at the root with
    keep_root_R = 0; no W^{-1} update product below the natural-order range (n3 < 200)."""
    g = hps.grid(0, 2, 0, 1, 4, 2)
    for keep in (1, 0):
        acts = hps.build_actions(g, 6, keep_root_R=bool(keep))
        got = [(a["level"], a["kind"], a["M"], a["N"], a["K"], a["batch"], a["cin"]) for a in acts]
        exp = []
        for d, n3, nbc in ((0, 8, 32), (1, 8, 24), (2, 4, 16)):
            n1, np_ = nbc - n3, 2 ** d
            exp += [(d, 6, n3, n1, n3, np_, 0), (d, 7, n3, n3, n3, np_, 0), (d, 8, n3, 2 * n1, n3, np_, 0),
                    (d, 10, n3, 2 * n1, n3, np_, 1)]
            if d > 0 or keep:
                exp.append((d, 9, n1, 2 * n1, n3, np_, 1))
        assert got == exp
    # C4's root level carries the 64-wide block-step update of its natural-order W^{-1}
    c4 = hps.build_actions(hps.grid(0, 1, 0, 1, 256, 256), 16)
    assert (0, 11, 3584, 3520, 64, 1, 1) in [(a["level"], a["kind"], a["M"], a["N"], a["K"], a["batch"], a["cin"])
                                             for a in c4]
