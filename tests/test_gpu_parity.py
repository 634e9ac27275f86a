"""CUDA path (through the C-ABI) vs the CPU oracle, element by element, on seeded inputs.

Tolerance: 1e-9 relative max-norm on R and u (BASELINE.json north_star)."""
import numpy as np
import pytest

import oracle
from paper_1812_07167_b200 import hps, inputs

pytestmark = pytest.mark.gpu
TOL = 1e-9


def rel(a, b):
    return np.max(np.abs(a - b)) / np.max(np.abs(b))


@pytest.fixture(scope="module", autouse=True)
def _built():
    import torch
    assert torch.cuda.is_available()
    import __graft_entry__
    __graft_entry__.build()


def problem(nx, ny, p, kappa, eta, x1=1.0, y1=1.0, nrhs=2, seed=0):
    g = hps.grid(0.0, x1, 0.0, y1, nx, ny)
    X, Y = hps.leaf_nodes(g, p)
    c = (1 + 0.3 * np.exp(-((X - 0.4 * x1) ** 2 + (Y - 0.6 * y1) ** 2) / 0.05)).astype(complex)
    rng = np.random.default_rng(seed)
    ni, nbr = (p - 2) ** 2, 2 * (nx + ny) * (p - 2)
    s = rng.standard_normal((nrhs, nx * ny, ni)) + 1j * rng.standard_normal((nrhs, nx * ny, ni))
    t = rng.standard_normal((nrhs, nbr)) + 1j * rng.standard_normal((nrhs, nbr))
    return g, c, s, t


@pytest.mark.parametrize("leaf_mode", [0, 1, 2])
@pytest.mark.parametrize("p", [4, 8, 10, 12, 14, 16, 20])
def test_leaf_parity(p, leaf_mode):
    """Leaf operators Psi, Y and the leaf R on non-square leaves (h_x = 0.5, h_y = 1): p = 12, 14,
    16 run the warp-specialised inverse (n_i = 100, 144, 196) with the fused epilogue in mode 0."""
    g, c, s, t = problem(2, 1, p, 7.0, 7.0 + 1j)
    S = hps.Solver(g, p, 7.0, 7.0 + 1j, c, keep_all_R=True, leaf_mode=leaf_mode)
    for leaf in range(2):
        Psi, Y = S.leaf_ops(leaf)
        lo = oracle.leaf(p, 0.5, 1.0, 7.0, 7.0 + 1j, c[leaf])
        assert rel(Psi, lo["Psi"]) < TOL
        assert rel(Y, lo["Y"]) < TOL
        assert rel(S.R(2 + leaf), lo["R"]) < TOL


@pytest.mark.parametrize("p", [4, 6, 8, 10, 12, 13, 14, 16])
def test_leaf_parity_real_elimination(p):
    """leaf_mode 3 (real A_ii^{-1} + complex n_b x n_b complement) on non-square
    leaves (h_x = 0.5, h_y = 1): Psi, Y and the leaf R vs the oracle's full-B inverse.  kappa = 4
    keeps kappa^2 c (<= 20.8) below the lowest Dirichlet eigenvalue of the leaf (49.3)."""
    g, c, s, t = problem(2, 1, p, 4.0, 4.0 + 1j)
    S = hps.Solver(g, p, 4.0, 4.0 + 1j, c, keep_all_R=True, leaf_mode=3)
    assert S.leaf_path() == 3
    for leaf in range(2):
        Psi, Y = S.leaf_ops(leaf)
        lo = oracle.leaf(p, 0.5, 1.0, 4.0, 4.0 + 1j, c[leaf])
        assert rel(Psi, lo["Psi"]) < TOL
        assert rel(Y, lo["Y"]) < TOL
        assert rel(S.R(2 + leaf), lo["R"]) < TOL


def test_leaf_real_elimination_pivoted():
    """leaf_mode 3 between the first two interior resonances (kappa^2 c in [50, 65], eigenvalues
    49.3 and 78.9): the gate fails, so the real Gauss-Jordan runs with partial pivoting."""
    kappa = np.sqrt(50.0)
    g, c, s, t = problem(2, 1, 12, kappa, kappa + 1j)
    S = hps.Solver(g, 12, kappa, kappa + 1j, c, keep_all_R=True, leaf_mode=3)
    assert S.leaf_path() == 3
    for leaf in range(2):
        Psi, Y = S.leaf_ops(leaf)
        lo = oracle.leaf(12, 0.5, 1.0, kappa, kappa + 1j, c[leaf])
        assert rel(Psi, lo["Psi"]) < TOL
        assert rel(Y, lo["Y"]) < TOL
        assert rel(S.R(2 + leaf), lo["R"]) < TOL


def test_leaf_real_elimination_forced_pivoting():
    """Fault injection (hps_debug_set): both real eliminations (A_ii and Sigma) with partial
    pivoting from the first step, and the natural-order attempt failing its first pivot check
    (the in-kernel fallback redoes the leaf with partial pivoting)."""
    g, c, s, t = problem(2, 1, 16, 4.0, 4.0 + 1j)
    lo = oracle.leaf(16, 0.5, 1.0, 4.0, 4.0 + 1j, c[1])
    for knobs in ({"dgj_pivot": 1}, {"dgj_force_bad": 1}):
        with hps.debug_knobs(**knobs):
            S = hps.Solver(g, 16, 4.0, 4.0 + 1j, c, keep_all_R=True, leaf_mode=3)
            Psi, Y = S.leaf_ops(1)
            err = max(rel(Psi, lo["Psi"]), rel(Y, lo["Y"]), rel(S.R(3), lo["R"]))
            S.close()
        assert err < TOL, (knobs, err)


def test_natural_order_merge_inverses_all_levels():
    """nat_min = 14: every merge W with n3 >= 14 is inverted in natural order —
    every box's R and u vs the oracle, complex eta included; second pass with every natural-order
    attempt forced to fail its pivot check (the pivoted fallback), third with the relative pivot
    threshold at 1.0 (any pivot smaller than its original diagonal falls back); the last two with
    the 64-wide block steps (nat_bb_min = 20: every W with n3 >= 20, one to two blocks)."""
    for knobs in ({"nat_min": 14}, {"nat_min": 14, "nat_force_fail": 1}, {"nat_min": 14, "nat_pivot_rel": 10000},
                  {"nat_min": 14, "nat_bb_min": 20}, {"nat_min": 14, "nat_bb_min": 20, "nat_pivot_rel": 10000}):
        worst = 0.0
        with hps.debug_knobs(**knobs):
            for nx, ny, p, kappa, eta in [(4, 4, 8, 9.0, 9.0 - 2j), (8, 4, 6, 9.0, 9.0), (4, 8, 10, 20.0, 20.0)]:
                g, c, s, t = problem(nx, ny, p, kappa, eta, x1=1.0, y1=ny / nx)
                S = hps.Solver(g, p, kappa, eta, c, keep_all_R=True)
                O = oracle.Oracle(0.0, 1.0, 0.0, ny / nx, nx, ny, p, kappa, eta, c, keep_all_R=True)
                for box in range(1, 2 * nx * ny):
                    worst = max(worst, rel(S.R(box), O.R(box)))
                worst = max(worst, rel(S.solve(s, t), O.solve(s, t)))
                S.close()
        assert worst < TOL, (knobs, worst)


def test_natural_blocked_lookahead():
    """Block-step natural-order W^{-1} (nat_bb_min = 100: the top levels' n3 = 160, three 64-wide
    blocks) with and without lookahead (knob nat_lookahead: block q + 1's D^{-1} and T on
    a second stream beside block q's trailing update): the same arithmetic per entry,
    so root R and u are bitwise equal; both vs the oracle."""
    nx, ny, p, kappa, eta = 16, 16, 12, 20.0, 20.0 + 2j
    g, c, s, t = problem(nx, ny, p, kappa, eta, nrhs=2)
    res = {}
    for la in (0, 1):
        with hps.debug_knobs(nat_min=100, nat_bb_min=100, nat_lookahead=la):
            S = hps.Solver(g, p, kappa, eta, c)
            res[la] = (S.R(1), S.solve(s, t), S.launches(0))
            S.close()
    # the lookahead splits each block step's update in two (one more launch per step): it ran
    assert res[1][2] > res[0][2], (res[0][2], res[1][2])
    assert np.array_equal(res[0][0], res[1][0]) and np.array_equal(res[0][1], res[1][1])
    O = oracle.Oracle(0.0, 1.0, 0.0, 1.0, nx, ny, p, kappa, eta, c)
    assert rel(res[1][0], O.R(1)) < TOL and rel(res[1][1], O.solve(s, t)) < TOL


@pytest.mark.parametrize("use_stream", [False, True])
def test_solve_graph_replay(use_stream):
    """Repeated solves with the same device buffers run as one CUDA graph launch from the third call
    on (knob solve_graph): new contents of s and t between the calls, a switch to
    other buffers and back, s = NULL, on the library's own stream and on a caller's torch stream; every
    result bitwise equal to the eager path (solve_graph = 0) and to the oracle at the suite's
    tolerance; the launch count of a replayed solve equals the eager one."""
    import torch
    nx, ny, p, kappa, eta = 8, 4, 8, 9.0, 9.0 - 1j
    g, c, s, t = problem(nx, ny, p, kappa, eta, nrhs=3)
    O = oracle.Oracle(0.0, 1.0, 0.0, 1.0, nx, ny, p, kappa, eta, c)
    d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    st = torch.cuda.Stream() if use_stream else None
    rng = np.random.default_rng(5)
    seq = []
    for k in range(6):
        sk = s * (1 + 0.5 * k) + rng.standard_normal(s.shape)
        tk = t * (1 - 0.3 * k) + 1j * rng.standard_normal(t.shape)
        seq.append((sk, tk))
    res = {}
    for graph in (0, 1):
        with hps.debug_knobs(solve_graph=graph):
            S = hps.Solver(g, p, kappa, eta, d(c), stream=st)
            sd, td = d(s), d(t)
            ud = torch.empty((3, nx * ny, p * p - 4), dtype=torch.complex128, device="cuda")
            s2, t2, u2 = d(s), d(t), torch.empty_like(ud)
            out, launches = [], []
            for k, (sk, tk) in enumerate(seq):
                if k == 4:  # other buffers once (a new key: eager), then back to the captured key (replay)
                    s2.copy_(d(sk))
                    t2.copy_(d(tk))
                    torch.cuda.synchronize()
                    S.solve(s2, t2, u2)
                    S.sync()
                    torch.cuda.synchronize()
                    out.append(u2.cpu().numpy())
                    launches.append(S.launches(1))
                    continue
                sd.copy_(d(sk))
                td.copy_(d(tk))
                torch.cuda.synchronize()
                S.solve(sd, td, ud)
                S.sync()
                torch.cuda.synchronize()
                out.append(ud.cpu().numpy())
                launches.append(S.launches(1))
            for _ in range(3):  # s = NULL, repeated (its own key)
                S.solve(None, td, ud)
                S.sync()
                torch.cuda.synchronize()
            out.append(ud.cpu().numpy())
            launches.append(S.launches(1))
            S.close()
        res[graph] = (out, launches)
    for k, (sk, tk) in enumerate(seq):
        assert rel(res[1][0][k], O.solve(sk, tk)) < TOL
    assert rel(res[1][0][-1], O.solve(np.zeros_like(s), seq[-1][1])) < TOL
    for a, b in zip(res[0][0], res[1][0]):
        assert np.array_equal(a, b)
    assert res[0][1] == res[1][1]


def test_leaf_schur_natural_and_pivoted_paths():
    """The complex interior Schur inverse (leaf_mode 0 with complex c) runs in natural order
    (DESIGN.md 3.12); the seq_pivot knob forces the pivoted path; leaf_panel switches the natural-order
    panels between the step-by-step and the block form; leaf_inplace 0 eliminates in the scratch matrix
    instead of the store's Y_i block; seq_force_bad makes the natural-order elimination fail at step 100
    (after it has overwritten its work matrix), so the pivoted fallback must redo the leaf.  All vs the
    oracle."""
    g, c, s, t = problem(2, 1, 16, 7.0, 7.0 + 1j)
    c = c + 0.05j
    for knobs in ({}, {"seq_pivot": 1}, {"leaf_panel": 1}, {"leaf_panel": 1 - hps.debug_get("leaf_panel")},
                  {"leaf_inplace": 0}, {"seq_force_bad": 1}, {"seq_force_bad": 1, "leaf_inplace": 0},
                  {"leaf_panel": 2}, {"leaf_panel": 2, "seq_force_bad": 1}):
        with hps.debug_knobs(**knobs):
            S = hps.Solver(g, 16, 7.0, 7.0 + 1j, c, keep_all_R=True)
            assert S.leaf_path() == 0
            w = 0.0
            for leaf in range(2):
                Psi, Y = S.leaf_ops(leaf)
                lo = oracle.leaf(16, 0.5, 1.0, 7.0, 7.0 + 1j, c[leaf])
                w = max(w, rel(Psi, lo["Psi"]), rel(Y, lo["Y"]), rel(S.R(2 + leaf), lo["R"]))
            S.close()
        assert w < TOL, (knobs, w)


def test_leaf_path_selection():
    """Auto mode takes the real elimination only for real c below the first interior resonance;
    leaf_mode 3 refuses complex c."""
    g, c, s, t = problem(2, 1, 8, 4.0, 4.0 + 1j)
    assert hps.Solver(g, 8, 4.0, 4.0 + 1j, c).leaf_path() == 3
    # complex Schur path (2: unfused at n_i = 36, below the fused kernels' range)
    assert hps.Solver(g, 8, 7.0, 7.0 + 1j, c).leaf_path() == 2   # 7^2 * 1.3 > 0.9 * 49.3
    cc = c + 1e-3j
    assert hps.Solver(g, 8, 4.0, 4.0 + 1j, cc).leaf_path() == 2
    g16, c16, _, _ = problem(2, 1, 16, 7.0, 7.0 + 1j)
    assert hps.Solver(g16, 16, 7.0, 7.0 + 1j, c16).leaf_path() == 0
    with pytest.raises(Exception):
        hps.Solver(g, 8, 4.0, 4.0 + 1j, cc, leaf_mode=3)


@pytest.mark.parametrize("knobs", [{}, {"dgj_nt": 256}, {"dgj_nt": 256, "dgj_pivot": 1},
                                   {"dgj_nt": 256, "dgj_force_bad": 1}])
def test_leaf_real_batched_p16_many_leaves(knobs):
    """64 leaves at p = 16 on the real path (several CTAs per SM wave), sampled leaves vs oracle; also
    with two 256-thread leaves per SM (dgj_nt), pivoting from the start, and the natural-order
    elimination failing its first check."""
    g, c, s, t = problem(8, 8, 16, 25.0, 25.0 + 3j)
    with hps.debug_knobs(**knobs):
        S = hps.Solver(g, 16, 25.0, 25.0 + 3j, c)
        assert S.leaf_path() == 3
        for leaf in [0, 17, 63]:
            Psi, Y = S.leaf_ops(leaf)
            lo = oracle.leaf(16, 0.125, 0.125, 25.0, 25.0 + 3j, c[leaf])
            assert rel(Psi, lo["Psi"]) < TOL
            assert rel(Y, lo["Y"]) < TOL


@pytest.mark.parametrize("nx,ny,p", [(1, 1, 8), (2, 1, 8), (1, 2, 6), (4, 4, 8), (8, 4, 6), (4, 8, 10)])
def test_every_R_and_u(nx, ny, p):
    kappa, eta = 9.0, 9.0 - 2j
    g, c, s, t = problem(nx, ny, p, kappa, eta, x1=1.0, y1=ny / nx)
    S = hps.Solver(g, p, kappa, eta, c, keep_all_R=True)
    O = oracle.Oracle(0.0, 1.0, 0.0, ny / nx, nx, ny, p, kappa, eta, c, keep_all_R=True)
    for box in range(1, 2 * nx * ny):
        assert rel(S.R(box), O.R(box)) < TOL, box
    u = S.solve(s, t)
    uo = O.solve(s, t)
    assert rel(u, uo) < TOL
    # s = None path (homogeneous: downward sweep only)
    u0 = S.solve(None, t)
    assert rel(u0, O.solve(np.zeros_like(s), t)) < TOL


def test_leaf_parity_batched_p16():
    """16 leaves at p = 16: the batched (fused) interior inversion path, several leaves vs oracle."""
    g, c, s, t = problem(4, 4, 16, 30.0, 30.0 + 3j)
    S = hps.Solver(g, 16, 30.0, 30.0 + 3j, c)
    for leaf in [0, 5, 15]:
        Psi, Y = S.leaf_ops(leaf)
        lo = oracle.leaf(16, 0.25, 0.25, 30.0, 30.0 + 3j, c[leaf])
        assert rel(Psi, lo["Psi"]) < TOL
        assert rel(Y, lo["Y"]) < TOL


def test_config1_plane_wave():
    cfg = inputs.CONFIGS[1]
    g = hps.grid(cfg.x0, cfg.x1, cfg.y0, cfg.y1, cfg.nx, cfg.ny)
    X, Y = hps.leaf_nodes(g, cfg.p)
    c, s, t = inputs.make_inputs(cfg, X, Y, *hps.root_boundary_nodes(g, cfg.p))
    S = hps.Solver(g, cfg.p, cfg.kappa, cfg.eta, c)
    u = S.solve(s, t)
    O = oracle.Oracle(cfg.x0, cfg.x1, cfg.y0, cfg.y1, cfg.nx, cfg.ny, cfg.p, cfg.kappa, cfg.eta, c)
    assert rel(u, O.solve(s, t)) < TOL
    assert rel(S.R(1), O.R(1)) < TOL
    # and the physics: plane wave to the C1 discretisation error (SURVEY: 2.8e-5 at p = 8)
    Xi, Yi = inputs.interior_of(cfg.p, X), inputs.interior_of(cfg.p, Y)
    exact_i = inputs.plane_wave(cfg.kappa, cfg.theta, Xi, Yi)
    assert np.max(np.abs(u[0][:, 4 * (cfg.p - 2):] - exact_i)) < 1e-4


@pytest.mark.parametrize("nx,ny,p", [(2, 2, 8), (4, 2, 12)])
def test_gl_boundary_basis_parity(nx, ny, p):
    """boundary_basis 1: t given at the Gauss-Legendre nodes; u equals the
    oracle's Chebyshev-basis solve of the oracle's own per-segment interpolation of t."""
    from oracle import gl
    kappa, eta = 9.0, 9.0 - 2j
    g, c, s, t = problem(nx, ny, p, kappa, eta, x1=1.0, y1=ny / nx)
    S = hps.Solver(g, p, kappa, eta, c, boundary_basis=1)
    u = S.solve(s, t)
    O = oracle.Oracle(0.0, 1.0, 0.0, ny / nx, nx, ny, p, kappa, eta, c)
    assert rel(u, O.solve(s, gl.t_to_cheb(p, t))) < TOL
    # the same data in the Chebyshev basis gives a different (correctly interpolated) problem
    assert rel(hps.Solver(g, p, kappa, eta, c).solve(s, t), u) > 1e-6


def test_gl_boundary_basis_plane_wave():
    """Plane wave with Robin data sampled at the Gauss-Legendre nodes: same accuracy as at the
    Chebyshev nodes (C1 geometry and discretisation)."""
    cfg = inputs.CONFIGS[1]
    g = hps.grid(cfg.x0, cfg.x1, cfg.y0, cfg.y1, cfg.nx, cfg.ny)
    X, Y = hps.leaf_nodes(g, cfg.p)
    c, s, t = inputs.make_inputs(cfg, X, Y, *hps.root_boundary_nodes(g, cfg.p, basis=1))
    u = hps.Solver(g, cfg.p, cfg.kappa, cfg.eta, c, boundary_basis=1).solve(s, t)
    Xi, Yi = inputs.interior_of(cfg.p, X), inputs.interior_of(cfg.p, Y)
    exact_i = inputs.plane_wave(cfg.kappa, cfg.theta, Xi, Yi)
    assert np.max(np.abs(u[0][:, 4 * (cfg.p - 2):] - exact_i)) < 1e-4


def test_gl_boundary_basis_sharded():
    """Gauss-Legendre root data through the subtree-sharded path (the top handle converts it):
    2 virtual ranks equal the single-handle GL solve."""
    import torch
    from paper_1812_07167_b200 import dist
    kappa, eta, nx, ny, p = 11.0, 11.0 + 2j, 4, 4, 8
    g, c, s, t = problem(nx, ny, p, kappa, eta, nrhs=2)
    u_ref = hps.Solver(g, p, kappa, eta, c, boundary_basis=1).solve(s, t)
    d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()

    def rank_fn(comm):
        rank, world = comm.info()
        sub, i0, j0 = dist.local_block(g, world, rank)
        D = dist.DistributedHPS(comm, g, p, kappa, eta, d(dist.slice_leaves(c, g, sub, i0, j0)), boundary_basis=1)
        u = D.solve(d(dist.slice_leaves(s, g, sub, i0, j0)), d(t)).cpu().numpy()
        D.close()
        return u, (sub, i0, j0)

    for u, (sub, i0, j0) in dist.run_virtual(2, rank_fn):
        assert rel(u, dist.slice_leaves(u_ref, g, sub, i0, j0)) < 1e-11


def gl_problem(nx, ny, p, q, kappa, eta, nrhs=2, seed=3):
    """problem() with root data at the q Gauss-Legendre nodes of every boundary segment."""
    g, c, s, _ = problem(nx, ny, p, kappa, eta, x1=1.0, y1=ny / nx, nrhs=nrhs, seed=seed)
    rng = np.random.default_rng(seed + 100)
    nbr = 2 * (nx + ny) * q
    t = rng.standard_normal((nrhs, nbr)) + 1j * rng.standard_normal((nrhs, nbr))
    return g, c, s, t


@pytest.mark.parametrize("leaf_mode", [0, 1])
@pytest.mark.parametrize("nx,ny,p,q,kappa", [(1, 1, 8, 4, 9.0), (2, 2, 8, 4, 9.0), (4, 2, 10, 5, 9.0),
                                             (4, 4, 16, 9, 9.0), (2, 1, 6, 2, 5.0), (8, 4, 16, 12, 30.0),
                                             (4, 4, 12, 10, 9.0)])
def test_gl_edges_parity(nx, ny, p, q, kappa, leaf_mode):
    """boundary_basis 2, the Gauss-Legendre EDGE representation with q independent of p (SURVEY
    8(f) NEXT-2): every box's R, the leaf Psi Pblk and Y, and u (with and without
    a body load) against the oracle's GL-edge tree (oracle.Oracle(..., qe=q)) at 1e-9.  Leaf mode 0
    covers the real interior elimination (4x4 and finer at kappa = 9) and the complex Schur path
    (1x1, 2x2, and 8x4 at kappa = 30); leaf mode 1 the full-B inverse."""
    eta = kappa - 2j
    g, c, s, t = gl_problem(nx, ny, p, q, kappa, eta)
    S = hps.Solver(g, p, kappa, eta, c, boundary_basis=2, q=q, keep_all_R=True, leaf_mode=leaf_mode)
    O = oracle.Oracle(0.0, 1.0, 0.0, ny / nx, nx, ny, p, kappa, eta, c, keep_all_R=True, qe=q)
    assert rel(S.solve(s, t), O.solve(s, t)) < TOL
    assert rel(S.solve(None, t), O.solve(np.zeros_like(s), t)) < TOL
    nbox, _ = oracle.tree_info(nx, ny)
    for box in range(1, nbox + 1):
        assert S.nb(box) == O.nb(box)
        assert rel(S.R(box), O.R(box)) < TOL, box
    for leaf in (0, nx * ny - 1):
        Psi, Y = S.leaf_ops(leaf)
        Po, Yo = O.leaf_ops(O.leaf_box(leaf % nx, leaf // nx))
        assert Psi.shape == (p * p - 4, 4 * q)
        assert rel(Psi, Po) < TOL and rel(Y, Yo) < TOL


def test_gl_edges_full_q_equals_gl_root_data():
    """q = p - 2: the GL-edge tree (basis 2) and the Chebyshev tree fed GL root data (basis 1)
    solve the same problem in two bases: u agrees to rounding."""
    nx, ny, p, kappa, eta = 4, 4, 10, 12.0, 12.0 + 1j
    g, c, s, t = gl_problem(nx, ny, p, p - 2, kappa, eta)
    u2 = hps.Solver(g, p, kappa, eta, c, boundary_basis=2, q=p - 2).solve(s, t)
    u1 = hps.Solver(g, p, kappa, eta, c, boundary_basis=1).solve(s, t)
    assert rel(u2, u1) < 1e-11


def test_gl_edges_polynomial_exact():
    """A global polynomial of degree q - 1 is reproduced to rounding through the GPU GL-edge tree
    (q = 6 < p - 2 = 10, 8x8 leaves); degree q is not (the representation truncates at q)."""
    from test_oracle_pins import Poly2D
    nx, ny, p, q, kappa, eta = 8, 8, 12, 6, 7.0, 7.0 + 1j
    g = hps.grid(0.0, 1.0, 0.0, 1.0, nx, ny)
    X, Y = hps.leaf_nodes(g, p)
    c = (1 + 0.25 * np.cos(3 * X) * np.sin(2 * Y)).astype(complex)
    Xi, Yi = inputs.interior_of(p, X), inputs.interior_of(p, Y)
    Xb, Yb, NX, NY = hps.root_boundary_nodes(g, p, basis=2, q=q)
    S = hps.Solver(g, p, kappa, eta, c, boundary_basis=2, q=q)
    errs = []
    for deg in (q - 1, q):
        P = Poly2D(deg, (0.0, 1.0, 0.0, 1.0), seed=5)
        s = -(P.val(Xi, Yi, dx=2) + P.val(Xi, Yi, dy=2)) - kappa ** 2 * inputs.interior_of(p, c) * P.val(Xi, Yi)
        t = NX * P.val(Xb, Yb, dx=1) + NY * P.val(Xb, Yb, dy=1) + 1j * eta * P.val(Xb, Yb)
        u = S.solve(s[None], t[None])[0]
        errs.append(np.max(np.abs(u[:, 4 * (p - 2):] - P.val(Xi, Yi))) / np.max(np.abs(P.val(Xi, Yi))))
    assert errs[0] < 1e-11 and errs[1] > 1e-9, errs   # measured 9.6e-14 and 3.1e-8


def test_gl_edges_sharded():
    """GL edges through the subtree-sharded path (4 virtual ranks, group split of the top levels)
    equal the single-GPU GL-edge solve."""
    import torch
    from paper_1812_07167_b200 import dist
    kappa, eta, nx, ny, p, q = 11.0, 11.0 + 2j, 4, 4, 10, 6
    g, c, s, t = gl_problem(nx, ny, p, q, kappa, eta)
    u_ref = hps.Solver(g, p, kappa, eta, c, boundary_basis=2, q=q).solve(s, t)
    d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()

    def rank_fn(comm):
        rank, world = comm.info()
        sub, i0, j0 = dist.local_block(g, world, rank)
        D = dist.DistributedHPS(comm, g, p, kappa, eta, d(dist.slice_leaves(c, g, sub, i0, j0)), boundary_basis=2,
                                q=q)
        u = D.solve(d(dist.slice_leaves(s, g, sub, i0, j0)), d(t)).cpu().numpy()
        D.close()
        return u, (sub, i0, j0)

    for u, (sub, i0, j0) in dist.run_virtual(4, rank_fn):
        assert rel(u, dist.slice_leaves(u_ref, g, sub, i0, j0)) < 1e-11


def test_block_cache_reuse_and_release():
    """Opt-in cache (hps_set_cache_limit): large device blocks (>= 256 MB: the 32x16-leaf store
    here) are parked by hps_free, re-used by the next handle and returned by hps_release_cache /
    a zero limit; without the opt-in nothing is parked.  Results are identical either way."""
    g, c, s, t = problem(32, 16, 16, 20.0, 20.0 + 1j, nrhs=1)
    u = []
    try:
        for k in range(4):
            if k == 1:
                hps.set_cache_limit(64 << 30)
            S = hps.Solver(g, 16, 20.0, 20.0 + 1j, c)
            u.append(S.solve(s, t))
            S.close()
            parked = hps.lib().hps_cache_bytes()
            assert (parked > 0) == (k >= 1), (k, parked)
            if k == 2:
                hps.release_cache()
                assert hps.lib().hps_cache_bytes() == 0
    finally:
        hps.set_cache_limit(0)
    assert hps.lib().hps_cache_bytes() == 0
    assert all(np.array_equal(u[0], x) for x in u[1:])


def test_torch_device_buffers():
    import torch
    g, c, s, t = problem(4, 2, 8, 5.0, 5.0)
    d = lambda a: torch.from_numpy(a).cuda()
    S = hps.Solver(g, 8, 5.0, 5.0, d(c))
    u = S.solve(d(s), d(t)).cpu().numpy()
    O = oracle.Oracle(0, 1, 0, 1, 4, 2, 8, 5.0, 5.0, c)
    assert rel(u, O.solve(s, t)) < TOL


@pytest.mark.parametrize("n,batch", [(14, 300), (20, 2), (33, 3), (60, 400), (100, 5), (196, 7), (196, 40), (252, 2),
                                     (252, 17), (230, 16), (57, 20),
                                     (257, 1), (300, 2), (448, 1), (700, 1), (1100, 1), (4200, 1)])
def test_batched_inverse(n, batch):
    """The Gauss-Jordan kernels (small, register panel, cluster panel) vs the oracle's LU."""
    rng = np.random.default_rng(n)
    A = rng.standard_normal((batch, n, n)) + 1j * rng.standard_normal((batch, n, n))
    A[:, 0, 0] = 0.0    # forces a pivot exchange on the first step
    X = hps.zinv_batched(A)
    if n <= 1500:
        for b in range(min(batch, 2)):
            ref = oracle.invert(A[b])
            assert rel(X[b], ref) < 1e-10 * max(1, n / 100)
    # residual, a property that holds at any size
    assert np.max(np.abs(A[-1] @ X[-1] - np.eye(n))) < 1e-9 * max(1, n / 500)


def test_batched_inverse_singular():
    A = np.zeros((2, 40, 40), complex)
    A[0] = np.eye(40)
    with pytest.raises(hps.HpsError):
        hps.zinv_batched(A)


def _sharded_run(world, g, p, kappa, eta, c, s, t, **kw):
    """Every virtual rank builds and solves its share; returns [(u_local, root R, flops, (sub, i0, j0))]."""
    import torch
    from paper_1812_07167_b200 import dist
    d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()

    def rank_fn(comm):
        rank, w = comm.info()
        sub, i0, j0 = dist.local_block(g, w, rank)
        D = dist.DistributedHPS(comm, g, p, kappa, eta, d(dist.slice_leaves(c, g, sub, i0, j0)), **kw)
        sl = None if s is None else d(dist.slice_leaves(s, g, sub, i0, j0))
        u = D.solve(sl, d(t)).cpu().numpy()
        R = D.root_R() if kw.get("keep_root_R", True) else None
        fl = (D.solver.flops(0), D.solver.flops(1))
        D.close()
        return u, R, fl, (sub, i0, j0)

    return dist.run_virtual(world, rank_fn)


@pytest.mark.parametrize("world,nx,ny,p,eta", [(2, 4, 4, 8, 11.0 + 2j), (4, 8, 4, 6, 11.0), (8, 8, 8, 6, 11.0 - 1j),
                                               (4, 32, 32, 16, 11.0 + 2j), (8, 16, 8, 10, 11.0)])
def test_virtual_ranks_match_single_gpu(world, nx, ny, p, eta):
    """Subtree sharding with the group split of the top levels (inside libhps) on
    `world` virtual ranks of one GPU equals the single-handle build/solve: the gathered root R and
    every rank's u, with and without body load; oracle check on the small grids."""
    from paper_1812_07167_b200 import dist
    kappa = 11.0
    g, c, s, t = problem(nx, ny, p, kappa, eta, x1=1.0, y1=ny / nx, nrhs=3)
    S = hps.Solver(g, p, kappa, eta, c)
    u_ref = S.solve(s, t)
    u0_ref = S.solve(None, t)
    R_ref = S.R(1)
    S.close()
    for u, R, fl, (sub, i0, j0) in _sharded_run(world, g, p, kappa, eta, c, s, t):
        assert rel(R, R_ref) < 1e-12
        assert rel(u, dist.slice_leaves(u_ref, g, sub, i0, j0)) < 1e-12
    for u, R, fl, (sub, i0, j0) in _sharded_run(world, g, p, kappa, eta, c, None, t, keep_root_R=False):
        assert R is None
        assert rel(u, dist.slice_leaves(u0_ref, g, sub, i0, j0)) < 1e-12
    if nx * ny <= 64:
        O = oracle.Oracle(0.0, 1.0, 0.0, ny / nx, nx, ny, p, kappa, eta, c)
        assert rel(u_ref, O.solve(s, t)) < TOL and rel(R_ref, O.R(1)) < TOL


def test_sharded_top_flops_split():
    """The group split divides the top levels' GEMM work: summed over the ranks, the build flops
    of a sharded run equal the single-GPU build flops plus (gs - 1) extra copies of the replicated
    W and W^{-1} (16 n3^3 per rank and level) -- i.e. each rank does 1 / gs of the Phi^a, Phi^b and
    R^tau products (hps_last_flops, algorithmic counts)."""
    nx, ny, p, kappa, eta, world = 16, 16, 8, 9.0, 9.0 + 1j, 8
    g, c, s, t = problem(nx, ny, p, kappa, eta, nrhs=1)
    S = hps.Solver(g, p, kappa, eta, c)
    S.solve(s, t)
    f_single = S.flops(0)
    S.close()
    res = _sharded_run(world, g, p, kappa, eta, c, s, t)
    plan = hps.dist_plan(g, p, world, 0)
    extra = sum((lv["gs"] - 1) * (1 << d) * 16.0 * lv["n3"] ** 3 for d, lv in enumerate(plan))
    f_sum = sum(fl[0] for _, _, fl, _ in res)
    assert abs(f_sum - (f_single + extra)) <= 1e-9 * f_single, (f_sum, f_single, extra)
    # per rank: the same work up to the first half of X = [R33b R31a | -R32b] (its I1 columns are a
    # product, its I2 columns a copy): at most 8 n3^2 w per level apart
    per = [fl[0] for _, _, fl, _ in res]
    slack = sum(8.0 * lv["n3"] ** 2 * lv["w"] for lv in plan)
    assert max(per) - min(per) <= slack * (1 + 1e-12), (per, slack)


@pytest.mark.parametrize("world", [2, 4, 8])
def test_config3_sharded_matches_single_gpu(world):
    """C3 (128 x 128 leaves, 10 ppw, 4 RHS here) sharded over `world` virtual ranks: the root R and
    u equal the single-GPU run (the top levels' products are split by columns only -- M/N
    splits -- so the build differs from the single-GPU one only where the GEMM tile choice does)."""
    from paper_1812_07167_b200 import dist
    cfg, g, c, s, t = _bench_inputs(3, nrhs=4)
    S = hps.Solver(g, cfg.p, cfg.kappa, cfg.eta, c)
    u_ref = S.solve(s, t)
    R_ref = S.R(1)
    S.close()
    res = _sharded_run(world, g, cfg.p, cfg.kappa, cfg.eta, c, s, t)
    worst_R = max(rel(R, R_ref) for _, R, _, _ in res)
    worst_u = max(rel(u, dist.slice_leaves(u_ref, g, sub, i0, j0)) for u, _, _, (sub, i0, j0) in res)
    bitwise_R = all(np.array_equal(R, R_ref) for _, R, _, _ in res)
    print(f"C3 sharded x{world}: root R rel {worst_R:.1e} (bitwise {bitwise_R}), u rel {worst_u:.1e}")
    assert worst_R < 1e-12 and worst_u < 1e-11


def test_stream_ordered_solve():
    """hps_opts.stream: the handle orders its work on the caller's (torch) stream; with device
    buffers hps_solve returns without waiting and hps_sync completes it; the result equals the
    synchronous solve.  Inputs produced by torch on that stream are consumed in order."""
    import torch
    g, c, s, t = problem(8, 8, 10, 9.0, 9.0 + 1j, nrhs=4)
    u_ref = hps.Solver(g, 10, 9.0, 9.0 + 1j, c).solve(s, t)
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        cd = torch.from_numpy(c).cuda()
        sd = torch.from_numpy(s).cuda() * 1.0          # produced on st, read by the library on st
        td = torch.from_numpy(t).cuda() * 1.0
        S = hps.Solver(g, 10, 9.0, 9.0 + 1j, cd, stream=st)
        u = torch.empty((4, 64, 96), dtype=torch.complex128, device="cuda")
        S.solve(sd, td, u)
        S.sync()
        assert S.time_ms(3) > 0
    st.synchronize()
    assert rel(u.cpu().numpy(), u_ref) < 1e-13
    S.close()


def test_nccl_single_rank_comm():
    """The NCCL transport on one rank: unique id -> ncclCommInitRank (run-time loaded NCCL) ->
    library wrapper; the all-gather self-test passes and a build with the communicator (G = 1:
    the plain single-GPU path) equals the plain build."""
    import torch
    import torch.distributed as tdist
    import socket
    from paper_1812_07167_b200 import dist
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    tdist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    try:
        comm = dist.init_nccl()
        assert comm.info() == (0, 1)
        comm.selftest(1)
        g, c, s, t = problem(4, 4, 8, 9.0, 9.0)
        u = hps.Solver(g, 8, 9.0, 9.0, c, comm=comm).solve(s, t)
        assert np.array_equal(u, hps.Solver(g, 8, 9.0, 9.0, c).solve(s, t))
        comm.close()
    finally:
        tdist.destroy_process_group()
    del torch


def test_virtual_comm_selftest():
    """The virtual transport's all-gather in every group size (8 virtual ranks)."""
    from paper_1812_07167_b200 import dist

    def fn(comm):
        for gs in (1, 2, 4, 8):
            comm.selftest(gs)
        return True

    assert all(dist.run_virtual(8, fn))


@pytest.mark.parametrize("m3", [1, 0])
@pytest.mark.parametrize("cfg", list(range(14)))
@pytest.mark.parametrize("M,N,K,batch", [(14, 84, 14, 3), (196, 168, 28, 2), (70, 9, 33, 1), (130, 200, 67, 1),
                                         (70, 1, 300, 2), (33, 3, 45, 3)])
def test_zgemm_configs(cfg, M, N, K, batch, m3):
    """Every DMMA tile configuration vs the oracle's triple-loop product (ragged edges, beta), in
    the 4M and the 3M form (knob gemm_3m)."""
    rng = np.random.default_rng(M * 1000 + N + K)
    A = rng.standard_normal((batch, M, K)) + 1j * rng.standard_normal((batch, M, K))
    B = rng.standard_normal((batch, K, N)) + 1j * rng.standard_normal((batch, K, N))
    Cin = rng.standard_normal((batch, M, N)) + 1j * rng.standard_normal((batch, M, N))
    if cfg == 9 and N > 4:
        pytest.skip("GEMV path is for N <= 4")
    with hps.debug_knobs(gemm_3m=m3):
        for alpha, beta in [(1.0, 1.0), (-1.0, 0.5 - 2j)]:
            C, _ = hps.zgemm_batched(A, B, Cin, alpha, beta, cfg=cfg)
            for b in range(batch):
                ref = alpha * oracle.matmul(A[b], B[b]) + beta * Cin[b]
                assert rel(C[b], ref) < 1e-13


@pytest.mark.parametrize("m3", [1, 0])
@pytest.mark.parametrize("cfg", [1 | 2 << 8, 2 | 4 << 8, 13 | 8 << 8, 5 | 2 << 8, 6 | 4 << 8])
@pytest.mark.parametrize("M,N,K,batch", [(196, 168, 28, 2), (70, 9, 33, 1), (130, 200, 671, 1), (33, 16, 1500, 3)])
def test_zgemm_split_k(cfg, M, N, K, batch, m3):
    """Split-K configurations (tile | slices << 8, zgemm.cu launch_cfg): partial tiles per K slice
    (whole BK stages; empty slices when K is short), Cin only in slice 0, slices summed in order by
    the reduction kernel -- vs the oracle's product with alpha, beta, in both product forms."""
    rng = np.random.default_rng(M * 7 + N + K)
    A = rng.standard_normal((batch, M, K)) + 1j * rng.standard_normal((batch, M, K))
    B = rng.standard_normal((batch, K, N)) + 1j * rng.standard_normal((batch, K, N))
    Cin = rng.standard_normal((batch, M, N)) + 1j * rng.standard_normal((batch, M, N))
    with hps.debug_knobs(gemm_3m=m3):
        for alpha, beta in [(1.0, 1.0), (-1.0, 0.5 - 2j), (0.5j, 0.0)]:
            C, _ = hps.zgemm_batched(A, B, Cin if beta != 0 else None, alpha, beta, cfg=cfg)
            for b in range(batch):
                ref = alpha * oracle.matmul(A[b], B[b]) + beta * Cin[b]
                assert rel(C[b], ref) < 1e-13


@pytest.mark.parametrize("cfg", [2, 5])
def test_zgemm_3m_error_bound(cfg):
    """3M vs 4M error against the oracle's product at long K and on operands whose imaginary parts
    are 1e-6 of their real parts (where Ci = T3 - T1 - T2 cancels): normwise, the 3M error stays
    within a small constant (Higham's bound for the 3M method) of the 4M error, and both <= 1e-14."""
    rng = np.random.default_rng(7)
    M, N, K = 96, 80, 3584
    A = rng.standard_normal((1, M, K)) + 1j * rng.standard_normal((1, M, K))
    B = rng.standard_normal((1, K, N)) + 1j * rng.standard_normal((1, K, N))
    As = A.real + 1e-6j * A.imag
    for a, b in [(A, B), (As, B), (As, B.real + 1e-6j * B.imag)]:
        ref = oracle.matmul(a[0], b[0])
        errs = []
        for m3 in (0, 1):
            with hps.debug_knobs(gemm_3m=m3):
                C, _ = hps.zgemm_batched(a, b, None, 1.0, 0.0, cfg=cfg)
            errs.append(np.linalg.norm(C[0] - ref) / (np.linalg.norm(a[0]) * np.linalg.norm(b[0])))
        assert errs[0] < 1e-15 and errs[1] < 1e-15
        assert errs[1] < 8 * errs[0] + 1e-17, errs


@pytest.mark.parametrize("ns,tol", [(6, 2e-10), (7, 2e-12), (8, 2e-14)])
@pytest.mark.parametrize("M,N,K,batch", [(130, 200, 671, 1), (96, 80, 3584, 2), (70, 12, 33, 3)])
def test_zgemm_integer_slices(M, N, K, batch, ns, tol):
    """Opt-in integer-slice form of the big products (knob gemm_slices = s, zgemm_slices.cu, DESIGN.md
    11): s 7-bit slices per real operand, slice products exact in int32 on the INT8 tensor path, folded
    in FP64 -- vs the oracle's triple-loop product with alpha, beta, operands whose rows span six
    decades; normwise error per slice count as tools/ozaki_probe.py measures it.  Off by default."""
    rng = np.random.default_rng(M + 3 * N + K)
    A = rng.standard_normal((batch, M, K)) + 1j * rng.standard_normal((batch, M, K))
    B = rng.standard_normal((batch, K, N)) + 1j * rng.standard_normal((batch, K, N))
    B = B * 10.0 ** rng.uniform(-6, 0, (batch, K, 1))
    Cin = rng.standard_normal((batch, M, N)) + 1j * rng.standard_normal((batch, M, N))
    with hps.debug_knobs(gemm_slices=ns, gemm_slices_min=12):
        for alpha, beta in [(1.0, 1.0), (-1.0, 0.5 - 2j), (0.5j, 0.0)]:
            C, _ = hps.zgemm_batched(A, B, Cin if beta != 0 else None, alpha, beta)
            for b in range(batch):
                P = oracle.matmul(A[b], B[b])
                ref = alpha * P + beta * Cin[b]
                scale = np.max(np.abs(A[b]), axis=1)[:, None] * np.max(np.abs(B[b]), axis=0)[None, :] * np.sqrt(K)
                assert np.max(np.abs(C[b] - ref) / scale) < tol


def test_config2_integer_slices():
    """C2 whole problem with every product of n >= 100 in the integer-slice form (s = 8): root R and u
    vs the oracle at the suite's tolerance and within 1e-11 of the default DMMA path."""
    cfg, g, c, s, t = _bench_inputs(2)
    with hps.debug_knobs(gemm_slices=8, gemm_slices_min=100):
        S = hps.Solver(g, cfg.p, cfg.kappa, cfg.eta, c)
        u = S.solve(s, t)
        R = S.R(1)
    S2 = hps.Solver(g, cfg.p, cfg.kappa, cfg.eta, c)
    u2 = S2.solve(s, t)
    O = oracle.Oracle(cfg.x0, cfg.x1, cfg.y0, cfg.y1, cfg.nx, cfg.ny, cfg.p, cfg.kappa, cfg.eta, c)
    assert rel(R, O.R(1)) < TOL
    assert rel(u, O.solve(s, t)) < TOL
    assert rel(u, u2) < 1e-11
    assert rel(R, S2.R(1)) < 1e-11


# ---------------------------------------------------------------------------
# BASELINE configurations at full size, in the bench's launch configuration
# ---------------------------------------------------------------------------
def _bench_inputs(cfgno, nrhs=None):
    import bench
    cfg = inputs.CONFIGS[cfgno]
    g, c, s, t = bench.setup(cfg, hps)
    if nrhs is not None:
        s, t = s[:nrhs], t[:nrhs]
    return cfg, g, c, s, t


def test_config2_full_vs_oracle():
    """C2 (the bench workload), whole problem: root R and u vs the oracle's Algorithm 1 + 2."""
    cfg, g, c, s, t = _bench_inputs(2)
    S = hps.Solver(g, cfg.p, cfg.kappa, cfg.eta, c)
    u = S.solve(s, t)
    O = oracle.Oracle(cfg.x0, cfg.x1, cfg.y0, cfg.y1, cfg.nx, cfg.ny, cfg.p, cfg.kappa, cfg.eta, c)
    assert rel(S.R(1), O.R(1)) < TOL
    assert rel(u, O.solve(s, t)) < TOL


@pytest.mark.parametrize("m3", [0, 1])
def test_config2_product_forms(m3):
    """C2 whole problem in each complex-product form (knob gemm_3m): root R and u vs
    the oracle at the suite's tolerance, and the two forms within 1e-12 of each other."""
    cfg, g, c, s, t = _bench_inputs(2)
    with hps.debug_knobs(gemm_3m=m3):
        S = hps.Solver(g, cfg.p, cfg.kappa, cfg.eta, c)
        u = S.solve(s, t)
        R = S.R(1)
    with hps.debug_knobs(gemm_3m=1 - m3):
        S2 = hps.Solver(g, cfg.p, cfg.kappa, cfg.eta, c)
        u2 = S2.solve(s, t)
    O = oracle.Oracle(cfg.x0, cfg.x1, cfg.y0, cfg.y1, cfg.nx, cfg.ny, cfg.p, cfg.kappa, cfg.eta, c)
    assert rel(R, O.R(1)) < TOL
    assert rel(u, O.solve(s, t)) < TOL
    assert rel(u, u2) < 1e-12


def test_config3_sampled_leaves_and_merges():
    """C3 (128x128 leaves, 10 ppw): sampled leaves vs oracle.leaf, and level-local merges — the
    GPU children's R fed to oracle.merge must give the GPU parent R — at EVERY level, one sampled
    box per level, up to the root (n3 = 1792, child n_b = 5376: about a minute of the oracle's
    row-parallel products on the host cores)."""
    cfg, g, c, s, t = _bench_inputs(3, nrhs=1)
    S = hps.Solver(g, cfg.p, cfg.kappa, cfg.eta, c, keep_all_R=True)
    h = 1.0 / 128
    rng = np.random.default_rng(3)
    for leaf in rng.choice(cfg.nleaf, 3, replace=False):
        Psi, Y = S.leaf_ops(int(leaf))
        lo = oracle.leaf(cfg.p, h, h, cfg.kappa, cfg.eta, c[leaf])
        assert rel(Psi, lo["Psi"]) < TOL and rel(Y, lo["Y"]) < TOL
    L = 14
    errs = {}
    for d in range(L - 1, -1, -1):
        box = (1 << d) + int(rng.integers(0, 1 << d))
        ci0, ci1, cj0, cj1, _ = oracle.box_rect(cfg.nx, cfg.ny, 2 * box)
        vertical = oracle.box_rect(cfg.nx, cfg.ny, box)[4]
        ref = oracle.merge(cfg.p, ci1 - ci0, cj1 - cj0, vertical, S.R(2 * box), S.R(2 * box + 1))["Rtau"]
        errs[d] = rel(S.R(box), ref)
    S.close()
    print("C3 level-local merge parity (depth: rel err):", {d: f"{e:.1e}" for d, e in errs.items()})
    assert max(errs.values()) < TOL, errs


def test_config3_polynomial_exact():
    """At C3 scale no oracle run is needed for u: a global polynomial of degree p-1 per variable
    is reproduced exactly by the discretisation, so the CUDA path's u must match
    it to rounding (bound derived from cond ~ 1e6 x eps x levels)."""
    import numpy.polynomial.chebyshev as npc
    cfg = inputs.CONFIGS[3]
    p = cfg.p
    g = hps.grid(cfg.x0, cfg.x1, cfg.y0, cfg.y1, cfg.nx, cfg.ny)
    X, Y = hps.leaf_nodes(g, p)
    Xb, Yb, NX, NY = hps.root_boundary_nodes(g, p)
    rng = np.random.default_rng(9)
    a = (rng.standard_normal((p, p)) + 1j * rng.standard_normal((p, p))) / np.outer(np.arange(1, p + 1), np.arange(1, p + 1))
    val = lambda x, y, dx=0, dy=0: npc.chebval2d(2 * x - 1, 2 * y - 1,
                                                 (npc.chebder(npc.chebder(a, dx, axis=0) * 2 ** dx, dy, axis=1) * 2 ** dy)
                                                 if (dx or dy) else a)
    c = inputs.c_at(cfg, X, Y)
    Xi, Yi, ci = inputs.interior_of(p, X), inputs.interior_of(p, Y), inputs.interior_of(p, c)
    s = (-(val(Xi, Yi, 2, 0) + val(Xi, Yi, 0, 2)) - cfg.kappa ** 2 * ci * val(Xi, Yi))[None]
    t = (NX * val(Xb, Yb, 1, 0) + NY * val(Xb, Yb, 0, 1) + 1j * cfg.eta * val(Xb, Yb))[None]
    S = hps.Solver(g, p, cfg.kappa, cfg.eta, c, keep_root_R=False)
    u = S.solve(np.ascontiguousarray(s), np.ascontiguousarray(t))[0]
    ex_i = val(Xi, Yi)
    scale = np.max(np.abs(ex_i))
    # measured 1.1e-13 .. 2.0e-13 over three seeds (tools/poly_errors.py, profiles/r02_poly_errors.txt);
    # bound = 10x the worst, see DESIGN.md 6 for the conditioning argument
    assert np.max(np.abs(u[:, 4 * (p - 2):] - ex_i)) / scale < 2e-12


def test_paper_experiment_convergence():
    """The paper's Sec. 4.1 experiment (NEXT-1): e_inf decays with N for each n_c, spectrally
    faster for larger n_c; at n_c = 16 it reaches the roundoff plateau."""
    from paper_1812_07167_b200 import experiments
    tab = experiments.convergence_table(ps=(6, 9, 16), sides=(8, 16, 32))
    for p, rows in tab.items():
        errs = [e for _, e in rows]
        assert errs[-1] < errs[0] / 10, (p, errs)
    assert tab[16][-1][1] < 1e-8, tab[16]
    assert tab[16][1][1] < tab[9][1][1] < tab[6][1][1]


def test_paper_experiment_matches_oracle_small():
    """Same manufactured problem through the oracle on a 4x4-leaf grid: GPU u == oracle u."""
    p, m, kappa = 9, 4, inputs.PAPER_KAPPA
    g = hps.grid(0.0, 1.0, 0.0, 1.0, m, m)
    X, Y = hps.leaf_nodes(g, p)
    Xb, Yb, NX, NY = hps.root_boundary_nodes(g, p)
    c = inputs.paper_c(X, Y)
    s = inputs.paper_s(inputs.interior_of(p, X), inputs.interior_of(p, Y))[None]
    t = inputs.paper_t(Xb, Yb, NX, NY)[None]
    S = hps.Solver(g, p, kappa, kappa, c)
    O = oracle.Oracle(0, 1, 0, 1, m, m, p, kappa, kappa, c)
    assert rel(S.solve(s, t), O.solve(s, t)) < TOL


def _root_R_device(S):
    import torch
    n = S.nb(1)
    R = torch.empty((n, n), dtype=torch.complex128, device="cuda")
    hps._check(hps.lib().hps_export_R(S.h, 1, R.data_ptr()))
    return R


@pytest.mark.parametrize("cfgno", [2, 3, 4])
def test_root_R_conj_unitary_full_size(cfgno):
    """Full-size pin with no oracle run (reading Q9): kappa, c, eta are real in C2-C4, so the
    composite DtN map is real and the root ItI map satisfies R conj(R) = I exactly; the CUDA
    path's R^1 (1792^2 at C2 ... 14336^2 at C4, built in the bench's launch configuration)
    must reproduce it to rounding.  The check product runs on the GPU through torch (test
    infrastructure only).  Measured: 1.4e-14 (C2), 2.7e-14 (C3), 4.1e-14 (C4)."""
    import torch
    cfg, g, c, s, t = _bench_inputs(cfgno, nrhs=1)
    assert np.isrealobj(c) or np.max(np.abs(np.imag(c))) == 0.0
    S = hps.Solver(g, cfg.p, cfg.kappa, cfg.eta, torch.from_numpy(np.ascontiguousarray(c)).cuda())
    R = _root_R_device(S)
    E = R @ R.conj() - torch.eye(R.shape[0], dtype=torch.complex128, device="cuda")
    err = E.abs().max().item()
    S.close()
    assert err < 1e-10, err


def test_config4_sampled_leaves_and_polynomial():
    """C4 (256 x 256 leaves, 16.7M Chebyshev nodes, kappa h = 10) on one GPU: sampled leaf
    operators vs oracle.leaf, and the polynomial manufactured solution reproduced through the
    whole 16-level tree (collocation is exact on degree <= p-1 polynomials)."""
    import numpy.polynomial.chebyshev as npc
    import torch
    cfg = inputs.CONFIGS[4]
    p = cfg.p
    g = hps.grid(cfg.x0, cfg.x1, cfg.y0, cfg.y1, cfg.nx, cfg.ny)
    X, Y = hps.leaf_nodes(g, p)
    Xb, Yb, NX, NY = hps.root_boundary_nodes(g, p)
    c = inputs.c_at(cfg, X, Y)
    rng = np.random.default_rng(11)
    a = (rng.standard_normal((p, p)) + 1j * rng.standard_normal((p, p))) / np.outer(np.arange(1, p + 1), np.arange(1, p + 1))
    val = lambda x, y, dx=0, dy=0: npc.chebval2d(2 * x - 1, 2 * y - 1,
                                                 (npc.chebder(npc.chebder(a, dx, axis=0) * 2 ** dx, dy, axis=1) * 2 ** dy)
                                                 if (dx or dy) else a)
    Xi, Yi, ci = inputs.interior_of(p, X), inputs.interior_of(p, Y), inputs.interior_of(p, c)
    s = (-(val(Xi, Yi, 2, 0) + val(Xi, Yi, 0, 2)) - cfg.kappa ** 2 * ci * val(Xi, Yi))[None]
    t = (NX * val(Xb, Yb, 1, 0) + NY * val(Xb, Yb, 0, 1) + 1j * cfg.eta * val(Xb, Yb))[None]
    dev = lambda z: torch.from_numpy(np.ascontiguousarray(z)).cuda()
    S = hps.Solver(g, p, cfg.kappa, cfg.eta, dev(c), keep_root_R=False)
    h = 1.0 / cfg.nx
    for leaf in rng.choice(cfg.nleaf, 2, replace=False):
        Psi, Yop = S.leaf_ops(int(leaf))
        lo = oracle.leaf(p, h, h, cfg.kappa, cfg.eta, c[leaf])
        assert rel(Psi, lo["Psi"]) < TOL and rel(Yop, lo["Y"]) < TOL
    u = S.solve(dev(s), dev(t))[0].cpu().numpy()
    S.close()
    ex_i = val(Xi, Yi)
    # measured 2.3e-13 / 2.7e-13 (two seeds, tools/poly_errors.py); bound = 10x the worst
    assert np.max(np.abs(u[:, 4 * (p - 2):] - ex_i)) / np.max(np.abs(ex_i)) < 3e-12


@pytest.mark.parametrize("nx,ny,p,nrhs", [(4, 4, 8, 37), (8, 4, 10, 64), (2, 2, 16, 9)])
def test_many_rhs(nx, ny, p, nrhs):
    """Batches of right-hand sides through the tiled layout kernels (nrhs >= 8, ragged tiles)
    and the GEMM sweeps: u for every RHS vs the oracle's Algorithm 2."""
    kappa, eta = 11.0, 11.0
    g, c, s, t = problem(nx, ny, p, kappa, eta, x1=1.0, y1=ny / nx, nrhs=nrhs, seed=5)
    S = hps.Solver(g, p, kappa, eta, c)
    O = oracle.Oracle(0.0, 1.0, 0.0, ny / nx, nx, ny, p, kappa, eta, c)
    assert rel(S.solve(s, t), O.solve(s, t)) < TOL


def test_planned_regimes_parity():
    """Representative-action planner (NEXT-3): plan every level of an 8 x 8-leaf, p = 12 tree
    (leaf n_i = 100, interface n3 = 10 ... 80), build with the plan, and with every feasible
    regime forced on the top interface inverse: R and u match the oracle in each case."""
    nx, ny, p, kappa, eta = 8, 8, 12, 12.0, 12.0 - 1j
    g, c, s, t = problem(nx, ny, p, kappa, eta)
    O = oracle.Oracle(0.0, 1.0, 0.0, 1.0, nx, ny, p, kappa, eta, c)
    Ro, uo = O.R(1), O.solve(s, t)
    try:
        rows = hps.plan_problem(g, p)
        assert len(rows) == 7
        for _, n, nb, reg, tab in rows:
            assert reg in tab and all(tab[reg][0] <= e for e, _, _ in tab.values())
            assert hps.plan_regime(n, nb) == reg
        S = hps.Solver(g, p, kappa, eta, c)
        assert rel(S.R(1), Ro) < TOL and rel(S.solve(s, t), uo) < TOL
        S.close()
        n_top, nb_top = hps.rep_actions(g, p)[-1]
        for reg in range(1, 8):
            if (reg == 1 and n_top > 112) or (reg in (3, 7) and n_top > 240):
                continue
            hps._check(hps.lib().hps_plan_set(n_top, nb_top, reg))
            S = hps.Solver(g, p, kappa, eta, c)
            assert rel(S.R(1), Ro) < TOL, reg
            S.close()
    finally:
        hps.plan_clear()


def test_plan_solve_parity():
    """Solve-stage planner (hps_plan_solve): every action's shape is timed with each candidate tile
    configuration and the fastest recorded; the planned solve still matches the oracle at 1e-9 and
    the unplanned solve to rounding (the configurations differ in tiling and, for the GEMV kernel of
    N <= 4 and the split-K configurations, in the summation order along K)."""
    nx, ny, p, kappa, eta = 8, 4, 12, 15.0, 15.0 - 1j
    g, c, s, t = problem(nx, ny, p, kappa, eta, x1=1.0, y1=0.5, nrhs=16)
    hps.plan_clear()
    u0 = hps.Solver(g, p, kappa, eta, c).solve(s, t)
    try:
        plan = hps.plan_solve(g, p, 16)
        assert len(plan) == len(hps.solve_actions(g, p, 16))
        assert all(a["rule_ms"] > 0 and a["best_ms"] <= a["rule_ms"] * 1.0001 for a in plan)
        u1 = hps.Solver(g, p, kappa, eta, c).solve(s, t)
    finally:
        hps.plan_clear()
    O = oracle.Oracle(0.0, 1.0, 0.0, 0.5, nx, ny, p, kappa, eta, c)
    assert rel(u1, O.solve(s, t)) < TOL
    assert rel(u1, u0) < 1e-12


def test_plan_build_parity():
    """Build-stage GEMM planner (hps_plan_build): the planned build's root R and u match the
    oracle at 1e-9 and the unplanned build to rounding."""
    nx, ny, p, kappa, eta = 16, 16, 12, 20.0, 20.0 + 2j
    g, c, s, t = problem(nx, ny, p, kappa, eta, nrhs=2)
    hps.plan_clear()
    S0 = hps.Solver(g, p, kappa, eta, c)
    u0, R0 = S0.solve(s, t), S0.R(1)
    try:
        plan = hps.plan_build(g, p)
        assert len(plan) == len(hps.build_actions(g, p)) and any(a["kind"] == 9 for a in plan)
        S1 = hps.Solver(g, p, kappa, eta, c)
        u1, R1 = S1.solve(s, t), S1.R(1)
    finally:
        hps.plan_clear()
    O = oracle.Oracle(0.0, 1.0, 0.0, 1.0, nx, ny, p, kappa, eta, c)
    assert rel(R1, O.R(1)) < TOL and rel(u1, O.solve(s, t)) < TOL
    assert rel(R1, R0) < 1e-12 and rel(u1, u0) < 1e-12


def test_rhs_chunks():
    """Right-hand sides in chunks (knob rhs_chunk; automatic by free memory otherwise, SURVEY hard
    part 7): 37 RHS in chunks of 8 (the last of 5) equal one 37-RHS sweep to rounding and the oracle
    at 1e-9, with host buffers (staged chunk by chunk) and with torch device buffers; the phase
    times are summed over the chunks."""
    import torch
    nx, ny, p, kappa, eta = 4, 4, 12, 11.0, 11.0 + 1j
    g, c, s, t = problem(nx, ny, p, kappa, eta, nrhs=37, seed=4)
    S = hps.Solver(g, p, kappa, eta, c)
    u_all = S.solve(s, t)
    with hps.debug_knobs(rhs_chunk=8):
        u_host = S.solve(s, t)
        assert S.time_ms(3) > 0 and abs(S.time_ms(3) - S.time_ms(4) - S.time_ms(5)) < 1e-6
        d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
        u_dev = S.solve(d(s), d(t)).cpu().numpy()
        u_nos = S.solve(None, t)
    assert rel(u_host, u_all) < 1e-12 and rel(u_dev, u_all) < 1e-12
    O = oracle.Oracle(0.0, 1.0, 0.0, 1.0, nx, ny, p, kappa, eta, c)
    assert rel(u_host, O.solve(s, t)) < TOL
    assert rel(u_nos, O.solve(np.zeros_like(s), t)) < TOL


@pytest.mark.parametrize("nx,ny,p", [(4, 4, 16), (8, 4, 10), (2, 2, 8), (16, 8, 6)])
def test_merge_small_levels(nx, ny, p):
    """Lowest merge levels (n3 <= 28) fused into one CTA per merge (merge_small.cu, knob merge_small):
    every box's R and u match the oracle at 1e-9 and the GEMM path to rounding, with and without a
    body load, complex eta."""
    kappa, eta = 13.0, 13.0 - 2j
    g, c, s, t = problem(nx, ny, p, kappa, eta, x1=1.0, y1=ny / nx)
    O = oracle.Oracle(0.0, 1.0, 0.0, ny / nx, nx, ny, p, kappa, eta, c, keep_all_R=True)
    res = {}
    for ms in (1, 0):
        with hps.debug_knobs(merge_small=ms):
            S = hps.Solver(g, p, kappa, eta, c, keep_all_R=True)
            res[ms] = (S.solve(s, t), S.solve(None, t), [S.R(b) for b in range(1, oracle.tree_info(nx, ny)[0] + 1)])
            S.close()
    u1, u1n, R1 = res[1]
    u0, u0n, R0 = res[0]
    assert rel(u1, O.solve(s, t)) < TOL and rel(u1n, O.solve(np.zeros_like(s), t)) < TOL
    assert rel(u1, u0) < 1e-12 and rel(u1n, u0n) < 1e-12
    for b, (r1, r0) in enumerate(zip(R1, R0), start=1):
        assert rel(r1, O.R(b)) < TOL, b
        assert rel(r1, r0) < 1e-12, b
