"""Multi-rank subtree sharding on CPU (no GPU): the partition geometry, and the SPMD driver
(paper_1812_07167_b200.dist) over real torch.distributed gloo ranks (world size 2 and 4) and
over virtual thread ranks.  The numerics of the build are the ORACLE's here (an oracle-backed
backend, test-only): subtree roots built by oracle.Oracle on each rank's rectangle, gathered,
merged upward with oracle.merge — and compared with the single-process oracle root R.  The
solve plumbing (gather order, own-slice selection) is checked with a tagging backend."""
import os
import socket

import numpy as np
import pytest

import oracle
from paper_1812_07167_b200 import dist, hps


@pytest.mark.parametrize("nx,ny", [(4, 4), (8, 4), (4, 8), (2, 1), (16, 8)])
def test_subtree_grid_matches_oracle_tree(nx, ny):
    g = hps.grid(0.0, 2.0, -1.0, 0.5, nx, ny)
    L = oracle.tree_info(nx, ny)[1]
    for depth in range(0, min(L, 4) + 1):
        cover = np.zeros((ny, nx), int)
        for r in range(1 << depth):
            sub, i0, j0 = hps.subtree_grid(g, depth, r)
            bi0, bi1, bj0, bj1, _ = oracle.box_rect(nx, ny, (1 << depth) + r)
            assert (i0, j0, i0 + sub.nx, j0 + sub.ny) == (bi0, bj0, bi1, bj1)
            assert abs(sub.x0 - (0.0 + 2.0 * i0 / nx)) < 1e-15 and abs(sub.y1 - (-1.0 + 1.5 * (j0 + sub.ny) / ny)) < 1e-15
            cover[j0:j0 + sub.ny, i0:i0 + sub.nx] += 1
        assert np.all(cover == 1)


class OracleBackend:
    """Test-only backend: oracle numerics for the build; tagging functions for the solve."""

    def __init__(self, g):
        self.g = g

    def build_subtree(self, g_sub, p, kappa, eta, c_local):
        return oracle.Oracle(g_sub.x0, g_sub.x1, g_sub.y0, g_sub.y1, g_sub.nx, g_sub.ny, p, kappa, eta, c_local)

    def root_R(self, sub, like):
        return sub.R(1)

    def build_top(self, g, p, kappa, eta, depth, R_all):
        Rs = {(1 << depth) + r: R_all[r] for r in range(1 << depth)}
        for d in range(depth - 1, -1, -1):
            for m in range(1 << d):
                box = (1 << d) + m
                ci0, ci1, cj0, cj1, _ = oracle.box_rect(g.nx, g.ny, 2 * box)
                vertical = oracle.box_rect(g.nx, g.ny, box)[4]
                Rs[box] = oracle.merge(p, ci1 - ci0, cj1 - cj0, vertical, Rs[2 * box], Rs[2 * box + 1])["Rtau"]
        return {"R": Rs[1]}

    def solve_up(self, sub, s_local, nrhs, like):
        return np.ones((nrhs, sub.nb(1)), complex) * s_local.sum()

    def solve_top(self, top, h_all, t_root):
        nb = h_all.shape[-1]
        return 2 * h_all + t_root[None, :, :nb]

    def solve_down(self, sub, t_sub):
        return t_sub


def problem(nx=4, ny=4, p=6):
    g = hps.grid(0.0, 1.0, 0.0, ny / nx, nx, ny)
    X, Y = oracle.leaf_nodes(0.0, 1.0, 0.0, ny / nx, nx, ny, p)
    c = (1 + 0.3 * np.exp(-((X - 0.3) ** 2 + (Y - 0.4) ** 2) / 0.05)).astype(complex)
    rng = np.random.default_rng(nx * ny)
    s = rng.standard_normal((2, nx * ny, (p - 2) ** 2)) + 0j
    t = rng.standard_normal((2, 2 * (nx + ny) * (p - 2))) + 0j
    return g, p, 7.0, 7.0 + 0.5j, c, s, t


def run_rank(comm):
    g, p, kappa, eta, c, s, t = problem()
    sub, i0, j0 = dist.local_block(g, comm.world, comm.rank)
    D = dist.DistributedHPS(comm, OracleBackend(g), g, p, kappa, eta, dist.slice_leaves(c, g, sub, i0, j0))
    s_loc = dist.slice_leaves(s, g, sub, i0, j0)
    out = D.solve(s_loc, t)
    nb = out.shape[-1]
    expect = 2 * np.ones((2, nb), complex) * s_loc.sum() + t[:, :nb]
    return D.top["R"], np.max(np.abs(out - expect))


def reference_root():
    g, p, kappa, eta, c, s, t = problem()
    return oracle.Oracle(g.x0, g.x1, g.y0, g.y1, g.nx, g.ny, p, kappa, eta, c).R(1)


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_thread_ranks_oracle_backend(world):
    res = dist.run_threads(world, run_rank)
    Rref = reference_root()
    for R, err in res:
        assert np.max(np.abs(R - Rref)) / np.max(np.abs(Rref)) < 1e-10
        assert err == 0.0


def _gloo_worker(rank, world, port, q):
    import torch.distributed as tdist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        R, err = run_rank(dist.TorchComm())
        q.put((rank, R, err))
    finally:
        tdist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.mark.parametrize("world", [2, 4])
def test_gloo_ranks_oracle_backend(world):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    out = [q.get(timeout=300) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    Rref = reference_root()
    assert sorted(o[0] for o in out) == list(range(world))
    for _, R, err in out:
        assert np.max(np.abs(R - Rref)) / np.max(np.abs(Rref)) < 1e-10
        assert err == 0.0
