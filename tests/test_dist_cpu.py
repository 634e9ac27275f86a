"""Multi-rank subtree sharding on CPU (no GPU): the partition geometry, the host plan of the
group split of the top levels (hps_dist_plan), and the communicator plumbing of
paper_1812_07167_b200.dist over real torch.distributed gloo ranks (world size 2 and 4): the NCCL
unique id made by the library on rank 0 reaches every rank, and the per-rank plans gathered over
gloo tile every top-level merge's columns exactly once.  The sharded numerics themselves run in
libhps on the GPU (tests/test_gpu_parity.py: virtual ranks vs the single-GPU build)."""
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


def check_plans(g, p, plans):
    """plans[r] = hps.dist_plan(g, p, G, r).  Every top-level merge (depth d, box m) is handled by
    the aligned group of gs = G >> d ranks above it; their column slices tile [0, ntau) exactly;
    the first half of the group sits under the alpha child; n3 / ntau are the oracle tree's."""
    G = len(plans)
    D = len(plans[0])
    assert 1 << D == G
    for d in range(D):
        gs = G >> d
        for m in range(1 << d):
            box = (1 << d) + m
            ci0, ci1, cj0, cj1, _ = oracle.box_rect(g.nx, g.ny, 2 * box)
            vertical = oracle.box_rect(g.nx, g.ny, box)[4]
            q = p - 2
            n3 = (cj1 - cj0) * q if vertical else (ci1 - ci0) * q
            nbc = 2 * ((ci1 - ci0) + (cj1 - cj0)) * q
            ranks = range(m * gs, (m + 1) * gs)
            cover = np.zeros(2 * (nbc - n3), int)
            for r in ranks:
                lv = plans[r][d]
                assert lv["gs"] == gs and lv["grank"] == r - m * gs
                assert lv["side"] == (1 if lv["grank"] >= gs // 2 else 0)
                assert lv["n3"] == n3 and lv["ntau"] == 2 * (nbc - n3) and lv["n1"] == nbc - n3
                cover[lv["j0"]:lv["j0"] + lv["w"]] += 1
            assert np.all(cover == 1), (d, m)
            # the alpha side's ranks own the subtrees inside child 2 box
            for r in ranks:
                sub, i0, j0 = hps.subtree_grid(g, D, r)
                inside_alpha = ci0 <= i0 < ci1 and cj0 <= j0 < cj1
                assert inside_alpha == (plans[r][d]["side"] == 0)


@pytest.mark.parametrize("nx,ny,G", [(256, 256, 8), (1024, 512, 8), (8, 8, 4), (16, 8, 2), (4, 4, 16)])
def test_dist_plan_tiles_every_top_merge(nx, ny, G):
    g = hps.grid(0.0, nx / max(nx, ny), 0.0, ny / max(nx, ny), nx, ny)
    check_plans(g, 16, [hps.dist_plan(g, 16, G, r) for r in range(G)])


def test_dist_plan_rejects_shallow_tree():
    with pytest.raises(hps.HpsError):
        hps.dist_plan(hps.grid(0, 1, 0, 1, 2, 1), 8, 4, 0)


def _gloo_worker(rank, world, port, q):
    import torch
    import torch.distributed as tdist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # the NCCL unique id made by the library on rank 0 travels over the process group
        uid = dist.broadcast_unique_id(hps.Comm.nccl_unique_id)
        # every rank's host plan of the split, gathered over gloo
        g = hps.grid(0.0, 2.0, 0.0, 1.0, 64, 32)
        plan = hps.dist_plan(g, 16, world, rank)
        flat = torch.tensor([[v for lv in plan for v in lv.values()]], dtype=torch.int64)
        out = [torch.zeros_like(flat) for _ in range(world)]
        tdist.all_gather(out, flat)
        keys = list(plan[0].keys())
        plans = [[dict(zip(keys, o[0, 8 * d:8 * d + 8].tolist())) for d in range(len(plan))] for o in out]
        # this rank's leaf slice of a natural-order array
        sub, i0, j0 = dist.local_block(g, world, rank)
        a = np.arange(g.nx * g.ny * 3).reshape(1, g.nx * g.ny, 3)
        loc = dist.slice_leaves(a, g, sub, i0, j0)
        q.put((rank, uid, plans, (sub.nx, sub.ny, i0, j0), loc.sum()))
    finally:
        tdist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.mark.parametrize("world", [2, 4])
def test_gloo_ranks_split_plumbing(world):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    out = sorted([q.get(timeout=300) for _ in range(world)], key=lambda o: o[0])
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    assert [o[0] for o in out] == list(range(world))
    uids = {o[1] for o in out}
    assert len(uids) == 1 and len(out[0][1]) == 128
    g = hps.grid(0.0, 2.0, 0.0, 1.0, 64, 32)
    for o in out:   # every rank saw the same gathered plans, and they tile the top merges
        assert o[2] == out[0][2]
    check_plans(g, 16, out[0][2])
    # the local leaf slices partition the leaves
    a = np.arange(g.nx * g.ny * 3)
    assert sum(o[4] for o in out) == a.sum()
    assert sum(o[3][0] * o[3][1] for o in out) == g.nx * g.ny
