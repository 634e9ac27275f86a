"""Subtree sharding of the HPS tree over G ranks (PAPER.md:1336-1338 names
distributed memory as the paper's next step).

The exchange itself runs INSIDE libhps (hps_build / hps_solve with a communicator in hps_opts,
csrc/comm.cu + the sharded top levels in csrc/hps_api.cu):
* partition: the top log2(G) splits of the tree (its own split rule) give G congruent rectangles;
  rank r owns the subtree of the depth-log2(G) box with heap index 2^log2(G) + r.  Its c, s and u
  slices are rank-local; t (the root boundary data) is passed whole on every rank;
* build: every rank builds its leaves and subtree with no communication; at the top level with
  2^k merges the G / 2^k ranks under a box all-gather the children's ItI maps, form W and W^-1
  (replicated) and each computes a 1 / (G / 2^k) column slice of Phi^a, Phi^b and R^tau (R^tau
  stays column-distributed until the next level's gather);
* solve: subtree up-sweep; per top level an all-gather of the group's box data h and a
  replicated t~ step; down-sweep with the column slices of Phi and an all-gather + ordered sum of
  the partial products; subtree down-sweep.

This module only creates communicators and slices arrays: `init_nccl` (NCCL over NVLink, one
process per GPU: the NCCL unique id travels over torch.distributed) and `run_virtual` (G ranks as
host threads of one process on one GPU, for tests).
"""
import math
import threading

import numpy as np

from . import hps


def depth_for(world):
    d = int(round(math.log2(world)))
    if 1 << d != world:
        raise ValueError("the number of ranks must be a power of two")
    return d


def local_block(g, world, rank):
    """(sub-grid, leaf i0, leaf j0) of rank's subtree."""
    return hps.subtree_grid(g, depth_for(world), rank)


def slice_leaves(arr, g, sub, i0, j0):
    """Select a rank's leaves from a natural-order array [..., nx*ny, k] (local natural order)."""
    lead = arr.shape[:-2]
    a = arr.reshape(lead + (g.ny, g.nx, arr.shape[-1]))
    a = a[..., j0:j0 + sub.ny, i0:i0 + sub.nx, :]
    return a.reshape(lead + (sub.nx * sub.ny, arr.shape[-1]))


def broadcast_unique_id(make_id, group=None):
    """Rank 0 makes the NCCL unique id (hps_nccl_unique_id); every rank receives it over the
    torch.distributed process group (gloo or NCCL).  Returns the 128 bytes."""
    import torch.distributed as tdist
    obj = [make_id() if tdist.get_rank(group) == 0 else None]
    tdist.broadcast_object_list(obj, src=0, group=group)
    return obj[0]


def init_nccl(group=None):
    """The library communicator of this process's rank: ncclCommInitRank on the current CUDA
    device from a unique id broadcast over torch.distributed, wrapped by hps_comm_wrap_nccl."""
    import torch.distributed as tdist
    uid = broadcast_unique_id(hps.Comm.nccl_unique_id, group)
    return hps.Comm.nccl(tdist.get_world_size(group), tdist.get_rank(group), uid)


def run_virtual(world, fn):
    """Run fn(comm) on `world` virtual ranks (host threads sharing the current GPU, each with its
    own library communicator); returns the per-rank results (re-raises the first error)."""
    grp = hps.VirtualGroup(world)
    res, err = [None] * world, [None] * world
    comms = [grp.comm(r) for r in range(world)]

    def body(r):
        try:
            import torch
            if torch.cuda.is_available():
                torch.cuda.set_device(torch.cuda.current_device())
            res[r] = fn(comms[r])
        except BaseException as e:  # noqa: BLE001 - propagate to the caller
            err[r] = e

    th = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for c in comms:
        c.close()
    grp.close()
    for e in err:
        if e is not None:
            raise e
    return res


class DistributedHPS:
    """SPMD driver: every rank constructs one with its communicator and its local leaf data."""

    def __init__(self, comm, g, p, kappa, eta, c_local, **kw):
        self.comm, self.g, self.p = comm, g, p
        rank, world = comm.info()
        self.rank, self.world = rank, world
        self.sub_grid, self.i0, self.j0 = local_block(g, world, rank)
        self.solver = hps.Solver(g, p, kappa, eta, c_local, comm=comm, **kw)

    def solve(self, s_local, t_root, u=None):
        return self.solver.solve(s_local, t_root, u)

    def root_R(self):
        return self.solver.R(1)

    def close(self):
        self.solver.close()
