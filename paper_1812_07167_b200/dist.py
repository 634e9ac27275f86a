"""Subtree sharding of the HPS tree over G ranks (PAPER.md:1336-1338 names
distributed memory as the paper's future work).

Partition: the top log2(G) splits of the tree (same split rule as the tree itself) give G
congruent rectangles; rank r owns the subtree of the depth-log2(G) box with heap index r.
* build: every rank runs the leaf build and all merges of its subtree with NO communication
  (hps_build on its rectangle); the subtree-root ItI operators are all-gathered (one
  collective, n_b^2 complex per rank) and every rank merges the top log2(G) levels
  (hps_build_top) — replicated, so the top operators needed by the solve are local.
* solve: hps_solve_up on every subtree; all-gather of the subtree-root outgoing data h
  (n_b x nrhs per rank); every rank runs the top upward and downward passes (hps_solve_top)
  and keeps the incoming data t of its own subtree root; hps_solve_down on every subtree.

`Comm` is the only thing that differs between a real multi-GPU run (TorchComm over
torch.distributed: NCCL for CUDA tensors, gloo for CPU tensors) and the single-GPU
virtual-rank mode (ThreadComm: G ranks as host threads of one process, gather by a host-side
barrier — no kernel waits on another).  The numerics are the library's; this module only moves
arguments.
"""
import math
import threading

import numpy as np

from . import hps


# ---------------------------------------------------------------------------
# Communicators
# ---------------------------------------------------------------------------
class TorchComm:
    """torch.distributed process group (NCCL for CUDA tensors, gloo for CPU tensors)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)

    def all_gather(self, x):
        import torch
        xt = x if hasattr(x, "data_ptr") else torch.from_numpy(np.ascontiguousarray(x))
        out = [torch.empty_like(xt) for _ in range(self.world)]
        self.dist.all_gather(out, xt.contiguous(), group=self.group)
        if xt.is_cuda:
            torch.cuda.current_stream().synchronize()   # the library reads these on its own stream
        return out if hasattr(x, "data_ptr") else [o.numpy() for o in out]

    def barrier(self):
        self.dist.barrier(group=self.group)


class _ThreadGroup:
    def __init__(self, world):
        self.world = world
        self.barrier = threading.Barrier(world)
        self.slots = [None] * world


class ThreadComm:
    """Virtual ranks: `world` host threads of one process sharing one GPU."""

    def __init__(self, group, rank):
        self.g = group
        self.rank = rank
        self.world = group.world

    def all_gather(self, x):
        self.g.slots[self.rank] = x
        self.g.barrier.wait()
        out = list(self.g.slots)
        self.g.barrier.wait()
        return out

    def barrier(self):
        self.g.barrier.wait()


def run_threads(world, fn):
    """Run fn(comm) on `world` virtual ranks; returns the per-rank results (re-raises)."""
    group = _ThreadGroup(world)
    res, err = [None] * world, [None] * world

    def body(r):
        try:
            res[r] = fn(ThreadComm(group, r))
        except BaseException as e:  # noqa: BLE001 - propagate to the caller
            err[r] = e
            group.barrier.abort()

    th = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for e in err:
        if e is not None and not isinstance(e, threading.BrokenBarrierError):
            raise e
    for e in err:
        if e is not None:
            raise e
    return res


# ---------------------------------------------------------------------------
# Partition helpers
# ---------------------------------------------------------------------------
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


def _stack(xs):
    if hasattr(xs[0], "data_ptr"):
        import torch
        out = torch.stack(xs).contiguous()
        if out.is_cuda:
            # the library reads this buffer on its own stream: the stack kernel (on torch's
            # current stream) must be complete first
            torch.cuda.current_stream(out.device).synchronize()
        return out
    return np.ascontiguousarray(np.stack(xs))


# ---------------------------------------------------------------------------
# Backend: the CUDA library (product path)
# ---------------------------------------------------------------------------
class CudaBackend:
    def __init__(self, device=-1, profile=False, boundary_basis=0):
        self.device = device
        self.profile = profile
        self.boundary_basis = boundary_basis  # 1: root t at Gauss-Legendre nodes (hps_solve_top converts)

    def build_subtree(self, g_sub, p, kappa, eta, c_local):
        return hps.Solver(g_sub, p, kappa, eta, c_local, keep_root_R=True, device=self.device, profile=self.profile)

    def root_R(self, sub, like):
        n = sub.nb(1)
        out = hps._empty_like_ref(like, (n, n))
        hps._check(hps.lib().hps_export_R(sub.h, 1, hps._ptr(out, n * n, "R")))
        return out

    def build_top(self, g, p, kappa, eta, depth, R_all):
        return hps.TopSolver(g, p, kappa, eta, depth, R_all, device=self.device, profile=self.profile,
                             boundary_basis=self.boundary_basis)

    def solve_up(self, sub, s_local, nrhs, like):
        return sub.solve_up(s_local, nrhs, hps._empty_like_ref(like, (nrhs, sub.nb_root)))

    def solve_top(self, top, h_all, t_root):
        return top.solve(h_all, t_root)

    def solve_down(self, sub, t_sub):
        return sub.solve_down(t_sub)


class DistributedHPS:
    """SPMD driver: every rank constructs one with its own comm and its local leaf data."""

    def __init__(self, comm, backend, g, p, kappa, eta, c_local):
        self.comm, self.be, self.g, self.p = comm, backend, g, p
        self.depth = depth_for(comm.world)
        self.sub_grid, self.i0, self.j0 = local_block(g, comm.world, comm.rank)
        self.sub = backend.build_subtree(self.sub_grid, p, kappa, eta, c_local)
        R = backend.root_R(self.sub, c_local)
        R_all = comm.all_gather(R)                          # the one build-time collective
        self.top = backend.build_top(g, p, kappa, eta, self.depth, _stack(R_all))

    def solve(self, s_local, t_root):
        nrhs = int(t_root.shape[0])
        h = self.be.solve_up(self.sub, s_local, nrhs, t_root)
        h_all = self.comm.all_gather(h)                      # the one solve-time collective
        t_all = self.be.solve_top(self.top, _stack(h_all), t_root)
        t_mine = t_all[self.comm.rank]
        if hasattr(t_mine, "contiguous"):
            t_mine = t_mine.contiguous()
        else:
            t_mine = np.ascontiguousarray(t_mine)
        return self.be.solve_down(self.sub, t_mine)

    def root_R(self):
        return self.top.R(1)

    def close(self):
        for o in (self.sub, self.top):
            if hasattr(o, "close"):
                o.close()
