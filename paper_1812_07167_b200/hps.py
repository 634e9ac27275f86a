"""Thin Python binding of libhps.so (include/hps.h) — argument marshalling only.

Every step of the build and solve runs in the library's sm_100a kernels.  Arrays may be
numpy (host) or torch CUDA tensors (device); the library detects which.  There is no CPU
fallback: if libhps.so is missing or no CUDA device is present, calls raise.
"""
import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libhps.so")
_lib = None

HPS_ERRORS = {-1: "EINVAL", -2: "ESINGULAR", -3: "ENOMEM", -4: "ECUDA", -5: "ENOTKEPT"}


class HpsError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{HPS_ERRORS.get(code, code)}: {msg}")
        self.code = code


class hps_grid(C.Structure):
    _fields_ = [("x0", C.c_double), ("x1", C.c_double), ("y0", C.c_double), ("y1", C.c_double),
                ("nx", C.c_int32), ("ny", C.c_int32)]


class hps_c128(C.Structure):
    _fields_ = [("re", C.c_double), ("im", C.c_double)]


class hps_opts(C.Structure):
    _fields_ = [("keep_root_R", C.c_int32), ("keep_all_R", C.c_int32), ("device", C.c_int32),
                ("leaf_chunk", C.c_int32), ("profile", C.c_int32), ("leaf_mode", C.c_int32),
                ("boundary_basis", C.c_int32), ("n_gpus", C.c_int32), ("nccl_comm", C.c_void_p),
                ("stream", C.c_void_p), ("comm", C.c_void_p)]


SYMBOLS = ["hps_build", "hps_solve", "hps_export_R", "hps_export_leaf", "hps_box_nb", "hps_num_boxes",
           "hps_leaf_nodes", "hps_root_boundary_nodes", "hps_boundary_nodes_gl", "hps_boundary_nodes_glq",
           "hps_last_time_ms", "hps_last_launches",
           "hps_last_flops", "hps_leaf_path", "hps_set_profiling", "hps_kernel_stats", "hps_reset_stats", "hps_zinv_batched", "hps_zinv_timed", "hps_debug_ws_trace", "hps_rep_actions", "hps_plan_inverse", "hps_plan_set", "hps_plan_clear", "hps_plan_regime", "hps_solve_actions", "hps_plan_solve",
           "hps_build_actions", "hps_plan_build", "hps_fp64_peak", "hps_subtree_grid", "hps_build_top", "hps_solve_up",
           "hps_solve_down", "hps_solve_top", "hps_zgemm_batched", "hps_free", "hps_release_cache",
           "hps_set_cache_limit", "hps_cache_bytes", "hps_debug_set", "hps_debug_get", "hps_last_error",
           "hps_sync", "hps_nccl_unique_id", "hps_nccl_comm_init", "hps_nccl_comm_destroy", "hps_comm_wrap_nccl",
           "hps_vcomm_create", "hps_vcomm_rank", "hps_vcomm_destroy", "hps_comm_info", "hps_comm_selftest",
           "hps_comm_free", "hps_dist_plan"]

KCLASSES = ["zgemm_dmma", "zgj_panel", "zgj_small", "zgj_aux", "leaf_assemble", "layout", "zgj_fused", "leaf_gj", "zgemv"]


def lib():
    """Load libhps.so (raises if it was not built — there is no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built; run __graft_entry__.build()")
        L = C.CDLL(LIB_PATH)
        vp, dp, i32, i64 = C.c_void_p, C.c_void_p, C.c_int, C.c_int64
        L.hps_build.argtypes = [C.POINTER(hps_grid), i32, i32, C.c_double, hps_c128, dp, C.POINTER(hps_opts),
                                C.POINTER(vp)]
        L.hps_solve.argtypes = [vp, i32, dp, dp, dp]
        L.hps_export_R.argtypes = [vp, i64, dp]
        L.hps_export_leaf.argtypes = [vp, i64, dp, dp]
        L.hps_box_nb.argtypes = [vp, i64]
        L.hps_box_nb.restype = i64
        L.hps_num_boxes.argtypes = [vp]
        L.hps_num_boxes.restype = i64
        L.hps_leaf_nodes.argtypes = [C.POINTER(hps_grid), i32, dp, dp]
        L.hps_root_boundary_nodes.argtypes = [C.POINTER(hps_grid), i32, dp, dp, dp, dp]
        L.hps_boundary_nodes_gl.argtypes = [C.POINTER(hps_grid), i32, dp, dp, dp, dp]
        L.hps_boundary_nodes_glq.argtypes = [C.POINTER(hps_grid), i32, dp, dp, dp, dp]
        L.hps_last_time_ms.argtypes = [vp, i32]
        L.hps_last_time_ms.restype = C.c_double
        L.hps_last_launches.argtypes = [vp, i32]
        L.hps_last_launches.restype = i64
        L.hps_last_flops.argtypes = [vp, i32]
        L.hps_last_flops.restype = C.c_double
        L.hps_set_profiling.argtypes = [vp, i32]
        L.hps_leaf_path.argtypes = [vp]
        L.hps_kernel_stats.argtypes = [vp, i32, C.POINTER(i64), C.POINTER(C.c_double), C.POINTER(C.c_double),
                                       C.POINTER(C.c_double)]
        L.hps_reset_stats.argtypes = [vp]
        L.hps_zinv_batched.argtypes = [i32, i32, dp, dp]
        L.hps_zinv_timed.argtypes = [i32, i32, i32, dp, dp, i32, C.POINTER(C.c_double)]
        L.hps_debug_ws_trace.argtypes = [i32, dp]
        L.hps_rep_actions.argtypes = [C.POINTER(hps_grid), i32, i32, dp, dp]
        L.hps_plan_inverse.argtypes = [i32, i32, dp, dp, dp]
        L.hps_plan_set.argtypes = [i32, i32, i32]
        L.hps_plan_regime.argtypes = [i32, i32]
        L.hps_solve_actions.argtypes = [C.POINTER(hps_grid), i32, i32, i32, dp]
        L.hps_plan_solve.argtypes = [C.POINTER(hps_grid), i32, i32, i32, dp, dp, dp, dp]
        L.hps_build_actions.argtypes = [C.POINTER(hps_grid), i32, i32, i32, dp]
        L.hps_fp64_peak.argtypes = [C.POINTER(C.c_double)]
        L.hps_plan_build.argtypes = [C.POINTER(hps_grid), i32, i32, i32, dp, dp, dp, dp]
        L.hps_zgemm_batched.argtypes = [i32, i32, i32, i32, i32, dp, dp, dp, dp, hps_c128, hps_c128, i32,
                                        C.POINTER(C.c_double)]
        L.hps_subtree_grid.argtypes = [C.POINTER(hps_grid), i32, i64, C.POINTER(hps_grid), C.POINTER(C.c_int32),
                                       C.POINTER(C.c_int32)]
        L.hps_build_top.argtypes = [C.POINTER(hps_grid), i32, i32, C.c_double, hps_c128, i32, dp,
                                    C.POINTER(hps_opts), C.POINTER(vp)]
        L.hps_solve_up.argtypes = [vp, i32, dp, dp]
        L.hps_solve_down.argtypes = [vp, i32, dp, dp]
        L.hps_solve_top.argtypes = [vp, i32, dp, dp, dp]
        L.hps_free.argtypes = [vp]
        L.hps_set_cache_limit.argtypes = [i64]
        L.hps_sync.argtypes = [vp]
        L.hps_nccl_unique_id.argtypes = [C.c_char_p]
        L.hps_nccl_comm_init.argtypes = [i32, i32, C.c_char_p, C.POINTER(vp)]
        L.hps_nccl_comm_destroy.argtypes = [vp]
        L.hps_comm_wrap_nccl.argtypes = [vp, C.POINTER(vp)]
        L.hps_vcomm_create.argtypes = [i32, C.POINTER(vp)]
        L.hps_vcomm_rank.argtypes = [vp, i32, C.POINTER(vp)]
        L.hps_vcomm_destroy.argtypes = [vp]
        L.hps_comm_info.argtypes = [vp, C.POINTER(C.c_int), C.POINTER(C.c_int)]
        L.hps_comm_selftest.argtypes = [vp, i32]
        L.hps_comm_free.argtypes = [vp]
        L.hps_dist_plan.argtypes = [C.POINTER(hps_grid), i32, i32, i32, dp, i32]
        L.hps_cache_bytes.restype = i64
        L.hps_debug_set.argtypes = [C.c_char_p, i32]
        L.hps_debug_get.argtypes = [C.c_char_p, C.POINTER(C.c_int)]
        L.hps_last_error.restype = C.c_char_p
        _lib = L
    return _lib


def _check(rc):
    if rc != 0:
        raise HpsError(rc, lib().hps_last_error().decode())


def _ptr(a, nelem, what):
    """Device pointer of a torch tensor or host pointer of a numpy array (complex128)."""
    if a is None:
        return None
    if hasattr(a, "data_ptr"):   # torch tensor
        import torch
        if a.dtype != torch.complex128 or not a.is_contiguous():
            raise TypeError(f"{what}: need a contiguous complex128 tensor")
        if a.numel() != nelem:
            raise ValueError(f"{what}: expected {nelem} elements, got {a.numel()}")
        return a.data_ptr()
    if not isinstance(a, np.ndarray) or a.dtype != np.complex128 or not a.flags.c_contiguous:
        raise TypeError(f"{what}: need a C-contiguous numpy complex128 array")
    if a.size != nelem:
        raise ValueError(f"{what}: expected {nelem} elements, got {a.size}")
    return a.ctypes.data


def _torch_ready(*arrays, stream=None):
    """Device inputs must be complete when the library reads them on its own stream: if any
    argument is a CUDA torch tensor and the handle does not order its work on torch's stream,
    wait for torch's current stream first (a torch.stack still running on torch's
    stream was read by the library's non-blocking stream)."""
    if stream is not None:
        return
    for a in arrays:
        if a is not None and hasattr(a, "is_cuda") and a.is_cuda:
            import torch
            torch.cuda.current_stream(a.device).synchronize()
            return


def grid(x0, x1, y0, y1, nx, ny):
    return hps_grid(x0, x1, y0, y1, nx, ny)


def leaf_nodes(g, p):
    n = g.nx * g.ny * p * p
    X = np.zeros((g.nx * g.ny, p * p))
    Y = np.zeros_like(X)
    del n
    _check(lib().hps_leaf_nodes(C.byref(g), p, X.ctypes.data, Y.ctypes.data))
    return X, Y


def release_cache():
    """Return the cached large device blocks of freed handles to the driver (hps_release_cache)."""
    _check(lib().hps_release_cache())


def set_cache_limit(nbytes):
    """Opt in (nbytes > 0) to the cross-handle cache of large blocks, or disable it (0)."""
    _check(lib().hps_set_cache_limit(int(nbytes)))


def debug_get(name):
    v = C.c_int()
    _check(lib().hps_debug_get(name.encode(), C.byref(v)))
    return v.value


class debug_knobs:
    """Context manager: set library debug/tuning knobs (hps_debug_set), restore them on exit."""

    def __init__(self, **kw):
        self.kw = kw
        self.old = {}

    def __enter__(self):
        for k, v in self.kw.items():
            self.old[k] = debug_get(k)
            _check(lib().hps_debug_set(k.encode(), int(v)))
        return self

    def __exit__(self, *a):
        for k, v in self.old.items():
            lib().hps_debug_set(k.encode(), int(v))


def root_boundary_nodes(g, p, basis=0, q=None):
    """Root boundary nodes and outward normals; basis 1: the p - 2 Gauss-Legendre nodes per leaf
    edge; basis 2: q Gauss-Legendre nodes per leaf edge (q defaults to p - 2)."""
    q = p - 2 if q is None else q
    n = 2 * (g.nx + g.ny) * (q if basis == 2 else p - 2)
    X, Y, NX, NY = (np.zeros(n) for _ in range(4))
    if basis == 2:
        _check(lib().hps_boundary_nodes_glq(C.byref(g), q, X.ctypes.data, Y.ctypes.data, NX.ctypes.data,
                                            NY.ctypes.data))
        return X, Y, NX, NY
    fn = lib().hps_boundary_nodes_gl if basis == 1 else lib().hps_root_boundary_nodes
    _check(fn(C.byref(g), p, X.ctypes.data, Y.ctypes.data, NX.ctypes.data, NY.ctypes.data))
    return X, Y, NX, NY


def subtree_grid(g, depth, index):
    """(sub-grid, leaf i0, leaf j0) of the depth-`depth` box with heap index `index`."""
    sub = hps_grid()
    i0, j0 = C.c_int32(), C.c_int32()
    _check(lib().hps_subtree_grid(C.byref(g), depth, index, C.byref(sub), C.byref(i0), C.byref(j0)))
    return sub, i0.value, j0.value


def nb_of(g, p):
    return 2 * (g.nx + g.ny) * (p - 2)


def _empty_like_ref(ref, shape):
    if hasattr(ref, "data_ptr"):
        import torch
        return torch.empty(shape, dtype=torch.complex128, device=ref.device)
    return np.zeros(shape, complex)


def zgemm_batched(A, B, Cin=None, alpha=1.0, beta=0.0, cfg=-1, reps=1):
    """C = alpha A B + beta Cin through the library's DMMA kernel; returns (C, ms per call).
    A [batch, M, K], B [batch, K, N] (numpy complex128 or torch CUDA tensors)."""
    batch, M, K = A.shape
    N = B.shape[2]
    out = _empty_like_ref(A, (batch, M, N))
    ms = C.c_double()
    a, b = complex(alpha), complex(beta)
    _check(lib().hps_zgemm_batched(cfg, M, N, K, batch, _ptr(A, batch * M * K, "A"), _ptr(B, batch * K * N, "B"),
                                   _ptr(Cin, batch * M * N, "Cin"), _ptr(out, batch * M * N, "C"),
                                   hps_c128(a.real, a.imag), hps_c128(b.real, b.imag), reps, C.byref(ms)))
    return out, ms.value


def zinv_batched(A):
    """Batched inverse through the library's Gauss-Jordan kernels (A: [batch, n, n] complex128)."""
    A = np.ascontiguousarray(A, dtype=np.complex128)
    out = np.zeros_like(A)
    _check(lib().hps_zinv_batched(A.shape[-1], A.shape[0], A.ctypes.data, out.ctypes.data))
    return out


REGIMES = {1: "smem", 2: "fused", 3: "warp-specialised", 4: "blocked-implicit", 5: "blocked-explicit",
           6: "blocked-recursive", 7: "sequential-phase"}


def rep_actions(g, p):
    """[(n, nbox)] of every level's representative action: the leaf inverse, then the merge
    levels' interface inverses bottom-up (Table 1)."""
    n = np.zeros(64, np.int32)
    nb = np.zeros(64, np.int32)
    k = lib().hps_rep_actions(C.byref(g), p, 64, n.ctypes.data, nb.ctypes.data)
    if k < 0:
        _check(k)
    return [(int(n[i]), int(nb[i])) for i in range(k)]


def plan_inverse(n, nbox):
    """Measure the regimes for nbox n x n inverses and record the argmin of
    eps = ceil(nbox / theta_o) r; returns (regime, {regime: (eps_ms, r_ms, theta_o)})."""
    eps = np.zeros(8)
    r = np.zeros(8)
    th = np.zeros(8, np.int32)
    reg = lib().hps_plan_inverse(n, nbox, eps.ctypes.data, r.ctypes.data, th.ctypes.data)
    if reg < 0:
        _check(reg)
    return reg, {k: (float(eps[k]), float(r[k]), int(th[k])) for k in range(1, 8) if eps[k] >= 0}


def plan_problem(g, p):
    """Plan every level of a problem (the paper's per-level theta choice); returns table rows
    (level label, n, nbox, chosen regime, {regime: (eps, r, theta_o)})."""
    rows = []
    for i, (n, nb) in enumerate(rep_actions(g, p)):
        reg, tab = plan_inverse(n, nb)
        rows.append(("leaf" if i == 0 else f"merge {i}", n, nb, reg, tab))
    return rows


GEMM_KINDS = ["leaf u~ = Y s", "leaf u = Psi t (+ u~)", "Upsilon R33 h", "W^-1", "Gamma^tau R13 t~",
              "Phi t (+ t~)", "R33b R31a", "W = I - R33b R33a", "Phi^a = W^-1 X", "R^tau rows", "Phi^b",
              "W^-1 block-step update"]
_KEYS = ("level", "kind", "M", "N", "K", "batch", "cin")


def _actions(fn, *args):
    n = fn(*args, 0, None)
    if n < 0:
        _check(n)
    out = np.zeros((n, 7), dtype=np.int32)
    _check(0 if fn(*args, n, out.ctypes.data) == n else -1)
    return out


def fp64_peak():
    """Live FP64 tensor (DMMA m8n8k4) throughput of the current device, TFLOP/s (hps_fp64_peak)."""
    v = C.c_double()
    _check(lib().hps_fp64_peak(C.byref(v)))
    return v.value


def build_actions(g, p, keep_root_R=True):
    """The build's batched products per merge level (host only): list of dicts."""
    acts = _actions(lib().hps_build_actions, C.byref(g), p, int(keep_root_R))
    return [dict(zip(_KEYS, map(int, r))) for r in acts]


def plan_build(g, p, keep_root_R=True):
    """Time every build product's shape with each GEMM tile configuration and record the fastest."""
    n = len(build_actions(g, p, keep_root_R))
    acts = np.zeros((n, 7), dtype=np.int32)
    ch = np.zeros(n, dtype=np.int32)
    tr, tb = np.zeros(n), np.zeros(n)
    rc = lib().hps_plan_build(C.byref(g), p, int(keep_root_R), n, acts.ctypes.data, ch.ctypes.data, tr.ctypes.data,
                              tb.ctypes.data)
    if rc < 0:
        _check(rc)
    return [dict(zip(_KEYS, map(int, acts[i])), cfg=int(ch[i]), rule_ms=float(tr[i]), best_ms=float(tb[i]))
            for i in range(n)]


def solve_actions(g, p, nrhs):
    """Solve-stage representative actions (host only): list of dicts (level, kind, M, N, K, batch, cin)."""
    n = lib().hps_solve_actions(C.byref(g), p, nrhs, 0, None)
    if n < 0:
        _check(n)
    out = np.zeros((n, 7), dtype=np.int32)
    _check(0 if lib().hps_solve_actions(C.byref(g), p, nrhs, n, out.ctypes.data) == n else -1)
    keys = ("level", "kind", "M", "N", "K", "batch", "cin")
    return [dict(zip(keys, map(int, r))) for r in out]


def plan_solve(g, p, nrhs):
    """Time every solve action's shape with each GEMM tile configuration and record the fastest
    (PAPER.md:881-953 applied to the solve's matvecs); returns the actions with the chosen
    configuration (-1: the fixed rule) and the rule's / chosen time in ms."""
    n = lib().hps_solve_actions(C.byref(g), p, nrhs, 0, None)
    if n < 0:
        _check(n)
    acts = np.zeros((n, 7), dtype=np.int32)
    ch = np.zeros(n, dtype=np.int32)
    tr, tb = np.zeros(n), np.zeros(n)
    rc = lib().hps_plan_solve(C.byref(g), p, nrhs, n, acts.ctypes.data, ch.ctypes.data, tr.ctypes.data,
                              tb.ctypes.data)
    if rc < 0:
        _check(rc)
    keys = ("level", "kind", "M", "N", "K", "batch", "cin")
    return [dict(zip(keys, map(int, acts[i])), cfg=int(ch[i]), rule_ms=float(tr[i]), best_ms=float(tb[i]))
            for i in range(n)]


def plan_clear():
    lib().hps_plan_clear()


def plan_regime(n, nbox):
    return lib().hps_plan_regime(n, nbox)


def zinv_timed(A, mode=0, reps=3):
    """Batched inverse of A [batch, n, n] (numpy or torch CUDA) with kernel family `mode`
    (0 library choice, 1 fused, 2 blocked); returns (A^{-1}, mean ms per inversion)."""
    batch, n, _ = A.shape
    out = _empty_like_ref(A, (batch, n, n))
    ms = C.c_double()
    _check(lib().hps_zinv_timed(mode, n, batch, _ptr(A, batch * n * n, "A"), _ptr(out, batch * n * n, "out"), reps,
                                C.byref(ms)))
    return out, ms.value


def dist_plan(g, p, G, rank):
    """Host-only plan of the sharded top levels (hps_dist_plan): one dict per top depth."""
    info = np.zeros(8 * 32, np.int32)
    k = lib().hps_dist_plan(C.byref(g), p, G, rank, info.ctypes.data, 32)
    if k < 0:
        _check(k)
    keys = ("gs", "grank", "side", "n3", "n1", "ntau", "j0", "w")
    return [dict(zip(keys, (int(v) for v in info[8 * d:8 * d + 8]))) for d in range(k)]


class Comm:
    """A library communicator (hps_comm): NCCL (one process per GPU) or a virtual rank."""

    def __init__(self, handle, owner=None, nccl_comm=None):
        self.h = handle
        self._owner = owner          # keeps a virtual group alive
        self._nccl = nccl_comm       # raw ncclComm_t we created (destroyed with us)

    @staticmethod
    def nccl_unique_id():
        buf = C.create_string_buffer(128)
        _check(lib().hps_nccl_unique_id(buf))
        return buf.raw

    @classmethod
    def nccl(cls, nranks, rank, uid):
        """ncclCommInitRank on the current device + the library wrapper (collective)."""
        raw = C.c_void_p()
        _check(lib().hps_nccl_comm_init(nranks, rank, C.c_char_p(uid), C.byref(raw)))
        h = C.c_void_p()
        _check(lib().hps_comm_wrap_nccl(raw, C.byref(h)))
        return cls(h, nccl_comm=raw)

    def info(self):
        r, n = C.c_int(), C.c_int()
        _check(lib().hps_comm_info(self.h, C.byref(r), C.byref(n)))
        return r.value, n.value

    def selftest(self, gs):
        _check(lib().hps_comm_selftest(self.h, gs))

    def close(self):
        if getattr(self, "h", None):
            lib().hps_comm_free(self.h)
            self.h = None
        if getattr(self, "_nccl", None):
            lib().hps_nccl_comm_destroy(self._nccl)
            self._nccl = None


class VirtualGroup:
    """G virtual ranks in one process (host threads sharing one GPU): hps_vcomm_create."""

    def __init__(self, G):
        self.g = C.c_void_p()
        _check(lib().hps_vcomm_create(G, C.byref(self.g)))
        self.G = G

    def comm(self, rank):
        h = C.c_void_p()
        _check(lib().hps_vcomm_rank(self.g, rank, C.byref(h)))
        return Comm(h, owner=self)

    def close(self):
        if getattr(self, "g", None):
            lib().hps_vcomm_destroy(self.g)
            self.g = None


class Solver:
    """hps_build on construction; solve() is hps_solve.  With comm (a Comm of G ranks) the build
    and solve are sharded by subtree (c, s, u: this rank's rectangle; t: the whole root boundary)."""

    def __init__(self, g, p, kappa, eta, c, keep_root_R=True, keep_all_R=False, device=-1, leaf_chunk=0,
                 profile=False, leaf_mode=0, boundary_basis=0, comm=None, stream=None, q=None):
        """q: boundary nodes per leaf edge (p - 2; any 2 <= q <= p - 2 with boundary_basis 2)."""
        self.g, self.p = g, p
        self.comm = comm
        G, rank = 1, 0
        if comm is not None:
            rank, G = comm.info()
        self.G, self.rank = G, rank
        self.sub = subtree_grid(g, int(round(np.log2(G))), rank)[0] if G > 1 else g
        self.nleaf = self.sub.nx * self.sub.ny
        self.q = p - 2 if q is None else int(q)
        self.nt, self.ni = p * p - 4, (p - 2) ** 2
        self.nb_root = 2 * (g.nx + g.ny) * self.q
        mask = -1 if profile is True else int(profile)
        st = None
        if stream is not None:
            st = stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)
        opts = hps_opts(int(keep_root_R), int(keep_all_R), int(device), int(leaf_chunk), mask, int(leaf_mode),
                        int(boundary_basis), int(G), None, st, comm.h if comm is not None else None)
        eta = complex(eta)
        h = C.c_void_p()
        cp = _ptr(c, self.nleaf * p * p, "c_samples")
        self._c = c   # keep alive during the call
        self._stream = st
        _torch_ready(c, stream=st)
        _check(lib().hps_build(C.byref(g), p, self.q, float(kappa), hps_c128(eta.real, eta.imag), cp,
                               C.byref(opts), C.byref(h)))
        self.h = h

    def solve(self, s, t, u=None):
        """s: [nrhs][nleaf][q*q] or None, t: [nrhs][nb_root]; returns u [nrhs][nleaf][p*p-4]."""
        nrhs = int(t.shape[0])
        if u is None:
            if hasattr(t, "data_ptr"):
                import torch
                u = torch.empty((nrhs, self.nleaf, self.nt), dtype=torch.complex128, device=t.device)
            else:
                u = np.zeros((nrhs, self.nleaf, self.nt), complex)
        _torch_ready(s, t, u, stream=self._stream)
        _check(lib().hps_solve(self.h, nrhs, _ptr(s, nrhs * self.nleaf * self.ni, "s"),
                               _ptr(t, nrhs * self.nb_root, "t"), _ptr(u, nrhs * self.nleaf * self.nt, "u")))
        return u

    def sync(self):
        """Wait for a stream-ordered solve (hps_sync)."""
        _check(lib().hps_sync(self.h))

    def solve_up(self, s, nrhs, h_root=None):
        """Upward pass only; returns the root's outgoing particular data [nrhs][nb_root]."""
        if h_root is None:
            h_root = _empty_like_ref(s if s is not None else np.zeros(1, complex), (nrhs, self.nb_root))
        _torch_ready(s, h_root, stream=self._stream)
        _check(lib().hps_solve_up(self.h, nrhs, _ptr(s, nrhs * self.nleaf * self.ni, "s"),
                                  _ptr(h_root, nrhs * self.nb_root, "h_root")))
        return h_root

    def solve_down(self, t, u=None):
        nrhs = int(t.shape[0])
        if u is None:
            u = _empty_like_ref(t, (nrhs, self.nleaf, self.nt))
        _torch_ready(t, u, stream=self._stream)
        _check(lib().hps_solve_down(self.h, nrhs, _ptr(t, nrhs * self.nb_root, "t"),
                                    _ptr(u, nrhs * self.nleaf * self.nt, "u")))
        return u

    def nb(self, box):
        return lib().hps_box_nb(self.h, box)

    def R(self, box=1):
        n = self.nb(box)
        out = np.zeros((n, n), complex)
        _check(lib().hps_export_R(self.h, box, out.ctypes.data))
        return out

    def leaf_ops(self, leaf):
        Psi = np.zeros((self.nt, 4 * self.q), complex)
        Y = np.zeros((self.nt, self.ni), complex)
        _check(lib().hps_export_leaf(self.h, leaf, Psi.ctypes.data, Y.ctypes.data))
        return Psi, Y

    def time_ms(self, which):
        return lib().hps_last_time_ms(self.h, which)

    def launches(self, which):
        return lib().hps_last_launches(self.h, which)

    def flops(self, which):
        return lib().hps_last_flops(self.h, which)

    def leaf_path(self):
        """Leaf path the build took: 0 complex Schur (fused), 1 full B, 2 complex Schur (unfused),
        3 real interior elimination (hps.h leaf_mode)."""
        return lib().hps_leaf_path(self.h)

    def set_profiling(self, mask):
        _check(lib().hps_set_profiling(self.h, -1 if mask is True else int(mask)))

    def reset_stats(self):
        _check(lib().hps_reset_stats(self.h))

    def kernel_stats(self):
        """{class name: dict(launches, ms, flops, bytes)} accumulated since build / reset."""
        out = {}
        for k, name in enumerate(KCLASSES):
            n, ms, fl, by = C.c_int64(), C.c_double(), C.c_double(), C.c_double()
            _check(lib().hps_kernel_stats(self.h, k, C.byref(n), C.byref(ms), C.byref(fl), C.byref(by)))
            out[name] = dict(launches=n.value, ms=ms.value, flops=fl.value, bytes=by.value)
        return out

    def close(self):
        if getattr(self, "h", None):
            lib().hps_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class TopSolver:
    """hps_build_top: the merge tree above `depth` from the gathered subtree-root operators."""

    def __init__(self, g, p, kappa, eta, depth, R_sub, keep_root_R=True, device=-1, profile=False, boundary_basis=0):
        self.g, self.p, self.depth = g, p, depth
        sub, _, _ = subtree_grid(g, depth, 0)
        self.nb_sub = nb_of(sub, p)
        self.nb_root = nb_of(g, p)
        self.nsub = 1 << depth
        opts = hps_opts(int(keep_root_R), 0, int(device), 0, -1 if profile is True else int(profile), 0,
                        int(boundary_basis))
        eta = complex(eta)
        h = C.c_void_p()
        _torch_ready(R_sub)
        _check(lib().hps_build_top(C.byref(g), p, p - 2, float(kappa), hps_c128(eta.real, eta.imag), depth,
                                   _ptr(R_sub, self.nsub * self.nb_sub ** 2, "R_sub"), C.byref(opts), C.byref(h)))
        self.h = h

    def solve(self, h_sub, t_root, t_sub=None):
        """h_sub [2^depth][nrhs][nb_sub] (or None), t_root [nrhs][nb_root] -> t_sub [2^depth][nrhs][nb_sub]."""
        nrhs = int(t_root.shape[0])
        if t_sub is None:
            t_sub = _empty_like_ref(t_root, (self.nsub, nrhs, self.nb_sub))
        _torch_ready(h_sub, t_root, t_sub)
        _check(lib().hps_solve_top(self.h, nrhs, _ptr(h_sub, self.nsub * nrhs * self.nb_sub, "h_sub"),
                                   _ptr(t_root, nrhs * self.nb_root, "t_root"),
                                   _ptr(t_sub, self.nsub * nrhs * self.nb_sub, "t_sub")))
        return t_sub

    def R(self, box=1):
        n = lib().hps_box_nb(self.h, box)
        out = np.zeros((n, n), complex)
        _check(lib().hps_export_R(self.h, box, out.ctypes.data))
        return out

    def time_ms(self, which):
        return lib().hps_last_time_ms(self.h, which)

    def close(self):
        if getattr(self, "h", None):
            lib().hps_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
