"""Seeded synthetic inputs for the HPS workloads (BASELINE.json configs 1-5).

This module is shared by the product path (bench.py) and the tests that feed
the oracle.  It holds NONE of the method's arithmetic: no discretisation, no
operator, no solve — only the PROBLEM DATA of eq. (1),
evaluated at coordinates the caller supplies:

* the coefficient c(x), the body load s(x), the impedance data t(x);
* the exact plane wave u = exp(i kappa d.x) and its Robin trace
  t = du/dnu + i eta u (used as boundary data, configs 1-2);
* SplitMix64 counter-based random numbers (SURVEY.md §8(d) recipe):
  uniform = (x >> 11) * 2^-53, complex normal CN(0,1) by Box-Muller
  (re, im ~ N(0, 1/2)).

Draw order per config: bumps (cx, cy[, a]) from the c-seed;
s as ``for r, for leaf (iy, ix), for interior node`` from the s-seed; t as
``for r, for boundary node`` (canonical [S,E,N,W]) from the t-seed.

Readings: Q13 "10 Chebyshev points per wavelength" means
kappa = 2 pi p / (10 h) with h the leaf side; Q14 a bump of "width 0.05" is
exp(-|x - x_k|^2 / (2 * 0.05^2)).
"""
from dataclasses import dataclass, field
import math

import numpy as np

_GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def splitmix64(seed, n, offset=0):
    """Outputs offset..offset+n-1 of SplitMix64 seeded with ``seed`` (uint64 array)."""
    with np.errstate(over="ignore"):
        i = np.arange(offset + 1, offset + n + 1, dtype=np.uint64)
        z = np.uint64(seed) + i * _GOLDEN
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        z = z ^ (z >> np.uint64(31))
    return z


def uniform(seed, n, offset=0):
    """U[0,1) doubles: (x >> 11) * 2^-53."""
    return (splitmix64(seed, n, offset) >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


def complex_normal(seed, n, offset=0):
    """CN(0,1): Box-Muller on consecutive uniform pairs, re, im ~ N(0, 1/2)."""
    u = uniform(seed, 2 * n, 2 * offset).reshape(n, 2)
    r = np.sqrt(-2.0 * np.log1p(-u[:, 0]))      # 1 - u1 in (0, 1]
    th = 2.0 * math.pi * u[:, 1]
    return (r * np.cos(th) + 1j * r * np.sin(th)) / math.sqrt(2.0)


@dataclass
class Config:
    name: str
    x0: float
    x1: float
    y0: float
    y1: float
    nx: int
    ny: int
    p: int
    kappa: float
    eta: complex
    nrhs: int
    c_kind: str                 # "one" | "dip" | "bumps"
    s_kind: str                 # "zero" | "gauss" | "cn"
    t_kind: str                 # "plane" | "cn"
    n_bumps: int = 0
    bump_amp: float = 0.3       # fixed amplitude, or max |a| when bump_random_amp
    bump_random_amp: bool = False
    seeds: tuple = (0, 0, 0)    # (c, s, t)
    theta: float = 0.3          # plane-wave angle
    n_gpus: tuple = (1,)
    extra: dict = field(default_factory=dict)

    @property
    def q(self):
        return self.p - 2

    @property
    def nleaf(self):
        return self.nx * self.ny

    @property
    def n_unique(self):
        """DOF N = unique nodes (reading Q16): q (nx ny q + (nx+1) ny + nx (ny+1))."""
        q, nx, ny = self.q, self.nx, self.ny
        return q * (nx * ny * q + (nx + 1) * ny + nx * (ny + 1))

    @property
    def nb_root(self):
        return 2 * (self.nx + self.ny) * self.q


def _ppw_kappa(p, h):
    """Reading Q13: 10 Chebyshev points per wavelength, lambda = 10 h / p."""
    return 2.0 * math.pi * p / (10.0 * h)


CONFIGS = {
    1: Config("C1: unit square 4x4 leaves p=8 kappa=10 plane wave", 0, 1, 0, 1, 4, 4, 8, 10.0, 10.0, 1,
              "one", "zero", "plane"),
    2: Config("C2: unit square 32x32 leaves p=16 kappa=40pi", 0, 1, 0, 1, 32, 32, 16, 40 * math.pi,
              40 * math.pi, 1, "dip", "gauss", "plane"),
    3: Config("C3: unit square 128x128 leaves p=16 10ppw 64 RHS", 0, 1, 0, 1, 128, 128, 16,
              _ppw_kappa(16, 1 / 128), _ppw_kappa(16, 1 / 128), 64, "bumps", "cn", "cn", n_bumps=8,
              seeds=(31, 32, 33), n_gpus=(1, 2, 4, 8)),
    4: Config("C4: unit square 256x256 leaves p=16 10ppw 16 RHS", 0, 1, 0, 1, 256, 256, 16,
              _ppw_kappa(16, 1 / 256), _ppw_kappa(16, 1 / 256), 16, "bumps", "cn", "cn", n_bumps=32,
              seeds=(41, 42, 43), n_gpus=(1, 2, 4, 8)),
    5: Config("C5: [0,2]x[0,1] 1024x512 leaves p=16 10ppw 128 RHS", 0, 2, 0, 1, 1024, 512, 16,
              _ppw_kappa(16, 1 / 512), _ppw_kappa(16, 1 / 512), 128, "bumps", "cn", "cn", n_bumps=64,
              bump_random_amp=True, seeds=(51, 52, 53), n_gpus=(8,)),
}


def bumps(cfg):
    """Bump centres (and amplitudes) drawn from the c-seed: cx, cy[, a] per bump."""
    per = 3 if cfg.bump_random_amp else 2
    u = uniform(cfg.seeds[0], per * cfg.n_bumps).reshape(cfg.n_bumps, per)
    cx = cfg.x0 + (cfg.x1 - cfg.x0) * u[:, 0]
    cy = cfg.y0 + (cfg.y1 - cfg.y0) * u[:, 1]
    a = (2 * u[:, 2] - 1) * cfg.bump_amp if cfg.bump_random_amp else np.full(cfg.n_bumps, cfg.bump_amp)
    return cx, cy, a


def c_at(cfg, X, Y):
    """c(x) at coordinates X, Y (any shape) -> complex array."""
    if cfg.c_kind == "one":
        return np.ones_like(X, dtype=complex)
    if cfg.c_kind == "dip":   # C2: 1 - 0.5 exp(-160 |x - (0.5, 0.5)|^2)
        return (1.0 - 0.5 * np.exp(-160.0 * ((X - 0.5) ** 2 + (Y - 0.5) ** 2))).astype(complex)
    if cfg.c_kind == "bumps":
        cx, cy, a = bumps(cfg)
        out = np.ones_like(X, dtype=float)
        w2 = 2.0 * 0.05 ** 2
        for k in range(cfg.n_bumps):
            out = out + a[k] * np.exp(-((X - cx[k]) ** 2 + (Y - cy[k]) ** 2) / w2)
        return out.astype(complex)
    raise ValueError(cfg.c_kind)


def s_interior(cfg, Xi, Yi, nrhs=None):
    """Body load at interior nodes.  Xi, Yi: [nleaf natural][q*q] coordinates.
    Returns [nrhs][nleaf][q*q]."""
    nrhs = cfg.nrhs if nrhs is None else nrhs
    shape = (nrhs,) + Xi.shape
    if cfg.s_kind == "zero":
        return np.zeros(shape, complex)
    if cfg.s_kind == "gauss":   # C2: exp(-500 |x - (0.3, 0.6)|^2)
        one = np.exp(-500.0 * ((Xi - 0.3) ** 2 + (Yi - 0.6) ** 2)).astype(complex)
        return np.broadcast_to(one, shape).copy()
    if cfg.s_kind == "cn":
        return complex_normal(cfg.seeds[1], int(np.prod(shape))).reshape(shape)
    raise ValueError(cfg.s_kind)


def plane_wave(kappa, theta, X, Y):
    d = (math.cos(theta), math.sin(theta))
    return np.exp(1j * kappa * (d[0] * X + d[1] * Y))


def plane_wave_robin(kappa, eta, theta, X, Y, NX, NY):
    """t = du/dnu + i eta u for u = exp(i kappa d.x): du/dnu = i kappa (nu.d) u."""
    u = plane_wave(kappa, theta, X, Y)
    nd = NX * math.cos(theta) + NY * math.sin(theta)
    return (1j * kappa * nd + 1j * eta) * u


def t_boundary(cfg, Xb, Yb, NXb, NYb, nrhs=None):
    """Root impedance data [nrhs][nb_root] at the canonical boundary nodes."""
    nrhs = cfg.nrhs if nrhs is None else nrhs
    if cfg.t_kind == "plane":
        one = plane_wave_robin(cfg.kappa, cfg.eta, cfg.theta, Xb, Yb, NXb, NYb)
        return np.broadcast_to(one, (nrhs, Xb.size)).copy()
    if cfg.t_kind == "cn":
        return complex_normal(cfg.seeds[2], nrhs * Xb.size).reshape(nrhs, Xb.size)
    raise ValueError(cfg.t_kind)


def interior_of(p, A):
    """Select the (p-2)^2 interior tensor nodes (x fastest) of [..., p*p] arrays."""
    A = A.reshape(A.shape[:-1] + (p, p))
    return A[..., 1:p - 1, 1:p - 1].reshape(A.shape[:-2] + ((p - 2) ** 2,))


def make_inputs(cfg, X, Y, Xb, Yb, NXb, NYb, nrhs=None):
    """Everything one workload needs, given node coordinates from the caller:
    X, Y [nleaf][p*p] (leaf tensor nodes), Xb.. root boundary nodes and normals.
    Returns (c [nleaf][p*p], s [nrhs][nleaf][q*q], t [nrhs][nb_root])."""
    c = c_at(cfg, X, Y)
    s = s_interior(cfg, interior_of(cfg.p, X), interior_of(cfg.p, Y), nrhs)
    t = t_boundary(cfg, Xb, Yb, NXb, NYb, nrhs)
    return c, s, t


# ---------------------------------------------------------------------------
# The paper's own experiment (Sec. 4): unit square, kappa = 16,
# c = exp(-8[(x-.5)^2 + (y-.5)^2]) (reading Q17), exact u = exp(i 2 pi kappa x) exp(i 2 pi kappa y),
# s = -Lap u - kappa^2 c u = (8 pi^2 kappa^2 - kappa^2 c) u, t = du/dnu + i eta u, eta = kappa.
# ---------------------------------------------------------------------------
PAPER_KAPPA = 16.0


def paper_c(X, Y):
    return np.exp(-8.0 * ((X - 0.5) ** 2 + (Y - 0.5) ** 2)).astype(complex)


def paper_u(X, Y, kappa=PAPER_KAPPA):
    return np.exp(2j * math.pi * kappa * X) * np.exp(2j * math.pi * kappa * Y)


def paper_s(X, Y, kappa=PAPER_KAPPA):
    return (8.0 * math.pi ** 2 * kappa ** 2 - kappa ** 2 * paper_c(X, Y)) * paper_u(X, Y, kappa)


def paper_t(X, Y, NX, NY, kappa=PAPER_KAPPA, eta=PAPER_KAPPA):
    du = 2j * math.pi * kappa * paper_u(X, Y, kappa)   # d/dx u = d/dy u
    return NX * du + NY * du + 1j * eta * paper_u(X, Y, kappa)
