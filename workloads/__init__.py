"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This module holds NO arithmetic of the method (no basis, no quadrature of
bilinear forms, no DtN, no multigrid).  It only produces the problem data a
user of the method hands to it -- the paper's problem statement
(Eq. `primal_elliptic`): per-element K, per-element
hybridized method tag and stabilisation tau, source samples f and Dirichlet
samples g_D -- for the five BASELINE.json configurations, plus seeded random
trace vectors for per-operator parity.

Sampling contract (shared with include/mgdtn.h, `mg_assemble_rhs`):
  * f is sampled per element at the tensor Gauss-Legendre points with
    nq = p + 4 points per direction, array shape [ny*nx][nq][nq], element id
    j*nx+i, point order [qy][qx] (qx runs along +x).
  * g_D is sampled on the 2*nx+2*ny boundary edges at nq Gauss points each,
    shape [2*nx+2*ny][nq], edge order: bottom H(i,0) i=0..nx-1, top H(i,ny),
    left V(0,j) j=0..ny-1, right V(nx,j); points along the edge's global
    orientation (+x for horizontal, +y for vertical).
The Gauss nodes are the sampling grid of the input format; they are computed
here with numpy's library routine (numpy.polynomial.legendre.leggauss).

Recipe (reading Q15 for the
random field, Q10 for the config-4 tile layout, Q9/Q21 for the SIPG-H penalty).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

HDG = 0
SIPG_H = 1
IIPG_H = 2
NIPG_H = 3
BLOCK_JACOBI = 0
CHEBYSHEV = 1


@dataclass
class Config:
    """One BASELINE.json configuration (index 1..5)."""
    index: int
    name: str
    n: int
    p: int
    nu: int
    smoother: int
    rtol: float = 1e-10
    seed_field: int = 0
    seed_vec: int = 0
    # free-form description
    desc: str = ""
    extras: dict = field(default_factory=dict)

    @property
    def ne(self) -> int:
        return self.n * self.n

    @property
    def trace_dofs(self) -> int:
        """Trace dofs as BASELINE.json counts them: all edges x (p+1)."""
        return 2 * self.n * (self.n + 1) * (self.p + 1)

    @property
    def h(self) -> float:
        return 1.0 / self.n


CONFIGS = {
    1: Config(1, "c1_8x8_p1_hdg_bj", n=8, p=1, nu=2, smoother=BLOCK_JACOBI,
              desc="2D Poisson unit square 8x8 quads, HDG p=1 tau=1 K=1, u=sin(pi x)sin(pi y), V(2,2) BJ"),
    2: Config(2, "c2_256x256_p4_hdg_cheb", n=256, p=4, nu=2, smoother=CHEBYSHEV,
              desc="2D Poisson 256x256 quads, HDG p=4 tau=1 K=1, u=sin(pi x)sin(pi y), V(2,2) Chebyshev"),
    3: Config(3, "c3_1024x1024_p2_darcy_bj", n=1024, p=2, nu=3, smoother=BLOCK_JACOBI,
              extras=dict(sigma=1.5, ell=16.0, clip=3.0),
              desc="heterogeneous Darcy 1024^2, HDG p=2, K=10^GRF(std 1.5, ell 16) clipped 1e6, f=1, V(3,3) BJ"),
    4: Config(4, "c4_512x512_p3_multinumerics_bj", n=512, p=3, nu=2, smoother=BLOCK_JACOBI,
              extras=dict(tile=64),
              desc="multinumerics 512^2 p=3, 64x64 tiles HDG(tau=1)/SIPG-H(10p^2K/h), K=10^U[-2,2] per tile"),
    5: Config(5, "c5_4096x4096_p4_scaling_cheb", n=4096, p=4, nu=2, smoother=CHEBYSHEV,
              extras=dict(sigma=1.0, ell=32.0, clip=None),
              desc="scaling run 4096^2 HDG p=4 tau=1, K=10^GRF(std 1, ell 32), f=1, V(2,2) Chebyshev"),
}
for _c in CONFIGS.values():
    _c.seed_field = 1000 + _c.index
    _c.seed_vec = 2000 + _c.index


def scaled_config(index: int, n: int) -> Config:
    """Same recipe as config `index` on an n x n mesh (parity-test sizes).

    Correlation lengths / tile sizes are scaled with n so the field keeps the
    same structure relative to the domain (tiles never smaller than 1 element).
    """
    base = CONFIGS[index]
    ex = dict(base.extras)
    if "ell" in ex:
        ex["ell"] = max(1.0, ex["ell"] * n / base.n)
    if "tile" in ex:
        ex["tile"] = max(1, ex["tile"] * n // base.n)
    c = Config(base.index, f"{base.name}@n{n}", n=n, p=base.p, nu=base.nu,
               smoother=base.smoother, rtol=base.rtol, desc=base.desc, extras=ex)
    c.seed_field = base.seed_field
    c.seed_vec = base.seed_vec
    return c


def config5_recipe(n: int) -> Config:
    """Config 5's recipe on an n x n mesh with its FULL-SIZE correlation length
    (32 elements, not scaled with n): the oracle-golden stand-in for config 5, whose
    4096^2 mesh is beyond the oracle's memory (tools/make_c5_golden.py)."""
    c = scaled_config(5, n)
    c.extras["ell"] = CONFIGS[5].extras["ell"]
    c.name = f"{CONFIGS[5].name}@n{n}_ell32"
    return c


def config3_recipe(n: int) -> Config:
    """Config 3's recipe on an n x n mesh with its FULL-SIZE correlation length (16
    elements, not scaled with n; std 1.5, clipped to a contrast of 1e6): the oracle-golden
    stand-in for config 3 under the GPU's readings, whose full-size oracle solve (1270
    PCG iterations on 6.3M dofs) takes the oracle ~4 h (tools/make_recipe_golden.py)."""
    c = scaled_config(3, n)
    c.extras["ell"] = CONFIGS[3].extras["ell"]
    c.name = f"{CONFIGS[3].name}@n{n}_ell16"
    return c


# --------------------------------------------------------------------------
# sampling grid of the input format
# --------------------------------------------------------------------------

def sample_points_1d(nq: int) -> np.ndarray:
    """Gauss-Legendre nodes on [0,1] (numpy library routine), ascending."""
    x, _ = np.polynomial.legendre.leggauss(nq)
    return 0.5 * (x + 1.0)


def n_samples(p: int) -> int:
    return p + 4


def element_sample_coords(n: int, p: int):
    """Physical coordinates of the f sample points, shape [n*n, nq, nq] each."""
    nq = n_samples(p)
    s = sample_points_1d(nq)
    h = 1.0 / n
    i = np.arange(n)
    j = np.arange(n)
    # X[e, qy, qx]
    xi = (i[:, None] + s[None, :]) * h          # [i, qx]
    yj = (j[:, None] + s[None, :]) * h          # [j, qy]
    X = np.broadcast_to(xi[None, :, None, :], (n, n, nq, nq))   # [j,i,qy,qx]
    Y = np.broadcast_to(yj[:, None, :, None], (n, n, nq, nq))
    return X.reshape(n * n, nq, nq), Y.reshape(n * n, nq, nq)


def boundary_sample_coords(n: int, p: int):
    """Coordinates of g_D samples, shape [4n, nq]: bottom, top, left, right."""
    nq = n_samples(p)
    s = sample_points_1d(nq)
    h = 1.0 / n
    t = (np.arange(n)[:, None] + s[None, :]) * h     # along-edge coordinate
    zeros = np.zeros_like(t)
    ones = np.ones_like(t)
    X = np.concatenate([t, t, zeros, ones], axis=0)
    Y = np.concatenate([zeros, ones, t, t], axis=0)
    return X, Y


# --------------------------------------------------------------------------
# random fields (reading Q15)
# --------------------------------------------------------------------------

def gaussian_random_field(n: int, sigma: float, ell: float, seed: int,
                          clip: float | None) -> np.ndarray:
    """Cell-centred n x n Gaussian field, squared-exponential covariance.

    White noise on a (2n)^2 periodic grid convolved (FFT) with exp(-r^2/ell^2);
    the self-convolution gives covariance ~ exp(-r^2/(2 ell^2)).  The n x n
    corner is standardised to empirical mean 0 / std sigma and clipped to
    [-clip, clip] if clip is given.  Returns g with shape [n*n] (id j*n+i).
    """
    rng = np.random.default_rng(seed)
    m = 2 * n
    w = rng.standard_normal((m, m))
    k = np.fft.fftfreq(m) * m                      # integer offsets, wrapped
    r2 = k[:, None] ** 2 + k[None, :] ** 2
    kern = np.exp(-r2 / (ell * ell))
    g = np.real(np.fft.ifft2(np.fft.fft2(w) * np.fft.fft2(kern)))[:n, :n]
    g = (g - g.mean()) / g.std() * sigma
    if clip is not None:
        g = np.clip(g, -clip, clip)
    return np.ascontiguousarray(g.reshape(n * n))


# --------------------------------------------------------------------------
# problem data per config
# --------------------------------------------------------------------------

@dataclass
class Problem:
    cfg: Config
    K: np.ndarray          # [ne] float64
    method: np.ndarray     # [ne] int8
    tau: np.ndarray        # [ne] float64
    f_qp: np.ndarray | None  # [ne, nq, nq] or None
    f_const: float
    gD_qp: np.ndarray | None  # [4n, nq] or None
    exact: object = None   # callable (x, y) -> u, or None


def _sin_sin(x, y):
    return np.sin(np.pi * x) * np.sin(np.pi * y)


def make_problem(cfg: Config, with_f: bool = True) -> Problem:
    n, p = cfg.n, cfg.p
    ne = n * n
    h = 1.0 / n
    method = np.full(ne, HDG, dtype=np.int8)
    tau = np.ones(ne)
    K = np.ones(ne)
    f_qp = None
    f_const = 0.0
    gD = None
    exact = None
    if cfg.index in (1, 2):
        if with_f:
            X, Y = element_sample_coords(n, p)
            f_qp = 2.0 * np.pi ** 2 * _sin_sin(X, Y)
        exact = _sin_sin
    elif cfg.index in (3, 5):
        ex = cfg.extras
        g = gaussian_random_field(n, ex["sigma"], ex["ell"], cfg.seed_field, ex["clip"])
        K = 10.0 ** g
        f_const = 1.0
    elif cfg.index == 4:
        tile = cfg.extras["tile"]
        nt = n // tile
        rng = np.random.default_rng(cfg.seed_field)
        gt = rng.uniform(-2.0, 2.0, size=(nt, nt))          # [J, I]
        jj, ii = np.divmod(np.arange(ne), n)
        TI, TJ = ii // tile, jj // tile
        K = 10.0 ** gt[TJ, TI]
        is_sipg = ((TI + TJ) % 2) == 1
        method[is_sipg] = SIPG_H
        tau = np.where(is_sipg, 10.0 * p * p * K / h, 1.0)
        def u4(x, y):
            return np.sin(2 * np.pi * x) * np.cos(np.pi * y)
        if with_f:
            X, Y = element_sample_coords(n, p)
            f_qp = 5.0 * np.pi ** 2 * K[:, None, None] * u4(X, Y)
        BX, BY = boundary_sample_coords(n, p)
        gD = u4(BX, BY)
    else:
        raise ValueError(cfg.index)
    return Problem(cfg, np.ascontiguousarray(K), method, np.ascontiguousarray(tau),
                   None if f_qp is None else np.ascontiguousarray(f_qp), f_const,
                   None if gD is None else np.ascontiguousarray(gD), exact)


def nonsymmetric_problem(cfg: Config, mix: str = "tiles") -> Problem:
    """The config's recipe (K field, f, g_D) with the nonsymmetric IPDG-H schemes
    (Eq. IPG_H) on its elements -- the SURVEY 8(f) f2 workload:
      mix = "nipg" / "iipg": that scheme everywhere;
      mix = "tiles": 8 x 8 tiles (at least 1 element) cycling HDG, SIPG-H, IIPG-H,
                     NIPG-H by (I + 2 J) mod 4 (multinumerics).
    tau = (p+1)(p+2) K_T / h on the IPDG-H elements (the kappa-scaled penalty of
    PAPER.md:1700-1701, 1391-1392), the config's tau on HDG elements."""
    pr = make_problem(cfg)
    n, p = cfg.n, cfg.p
    ne = n * n
    if mix in ("nipg", "iipg"):
        method = np.full(ne, NIPG_H if mix == "nipg" else IIPG_H, dtype=np.int8)
    else:
        tile = max(1, n // 8)
        jj, ii = np.divmod(np.arange(ne), n)
        method = np.array([HDG, SIPG_H, IIPG_H, NIPG_H], np.int8)[((ii // tile) + 2 * (jj // tile)) % 4]
    tau = np.where(method == HDG, np.where(pr.method == HDG, pr.tau, 1.0),
                   (p + 1) * (p + 2) * pr.K * n)
    return Problem(cfg, pr.K, method, np.ascontiguousarray(tau), pr.f_qp, pr.f_const, pr.gD_qp,
                   pr.exact)


def random_trace_vector(ndof: int, seed: int) -> np.ndarray:
    """x ~ U[-1,1] on every dof (reading Q19); Dirichlet entries are ignored
    by both implementations."""
    return np.random.default_rng(seed).uniform(-1.0, 1.0, size=ndof)


def trace_ndof(n: int, p: int) -> int:
    return 2 * n * (n + 1) * (p + 1)


# ---------------------------------------------------------------- element-block partitions
# (multi-GPU layout of include/mgdtn.h `mg_partition`: rank r = ry*px + rx holds the
# global elements [rx*bx, (rx+1)*bx) x [ry*by, (ry+1)*by), bx = n/px, by = n/py, in
# local element order jl*bx + il, and the edges of those elements in the local
# numbering of a bx x by mesh.)

def block_of(n: int, px: int, py: int, rank: int):
    """(ox, oy, bx, by) of a rank's element block of an n x n mesh."""
    bx, by = n // px, n // py
    return (rank % px) * bx, (rank // px) * by, bx, by


def block_edge_ids(n: int, px: int, py: int, rank: int) -> np.ndarray:
    """Global edge id of every local edge of a rank's block (local edge order)."""
    return block_edge_ids_at(n, *block_of(n, px, py, rank))


def block_edge_ids_at(n: int, ox: int, oy: int, bx: int, by: int) -> np.ndarray:
    """Global edge ids (n x n mesh) of the local edges of the block at (ox, oy), bx x by."""
    jh, ih = np.divmod(np.arange(bx * (by + 1)), bx)
    hid = (oy + jh) * n + (ox + ih)
    jv, iv = np.divmod(np.arange((bx + 1) * by), bx + 1)
    vid = n * (n + 1) + (oy + jv) * (n + 1) + (ox + iv)
    return np.concatenate([hid, vid]).astype(np.int64)


def block_dof_ids(n: int, p: int, px: int, py: int, rank: int) -> np.ndarray:
    """Global trace-dof id of every local dof of a rank's block."""
    return dof_ids(block_edge_ids(n, px, py, rank), p)


def dof_ids(edges: np.ndarray, p: int) -> np.ndarray:
    k1 = p + 1
    return (edges[:, None] * k1 + np.arange(k1)[None, :]).reshape(-1)


def block_problem(pr: Problem, px: int, py: int, rank: int) -> Problem:
    """A rank's share of a problem: its elements' K / method / tau / f samples and
    the g_D samples of its block's 2*bx + 2*by boundary edges (sides that are
    partition interfaces get zeros; the library ignores them)."""
    n = pr.cfg.n
    ox, oy, bx, by = block_of(n, px, py, rank)
    jj, ii = np.divmod(np.arange(bx * by), bx)
    ge = (oy + jj) * n + (ox + ii)
    f = None if pr.f_qp is None else np.ascontiguousarray(pr.f_qp[ge])
    gD = None
    if pr.gD_qp is not None:
        nq = pr.gD_qp.shape[1]
        gD = np.zeros((2 * bx + 2 * by, nq))
        if oy == 0:
            gD[:bx] = pr.gD_qp[ox:ox + bx]                                    # bottom
        if oy + by == n:
            gD[bx:2 * bx] = pr.gD_qp[n + ox:n + ox + bx]                      # top
        if ox == 0:
            gD[2 * bx:2 * bx + by] = pr.gD_qp[2 * n + oy:2 * n + oy + by]     # left
        if ox + bx == n:
            gD[2 * bx + by:] = pr.gD_qp[3 * n + oy:3 * n + oy + by]           # right
    return Problem(pr.cfg, np.ascontiguousarray(pr.K[ge]), np.ascontiguousarray(pr.method[ge]),
                   np.ascontiguousarray(pr.tau[ge]), f, pr.f_const, gD, pr.exact)


# ---------------------------------------------------------------- the paper's Example I
def example1_problem(n: int, p: int, tau_mode: str, method: int = HDG) -> Problem:
    """Example I: q = x y exp(x^2 y^3) on the unit square, K = 1,
    f = -Laplace(q) sampled on the f grid, strong Dirichlet data g_D = q.  One scheme
    on every element (`method`, default HDG); tau = 1 (tau_mode "1"), 1/h_min
    ("1/h_min") or (p+1)(p+2)/h_min ("(p+1)(p+2)/h_min", the NIPG-H tables,
    PAPER.md:1391-1392), h_min = 1/n."""
    X, Y = element_sample_coords(n, p)
    e = np.exp(X ** 2 * Y ** 3)
    f = -(e * (6 * X * Y ** 4 + 4 * X ** 3 * Y ** 7) + e * (12 * X ** 3 * Y ** 2 + 9 * X ** 5 * Y ** 5))
    BX, BY = boundary_sample_coords(n, p)
    gD = BX * BY * np.exp(BX ** 2 * BY ** 3)
    ne = n * n
    tv = {"1": 1.0, "1/h_min": float(n), "(p+1)(p+2)/h_min": float((p + 1) * (p + 2) * n)}
    tau = np.full(ne, tv[tau_mode])
    cfg = Config(0, f"exampleI_n{n}_p{p}_tau{tau_mode}_m{method}", n=n, p=p, nu=3,
                 smoother=BLOCK_JACOBI, rtol=1e-9)
    return Problem(cfg, np.ones(ne), np.full(ne, method, np.int8), tau, np.ascontiguousarray(f), 0.0,
                   np.ascontiguousarray(gD), lambda x, y: x * y * np.exp(x ** 2 * y ** 3))
