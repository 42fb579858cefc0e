"""Element-local hybridized solvers and their DtN maps (static condensation).

PAPER.md:184-199 (Eqs. `HDG`, `HDG_flux`), 230-233 (Eq. `SIPG_H`),
305-316 ("express the local volume unknowns u and/or q, element-by-element,
as a function of the skeletal unknowns lambda ... use the conservation
condition to construct a global linear system").

Element T = [x0, x0+h] x [y0, y0+h], volume space Q^p (reading Q1), trace
space P^p per edge, GLL nodal bases, exact Gauss quadrature (reading Q2).
Local edge order {0 bottom, 1 right, 2 top, 3 left}, each parameterised in
its global orientation (+x / +y, reading Q3).  Volume node index
i = b*(p+1) + a (a along x).  Local trace dof (f, a) -> f*(p+1) + a.

For each element the oracle solves the *full* local system literally as the
paper writes it (no staged elimination): HDG unknowns (u_x, u_y, q) from
Eq. HDG_local1 (tested with v = (phi_i, 0) and (0, phi_i)) and Eq.
HDG_local2 (tested with w = phi_i, *without* integrating -(u, grad w) by
parts), SIPG-H unknown q from Eq. SIPG_H.  The element's conservation rows
<u_hat . n, mu>_{dT} (Eq. `conservation`) are affine in lambda:
    flux_T(lambda, f) = b_T - S_T lambda,
so S_T = -d flux / d lambda (the discrete DtN map) and
b_T = flux_T(0, f).  Summing over elements gives A = sum G^T S_T G and
g = sum G^T b_T (Eq. 3.1).
"""
from __future__ import annotations

from functools import lru_cache

import numpy as np

from .basis import gauss, gll_nodes, lagrange, lagrange_deriv

HDG = 0
SIPG_H = 1
IIPG_H = 2      # s_f = 0  (Eq. IPG_H)
NIPG_H = 3      # s_f = -1
S_F = {SIPG_H: 1.0, IIPG_H: 0.0, NIPG_H: -1.0}

# outward unit normals of the local edges {bottom, right, top, left}
NORMALS = np.array([[0.0, -1.0], [1.0, 0.0], [0.0, 1.0], [-1.0, 0.0]])


def _edge_param(f: int, s: np.ndarray):
    """Reference coordinates (xi, eta) of local edge f at parameter s."""
    z = np.zeros_like(s)
    o = np.ones_like(s)
    return [(s, z), (o, s), (s, o), (z, s)][f]


class RefElement:
    """Reference-element (unit square) matrices for order p.  Hats: h = 1."""

    def __init__(self, p: int):
        self.p = p
        k = p + 1
        self.nv = k * k
        self.m = 4 * k
        self.nodes = gll_nodes(p)
        nodes = self.nodes
        # --- volume quadrature (exact for products of Q^p functions) ---
        xq, wq = gauss(p + 2)
        V = lagrange(nodes, xq)          # [q, a]
        dV = lagrange_deriv(nodes, xq)
        # phi_i(xi_qx, eta_qy) with i = b*k + a
        PHI = np.einsum("xa,yb->yxba", V, V).reshape(len(xq), len(xq), self.nv)
        PX = np.einsum("xa,yb->yxba", dV, V).reshape(len(xq), len(xq), self.nv)
        PY = np.einsum("xa,yb->yxba", V, dV).reshape(len(xq), len(xq), self.nv)
        W2 = np.outer(wq, wq)            # [qy, qx]
        self.M = np.einsum("yx,yxi,yxj->ij", W2, PHI, PHI)
        # Dx_ij = (d_x phi_j, phi_i)
        self.Dx = np.einsum("yx,yxj,yxi->ij", W2, PX, PHI)
        self.Dy = np.einsum("yx,yxj,yxi->ij", W2, PY, PHI)
        self.L = np.einsum("yx,yxi,yxj->ij", W2, PX, PX) + np.einsum("yx,yxi,yxj->ij", W2, PY, PY)
        # --- edge quadrature ---
        sq, ws = gauss(p + 2)
        MU = lagrange(nodes, sq)          # trace basis mu_a(s_q)
        nv, m = self.nv, self.m
        E = np.zeros((nv, m))
        F = np.zeros((nv, nv))
        Fx = np.zeros((nv, nv))
        Fy = np.zeros((nv, nv))
        H = np.zeros((m, m))
        N = np.zeros((nv, nv))
        Nl = np.zeros((nv, m))
        for f in range(4):
            xi, eta = _edge_param(f, sq)
            nx, ny = NORMALS[f]
            Vx = lagrange(nodes, xi)
            Vy = lagrange(nodes, eta)
            dVx = lagrange_deriv(nodes, xi)
            dVy = lagrange_deriv(nodes, eta)
            ph = np.einsum("qa,qb->qba", Vx, Vy).reshape(len(sq), nv)
            gx = np.einsum("qa,qb->qba", dVx, Vy).reshape(len(sq), nv)
            gy = np.einsum("qa,qb->qba", Vx, dVy).reshape(len(sq), nv)
            gn = nx * gx + ny * gy       # grad phi . n
            sl = slice(f * (p + 1), (f + 1) * (p + 1))
            E[:, sl] += np.einsum("q,qi,qa->ia", ws, ph, MU)
            F += np.einsum("q,qi,qj->ij", ws, ph, ph)
            Fx += nx * np.einsum("q,qi,qj->ij", ws, ph, ph)
            Fy += ny * np.einsum("q,qi,qj->ij", ws, ph, ph)
            H[sl, sl] += np.einsum("q,qa,qb->ab", ws, MU, MU)
            N += np.einsum("q,qj,qi->ij", ws, gn, ph)       # <grad phi_j . n, phi_i>
            Nl[:, sl] += np.einsum("q,qa,qi->ia", ws, MU, gn)  # <mu_a, grad phi_i . n>
        self.E, self.F, self.Fx, self.Fy, self.H, self.N, self.Nl = E, F, Fx, Fy, H, N, Nl
        self.Cx = E * np.repeat(NORMALS[:, 0], p + 1)[None, :]
        self.Cy = E * np.repeat(NORMALS[:, 1], p + 1)[None, :]
        # --- source quadrature on the input sampling grid (p+4 Gauss) ---
        sf, wf = gauss(p + 4)
        Vf = lagrange(nodes, sf)
        self.f_weights = np.outer(wf, wf)                         # [qy, qx]
        self.f_basis = np.einsum("xa,yb->yxba", Vf, Vf).reshape(len(sf), len(sf), nv)
        self.edge_f_weights = wf
        self.edge_f_basis = Vf                                     # [q, a]
        self.Hhat1 = np.einsum("q,qa,qb->ab", ws, MU, MU)          # 1D edge mass


@lru_cache(maxsize=None)
def ref(p: int) -> RefElement:
    return RefElement(p)


def _local_systems_hdg(R: RefElement, K: np.ndarray, tau: np.ndarray, h: float):
    """Full HDG local system per element (batched over elements).

    Z z = Y lambda + [0; 0; f_w],  flux = Bf z - tau H lambda,
    z = (u_x, u_y, q):
      Eq. HDG_local1:  (K^-1 u, v) - (q, div v) + <lambda, v.n> = 0
      Eq. HDG_local2:  -(u, grad w) + <u.n + tau (q - lambda), w> = (f, w)
    Physical matrices: M = h^2 Mhat, Dx = h Dxhat, boundary terms = h * hat.
    """
    ne = len(K)
    nv, m = R.nv, R.m
    M = h * h * R.M
    Dx, Dy = h * R.Dx, h * R.Dy
    Fx, Fy, F = h * R.Fx, h * R.Fy, h * R.F
    E, Cx, Cy, H = h * R.E, h * R.Cx, h * R.Cy, h * R.H
    Z = np.zeros((ne, 3 * nv, 3 * nv))
    Y = np.zeros((ne, 3 * nv, m))
    Bf = np.zeros((ne, m, 3 * nv))
    a, b, c = slice(0, nv), slice(nv, 2 * nv), slice(2 * nv, 3 * nv)
    Kinv = (1.0 / K)[:, None, None]
    t = tau[:, None, None]
    Z[:, a, a] = Kinv * M
    Z[:, b, b] = Kinv * M
    Z[:, a, c] = -Dx.T           # -(q, d_x phi_i) = -(Dx^T q)_i
    Z[:, b, c] = -Dy.T
    Z[:, c, a] = -Dx.T + Fx      # -(u_x, d_x w_i) + <u_x n_x, w_i>
    Z[:, c, b] = -Dy.T + Fy
    Z[:, c, c] = t * F           # tau <q, w>
    Y[:, a, :] = -Cx             # -<lambda, v.n>
    Y[:, b, :] = -Cy
    Y[:, c, :] = t * E           # + tau <lambda, w>
    Bf[:, :, a] = Cx.T           # <u.n, mu>
    Bf[:, :, b] = Cy.T
    Bf[:, :, c] = t * E.T        # tau <q, mu>
    tH = t * H                   # tau <lambda, mu>
    return Z, Y, Bf, tH


def _local_systems_ipdg(R: RefElement, K: np.ndarray, tau: np.ndarray, h: float,
                        s_f: float = 1.0):
    """Hybridized IPDG local system (Eq. IPG_H) per element;
    s_f = 1 SIPG-H (Eq. SIPG_H), 0 IIPG-H, -1 NIPG-H.

    (K grad q, grad w) - s_f <q - lambda, K grad w.n> - <K grad q.n, w>
        + <tau (q - lambda), w> = (f, w)
    flux (Eq. IPDG_flux): u_hat.n = -K grad q.n + tau (q - lambda).
    With N_ij = <grad phi_j.n, phi_i>, Nl_(i,(f,a)) = <mu_a, grad phi_i.n_f>:
    <K grad q.n, w_i> = K (N q)_i,  s_f <q, K grad w_i.n> = s_f K (N^T q)_i,
    s_f <lambda, K grad w_i.n> = s_f K (Nl lambda)_i.
    Physical: L = Lhat, N = Nhat, Nl = Nlhat, F = h Fhat, E = h Ehat.
    """
    Kb = K[:, None, None]
    t = tau[:, None, None]
    L, N, Nl = R.L, R.N, R.Nl
    F, E, H = h * R.F, h * R.E, h * R.H
    Z = Kb * (L - s_f * N.T - N) + t * F
    Y = t * E - s_f * Kb * Nl
    Bf = -Kb * Nl.T + t * E.T
    tH = t * H
    return Z, Y, Bf, tH


def _local_systems_sipg(R, K, tau, h):
    return _local_systems_ipdg(R, K, tau, h, S_F[SIPG_H])


def _builders():
    """(method code, local-system builder) for every hybridized scheme."""
    out = [(HDG, _local_systems_hdg)]
    for code, sf in S_F.items():
        out.append((code, lambda R, K, tau, h, sf=sf: _local_systems_ipdg(R, K, tau, h, sf)))
    return out


def element_dtn(p: int, K, method, tau, h: float, chunk: int = 2048):
    """Element DtN maps S_T [ne, m, m] (Schur complement of the local solve).

    S_T = tau H - Bf Z^{-1} Y  (= -d flux_T / d lambda), per element.  Row a
    is the flux moment on local dof a; nonsymmetric for IIPG-H / NIPG-H.
    """
    R = ref(p)
    K = np.asarray(K, float)
    tau = np.asarray(tau, float)
    method = np.asarray(method)
    ne = len(K)
    S = np.empty((ne, R.m, R.m))
    for mcode, builder in _builders():
        idx = np.nonzero(method == mcode)[0]
        for s in range(0, len(idx), chunk):
            ids = idx[s:s + chunk]
            Z, Y, Bf, tH = builder(R, K[ids], tau[ids], h)
            S[ids] = tH - Bf @ np.linalg.solve(Z, Y)
    return S


def load_vectors(p: int, h: float, f_qp):
    """f_w,i = (f, phi_i)_T from the input samples (p+4 Gauss points)."""
    R = ref(p)
    return h * h * np.einsum("yx,eyx,yxi->ei", R.f_weights, f_qp, R.f_basis)


def element_rhs(p: int, K, method, tau, h: float, f_qp=None, f_const=0.0,
                chunk: int = 2048):
    """b_T = flux_T(lambda = 0, f) = Bf Z^{-1} [0; 0; f_w] per element."""
    R = ref(p)
    K = np.asarray(K, float)
    tau = np.asarray(tau, float)
    method = np.asarray(method)
    ne = len(K)
    if f_qp is None:
        fw = np.broadcast_to(f_const * h * h * np.einsum("yx,yxi->i", R.f_weights, R.f_basis),
                             (ne, R.nv))
    else:
        fw = load_vectors(p, h, f_qp)
    b = np.empty((ne, R.m))
    nv = R.nv
    for mcode, builder in _builders():
        idx = np.nonzero(method == mcode)[0]
        for s in range(0, len(idx), chunk):
            ids = idx[s:s + chunk]
            Z, Y, Bf, tH = builder(R, K[ids], tau[ids], h)
            rhs = np.zeros((len(ids), Z.shape[1]))
            rhs[:, Z.shape[1] - nv:] = fw[ids]          # q-equation rows are last
            b[ids] = np.einsum("eij,ej->ei", Bf, np.linalg.solve(Z, rhs[..., None])[..., 0])
    return b


def recover_q(p: int, K, method, tau, h: float, lam_T, f_qp=None, f_const=0.0):
    """Volume recovery q_T (nodal coefficients) from the element traces lam_T.

    PAPER.md:310-312: "the local volume unknowns can be recovered in an
    element-by-element fashion completely independent of each other".
    """
    R = ref(p)
    K = np.asarray(K, float)
    tau = np.asarray(tau, float)
    method = np.asarray(method)
    ne = len(K)
    nv = R.nv
    if f_qp is None:
        fw = np.broadcast_to(f_const * h * h * np.einsum("yx,yxi->i", R.f_weights, R.f_basis),
                             (ne, nv))
    else:
        fw = load_vectors(p, h, f_qp)
    q = np.empty((ne, nv))
    for mcode, builder in _builders():
        idx = np.nonzero(method == mcode)[0]
        if len(idx) == 0:
            continue
        Z, Y, Bf, tH = builder(R, K[idx], tau[idx], h)
        rhs = np.einsum("eij,ej->ei", Y, lam_T[idx])
        rhs[:, Z.shape[1] - nv:] += fw[idx]
        z = np.linalg.solve(Z, rhs[..., None])[..., 0]
        q[idx] = z[:, Z.shape[1] - nv:]
    return q
