"""DtN-based geometric multigrid hierarchy and V-cycle (Section 3).

Levels are numbered k = N (finest, order p) down to 1 (coarsest).  Every
operator is a global sparse matrix over the *free* trace dofs of its level,
built literally from the paper's formulas:

  p-coarsening, for p > 1:
      I_N = J_N, Q_{N-1} = J_N^*, A_{N-1} = J_N^* A_N J_N      (Eq. ANm1)
  h-coarsening by 2x2 agglomeration:
      E_k = E_{k,I} (+) E_{k,B}, M_{k-1} subset M_{k,B}        (Eq. 3.2)
      I_k = [-A_II^-1 A_IB J_k ; J_k]                          (Eq. 3.3)
      Q_{k-1} = [-J_k^* A_BI A_II^-1 , J_k^*]                  (Eq. 3.5)
      A_{k-1} = J_k^*(A_BB - A_BI A_II^-1 A_IB) J_k            (Eq. Akm1)
  local correction T_k = [A_II^-1 0; 0 0]                      (Eq. 3.11)
  V-cycle = Algorithm 1, B_1 = A_1^-1 by a direct solver.

Readings: adjoints are matrix transposes (Q5); J_k is nodal P1
interpolation along straight macro-edges split in halves (O7); coarse
macro-edges on dOmega carry no dofs (Dirichlet); A_II^-1 is formed per
macro-element block because A_II is block diagonal across macros
("completely local to each macro-element"); smoothers:
edge block-Jacobi and Chebyshev on D_B^-1 A with
bounds [lambda_max/30, lambda_max] (Q8, Q11).
"""
from __future__ import annotations

import numpy as np
import scipy.linalg as sla
import scipy.sparse as sp

from . import mesh
from .basis import gll_nodes

BLOCK_JACOBI = 0
CHEBYSHEV = 1
LUSGS = 2       # symmetric block Gauss-Seidel on edge blocks, 4-colour order


# --------------------------------------------------------------------------
# injections J
# --------------------------------------------------------------------------

def p_injection_full(n: int, p: int) -> sp.csr_matrix:
    """J_N: P^1 -> P^p on every edge (nodal interpolation at GLL nodes).

    Fine dof (e, a) = (1 - s_a) * coarse (e, 0) + s_a * coarse (e, 1).
    """
    s = gll_nodes(p)
    E = mesh.n_edges(n)
    k = p + 1
    rows, cols, vals = [], [], []
    for a in range(k):
        rows += [np.arange(E) * k + a] * 2
        cols += [np.arange(E) * 2 + 0, np.arange(E) * 2 + 1]
        vals += [np.full(E, 1.0 - s[a]), np.full(E, s[a])]
    return sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                         shape=(E * k, E * 2)).tocsr()


def p_coarsen_element(S: np.ndarray, p: int) -> np.ndarray:
    """Element form of Eq. ANm1: S^(1)_T = J_p^T S_T J_p for
    a batch S [ne, 4(p+1), 4(p+1)] of order-p element DtN maps, J_p the
    per-edge P1 -> P^p nodal injection of p_injection_full (local dof f*(p+1)+a
    <- (1 - s_a) c_(f,0) + s_a c_(f,1)).  Summed over elements this is the
    global J_N^T A_N J_N (pinned against it in tests/test_oracle_multigrid.py).
    """
    s = gll_nodes(p)
    j1 = np.stack([1.0 - s, s], axis=1)            # [(p+1), 2]
    J = np.kron(np.eye(4), j1)                     # [4(p+1), 8]
    return np.einsum("ai,eab,bj->eij", J, S, J)


def h_injection_full(n: int) -> sp.csr_matrix:
    """J_k: coarse P1 macro-edge functions -> fine P1 on its two halves.

    Coarse H_c(I,J) = fine H(2I,2J) u H(2I+1,2J); V_c(I,J) = V(2I,2J) u V(2I,2J+1)
    (first half = lower coordinate).  Nodal evaluation at the fine nodes:
    first half gets (c0, (c0+c1)/2), second half ((c0+c1)/2, c1).
    """
    nc = n // 2
    rows, cols, vals = [], [], []
    I, J = np.meshgrid(np.arange(nc), np.arange(nc + 1), indexing="xy")
    I, J = I.ravel(), J.ravel()
    halves = []
    # horizontal coarse edges
    ce = mesh.hedge(nc, I, J)
    halves.append((ce, mesh.hedge(n, 2 * I, 2 * J), mesh.hedge(n, 2 * I + 1, 2 * J)))
    I, J = np.meshgrid(np.arange(nc + 1), np.arange(nc), indexing="xy")
    I, J = I.ravel(), J.ravel()
    ce = mesh.vedge(nc, I, J)
    halves.append((ce, mesh.vedge(n, 2 * I, 2 * J), mesh.vedge(n, 2 * I, 2 * J + 1)))
    for ce, f0, f1 in halves:
        c0, c1 = 2 * ce, 2 * ce + 1
        entries = [(2 * f0, c0, 1.0), (2 * f0 + 1, c0, 0.5), (2 * f0 + 1, c1, 0.5),
                   (2 * f1, c0, 0.5), (2 * f1, c1, 0.5), (2 * f1 + 1, c1, 1.0)]
        for r, c, v in entries:
            rows.append(r)
            cols.append(c)
            vals.append(np.full(len(r), v))
    return sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                         shape=(mesh.n_edges(n) * 2, mesh.n_edges(nc) * 2)).tocsr()


def interior_edge_mask(n: int) -> np.ndarray:
    """Fine edges interior to the 2x2 macro-elements of the coarser level:
    vertical lines x = odd, horizontal lines y = odd (E_{k,I})."""
    mask = np.zeros(mesh.n_edges(n), dtype=bool)
    i = np.arange(n)
    odd = np.arange(1, n, 2)
    J, I = np.meshgrid(odd, i, indexing="ij")
    mask[mesh.hedge(n, I.ravel(), J.ravel())] = True
    J, I = np.meshgrid(i, odd, indexing="ij")
    mask[mesh.vedge(n, I.ravel(), J.ravel())] = True
    return mask


def macro_interior_edges(n: int) -> np.ndarray:
    """[nmacro, 4] interior fine edge ids per macro (I,J), macro id J*nc+I."""
    nc = n // 2
    J, I = np.divmod(np.arange(nc * nc), nc)
    return np.stack([mesh.hedge(n, 2 * I, 2 * J + 1), mesh.hedge(n, 2 * I + 1, 2 * J + 1),
                     mesh.vedge(n, 2 * I + 1, 2 * J), mesh.vedge(n, 2 * I + 1, 2 * J + 1)], axis=1)


# --------------------------------------------------------------------------
# levels
# --------------------------------------------------------------------------

class Level:
    def __init__(self, n, p, A, free):
        self.n, self.p = n, p
        self.A = A.tocsr()
        self.free = free                # full dof ids of the free dofs (sorted)
        self.kind = None                # transfer to the coarser level: 'p' | 'h' | None
        self.lam_max = None

    @property
    def k1(self):
        return self.p + 1

    # ---- edge blocks for block-Jacobi ----
    def build_edge_blocks(self):
        k = self.k1
        nfe = len(self.free) // k
        A = self.A
        idx = np.arange(len(self.free)).reshape(nfe, k)
        D = np.empty((nfe, k, k))
        Ad = A.toarray() if A.shape[0] <= 4096 else None
        for a in range(k):
            for b in range(k):
                if Ad is not None:
                    D[:, a, b] = Ad[idx[:, a], idx[:, b]]
                else:
                    D[:, a, b] = np.asarray(A[idx[:, a], idx[:, b]]).ravel()
        self.D = D

    def apply_Dinv(self, r):
        k = self.k1
        return np.linalg.solve(self.D, r.reshape(-1, k, 1)).reshape(-1)

    def apply_D(self, v):
        k = self.k1
        return np.einsum("eab,eb->ea", self.D, v.reshape(-1, k)).reshape(-1)

    # ---- 4-colour edge partition for LU-SGS (reading F3) ----
    def colour_sets(self):
        """[4] arrays of free-edge positions (into the free-edge list): colour 0/1 =
        horizontal edges of even / odd rows j, colour 2/3 = vertical edges of even /
        odd columns i.  An element's 4 edges have 4 different colours, so the edges
        of one colour share no element: their blocks are mutually uncoupled."""
        if getattr(self, "_colours", None) is None:
            k = self.k1
            edges = self.free[::k] // k
            nh = self.n * (self.n + 1)
            col = np.where(edges < nh, (edges // self.n) % 2, 2 + ((edges - nh) % (self.n + 1)) % 2)
            self._colours = [np.nonzero(col == c)[0] for c in range(4)]
        return self._colours


def _block_inverse(A_II: sp.csr_matrix, blocks: np.ndarray) -> sp.csr_matrix:
    """A_II^-1 for a block-diagonal A_II; `blocks` [nb, bs] are positions."""
    nb, bs = blocks.shape
    Ad = np.empty((nb, bs, bs))
    for a in range(bs):
        row = A_II[blocks[:, a]]
        for b in range(bs):
            Ad[:, a, b] = np.asarray(row[np.arange(nb), blocks[:, b]]).ravel()
    inv = np.linalg.inv(Ad)
    rows = np.repeat(blocks, bs, axis=1).ravel()
    cols = np.tile(blocks, (1, bs)).ravel()
    return sp.coo_matrix((inv.ravel(), (rows, cols)), shape=A_II.shape).tocsr()


def assembly_free(S: np.ndarray, n: int, p: int, free: np.ndarray) -> sp.csr_matrix:
    """sum_T G_T^T S_T G_T restricted to the free dofs (oracle.assembly.assemble_full)."""
    from .assembly import assemble_full
    return assemble_full(n, p, S)[free][:, free].tocsr()


def _positions(sub: np.ndarray, full_sorted: np.ndarray) -> np.ndarray:
    pos = np.searchsorted(full_sorted, sub)
    assert np.all(full_sorted[pos] == sub)
    return pos


# child local edge -> macro edge: macro edges 0..3 are the interior cross
# [H(2I,2J+1), H(2I+1,2J+1), V(2I+1,2J), V(2I+1,2J+1)] (macro_interior_edges order),
# 4..11 the boundary halves [bottom (2I), (2I+1); right (2J), (2J+1); top; left], each
# pair with the lower coordinate first; children (2I,2J), (2I+1,2J), (2I,2J+1), (2I+1,2J+1);
# child local edges {bottom, right, top, left}
_MACRO_EDGE = np.array([[4, 2, 0, 10], [5, 6, 1, 2], [0, 3, 8, 11], [1, 7, 9, 3]])


def project_constants(S: np.ndarray) -> np.ndarray:
    """P S P with P = I - 11^T/m: the nearest map (Frobenius) that annihilates constant
    traces, as the exact DtN map of every level does (fine level: u = 0, q = lambda = c
    solves the local problem; coarse levels: the macro's harmonic
    extension of a constant is that constant and J_M maps constants to constants)."""
    m = S.shape[1]
    P = np.eye(m) - np.ones((m, m)) / m
    return np.einsum("ab,ebc,cd->ead", P, S, P)


def galerkin_per_macro(S: np.ndarray, n: int, schur_inv: bool = False) -> np.ndarray:
    """Coarse element DtN maps by Prop. DtN macro by macro: for each
    2x2 macro assemble its 24x24 map S^M from its four children's 8x8 maps (P1 level),
    eliminate its interior edges, and inject its boundary halves:
        S_c^M = J_M^T (S_BB - S_BI S_II^-1 S_IB) J_M            (Eq. Akm1, per macro),
    J_M the nodal P1 injection of O7.  Summed over macros this is the same A_{k-1} as
    the global product J^T (A_BB - A_BI A_II^-1 A_IB) J (A_II and A_IB are macro-local,
    A_BB is the sum of the macros' S_BB), with the sums taken in another order -- a second
    valid FP64 evaluation used to measure the per-V-cycle noise floor.
    S: [n*n, 8, 8] element maps of the level (element id j*n+i); returns [(n/2)^2, 8, 8]."""
    nc = n // 2
    J, I = np.divmod(np.arange(nc * nc), nc)
    kids = [(2 * I) + n * (2 * J), (2 * I + 1) + n * (2 * J), (2 * I) + n * (2 * J + 1),
            (2 * I + 1) + n * (2 * J + 1)]
    SM = np.zeros((nc * nc, 24, 24))
    for c in range(4):
        loc = (_MACRO_EDGE[c][:, None] * 2 + np.arange(2)[None, :]).reshape(-1)
        SM[:, loc[:, None], loc[None, :]] += S[kids[c]]
    Iq, Bq = np.arange(8), np.arange(8, 24)
    SII = SM[:, Iq[:, None], Iq[None, :]]
    SIB = SM[:, Iq[:, None], Bq[None, :]]
    SBI = SM[:, Bq[:, None], Iq[None, :]]
    SBB = SM[:, Bq[:, None], Bq[None, :]]
    schur = SBB - (SBI @ np.linalg.inv(SII)) @ SIB if schur_inv else SBB - SBI @ np.linalg.solve(SII, SIB)
    h = np.array([[1.0, 0.0], [0.5, 0.5], [0.5, 0.5], [0.0, 1.0]])
    JM = np.kron(np.eye(4), h)          # [16, 8]: 4 sides x (2 halves x 2 dofs) -> 4 x 2
    return np.einsum("ba,ebc,cd->ead", JM, schur, JM)


class Hierarchy:
    """MG hierarchy from the finest trace operator A_N (free dofs)."""

    def __init__(self, A_N, n, p, n_h_levels=0, smoother=BLOCK_JACOBI, nu_pre=2, nu_post=2,
                 omega=1.0, cheb_ratio=30.0, lmax_iters=20, lmax_safety=1.05,
                 step3=True, step5=False, nu_doubling=False, all_free=False,
                 element_maps=None, galerkin="global", project_levels=False, schur_inv=False):
        """galerkin="macro" (needs element_maps, the fine level's [n*n, m, m] maps): every
        coarse operator is assembled from per-macro coarse maps (galerkin_per_macro)
        instead of the global sparse product -- the same operators summed in another
        order (P17 noise floor)."""
        self.smoother = smoother
        self.nu_pre, self.nu_post = nu_pre, nu_post
        self.omega = omega
        self.cheb_ratio = cheb_ratio
        self.step3, self.step5 = step3, step5
        self.nu_doubling = nu_doubling
        # all_free=True: no Dirichlet elimination (Neumann-type patch, used by
        # the DtN pins); the coarsest operator is then singular (constants).
        free_of = (lambda nn, pp: np.arange(mesh.n_edges(nn) * (pp + 1))) if all_free else mesh.free_dofs
        self.all_free = all_free
        levels = [Level(n, p, A_N, free_of(n, p))]
        # p-coarsening: Eq. ANm1
        if p > 1:
            fine = levels[-1]
            Jf = p_injection_full(n, p)
            cfree = free_of(n, 1)
            J = Jf[fine.free][:, cfree].tocsr()
            fine.kind, fine.J = "p", J
            A1 = (J.T @ fine.A @ J).tocsr()
            if galerkin == "macro":
                element_maps = p_coarsen_element(element_maps, p)
                if project_levels:
                    element_maps = project_constants(element_maps)
                A1 = assembly_free(element_maps, n, 1, cfree)
            levels.append(Level(n, 1, A1, cfree))
        # h-coarsening: Eq. Akm1 down to a 2x2 macro mesh (or n_h_levels)
        nh = 0
        # agglomerate while the coarse mesh stays even (n % 4 == 0) -- a 2x2
        # macro mesh at the bottom for n = 2^L (reading Q14)
        while levels[-1].n > 2 and levels[-1].n % 4 == 0 and (n_h_levels <= 0 or nh < n_h_levels):
            fine = levels[-1]
            nf = fine.n
            nc = nf // 2
            dof_edge = fine.free // 2
            imask = interior_edge_mask(nf)[dof_edge]
            I_pos = np.nonzero(imask)[0]
            B_pos = np.nonzero(~imask)[0]
            A = fine.A
            A_II = A[I_pos][:, I_pos].tocsr()
            A_IB = A[I_pos][:, B_pos].tocsr()
            A_BI = A[B_pos][:, I_pos].tocsr()
            A_BB = A[B_pos][:, B_pos].tocsr()
            # A_II is block diagonal over macros: 4 interior edges x 2 dofs each
            medges = macro_interior_edges(nf)
            mdofs = (medges[:, :, None] * 2 + np.arange(2)[None, None, :]).reshape(-1, 8)
            blocks = _positions(mdofs.ravel(), fine.free[I_pos]).reshape(-1, 8)
            AII_inv = _block_inverse(A_II, blocks)
            cfree = free_of(nc, 1)
            J = h_injection_full(nf)[fine.free[B_pos]][:, cfree].tocsr()
            Ac = J.T @ (A_BB - A_BI @ AII_inv @ A_IB) @ J
            fine.kind = "h"
            fine.I_pos, fine.B_pos = I_pos, B_pos
            fine.A_II, fine.A_IB, fine.A_BI, fine.A_BB = A_II, A_IB, A_BI, A_BB
            fine.AII_inv, fine.J, fine.macro_blocks = AII_inv, J, blocks
            if galerkin == "macro":
                if p == 1 and nh == 0 and element_maps is not None and element_maps.shape[1] != 8:
                    raise ValueError("element_maps must be the fine level's maps")
                element_maps = galerkin_per_macro(element_maps, nf, schur_inv)
                if project_levels:
                    element_maps = project_constants(element_maps)
                Ac = assembly_free(element_maps, nc, 1, cfree)
            levels.append(Level(nc, 1, Ac.tocsr(), cfree))
            nh += 1
        self.levels = levels                 # levels[0] = finest (k = N)
        coarsest = levels[-1]
        self.A1_dense = coarsest.A.toarray()
        # A_N nonsymmetric (IIPG-H / NIPG-H elements): every level is (the
        # Galerkin Q A I of a nonsymmetric A); B_1 = A_1^-1 by LU instead of Cholesky
        dA = A_N - A_N.T
        self.symmetric = (abs(dA).max() if dA.nnz else 0.0) <= 1e-13 * abs(A_N).max()
        self.A1_chol = self.A1_lu = None
        if not all_free:
            if self.symmetric:
                self.A1_chol = sla.cho_factor(self.A1_dense, lower=True)
            else:
                self.A1_lu = sla.lu_factor(self.A1_dense)
        if smoother == CHEBYSHEV and not self.symmetric:
            raise ValueError("Chebyshev needs a symmetric A (real spectrum of D^-1 A)")
        for L in levels[:-1]:
            L.build_edge_blocks()
            if smoother == CHEBYSHEV:
                L.lam_max = lmax_safety * self.estimate_lambda_max(L, lmax_iters)

    # ---- Q11: power iteration on D_B^-1 A ----
    @staticmethod
    def estimate_lambda_max(L: Level, iters: int) -> float:
        i = L.free
        v = 1.0 + (i % 7) / 7.0
        for _ in range(iters):
            v = L.apply_Dinv(L.A @ v)
            v = v / np.linalg.norm(v)
        return float(v @ (L.A @ v)) / float(v @ L.apply_D(v))

    @property
    def N(self):
        return len(self.levels)

    # ---- transfers ----
    def prolong(self, li, ec):
        """I_k e_c (Eq. 3.3 / 3.4); li indexes self.levels (0 = finest)."""
        L = self.levels[li]
        if L.kind == "p":
            return L.J @ ec
        e = np.zeros(len(L.free))
        eB = L.J @ ec
        e[L.B_pos] = eB
        e[L.I_pos] = -(L.AII_inv @ (L.A_IB @ eB))
        return e

    def restrict(self, li, r):
        """Q_{k-1} r (Eq. 3.5 / 3.6) -- full formula incl. the interior term."""
        L = self.levels[li]
        if L.kind == "p":
            return L.J.T @ r
        rI, rB = r[L.I_pos], r[L.B_pos]
        return L.J.T @ (rB - L.A_BI @ (L.AII_inv @ rI))

    def local_correction(self, li, r):
        """T_k r = [A_II^-1 r_I ; 0] (Eq. 3.11)."""
        L = self.levels[li]
        e = np.zeros(len(L.free))
        e[L.I_pos] = L.AII_inv @ r[L.I_pos]
        return e

    def coarse_solve(self, r):
        if self.A1_lu is not None:
            return sla.lu_solve(self.A1_lu, r)
        return sla.cho_solve(self.A1_chol, r)

    # ---- smoothers G_{k,m} ----
    def smooth(self, li, e, r, steps):
        """`steps` smoothing iterations on A_k e = r starting from e."""
        L = self.levels[li]
        A = L.A
        if self.smoother == BLOCK_JACOBI:
            for _ in range(steps):
                e = e + self.omega * L.apply_Dinv(r - A @ e)
            return e
        if self.smoother == LUSGS:
            # LU-SGS (one forward and one backward Gauss-Seidel
            # sweep) on edge blocks, in the 4-colour order: forward colours 0,1,2,3,
            # backward 3,2,1,0; each colour's blocks update together (reading F3)
            k = L.k1
            sets = L.colour_sets()
            for _ in range(steps):
                for c in (0, 1, 2, 3, 3, 2, 1, 0):
                    ed = sets[c]
                    pos = (ed[:, None] * k + np.arange(k)[None, :]).reshape(-1)
                    res = (r[pos] - A[pos] @ e).reshape(-1, k, 1)
                    e = e.copy()
                    e[pos] += self.omega * np.linalg.solve(L.D[ed], res).reshape(-1)
            return e
        # Chebyshev on D^-1 A over [b/ratio, b] (O8)
        b = L.lam_max
        a = b / self.cheb_ratio
        theta, delta = 0.5 * (b + a), 0.5 * (b - a)
        sigma = theta / delta
        rho = 1.0 / sigma
        d = L.apply_Dinv(r - A @ e) / theta
        e = e + d
        for _ in range(1, steps):
            rho_new = 1.0 / (2.0 * sigma - rho)
            d = rho_new * rho * d + (2.0 * rho_new / delta) * L.apply_Dinv(r - A @ e)
            e = e + d
            rho = rho_new
        return e

    def _nu(self, li, nu):
        if not self.nu_doubling:
            return nu
        return nu * (2 ** li)       # m_{k-1} = 2 m_k (beta_0 = beta_1 = 2)

    # ---- Algorithm 1 ----
    def vcycle(self, r, li=0):
        """B_k(r_k), Algorithm 1 steps 1-6 (step 5 only if self.step5)."""
        if li == self.N - 1:
            return self.coarse_solve(r)
        L = self.levels[li]
        A = L.A
        e = np.zeros_like(r)                                          # step 1
        e = self.smooth(li, e, r, self._nu(li, self.nu_pre))          # step 2
        has_interior = L.kind == "h"
        if has_interior and self.step3:
            e = e + self.local_correction(li, r - A @ e)              # step 3
        ec = self.vcycle(self.restrict(li, r - A @ e), li + 1)        # step 4
        e = e + self.prolong(li, ec)
        if has_interior and self.step5:
            e = e + self.local_correction(li, r - A @ e)              # step 5
        e = self.smooth(li, e, r, self._nu(li, self.nu_post))         # step 6
        return e
