"""Trace system A lambda = g (Eq. `trace_linear_system`).

A = sum_T G_T^T S_T G_T and g = sum_T G_T^T b_T follow from the conservation
condition <[[u_hat . n]], mu>_e = 0 (Eq. `conservation`) after the element
solves of oracle.element.  Dirichlet data are imposed strongly through the
trace unknowns as the per-edge L2 projection of g_D
onto P^p (reading Q4) and moved to the right-hand side:
    A_FF lambda_F = g_F - A_FD lambda_D.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp

from . import element as el
from . import mesh


def assemble_full(n: int, p: int, S: np.ndarray) -> sp.csr_matrix:
    """Global A over all trace dofs (incl. dOmega), from element DtN maps."""
    dofs = mesh.element_dofs(n, p)
    m = dofs.shape[1]
    rows = np.repeat(dofs, m, axis=1).reshape(-1)
    cols = np.tile(dofs, (1, m)).reshape(-1)
    N = mesh.n_edges(n) * (p + 1)
    return sp.coo_matrix((S.reshape(-1), (rows, cols)), shape=(N, N)).tocsr()


def assemble_vector(n: int, p: int, b: np.ndarray) -> np.ndarray:
    dofs = mesh.element_dofs(n, p)
    g = np.zeros(mesh.n_edges(n) * (p + 1))
    np.add.at(g, dofs.reshape(-1), b.reshape(-1))
    return g


def dirichlet_values(n: int, p: int, gD_qp) -> np.ndarray:
    """lambda_D: per-edge L2 projection of g_D onto P^p (Gauss p+4 samples).

    <lambda_D, mu>_e = <g_D, mu>_e on each boundary edge; the edge length
    cancels on both sides.  Returns a full-length vector (0 off dOmega).
    """
    k = p + 1
    lam = np.zeros(mesh.n_edges(n) * k)
    if gD_qp is None:
        return lam
    R = el.ref(p)
    rhs = np.einsum("q,eq,qa->ea", R.edge_f_weights, gD_qp, R.edge_f_basis)
    vals = np.linalg.solve(R.Hhat1, rhs.T).T
    be = mesh.boundary_edges(n)
    lam[(be[:, None] * k + np.arange(k)[None, :]).reshape(-1)] = vals.reshape(-1)
    return lam


class TraceSystem:
    """Assembled trace system of one problem (full + free-dof views)."""

    def __init__(self, n, p, K, method, tau, f_qp=None, f_const=0.0, gD_qp=None):
        h = 1.0 / n
        self.n, self.p, self.h = n, p, h
        self.K, self.method, self.tau = np.asarray(K, float), np.asarray(method), np.asarray(tau, float)
        self.S = el.element_dtn(p, K, method, tau, h)
        self.b = el.element_rhs(p, K, method, tau, h, f_qp, f_const)
        self.f_qp, self.f_const = f_qp, f_const
        self.A_full = assemble_full(n, p, self.S)
        self.free = mesh.free_dofs(n, p)
        self.dir = mesh.dirichlet_dofs(n, p)
        self.lam_D = dirichlet_values(n, p, gD_qp)
        g_full = assemble_vector(n, p, self.b)
        self.A = self.A_full[self.free][:, self.free].tocsr()
        self.g = g_full[self.free] - self.A_full[self.free][:, self.dir] @ self.lam_D[self.dir]
        self.ndof = mesh.n_edges(n) * (p + 1)

    def to_full(self, lam_free: np.ndarray) -> np.ndarray:
        """Full trace vector: free part + Dirichlet values."""
        out = self.lam_D.copy()
        out[self.free] = lam_free
        return out

    def g_full(self) -> np.ndarray:
        out = np.zeros(self.ndof)
        out[self.free] = self.g
        return out
