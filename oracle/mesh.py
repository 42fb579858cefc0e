"""Structured n x n quadrilateral mesh of the unit square and its skeleton.

Canonical numbering (reading Q3), shared with the
C-ABI as the *layout contract* of trace vectors:
  element (i,j) id = j*n + i
  horizontal edge H(i,j), 0<=i<n, 0<=j<=n: id = j*n + i
  vertical   edge V(i,j), 0<=i<=n, 0<=j<n: id = n*(n+1) + j*(n+1) + i
  dof (edge e, node a) = e*(p+1) + a, nodes along the edge's global orientation
  element local edges: 0 = H(i,j), 1 = V(i+1,j), 2 = H(i,j+1), 3 = V(i,j)
Skeleton E_h = union of element boundaries; boundary edges
(on dOmega) carry Dirichlet data.
"""
from __future__ import annotations

import numpy as np


def n_edges(n: int) -> int:
    return 2 * n * (n + 1)


def hedge(n, i, j):
    return j * n + i


def vedge(n, i, j):
    return n * (n + 1) + j * (n + 1) + i


def element_edges(n: int) -> np.ndarray:
    """[n*n, 4] global edge ids of each element's {bottom, right, top, left}."""
    j, i = np.divmod(np.arange(n * n), n)
    return np.stack([hedge(n, i, j), vedge(n, i + 1, j), hedge(n, i, j + 1), vedge(n, i, j)], axis=1)


def element_dofs(n: int, p: int) -> np.ndarray:
    """[n*n, 4(p+1)] global dof ids of each element's local trace dofs."""
    k = p + 1
    ed = element_edges(n)
    return (ed[:, :, None] * k + np.arange(k)[None, None, :]).reshape(n * n, 4 * k)


def boundary_edges(n: int) -> np.ndarray:
    """Edge ids on dOmega in the g_D input order: bottom, top, left, right."""
    i = np.arange(n)
    return np.concatenate([hedge(n, i, 0), hedge(n, i, n), vedge(n, 0, i), vedge(n, n, i)])


def boundary_edge_mask(n: int) -> np.ndarray:
    mask = np.zeros(n_edges(n), dtype=bool)
    mask[boundary_edges(n)] = True
    return mask


def free_dofs(n: int, p: int) -> np.ndarray:
    """Sorted global dof ids not on dOmega (the unknowns of Eq. 3.1)."""
    k = p + 1
    fe = np.nonzero(~boundary_edge_mask(n))[0]
    return (fe[:, None] * k + np.arange(k)[None, :]).reshape(-1)


def dirichlet_dofs(n: int, p: int) -> np.ndarray:
    k = p + 1
    be = np.nonzero(boundary_edge_mask(n))[0]
    return (be[:, None] * k + np.arange(k)[None, :]).reshape(-1)
