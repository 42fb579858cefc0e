"""1D nodal bases and quadrature on [0,1] (reading Q2: GLL nodal Lagrange
bases for volume Q^p and trace P^p spaces, Gauss-Legendre quadrature).

PAPER.md:201-211 defines the spaces (P^p per element / per edge) but not the
basis or quadrature; SURVEY.md 8(c) Q1/Q2 fix Q^p on quads with GLL nodes.
"""
from __future__ import annotations

import numpy as np


def gll_nodes(p: int) -> np.ndarray:
    """Gauss-Lobatto-Legendre nodes on [0,1]: 0, roots of P_p', 1."""
    if p < 1:
        raise ValueError("p >= 1")
    if p == 1:
        return np.array([0.0, 1.0])
    inner = np.polynomial.legendre.Legendre.basis(p).deriv().roots()
    x = np.concatenate([[-1.0], np.sort(inner.real), [1.0]])
    return 0.5 * (x + 1.0)


def gauss(nq: int):
    """Gauss-Legendre nodes/weights on [0,1] (numpy library routine)."""
    x, w = np.polynomial.legendre.leggauss(nq)
    return 0.5 * (x + 1.0), 0.5 * w


def lagrange(nodes: np.ndarray, x: np.ndarray) -> np.ndarray:
    """V[q, a] = l_a(x_q) for the Lagrange basis on `nodes` (product form)."""
    x = np.atleast_1d(np.asarray(x, dtype=float))
    k = len(nodes)
    V = np.ones((len(x), k))
    for a in range(k):
        for b in range(k):
            if b != a:
                V[:, a] *= (x - nodes[b]) / (nodes[a] - nodes[b])
    return V


def lagrange_deriv(nodes: np.ndarray, x: np.ndarray) -> np.ndarray:
    """dV[q, a] = l_a'(x_q) (product rule, no shortcuts)."""
    x = np.atleast_1d(np.asarray(x, dtype=float))
    k = len(nodes)
    dV = np.zeros((len(x), k))
    for a in range(k):
        for c in range(k):
            if c == a:
                continue
            term = np.full(len(x), 1.0 / (nodes[a] - nodes[c]))
            for b in range(k):
                if b != a and b != c:
                    term = term * (x - nodes[b]) / (nodes[a] - nodes[b])
            dV[:, a] += term
    return dV
