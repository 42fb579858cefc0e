"""Krylov drivers: PCG (north star), left-preconditioned GMRES and MG as a
fixed-point solver.

Stopping rule (reading Q16): normalised residual
||r||_2 / ||g||_2 over the free dofs.  PCG uses the recursive residual with
rtol 1e-10 and lambda_0 = 0; it returns the true residual at exit as well.
"""
from __future__ import annotations

import numpy as np


def pcg(A, B, g, rtol=1e-10, maxit=2000, x0=None):
    """Standard preconditioned CG (Hestenes-Stiefel form).

    A: callable or matrix with @; B: callable preconditioner (one V-cycle).
    Returns dict(x, iters, relres, hist, status, true_relres).
    status: 0 converged, 1 maxit, 2 diverged, 3 breakdown (p.Ap <= 0).
    """
    Aop = A if callable(A) else (lambda v: A @ v)
    gn = float(np.linalg.norm(g))
    x = np.zeros_like(g) if x0 is None else x0.copy()
    if gn == 0.0:
        return dict(x=x, iters=0, relres=0.0, hist=[0.0], status=0, true_relres=0.0)
    r = g - Aop(x)
    hist = [float(np.linalg.norm(r)) / gn]
    if hist[-1] <= rtol:
        return dict(x=x, iters=0, relres=hist[-1], hist=hist, status=0, true_relres=hist[-1])
    z = B(r)
    p = z.copy()
    rz = float(r @ z)
    status = 1
    it = 0
    for it in range(1, maxit + 1):
        Ap = Aop(p)
        pAp = float(p @ Ap)
        if not pAp > 0.0:
            status = 3
            break
        alpha = rz / pAp
        x = x + alpha * p
        r = r - alpha * Ap
        rel = float(np.linalg.norm(r)) / gn
        hist.append(rel)
        if rel <= rtol:
            status = 0
            break
        if rel > 1e6:
            status = 2
            break
        z = B(r)
        rz_new = float(r @ z)
        beta = rz_new / rz
        p = z + beta * p
        rz = rz_new
    true_rel = float(np.linalg.norm(g - Aop(x))) / gn
    return dict(x=x, iters=it, relres=hist[-1], hist=hist, status=status, true_relres=true_rel)


def mg_solver(A, B, g, tol=1e-9, maxit=200):
    """lambda^{i+1} = lambda^i + B_N(g - A lambda^i)."""
    Aop = A if callable(A) else (lambda v: A @ v)
    gn = float(np.linalg.norm(g))
    x = np.zeros_like(g)
    r = g.copy()
    for it in range(1, maxit + 1):
        x = x + B(r)
        r = g - Aop(x)
        rel = float(np.linalg.norm(r)) / gn
        if rel <= tol:
            return dict(x=x, iters=it, relres=rel, status=0)
        if not np.isfinite(rel) or rel > 1e6:
            return dict(x=x, iters=it, relres=rel, status=2)
    return dict(x=x, iters=maxit, relres=rel, status=1)


def gmres(A, B, g, tol=1e-9, maxit=200):
    """Full (unrestarted) GMRES, left preconditioned by B, modified
    Gram-Schmidt; stops on the true residual ||g - A x|| / ||g|| (SPEC
    krylov reading; PAPER.md:1012-1015 normalises by ||g||)."""
    Aop = A if callable(A) else (lambda v: A @ v)
    gn = float(np.linalg.norm(g))
    n = len(g)
    z0 = B(g)
    beta = float(np.linalg.norm(z0))
    V = np.zeros((maxit + 1, n))
    Hm = np.zeros((maxit + 1, maxit))
    V[0] = z0 / beta
    x = np.zeros(n)
    for j in range(maxit):
        w = B(Aop(V[j]))
        for i in range(j + 1):
            Hm[i, j] = float(w @ V[i])
            w = w - Hm[i, j] * V[i]
        Hm[j + 1, j] = float(np.linalg.norm(w))
        if Hm[j + 1, j] > 0:
            V[j + 1] = w / Hm[j + 1, j]
        e1 = np.zeros(j + 2)
        e1[0] = beta
        y, *_ = np.linalg.lstsq(Hm[:j + 2, :j + 1], e1, rcond=None)
        x = V[:j + 1].T @ y
        rel = float(np.linalg.norm(g - Aop(x))) / gn
        if rel <= tol or Hm[j + 1, j] == 0:
            return dict(x=x, iters=j + 1, relres=rel, status=0)
    return dict(x=x, iters=maxit, relres=rel, status=1)
