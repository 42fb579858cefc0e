#!/usr/bin/env python3
"""Per-level accuracy of the GPU's 2x2 Galerkin agglomeration (k_agglomerate):
each coarse level's element DtN maps from the GPU vs a long-double per-macro
Schur complement (Prop. DtN) of the GPU's OWN finer level,
so every level's error is the agglomeration step's alone.

    python tools/agglomeration_probe.py --config 2 --n 128"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import workloads as W  # noqa: E402
from paper_1811_09909_b200 import MGSolver, smoother_from_config  # noqa: E402


def child_G(dtype):
    """G_c [4][8][16]: child local dof -> macro (interior 0..7 | coarse 8..15)."""
    G = np.zeros((4, 8, 16), dtype=dtype)
    m = {0: [("C", 0, 0), ("I", 2), ("I", 0), ("C", 3, 0)],
         1: [("C", 0, 1), ("C", 1, 0), ("I", 1), ("I", 2)],
         2: [("I", 0), ("I", 3), ("C", 2, 0), ("C", 3, 1)],
         3: [("I", 1), ("C", 1, 1), ("C", 2, 1), ("I", 3)]}
    for c in range(4):
        for f, t in enumerate(m[c]):
            for a in range(2):
                r = 2 * f + a
                if t[0] == "I":
                    G[c, r, 2 * t[1] + a] = 1
                else:
                    _, E, half = t
                    sp = (half + a) / 2
                    G[c, r, 8 + 2 * E] = 1 - sp
                    G[c, r, 8 + 2 * E + 1] = sp
    return G


def chol_solve(A, B):
    n = A.shape[1]
    L = np.zeros_like(A)
    for j in range(n):
        d = np.sqrt(A[:, j, j] - np.sum(L[:, j, :j] ** 2, axis=1))
        L[:, j, j] = d
        for i in range(j + 1, n):
            L[:, i, j] = (A[:, i, j] - np.sum(L[:, i, :j] * L[:, j, :j], axis=1)) / d
    Y = np.zeros_like(B)
    for i in range(n):
        Y[:, i, :] = (B[:, i, :] - np.einsum("mk,mkc->mc", L[:, i, :i], Y[:, :i, :])) / L[:, i, i][:, None]
    X = np.zeros_like(B)
    for i in reversed(range(n)):
        X[:, i, :] = (Y[:, i, :] - np.einsum("mk,mkc->mc", L[:, i + 1:, i], X[:, i + 1:, :])) / L[:, i, i][:, None]
    return X


def agglomerate(S, n):
    G = child_G(S.dtype)
    nc = n // 2
    J, I = np.divmod(np.arange(nc * nc), nc)
    Kr = np.zeros((nc * nc, 16, 16), dtype=S.dtype)
    for c in range(4):
        Sc = S[(2 * J + (c >> 1)) * n + 2 * I + (c & 1)]
        Kr += np.einsum("ra,mrs,sb->mab", G[c], Sc, G[c])
    X = chol_solve(Kr[:, :8, :8], Kr[:, :8, 8:])
    return Kr[:, 8:, 8:] - np.einsum("mia,mib->mab", Kr[:, :8, 8:], X)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--n", type=int, default=128)
    a = ap.parse_args()
    cfg = W.scaled_config(a.config, a.n)
    pr = W.make_problem(cfg, with_f=False)
    s = MGSolver(cfg.n, p=cfg.p)
    s.setup(pr.K, pr.method, pr.tau, smoother_from_config(cfg))
    out = {"config": cfg.name}
    k = s.nlevels - (1 if cfg.p > 1 else 0)
    while k > 1:
        nf = s.level_info(k)["nx"]
        Sf = s.element_dtn(k).cpu().numpy()
        Sc = s.element_dtn(k - 1).cpu().numpy()
        ref = agglomerate(Sf.astype(np.longdouble), nf)
        ref64 = ref.astype(np.float64)
        scale = np.abs(ref64).max(axis=(1, 2))
        err = (np.abs(Sc - ref64).max(axis=(1, 2)) / scale).max()
        err64 = (np.abs(agglomerate(Sf, nf) - ref64).max(axis=(1, 2)) / scale).max()
        out[f"lev{k - 1}_n{nf // 2}"] = {"gpu_vs_ld": float(err), "cpu64_vs_ld": float(err64)}
        k -= 1
    print(json.dumps(out))


if __name__ == "__main__":
    main()
