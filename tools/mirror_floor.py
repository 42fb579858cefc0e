#!/usr/bin/env python3
"""Evaluation-order floor of a converged MG-PCG solution: solve a config (or a recipe at
size n) and its mirror image x -> 1 - x (tests/mirror.py: the same discrete problem up to a
relabelling of elements, edges and dofs, so only the order of every sum changes), map the
mirrored solution back and report how far the two FP64 solutions are apart.  Runs on the
GPU path; the oracle at the same recipe sizes is compared by tests/test_gpu_recipe_goldens.py.

    python tools/mirror_floor.py --config 3            # full size
    python tools/mirror_floor.py --config 3 --n 512    # W.config3_recipe(512)
"""
import argparse
import copy
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402

import workloads as W  # noqa: E402
from mirror import mirror_elements, mirror_trace_perm  # noqa: E402


def solve(cfg, pr):
    from paper_1811_09909_b200 import MGSolver, smoother_from_config
    s = MGSolver(cfg.n, p=cfg.p)
    s.setup(pr.K, pr.method, pr.tau, smoother_from_config(cfg))
    g, lam_bc = s.assemble_rhs(pr.f_qp, pr.f_const, pr.gD_qp)
    lam, info = s.pcg_solve(g, rtol=cfg.rtol, maxit=4000)
    return (lam + lam_bc).cpu().numpy(), info


def floor(cfg):
    pr = W.make_problem(cfg)
    if pr.f_qp is not None or pr.gD_qp is not None:
        raise SystemExit("mirror floor: constant-source, homogeneous-Dirichlet recipes only")
    n = cfg.n
    pm = copy.copy(pr)
    pm.K, pm.method, pm.tau = (mirror_elements(a, n) for a in (pr.K, pr.method, pr.tau))
    l1, i1 = solve(cfg, pr)
    l2, i2 = solve(cfg, pm)
    d = l2[mirror_trace_perm(n, cfg.p + 1)] - l1
    return {"config": cfg.index, "n": n, "name": cfg.name, "iters": [i1["iters"], i2["iters"]],
            "rel_l2": float(np.linalg.norm(d) / np.linalg.norm(l1)),
            "rel_max": float(np.abs(d).max() / np.abs(l1).max())}


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--n", type=int, default=0)
    a = ap.parse_args()
    if a.n:
        cfg = W.config3_recipe(a.n) if a.config == 3 else W.config5_recipe(a.n)
    else:
        cfg = W.CONFIGS[a.config]
    print(json.dumps(floor(cfg)), flush=True)
