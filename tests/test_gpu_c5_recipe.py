"""Config 5's recipe (HDG p=4, tau=1, K = 10^g with a Gaussian field of std 1 and
correlation length 32 elements, V(2,2) Chebyshev, PCG to 1e-10) against a whole-vector
oracle golden at the largest mesh the oracle solves (tests/golden/c5_recipe_n<n>.json +
.npy, tools/make_c5_golden.py; oracle on its R5/R9-projected maps, tests/oracle_proj.py).
North star: iterations within +-1, the converged trace within 1e-9 -- here on every dof,
not a sample."""
import json
import os

import numpy as np
import pytest
import torch

import workloads as W

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("n", [512])
def test_c5_recipe_whole_vector_golden(n):
    base = os.path.join(ROOT, "tests", "golden", f"c5_recipe_n{n}")
    if not os.path.exists(base + ".json"):
        pytest.skip("golden not generated")
    from paper_1811_09909_b200 import MGSolver, smoother_from_config
    gold = json.load(open(base + ".json"))
    lam_o = np.load(base + ".npy")
    c = W.config5_recipe(n)
    pr = W.make_problem(c)
    assert abs(float(np.log10(pr.K).max()) - gold["log10K_max"]) < 1e-12   # same recipe
    s = MGSolver(n, p=c.p)
    s.setup(pr.K, pr.method, pr.tau, smoother_from_config(c))
    g, lam_bc = s.assemble_rhs(pr.f_qp, pr.f_const, pr.gD_qp)
    lam, info = s.pcg_solve(g, rtol=c.rtol, maxit=4000)
    assert info["status"] == "converged"
    assert abs(info["iters"] - gold["iters"]) <= 1, (info["iters"], gold["iters"])
    lam_g = (lam + lam_bc).cpu().numpy()
    d = lam_g - lam_o
    assert np.linalg.norm(d) <= 1e-9 * np.linalg.norm(lam_o), np.linalg.norm(d) / np.linalg.norm(lam_o)
    assert np.abs(d).max() <= 1e-9 * np.abs(lam_o).max(), np.abs(d).max() / np.abs(lam_o).max()
