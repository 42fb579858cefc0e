"""The heterogeneous configs' recipes against whole-vector oracle goldens at the largest
meshes the oracle solves in reasonable time (tests/golden/c<k>_recipe_n<n>.json + .npy,
tools/make_recipe_golden.py; the oracle under the GPU's readings R5 / R9 on the fine maps,
tests/oracle_proj.py, and R10 on every coarse level, oracle/multigrid.py; `_plain`: the
oracle as it stands):
  config 5's recipe (HDG p=4, tau=1, K = 10^g, Gaussian field of std 1 and correlation
    length 32 elements, V(2,2) Chebyshev) at n = 512 -- config 5 itself is beyond the
    oracle's memory;
  config 3's recipe (HDG p=2, std 1.5, length 16 elements, contrast 1e6, V(3,3)
    block-Jacobi) at n = 256 and 512 -- config 3's full-size oracle solve takes ~4 h.
North star: iterations within +-1, the converged trace within 1e-9 -- here on every dof.

Config 3's recipe at n >= 512 is the one case whose converged solution FP64 does not pin to
1e-9 (tools/map_floor.py): the GPU's element maps (staged Schur) and the
oracle's (full local solve) differ by ~4 ulp (median; 20 ulp max), and at contrast 1e6 after
830 iterations that alone moves the solution by 1.3e-9.  There the test checks the pieces
separately: the element maps to 1e-14, the GPU's whole setup + solve run on the ORACLE's
element maps (mg_debug_set_element_dtn + MG_OPT_KEEP_FINE_MAPS) against the oracle at the
north star's 1e-9, and the end-to-end solution at the measured floor (3e-9)."""
import json
import os

import numpy as np
import pytest
import torch

import workloads as W

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CASES = [(5, 512, ""), (3, 256, ""), (3, 256, "_plain"), (3, 512, ""), (3, 512, "_plain")]
TOL = 1e-9
TOL_C3_MAPS_FLOOR = 3e-9   # config-3 recipe, n >= 512: element-map rounding x conditioning


def recipe(idx, n):
    return W.config5_recipe(n) if idx == 5 else W.config3_recipe(n)


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def solve(s, c, pr):
    g, lam_bc = s.assemble_rhs(pr.f_qp, pr.f_const, pr.gD_qp)
    lam, info = s.pcg_solve(g, rtol=c.rtol, maxit=4000)
    assert info["status"] == "converged"
    return (lam + lam_bc).cpu().numpy(), info["iters"]


@pytest.mark.parametrize("case", CASES, ids=[f"c{a}n{b}{c}" for a, b, c in CASES])
def test_recipe_whole_vector_golden(case):
    idx, n, kind = case
    base = os.path.join(ROOT, "tests", "golden", f"c{idx}_recipe_n{n}{kind}")
    if not os.path.exists(base + ".json"):
        pytest.skip("golden not generated")
    from paper_1811_09909_b200 import MGSolver, smoother_from_config
    gold = json.load(open(base + ".json"))
    lam_o = np.load(base + ".npy")
    c = recipe(idx, n)
    pr = W.make_problem(c)
    assert abs(float(np.log10(pr.K).max()) - gold["log10K_max"]) < 1e-12   # same recipe
    s = MGSolver(n, p=c.p)
    sm = smoother_from_config(c)
    s.setup(pr.K, pr.method, pr.tau, sm)
    lam_g, it = solve(s, c, pr)
    assert abs(it - gold["iters"]) <= 1, (it, gold["iters"])
    floor = idx == 3 and n >= 512
    tol = TOL_C3_MAPS_FLOOR if floor else TOL
    d = lam_g - lam_o
    assert np.linalg.norm(d) <= tol * np.linalg.norm(lam_o), rel(lam_g, lam_o)
    assert np.abs(d).max() <= tol * np.abs(lam_o).max(), np.abs(d).max() / np.abs(lam_o).max()
    if floor and kind == "":
        # the same solve on the oracle's element maps: setup + solve pipeline at 1e-9
        from oracle import assembly
        from oracle_proj import project_maps
        ts = assembly.TraceSystem(n, c.p, pr.K, pr.method, pr.tau, pr.f_qp, pr.f_const, pr.gD_qp)
        So = project_maps(ts.S, c.p)
        N = s.nlevels
        Sg = s.element_dtn(N).cpu().numpy()
        dm = np.abs(Sg - So).max(axis=(1, 2)) / np.abs(So).max(axis=(1, 2))
        assert dm.max() <= 1e-14, dm.max()
        s.set_option(s.OPT_KEEP_FINE_MAPS, 1)
        s.set_element_dtn(N, torch.from_numpy(So))
        s.setup(pr.K, pr.method, pr.tau, sm)
        lam_i, it_i = solve(s, c, pr)
        s.set_option(s.OPT_KEEP_FINE_MAPS, 0)
        assert abs(it_i - gold["iters"]) <= 1, (it_i, gold["iters"])
        assert rel(lam_i, lam_o) <= TOL, rel(lam_i, lam_o)
