"""tests/mirror.py (the x -> 1 - x relabelling used by tools/mirror_floor.py): a
permutation of the trace dofs, an involution together with the element mirror, and the
oracle's solution of the mirrored config-3 recipe is the mirrored solution (to rounding)."""
import copy

import numpy as np

import workloads as W
from mirror import mirror_elements, mirror_trace_perm
from oracle import driver


def test_mirror_perm_is_an_involution():
    for n, k1 in ((4, 2), (6, 3), (8, 5)):
        P = mirror_trace_perm(n, k1)
        assert np.array_equal(np.sort(P), np.arange(len(P)))
        assert np.array_equal(P[P], np.arange(len(P)))
        a = np.arange(n * n)
        assert np.array_equal(mirror_elements(mirror_elements(a, n), n), a)


def test_oracle_mirrored_solution():
    c = W.config3_recipe(8)
    pr = W.make_problem(c)
    pm = copy.copy(pr)
    pm.K, pm.method, pm.tau = (mirror_elements(a, 8) for a in (pr.K, pr.method, pr.tau))
    r1 = driver.solve_problem(pr, maxit=4000)
    r2 = driver.solve_problem(pm, maxit=4000)
    assert r1["iters"] == r2["iters"]
    l1, l2 = r1["lam_full"], r2["lam_full"]
    assert np.linalg.norm(l2[mirror_trace_perm(8, c.p + 1)] - l1) <= 1e-12 * np.linalg.norm(l1)
