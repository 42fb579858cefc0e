"""bench.py's per-iteration byte model (reported as solve_roofline):
host-only checks of its bookkeeping on the config-2 level structure."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_1811_09909_b200.mgdtn import SmootherConfig  # noqa: E402


class _Levels:
    """The level structure of an n x n, order-p hierarchy (p-level + 2x2 agglomeration to 2x2)."""

    def __init__(self, n, p):
        self.L = []
        nn = n
        while nn >= 2:
            self.L.append((nn, 1))
            nn //= 2
        self.L = self.L[::-1]
        if p > 1:
            self.L.append((n, p))
        self.nlevels = len(self.L)

    def level_info(self, level):
        n, p = self.L[level - 1]
        return dict(nx=n, ny=n, p=p, ndof=2 * n * (n + 1) * (p + 1))


def test_fine_apply_dominates_and_counts():
    s = _Levels(256, 4)
    sm = SmootherConfig(kind=1, nu_pre=2, nu_post=2)
    b = bench.bytes_per_iteration(s, sm)
    # fine level in D4-orbit storage (reading R9): 65536 elements x 33 doubles per apply;
    # 5 fine applies per iteration (3 smoothing steps with an apply, the residual, the PCG
    # apply), each with 16 B per trace dof of x / y, D_e^-1 orbits (9 per edge) and the
    # smoothing vectors (r, e, Chebyshev d: 40 B per dof), transfers 32 B per dof, and
    # the PCG's 6 vector passes
    ne, nd, ned = 65536, 657920, 131584
    fine_S = ne * 33 * 8
    ap = fine_S + 16 * nd
    fine = 4 * (ap + 8 * ned * 9 + 40 * nd) + 8 * nd + 24 * nd + (ap + 48 * nd)
    assert 5 * fine_S < fine < b < 2 * fine
    assert abs(b - 4.77434112e8) / 4.77434112e8 < 1e-6
    # full storage (nonsymmetric) moves more; block-Jacobi drops the Chebyshev d traffic
    assert bench.bytes_per_iteration(s, sm, ns=True) > b
    assert bench.bytes_per_iteration(s, SmootherConfig(kind=0, nu_pre=2, nu_post=2)) < b


def test_more_smoothing_more_bytes():
    s = _Levels(64, 2)
    b2 = bench.bytes_per_iteration(s, SmootherConfig(kind=0, nu_pre=2, nu_post=2))
    b3 = bench.bytes_per_iteration(s, SmootherConfig(kind=0, nu_pre=3, nu_post=3))
    assert b3 > b2
