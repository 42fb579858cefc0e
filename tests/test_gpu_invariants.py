"""mg_check_invariants (SURVEY 5 debug mode): on set-up hierarchies of the five config
recipes every level's element maps annihilate constants (readings R5 /
R10), nothing is NaN / Inf, and the two-colour apply equals an independent atomicAdd
scatter apply; corrupted maps are reported, not silently used."""
import numpy as np
import pytest
import torch

import workloads as W

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _built():
    from paper_1811_09909_b200 import build
    build.build()
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.mark.parametrize("cfg,n", [(1, 8), (2, 32), (3, 64), (4, 64), (5, 64), (2, 256)])
def test_invariants_hold(cfg, n):
    from paper_1811_09909_b200 import MGSolver, smoother_from_config
    c = W.scaled_config(cfg, n) if W.CONFIGS[cfg].n != n else W.CONFIGS[cfg]
    pr = W.make_problem(c, with_f=False)
    s = MGSolver(n, p=c.p)
    s.setup(pr.K, pr.method, pr.tau, smoother_from_config(c))
    rep = s.check_invariants()
    assert rep["nonfinite"] == 0
    assert rep["const_mode"] <= 1e-12
    assert 0.0 <= rep["atomic_apply_diff"] <= 1e-13


def test_invariants_report_corruption():
    from paper_1811_09909_b200 import MGError, MGSolver, smoother_from_config
    c = W.scaled_config(2, 16)
    pr = W.make_problem(c, with_f=False)
    s = MGSolver(16, p=c.p)
    s.setup(pr.K, pr.method, pr.tau, smoother_from_config(c))
    S = s.element_dtn(s.nlevels).clone()
    m = S.shape[1]
    bad = S + torch.eye(m, dtype=S.dtype, device=S.device)   # no longer annihilates constants
    s.set_element_dtn(s.nlevels, bad)
    with pytest.raises(MGError, match="constants"):
        s.check_invariants()
    bad[3, 0, 0] = float("nan")
    s.set_element_dtn(s.nlevels, bad)
    with pytest.raises(MGError, match="non-finite"):
        s.check_invariants()
