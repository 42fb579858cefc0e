"""SURVEY.md 8(f) f3 on the GPU: the LU-SGS smoother on edge
blocks in the 4-colour order (forward colour sweeps 0,1,2,3, backward 3,2,1,0),
each colour sweep one apply whose colour-1 epilogue updates only that colour's
edges (AM_GSC).  Parity against oracle/multigrid.py (smoother LUSGS): every
smoothing step and one V-cycle at 1e-12, MG-PCG iterations +-1 and lambda at 1e-9."""
import numpy as np
import pytest
import torch

import workloads as W
from oracle import assembly, krylov, mesh, multigrid

pytestmark = pytest.mark.gpu
TOL = 1e-12


@pytest.fixture(scope="module", autouse=True)
def _built():
    from paper_1811_09909_b200 import build
    build.build()
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.mark.parametrize("idx,n", [(1, 8), (2, 16), (4, 16), (3, 32), (4, 64)])
def test_lusgs_parity(idx, n):
    from paper_1811_09909_b200 import MGSolver, SmootherConfig
    cfg = W.scaled_config(idx, n)
    pr = W.make_problem(cfg)
    s = MGSolver(n, p=cfg.p)
    s.setup(pr.K, pr.method, pr.tau, SmootherConfig(kind=2, nu_pre=1, nu_post=1))
    ts = assembly.TraceSystem(n, cfg.p, pr.K, pr.method, pr.tau, pr.f_qp, pr.f_const, pr.gD_qp)
    H = multigrid.Hierarchy(ts.A, n, cfg.p, smoother=multigrid.LUSGS, nu_pre=1, nu_post=1)
    N = s.nlevels
    rng = np.random.default_rng(77)
    for level in range(N, 1, -1):   # every level with a smoother
        Lo = H.levels[N - level]
        nd = s.ndof(level)
        r = rng.uniform(-1, 1, nd)
        e = rng.uniform(-1, 1, nd)
        free = Lo.free
        for steps in (1, 2):
            eg = s.smooth(level, torch.from_numpy(r), torch.from_numpy(e), steps).cpu().numpy()
            eo = H.smooth(N - level, e[free], r[free], steps)
            assert rel(eg[free], eo) <= TOL, (level, steps, rel(eg[free], eo))
    x = rng.uniform(-1, 1, s.ndof())
    z = s.vcycle(torch.from_numpy(x)).cpu().numpy()[ts.free]
    zo = H.vcycle(x[ts.free])
    assert rel(z, zo) <= TOL, rel(z, zo)
    g, lam_bc = s.assemble_rhs(pr.f_qp, pr.f_const, pr.gD_qp)
    lam, info = s.pcg_solve(g, rtol=cfg.rtol, maxit=2000)
    ref = krylov.pcg(ts.A, H.vcycle, ts.g, rtol=cfg.rtol, maxit=2000)
    assert info["status"] == "converged"
    assert abs(info["iters"] - ref["iters"]) <= 1, (info["iters"], ref["iters"])
    assert rel(lam.cpu().numpy()[ts.free], ref["x"]) <= 1e-9

