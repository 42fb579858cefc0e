"""SURVEY.md 8(f) f2 on the GPU: the nonsymmetric hybridized IPDG schemes IIPG-H
(s_f = 0) and NIPG-H (s_f = -1) of Eq. IPG_H, alone and mixed
with HDG / SIPG-H (multinumerics), through a
MG_BUILD_NONSYMMETRIC context: full element maps, LU blocks, the Eq. 3.5
restriction Q_{k-1} = [-J^T A_BI A_II^-1, J^T] (not I_k^T), block-Jacobi,
GMRES / MG as a solver.

Parity against oracle/ (element.py Eq. IPG_H, multigrid.py with LU coarsest):
every operator and the V-cycle at 1e-12, solver iterations +-1 and the solution
at 1e-9 -- the north-star bars -- plus the paper's tab:NIPG_bj counts."""
import json
import os

import numpy as np
import pytest
import torch

import workloads as W
from oracle import assembly, element, krylov, multigrid

pytestmark = pytest.mark.gpu
TOL_OP = 1e-12
TOL_SOL = 1e-9
GOLD = os.path.join(os.path.dirname(__file__), "golden", "paper_exampleI_tables.json")


@pytest.fixture(scope="module", autouse=True)
def _built():
    from paper_1811_09909_b200 import build
    build.build()
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def rel(a, b):
    a = np.asarray(a, float)
    b = np.asarray(b, float)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


class NSCase:
    def __init__(self, cfg_index, n, p, mix):
        from paper_1811_09909_b200 import MGSolver, SmootherConfig
        c = W.scaled_config(cfg_index, n)
        c.p = p
        self.cfg = c
        pr = W.nonsymmetric_problem(c, mix)
        self.pr = pr
        self.ts = assembly.TraceSystem(n, p, pr.K, pr.method, pr.tau, pr.f_qp, pr.f_const, pr.gD_qp)
        self.H = multigrid.Hierarchy(self.ts.A, n, p, smoother=0, nu_pre=c.nu, nu_post=c.nu)
        assert not self.H.symmetric
        self.gpu = MGSolver(n, p=p, nonsymmetric=True)
        self.sm = SmootherConfig(kind=0, nu_pre=c.nu, nu_post=c.nu)
        self.gpu.setup(pr.K, pr.method, pr.tau, self.sm)
        self.N = self.gpu.nlevels
        assert self.N == self.H.N

    def olev(self, level):
        return self.H.levels[self.N - level]

    def vec(self, level, seed):
        return W.random_trace_vector(self.gpu.ndof(level), seed)


CASES = [(1, 8, 1, "nipg"), (4, 16, 3, "tiles"), (2, 16, 4, "iipg"), (4, 16, 2, "nipg"),
         (4, 64, 3, "tiles"), (2, 32, 4, "tiles"), (2, 64, 2, "nipg")]
# n <= 64 as in test_gpu_parity.py: at n = 128 the per-V-cycle gap reaches the FP64 floor of two
# valid eliminations amplified through 7 Galerkin levels (3.1e-12 here, 1.8e-12 for config 2's
# symmetric recipe), above the 1e-12 per-V-cycle gate


@pytest.fixture(scope="module", params=CASES, ids=[f"c{a}n{b}p{c}{d}" for a, b, c, d in CASES])
def case(request):
    return NSCase(*request.param)


def test_ns_element_dtn_parity(case):
    """H1 with s_f in {1, 0, -1} and HDG in the generic LU form vs the oracle's
    literal local elimination."""
    S = case.gpu.element_dtn(case.N).cpu().numpy()
    So = case.ts.S
    err = np.abs(S - So).max(axis=(1, 2)) / np.abs(So).max(axis=(1, 2))
    assert err.max() <= TOL_OP, err.max()
    ipdg = np.isin(case.pr.method, (W.IIPG_H, W.NIPG_H))
    asym = np.abs(S[ipdg] - S[ipdg].transpose(0, 2, 1)).max(axis=(1, 2))
    assert np.all(asym > 1e-6 * np.abs(S[ipdg]).max(axis=(1, 2)))


def test_ns_apply_parity_every_level(case):
    for level in range(case.N, 0, -1):
        x = case.vec(level, 11 + level)
        y = case.gpu.apply(level, torch.from_numpy(x)).cpu().numpy()
        L = case.olev(level)
        yo = L.A @ x[L.free]
        assert rel(y[L.free], yo) <= TOL_OP, (level, rel(y[L.free], yo))
        bd = np.setdiff1d(np.arange(len(y)), L.free)
        assert np.all(y[bd] == 0.0)


def test_ns_smoother_parity(case):
    for level in range(case.N, 1, -1):
        L = case.olev(level)
        r = case.vec(level, 100 + level)
        e0 = case.vec(level, 200 + level)
        for steps in (1, 2):
            e = case.gpu.smooth(level, torch.from_numpy(r), torch.from_numpy(e0), steps).cpu().numpy()
            eo = case.H.smooth(case.N - level, e0[L.free], r[L.free], steps)
            assert rel(e[L.free], eo) <= TOL_OP, (level, steps, rel(e[L.free], eo))


def test_ns_transfer_parity(case):
    """Restriction by Eq. 3.5 (A_BI, not A_IB^T), prolongation by Eq. 3.3, local
    correction by Eq. 3.11 -- on every level."""
    for level in range(case.N, 1, -1):
        li = case.N - level
        L = case.olev(level)
        Lc = case.olev(level - 1)
        res = case.vec(level, 300 + level)
        rc = case.gpu.restrict(level, torch.from_numpy(res)).cpu().numpy()
        assert rel(rc[Lc.free], case.H.restrict(li, res[L.free])) <= TOL_OP, level
        ec = case.vec(level - 1, 400 + level)
        e0 = case.vec(level, 500 + level)
        e = case.gpu.prolong(level, torch.from_numpy(ec), torch.from_numpy(e0)).cpu().numpy()
        assert rel(e[L.free], e0[L.free] + case.H.prolong(li, ec[Lc.free])) <= TOL_OP, level
        if L.kind == "h":
            e = case.gpu.local_correct(level, torch.from_numpy(res), torch.from_numpy(e0)).cpu().numpy()
            eo = e0[L.free] + case.H.local_correction(li, res[L.free])
            assert rel(e[L.free], eo) <= TOL_OP, level


def test_ns_vcycle_parity(case):
    r = case.vec(case.N, 600)
    z = case.gpu.vcycle(torch.from_numpy(r)).cpu().numpy()
    fr = case.ts.free
    assert rel(z[fr], case.H.vcycle(r[fr])) <= TOL_OP


def test_ns_rhs_and_recovery_parity(case):
    pr = case.pr
    g, lam_bc = case.gpu.assemble_rhs(pr.f_qp, pr.f_const, pr.gD_qp)
    fr = case.ts.free
    assert rel(g.cpu().numpy()[fr], case.ts.g) <= TOL_OP
    lam_full = case.vec(case.N, 700)
    q, _ = case.gpu.recover_volume(torch.from_numpy(lam_full), pr.f_qp, pr.f_const)
    from oracle import mesh
    lamT = lam_full[mesh.element_dofs(case.cfg.n, case.cfg.p)]
    qo = element.recover_q(case.cfg.p, pr.K, pr.method, pr.tau, 1.0 / case.cfg.n, lamT, pr.f_qp,
                           pr.f_const)
    assert rel(q.cpu().numpy(), qo) <= TOL_OP


def test_ns_gmres_and_mg_solver_parity(case):
    pr = case.pr
    g, lam_bc = case.gpu.assemble_rhs(pr.f_qp, pr.f_const, pr.gD_qp)
    lam, info = case.gpu.gmres_solve(g, tol=1e-10, maxit=300)
    ref = krylov.gmres(case.ts.A, case.H.vcycle, case.ts.g, 1e-10, 300)
    assert info["status"] == "converged" and ref["status"] == 0
    assert abs(info["iters"] - ref["iters"]) <= 1, (info, ref["iters"])
    fr = case.ts.free
    x = lam.cpu().numpy()[fr]
    if info["iters"] == ref["iters"]:
        assert rel(x, ref["x"]) <= TOL_SOL
    assert np.linalg.norm(case.ts.g - case.ts.A @ x) <= 2e-10 * np.linalg.norm(case.ts.g)
    if case.cfg.n <= 16:
        lam2, a = case.gpu.mg_solve(g, tol=1e-10, maxit=300)
        ao = krylov.mg_solver(case.ts.A, case.H.vcycle, case.ts.g, 1e-10, 300)
        assert a["status"] == "converged" and abs(a["iters"] - ao["iters"]) <= 1, (a, ao["iters"])
        assert rel(lam2.cpu().numpy()[fr], ao["x"]) <= TOL_SOL


def test_ns_refusals():
    """PCG and Chebyshev need a symmetric A; IIPG-H / NIPG-H need a nonsymmetric ctx."""
    from paper_1811_09909_b200 import MGError, MGSolver, SmootherConfig
    c = W.scaled_config(1, 8)
    pr = W.nonsymmetric_problem(c, "nipg")
    s = MGSolver(8, p=1, nonsymmetric=True)
    with pytest.raises(MGError, match="UNSUPPORTED"):
        s.setup(pr.K, pr.method, pr.tau, SmootherConfig(kind=1, nu_pre=2, nu_post=2))
    s.setup(pr.K, pr.method, pr.tau, SmootherConfig(kind=0, nu_pre=2, nu_post=2))
    g, _ = s.assemble_rhs(pr.f_qp, pr.f_const, pr.gD_qp)
    with pytest.raises(MGError, match="UNSUPPORTED"):
        s.pcg_solve(g)
    sym = MGSolver(8, p=1)
    with pytest.raises(MGError, match="MG_ERR_ARG"):
        sym.setup(pr.K, pr.method, pr.tau, SmootherConfig(kind=0, nu_pre=2, nu_post=2))
        sym.assemble_rhs(pr.f_qp, pr.f_const, pr.gD_qp)
        sym.mg_solve(torch.zeros(sym.ndof(), dtype=torch.float64), maxit=1)


def test_ns_symmetric_methods_match_symmetric_context():
    """HDG / SIPG-H elements in a nonsymmetric context (generic LU local solves, full
    storage) give the symmetric context's operators."""
    from paper_1811_09909_b200 import MGSolver, SmootherConfig
    c = W.scaled_config(4, 16)
    pr = W.make_problem(c)
    sm = SmootherConfig(kind=0, nu_pre=2, nu_post=2)
    a = MGSolver(16, p=c.p)
    a.setup(pr.K, pr.method, pr.tau, sm)
    b = MGSolver(16, p=c.p, nonsymmetric=True)
    b.setup(pr.K, pr.method, pr.tau, sm)
    x = torch.from_numpy(W.random_trace_vector(a.ndof(), 5))
    for level in range(a.nlevels, 0, -1):
        xl = torch.from_numpy(W.random_trace_vector(a.ndof(level), level))
        assert rel(b.apply(level, xl).cpu().numpy(), a.apply(level, xl).cpu().numpy()) <= TOL_OP
    assert rel(b.vcycle(x).cpu().numpy(), a.vcycle(x).cpu().numpy()) <= TOL_OP


@pytest.mark.parametrize("p", [1, 2, 3, 4])
def test_gpu_reproduces_tab_nipg_bj(p):
    """tab:NIPG_bj: NIPG-H, tau = (p+1)(p+2)/h_min, block-Jacobi
    with beta = 2 doubling from m_N = 3, MG as solver and GMRES, Levels 2..4: the
    oracle's counts +-1 and the printed ones +-1 (p = 1 Level 2: +-2, F2)."""
    from paper_1811_09909_b200 import MGSolver, SmootherConfig
    gold = json.load(open(GOLD))["tab:NIPG_bj"]
    for li, L in enumerate((2, 3, 4)):
        n = 2 ** L
        pr = W.example1_problem(n, p, gold["tau"], gold["method"])
        s = MGSolver(n, p=p, nonsymmetric=True)
        s.setup(pr.K, pr.method, pr.tau, SmootherConfig(kind=0, nu_pre=3, nu_post=3, nu_doubling=True))
        g, _ = s.assemble_rhs(pr.f_qp, pr.f_const, pr.gD_qp)
        _, a = s.mg_solve(g, tol=1e-9, maxit=200)
        _, b = s.gmres_solve(g, tol=1e-9, maxit=200)
        ts = assembly.TraceSystem(n, p, pr.K, pr.method, pr.tau, pr.f_qp, 0.0, pr.gD_qp)
        H = multigrid.Hierarchy(ts.A, n, p, smoother=0, nu_pre=3, nu_post=3, nu_doubling=True)
        ao = krylov.mg_solver(ts.A, H.vcycle, ts.g, 1e-9, 200)
        bo = krylov.gmres(ts.A, H.vcycle, ts.g, 1e-9, 200)
        assert abs(a["iters"] - ao["iters"]) <= 1 and abs(b["iters"] - bo["iters"]) <= 1
        tol_mg = 2 if (p, L) == (1, 2) else 1
        assert abs(a["iters"] - gold["mg"][str(p)][li]) <= tol_mg, (p, L, a["iters"])
        assert abs(b["iters"] - gold["gmres"][str(p)][li]) <= 1, (p, L, b["iters"])
