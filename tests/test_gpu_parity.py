"""GPU parity: the CUDA path (through the C ABI) against the oracle on the
same seeded inputs (BASELINE.json north star: <= 1e-12 relative L2 per
operator apply and per V-cycle; <= 1e-9 on the converged trace solution with
iteration counts within +-1)."""
import numpy as np
import pytest
import torch

import workloads as W
from oracle import assembly, krylov, multigrid
from oracle import element as el

pytestmark = pytest.mark.gpu

TOL_OP = 1e-12
TOL_SOL = 1e-9


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


class Case:
    """One problem set up identically on both sides."""

    def __init__(self, cfg_index, n, p=None, smoother=None, nu=None, proj=False):
        from oracle_proj import project_maps
        from paper_1811_09909_b200 import MGSolver, SmootherConfig
        c = W.scaled_config(cfg_index, n) if W.CONFIGS[cfg_index].n != n else W.CONFIGS[cfg_index]
        if p is not None:
            c.p = p
        if smoother is not None:
            c.smoother = smoother
        if nu is not None:
            c.nu = nu
        self.cfg = c
        pr = W.make_problem(c)
        self.pr = pr
        self.ts = assembly.TraceSystem(c.n, c.p, pr.K, pr.method, pr.tau, pr.f_qp, pr.f_const, pr.gD_qp)
        self.proj = proj
        if proj:   # the oracle on its maps projected by readings R5 / R9 (tests/oracle_proj.py)
            ts = self.ts
            ts.S = project_maps(ts.S, c.p)
            ts.A_full = assembly.assemble_full(c.n, c.p, ts.S)
            ts.A = ts.A_full[ts.free][:, ts.free].tocsr()
            g_full = assembly.assemble_vector(c.n, c.p, ts.b)
            ts.g = g_full[ts.free] - ts.A_full[ts.free][:, ts.dir] @ ts.lam_D[ts.dir]
        # proj: readings R5 / R9 on the fine maps and R10 (constants annihilated) on every
        # coarse level's maps, built macro by macro (Prop. DtN) as the GPU builds them
        extra = dict(element_maps=self.ts.S, galerkin="macro", project_levels=True) if proj else {}
        self.H = multigrid.Hierarchy(self.ts.A, c.n, c.p, smoother=c.smoother, nu_pre=c.nu,
                                     nu_post=c.nu, **extra)
        self.gpu = MGSolver(c.n, p=c.p)
        self.sm = SmootherConfig(kind=c.smoother, nu_pre=c.nu, nu_post=c.nu)
        self.gpu.setup(pr.K, pr.method, pr.tau, self.sm)
        self.N = self.gpu.nlevels
        assert self.N == self.H.N

    def olev(self, level):
        return self.H.levels[self.N - level]

    def vec(self, level, seed):
        return W.random_trace_vector(self.gpu.ndof(level), seed)

    def free(self, level):
        return self.olev(level).free


# (config, n, compare against the projected oracle): up to n = 64 against the oracle
# as it stands; from n = 128 on (and the config-5 recipe at 64), the oracle's
# constant-mode rounding, accumulated coherently through its Galerkin chain, moves a
# V-cycle by more than the gate (2e-11 at config 2, n = 128: DESIGN.md 2b), so there the
# reference is the oracle under the same readings as the GPU -- R5 / R9 on the fine maps
# (tests/oracle_proj.py) and R10 on every coarse level (oracle/multigrid.py,
# galerkin="macro", project_levels=True), whose two evaluation orders agree to ~5e-15
CASES = [(1, 8, False), (2, 16, False), (3, 16, False), (4, 16, False), (5, 16, False),
         (2, 64, False), (3, 64, False), (4, 64, False), (5, 64, False), (5, 64, True),
         (2, 128, True), (5, 128, True), (2, 256, True)]


@pytest.fixture(scope="module", params=CASES,
                ids=[f"c{a}n{b}" + ("proj" if c else "") for a, b, c in CASES])
def case(request):
    a, b, c = request.param
    return Case(a, b, proj=c)


def test_element_dtn_parity(case):
    """H1: element DtN maps S_T (batched local solves) vs the oracle."""
    S = case.gpu.element_dtn(case.N).cpu().numpy()
    So = case.ts.S
    err = np.abs(S - So).max(axis=(1, 2)) / np.abs(So).max(axis=(1, 2))
    assert err.max() <= TOL_OP, err.max()


def test_apply_parity_every_level(case):
    """H6 on every level (fine DtN maps, p-coarsened and Galerkin coarse DtN)."""
    for level in range(case.N, 0, -1):
        x = case.vec(level, case.cfg.seed_vec + level)
        y = case.gpu.apply(level, torch.from_numpy(x)).cpu().numpy()
        L = case.olev(level)
        fr = L.free
        yo = L.A @ x[fr]
        assert rel(y[fr], yo) <= TOL_OP, (level, rel(y[fr], yo))
        bd = np.setdiff1d(np.arange(len(y)), fr)
        assert np.all(y[bd] == 0.0)


def test_apply_with_oracle_dtn_injected(case):
    """The fine apply alone, fed the oracle's S_T through the test hook."""
    gpu = case.gpu
    gpu.set_element_dtn(case.N, torch.from_numpy(case.ts.S))
    x = case.vec(case.N, 7)
    y = gpu.apply(case.N, torch.from_numpy(x)).cpu().numpy()
    fr = case.ts.free
    assert rel(y[fr], case.ts.A @ x[fr]) <= TOL_OP
    case.gpu.setup(case.pr.K, case.pr.method, case.pr.tau, case.sm)   # restore


def test_smoother_parity(case):
    for level in range(case.N, 1, -1):
        L = case.olev(level)
        r = case.vec(level, 100 + level)
        e0 = case.vec(level, 200 + level)
        for steps in (1, 2, 3):
            e = case.gpu.smooth(level, torch.from_numpy(r), torch.from_numpy(e0), steps).cpu().numpy()
            eo = case.H.smooth(case.N - level, e0[L.free], r[L.free], steps)
            assert rel(e[L.free], eo) <= TOL_OP, (level, steps, rel(e[L.free], eo))


def test_transfer_parity(case):
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
        eo = e0[L.free] + case.H.prolong(li, ec[Lc.free])
        assert rel(e[L.free], eo) <= TOL_OP, level
        if L.kind == "h":
            e = case.gpu.local_correct(level, torch.from_numpy(res), torch.from_numpy(e0)).cpu().numpy()
            eo = e0[L.free] + case.H.local_correction(li, res[L.free])
            assert rel(e[L.free], eo) <= TOL_OP, level


def test_chebyshev_lambda_max_parity(case):
    if case.cfg.smoother != 1:
        pytest.skip("block-Jacobi")
    for level in range(case.N, 1, -1):
        lam = case.gpu.lambda_max(level)
        assert abs(lam - case.olev(level).lam_max) <= 1e-12 * lam, level


def test_vcycle_parity(case):
    r = case.vec(case.N, 600)
    z = case.gpu.vcycle(torch.from_numpy(r)).cpu().numpy()
    fr = case.ts.free
    zo = case.H.vcycle(r[fr])
    assert rel(z[fr], zo) <= TOL_OP, rel(z[fr], zo)
    bd = np.setdiff1d(np.arange(len(z)), fr)
    assert np.all(z[bd] == 0.0)


EXEC_PATHS = [("sweep", 1, 1), ("grid_cap", 2, 1), ("grid_cap", 2, 3)]


@pytest.mark.parametrize("path", EXEC_PATHS, ids=[f"{a}{c}" for a, _, c in EXEC_PATHS])
def test_exec_paths_parity(case, path):
    """The same operators through the other kernel paths (mg_set_option): the
    single-pass streamed smoothing kernel forced onto the small orbit levels
    (MG_OPT_SWEEP = 1, nx % 64 == 0), and apply grids capped at 1 or 3 CTAs, so every
    CTA walks many chunks and the TMA / segment rings wrap around (MG_OPT_APPLY_GRID_CAP)."""
    name, key, val = path
    if name == "sweep" and case.cfg.n % 64:
        pytest.skip("the streamed kernel needs nx % 64 == 0")
    if case.cfg.n > 128:
        pytest.skip("exec-path sweep at n <= 128")
    gpu = case.gpu
    gpu.set_option(key, val)
    try:
        for level in range(case.N, 0, -1):
            L = case.olev(level)
            x = case.vec(level, case.cfg.seed_vec + level)
            y = gpu.apply(level, torch.from_numpy(x)).cpu().numpy()
            assert rel(y[L.free], L.A @ x[L.free]) <= TOL_OP, (level, "apply")
            if level > 1:
                r = case.vec(level, 100 + level)
                e0 = case.vec(level, 200 + level)
                for steps in (1, 2, 3):
                    e = gpu.smooth(level, torch.from_numpy(r), torch.from_numpy(e0), steps).cpu().numpy()
                    eo = case.H.smooth(case.N - level, e0[L.free], r[L.free], steps)
                    assert rel(e[L.free], eo) <= TOL_OP, (level, steps, "smooth")
        r = case.vec(case.N, 600)
        z = gpu.vcycle(torch.from_numpy(r)).cpu().numpy()
        assert rel(z[case.ts.free], case.H.vcycle(r[case.ts.free])) <= TOL_OP
        pr = case.pr
        g, lam_bc = gpu.assemble_rhs(pr.f_qp, pr.f_const, pr.gD_qp)
        lam, info = gpu.pcg_solve(g, rtol=case.cfg.rtol, maxit=2000)
        res = krylov.pcg(case.ts.A, case.H.vcycle, case.ts.g, rtol=case.cfg.rtol, maxit=2000)
        assert abs(info["iters"] - res["iters"]) <= 1
        assert rel((lam + lam_bc).cpu().numpy(), case.ts.to_full(res["x"])) <= TOL_SOL
    finally:
        gpu.set_option(key, 0)


def test_gather_apply_bitwise(case):
    """The one-pass gather-form apply (k_apply_gather, MG_OPT_GATHER_NE) against the pair
    of colour passes on every packed P1 level: apply, 1-3 smoothing steps and the whole
    V-cycle agree bit for bit (same row sums in the same order, same combination order),
    and the gather-form V-cycle matches the oracle."""
    if case.cfg.n > 256:
        pytest.skip("bitwise gather check at n <= 256")
    gpu = case.gpu
    big = 1 << 40

    def run():
        out = []
        for level in range(case.N, 0, -1):
            x = case.vec(level, case.cfg.seed_vec + level)
            out.append(gpu.apply(level, torch.from_numpy(x)).cpu().numpy())
            if level > 1:
                r = case.vec(level, 100 + level)
                e0 = case.vec(level, 200 + level)
                for steps in (1, 2, 3):
                    out.append(gpu.smooth(level, torch.from_numpy(r), torch.from_numpy(e0), steps).cpu().numpy())
        out.append(gpu.vcycle(torch.from_numpy(case.vec(case.N, 600))).cpu().numpy())
        return out

    try:
        gpu.set_option(gpu.OPT_GATHER_NE, 0)
        pair = run()
        gpu.set_option(gpu.OPT_GATHER_NE, big)
        gath = run()
    finally:
        gpu.set_option(gpu.OPT_GATHER_NE, 1 << 16)
    assert len(pair) == len(gath)
    for k, (a, b) in enumerate(zip(pair, gath)):
        assert np.array_equal(a, b), (k, np.max(np.abs(a - b)))
    r = case.vec(case.N, 600)
    assert rel(gath[-1][case.ts.free], case.H.vcycle(r[case.ts.free])) <= TOL_OP


@pytest.mark.parametrize("knob", ["MGDTN_W0U", "MGDTN_DFX", "MGDTN_W0H"])
def test_pcg_fold_bitwise(case, knob):
    """Two bitwise-neutral rearrangements of the PCG / V-cycle on the orbit levels against
    the plain sequence, over a whole solve and one V-cycle:
    MGDTN_W0U -- the direction update p = z + beta p folded into the colour-0 pass of the
    next apply (AM_W0U) instead of the k_pcg_pupdate pass (the same fma per entry);
    MGDTN_DFX -- Chebyshev step 1 after a first step from e = 0 reads d_0 from the iterate
    x_1 = 0 + d_0 (STEP_D_FROM_X) and the first step stores no d;
    MGDTN_W0H -- the h-prolongation of the P1 orbit level folded into its first
    post-smoothing step's colour-0 pass (AM_W0H) instead of k_prolong_edges."""
    import os
    gpu = case.gpu
    pr = case.pr
    g, _ = gpu.assemble_rhs(pr.f_qp, pr.f_const, pr.gD_qp)
    r = torch.from_numpy(case.vec(case.N, 600))
    out = {}
    try:
        for v in ("0", "1"):
            os.environ[knob] = v
            gpu.set_option(gpu.OPT_GATHER_NE, 1 << 16)   # (drops the captured graphs)
            lam, info = gpu.pcg_solve(g, rtol=case.cfg.rtol, maxit=2000)
            z = gpu.vcycle(r).cpu().numpy()
            out[v] = (lam.cpu().numpy(), info["iters"], z)
    finally:
        os.environ.pop(knob, None)
        gpu.set_option(gpu.OPT_GATHER_NE, 1 << 16)
    assert out["0"][1] == out["1"][1]
    assert np.array_equal(out["0"][0], out["1"][0])
    assert np.array_equal(out["0"][2], out["1"][2])


def test_pcg_zdot_fold(case):
    """MGDTN_ZDOT: the PCG's r.z accumulated in the colour-1 epilogue of the V-cycle's last
    fine smoothing step (orbit fine level) instead of a k_dot pass -- the same products
    summed in another order: the same iteration count and the solution to 1e-12."""
    import os
    gpu = case.gpu
    pr = case.pr
    g, _ = gpu.assemble_rhs(pr.f_qp, pr.f_const, pr.gD_qp)
    out = {}
    try:
        for v in ("0", "1"):
            os.environ["MGDTN_ZDOT"] = v
            gpu.set_option(gpu.OPT_GATHER_NE, 1 << 16)   # (drops the captured graphs)
            lam, info = gpu.pcg_solve(g, rtol=case.cfg.rtol, maxit=2000)
            out[v] = (lam.cpu().numpy(), info["iters"])
    finally:
        os.environ.pop("MGDTN_ZDOT", None)
        gpu.set_option(gpu.OPT_GATHER_NE, 1 << 16)
    assert abs(out["0"][1] - out["1"][1]) <= 1
    assert rel(out["1"][0], out["0"][0]) <= 1e-12


def test_rhs_parity(case):
    pr = case.pr
    g, lam_bc = case.gpu.assemble_rhs(pr.f_qp, pr.f_const, pr.gD_qp)
    g = g.cpu().numpy()
    lam_bc = lam_bc.cpu().numpy()
    fr = case.ts.free
    assert rel(g[fr], case.ts.g) <= TOL_OP
    assert np.allclose(lam_bc, case.ts.lam_D, rtol=0, atol=1e-13 * max(1, np.abs(case.ts.lam_D).max()))


def test_pcg_parity(case):
    pr = case.pr
    g, lam_bc = case.gpu.assemble_rhs(pr.f_qp, pr.f_const, pr.gD_qp)
    lam, info = case.gpu.pcg_solve(g, rtol=case.cfg.rtol, maxit=2000)
    res = krylov.pcg(case.ts.A, case.H.vcycle, case.ts.g, rtol=case.cfg.rtol, maxit=2000)
    assert info["status"] == "converged"
    assert abs(info["iters"] - res["iters"]) <= 1, (info, res["iters"])
    lam_full = (lam + lam_bc).cpu().numpy()
    ref = case.ts.to_full(res["x"])
    assert rel(lam_full, ref) <= TOL_SOL, rel(lam_full, ref)
    # the GPU solution solves the oracle's system to the requested tolerance, up to the
    # drift of the recursive residual (the stopping test, reading Q16) that the oracle's
    # own PCG shows at this conditioning (c3n64: oracle 2.75e-10 at rtol 1e-10)
    fr = case.ts.free
    lf = lam.cpu().numpy()[fr]
    true_rel = np.linalg.norm(case.ts.g - case.ts.A @ lf) / np.linalg.norm(case.ts.g)
    # finite-precision CG: ||g - A x_k - r_k|| <= eps O(k) ||A|| max_j ||x_j|| (Greenbaum,
    # "Iterative methods for solving linear systems", ch. 7.3), ||A||_2 <= ||A||_1 (symmetric)
    import scipy.sparse.linalg as spla
    m = 4 * (case.cfg.p + 1)
    gap = info["iters"] * np.finfo(float).eps * 4 * m * spla.norm(case.ts.A, 1) * \
        np.linalg.norm(lf) / np.linalg.norm(case.ts.g)
    assert true_rel <= max(3 * case.cfg.rtol, 2 * res["true_relres"], case.cfg.rtol + gap), \
        (true_rel, res["true_relres"], gap)


def test_pcg_eager_equals_graph_replay(case):
    """The CUDA-graph replay of an iteration and eager launches give bit-identical
    results (deterministic reductions, same kernel sequence)."""
    pr = case.pr
    g, _ = case.gpu.assemble_rhs(pr.f_qp, pr.f_const, pr.gD_qp)
    lam1, i1 = case.gpu.pcg_solve(g, rtol=case.cfg.rtol, history=True)
    case.gpu.use_graphs(False)
    try:
        lam2, i2 = case.gpu.pcg_solve(g, rtol=case.cfg.rtol, history=True)
    finally:
        case.gpu.use_graphs(True)
    assert i1["iters"] == i2["iters"]
    assert torch.equal(lam1, lam2)
    assert np.array_equal(i1["hist"], i2["hist"])


def test_solve_host_matches_device_path(case):
    pr = case.pr
    lam_h, info = case.gpu.solve_host(pr.K, pr.method, pr.tau, pr.f_qp, pr.f_const, pr.gD_qp,
                                      case.sm, rtol=case.cfg.rtol)
    g, lam_bc = case.gpu.assemble_rhs(pr.f_qp, pr.f_const, pr.gD_qp)
    lam, info2 = case.gpu.pcg_solve(g, rtol=case.cfg.rtol)
    assert info["iters"] == info2["iters"]
    assert np.array_equal(lam_h, (lam + lam_bc).cpu().numpy())


# ---------------------------------------------------------------- edge cases
def test_zero_rhs_zero_iterations():
    from paper_1811_09909_b200 import MGSolver, SmootherConfig
    s = MGSolver(8, p=2)
    s.setup(np.ones(64), np.zeros(64, np.int8), np.ones(64), SmootherConfig())
    lam, info = s.pcg_solve(torch.zeros(s.ndof(), dtype=torch.float64, device="cuda"))
    assert info["iters"] == 0 and info["status"] == "converged"
    assert torch.count_nonzero(lam).item() == 0


@pytest.mark.parametrize("n,p", [(2, 1), (2, 3), (4, 2), (6, 1), (12, 2), (10, 4)])
def test_small_and_ragged_meshes(n, p):
    """n = 2 (the direct level only), n = 6 / 10 / 12 (coarsening stops at an
    odd or non-2x2 macro mesh, dense coarsest), element counts that are not a
    multiple of 32 (ragged chunk tails)."""
    from paper_1811_09909_b200 import MGSolver, SmootherConfig
    c = W.Config(1, "edge", n=n, p=p, nu=2, smoother=0)
    pr = W.make_problem(c)
    ts = assembly.TraceSystem(n, p, pr.K, pr.method, pr.tau, pr.f_qp)
    H = multigrid.Hierarchy(ts.A, n, p, smoother=0, nu_pre=2, nu_post=2)
    s = MGSolver(n, p=p)
    assert s.nlevels == H.N
    s.setup(pr.K, pr.method, pr.tau, SmootherConfig())
    x = W.random_trace_vector(s.ndof(), 5)
    y = s.apply(s.nlevels, torch.from_numpy(x)).cpu().numpy()
    assert rel(y[ts.free], ts.A @ x[ts.free]) <= TOL_OP
    z = s.vcycle(torch.from_numpy(x)).cpu().numpy()
    assert rel(z[ts.free], H.vcycle(x[ts.free])) <= TOL_OP
    g, _ = s.assemble_rhs(pr.f_qp)
    lam, info = s.pcg_solve(g)
    res = krylov.pcg(ts.A, H.vcycle, ts.g)
    assert abs(info["iters"] - res["iters"]) <= 1
    assert rel(lam.cpu().numpy()[ts.free], res["x"]) <= TOL_SOL


def test_sipg_not_spd_is_reported():
    """An under-penalised SIPG-H element makes a local or edge block
    indefinite: the setup returns MG_ERR_NOT_SPD instead of producing garbage."""
    from paper_1811_09909_b200 import MGError, MGSolver, SmootherConfig
    s = MGSolver(8, p=3)
    ne = 64
    tau = np.full(ne, 1e-3)
    with pytest.raises(MGError, match="NOT_SPD"):
        s.setup(np.ones(ne), np.ones(ne, np.int8), tau, SmootherConfig())


def test_launch_counts_reported():
    from paper_1811_09909_b200 import MGSolver, SmootherConfig
    c = W.CONFIGS[1]
    pr = W.make_problem(c)
    s = MGSolver(8, p=1)
    s.setup(pr.K, pr.method, pr.tau, SmootherConfig())
    g, _ = s.assemble_rhs(pr.f_qp)
    _, info = s.pcg_solve(g)
    assert s.last_launch_count() >= 3 * info["iters"]
