"""Pins of oracle/assembly.py + the discretisation as a whole (SURVEY 8(c)
P5, P7, P8): exact special cases, global SPD structure and the convergence
law of the hybridized methods (PAPER.md:1083-1084 cites O(h^{p+1}))."""
import numpy as np
import pytest
import scipy.sparse.linalg as spla

import workloads as W
from oracle import assembly, basis, mesh
from oracle import element as el


def _solve_direct(ts):
    return ts.to_full(spla.spsolve(ts.A.tocsc(), ts.g))


def test_numbering_counts():
    # SPEC.md:53 n=4 -> 40 edges; SPEC.md:229 2x2 p=1 -> 8 free dofs
    assert mesh.n_edges(4) == 40
    assert len(mesh.free_dofs(2, 1)) == 8
    assert len(mesh.boundary_edges(4)) == 16
    ed = mesh.element_edges(3)
    # each interior edge shared by exactly two elements, boundary by one
    cnt = np.bincount(ed.ravel(), minlength=mesh.n_edges(3))
    assert np.all(cnt[mesh.boundary_edge_mask(3)] == 1)
    assert np.all(cnt[~mesh.boundary_edge_mask(3)] == 2)
    # checkerboard: same-colour elements share no edge
    j, i = np.divmod(np.arange(9), 3)
    for c in (0, 1):
        e = ed[((i + j) % 2) == c].ravel()
        assert len(np.unique(e)) == len(e)


def test_global_A_spd_config1():
    c = W.CONFIGS[1]
    pr = W.make_problem(c)
    ts = assembly.TraceSystem(c.n, c.p, pr.K, pr.method, pr.tau, pr.f_qp)
    A = ts.A.toarray()
    assert A.shape == (224, 224)
    assert np.abs(A - A.T).max() <= 1e-14 * np.abs(A).max()
    assert np.linalg.eigvalsh(A).min() > 0
    # full operator without Dirichlet elimination annihilates constants
    assert np.abs(ts.A_full @ np.ones(ts.ndof)).max() < 1e-12


@pytest.mark.parametrize("p", [1, 2, 3])
@pytest.mark.parametrize("method", [el.HDG, el.SIPG_H, el.IIPG_H, el.NIPG_H])
def test_constant_and_linear_solution_exact(p, method):
    """f = 0, g_D = linear -> lambda = trace of that linear function."""
    n = 4
    h = 1.0 / n
    K = np.full(n * n, 3.0)          # uniform K: a linear q is the exact solution
    tau = np.full(n * n, 2.0) if method == el.HDG else 10 * p * p * K / h
    BX, BY = W.boundary_sample_coords(n, p)
    lin = lambda x, y: 1.0 + 0.5 * x - 0.25 * y
    ts = assembly.TraceSystem(n, p, K, np.full(n * n, method), tau, None, 0.0, lin(BX, BY))
    lam = _solve_direct(ts)
    # nodal trace of the linear function on every edge
    s = basis.gll_nodes(p)
    ne = mesh.n_edges(n)
    ref = np.zeros(ne * (p + 1))
    for e in range(ne):
        if e < n * (n + 1):
            j, i = divmod(e, n)
            x, y = (i + s) * h, j * h + 0 * s
        else:
            j, i = divmod(e - n * (n + 1), n + 1)
            x, y = i * h + 0 * s, (j + s) * h
        ref[e * (p + 1):(e + 1) * (p + 1)] = lin(x, y)
    assert np.allclose(lam, ref, atol=1e-12)


def _l2_error(ts, lam_full, exact):
    n, p, h = ts.n, ts.p, ts.h
    lamT = lam_full[mesh.element_dofs(n, p)]
    q = el.recover_q(p, ts.K, ts.method, ts.tau, h, lamT, ts.f_qp, ts.f_const)
    R = el.ref(p)
    X, Y = W.element_sample_coords(n, p)
    qh = np.einsum("yxi,ei->eyx", R.f_basis, q)
    err2 = h * h * np.einsum("yx,eyx->", R.f_weights, (qh - exact(X, Y)) ** 2)
    return np.sqrt(err2)


@pytest.mark.parametrize("p,ns", [(1, (8, 16, 32)), (2, (4, 8, 16)), (3, (4, 8, 16)), (4, (4, 8))])
def test_hdg_convergence_order(p, ns):
    """P8: manufactured u = sin(pi x) sin(pi y), K = 1, tau = 1 (configs 1/2
    recipe): ||q - q_h||_L2 = O(h^{p+1}) (order p+1 +- 0.25)."""
    errs = []
    for n in ns:
        c = W.Config(0, "conv", n=n, p=p, nu=2, smoother=0)
        c.index = 1
        pr = W.make_problem(c)
        ts = assembly.TraceSystem(n, p, pr.K, pr.method, pr.tau, pr.f_qp)
        errs.append(_l2_error(ts, _solve_direct(ts), pr.exact))
    orders = np.log2(np.array(errs[:-1]) / np.array(errs[1:]))
    assert abs(orders[-1] - (p + 1)) < 0.25, (errs, orders)


@pytest.mark.parametrize("p", [1, 2, 3])
def test_sipg_convergence_order(p):
    errs = []
    for n in (8, 16, 32) if p == 1 else (4, 8, 16):
        h = 1.0 / n
        X, Y = W.element_sample_coords(n, p)
        u = lambda x, y: np.sin(np.pi * x) * np.sin(np.pi * y)
        ts = assembly.TraceSystem(n, p, np.ones(n * n), np.full(n * n, el.SIPG_H),
                                  np.full(n * n, 10 * p * p / h), 2 * np.pi ** 2 * u(X, Y))
        errs.append(_l2_error(ts, _solve_direct(ts), u))
    orders = np.log2(np.array(errs[:-1]) / np.array(errs[1:]))
    assert abs(orders[-1] - (p + 1)) < 0.25, (errs, orders)


def test_dirichlet_projection_exact_for_polynomials():
    """Q4: L2 projection reproduces P^p boundary data exactly."""
    n, p = 4, 3
    BX, BY = W.boundary_sample_coords(n, p)
    cub = lambda x, y: x ** 3 - 2 * y ** 2 + x * y
    lam = assembly.dirichlet_values(n, p, cub(BX, BY))
    s = basis.gll_nodes(p)
    h = 1.0 / n
    e = mesh.hedge(n, 1, 0)
    assert np.allclose(lam[e * 4:(e + 1) * 4], cub((1 + s) * h, 0 * s), atol=1e-13)
    e = mesh.vedge(n, n, 2)
    assert np.allclose(lam[e * 4:(e + 1) * 4], cub(1 + 0 * s, (2 + s) * h), atol=1e-13)
