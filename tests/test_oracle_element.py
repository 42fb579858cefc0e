"""Pins of oracle/basis.py and oracle/element.py against closed forms,
textbook values and an independent elimination."""
import numpy as np
import pytest

from oracle import basis
from oracle import element as el


# ---------------------------------------------------------------- P1 basis
def test_gll_nodes_closed_form():
    assert np.allclose(basis.gll_nodes(1), [0, 1])
    assert np.allclose(basis.gll_nodes(2), [0, 0.5, 1])
    a = 1 / np.sqrt(5)
    assert np.allclose(basis.gll_nodes(3), [0, (1 - a) / 2, (1 + a) / 2, 1], atol=1e-15)
    b = np.sqrt(3 / 7)
    assert np.allclose(basis.gll_nodes(4), [0, (1 - b) / 2, 0.5, (1 + b) / 2, 1], atol=1e-15)


@pytest.mark.parametrize("nq", [1, 2, 3, 5, 8])
def test_gauss_exactness(nq):
    x, w = basis.gauss(nq)
    for k in range(2 * nq):
        assert abs(w @ x ** k - 1.0 / (k + 1)) < 1e-14


@pytest.mark.parametrize("p", [1, 2, 3, 4])
def test_lagrange_nodal_partition_of_unity(p):
    nodes = basis.gll_nodes(p)
    assert np.allclose(basis.lagrange(nodes, nodes), np.eye(p + 1), atol=1e-14)
    x = np.linspace(0, 1, 17)
    assert np.allclose(basis.lagrange(nodes, x).sum(1), 1.0, atol=1e-13)
    assert np.allclose(basis.lagrange_deriv(nodes, x).sum(1), 0.0, atol=1e-11)
    # derivative vs finite differences (SPEC fem_basis invariant)
    eps = 1e-6
    fd = (basis.lagrange(nodes, x + eps) - basis.lagrange(nodes, x - eps)) / (2 * eps)
    assert np.allclose(basis.lagrange_deriv(nodes, x), fd, atol=1e-7)


def test_edge_mass_p1():
    # p=1, length 1 -> [[1/3, 1/6], [1/6, 1/3]]
    assert np.allclose(el.ref(1).Hhat1, [[1 / 3, 1 / 6], [1 / 6, 1 / 3]], atol=1e-15)


def test_q1_mass_closed_form():
    # bilinear mass on the unit square: 1/36 * [4 2 2 1; 2 4 1 2; 2 1 4 2; 1 2 2 4]
    M = el.ref(1).M
    ref = np.array([[4, 2, 2, 1], [2, 4, 1, 2], [2, 1, 4, 2], [1, 2, 2, 4]]) / 36.0
    assert np.allclose(M, ref, atol=1e-15)


@pytest.mark.parametrize("p", [1, 2, 3, 4])
def test_divergence_theorem_and_stiffness(p):
    R = el.ref(p)
    # int_T d_x phi_j = oint phi_j n_x
    assert np.allclose(R.Dx.sum(0), R.Fx.sum(0), atol=1e-13)
    assert np.allclose(R.Dy.sum(0), R.Fy.sum(0), atol=1e-13)
    # integration by parts, exact quadrature: Dx + Dx^T = Fx
    assert np.allclose(R.Dx + R.Dx.T, R.Fx, atol=1e-13)
    # stiffness row sums vanish
    assert np.allclose(R.L.sum(1), 0.0, atol=1e-12)
    # total edge length 4, area 1
    assert abs(R.E.sum() - 4.0) < 1e-13 and abs(R.M.sum() - 1.0) < 1e-13


# ---------------------------------------------------------------- P2-P6
def _rand_elems(p, ne, seed, method):
    rng = np.random.default_rng(seed)
    K = 10.0 ** rng.uniform(-2, 2, ne)
    h = 1.0 / 8
    if method == el.HDG:
        tau = 10.0 ** rng.uniform(-1, 1, ne)
    else:
        tau = 10.0 * p * p * K / h
    return K, tau, h


def _nodal_trace(p, h, fun, x0=0.0, y0=0.0):
    """Nodal values of fun on the 4 local edges (global orientation)."""
    s = basis.gll_nodes(p)
    pts = [(x0 + s * h, y0 + 0 * s), (x0 + h + 0 * s, y0 + s * h), (x0 + s * h, y0 + h + 0 * s),
           (x0 + 0 * s, y0 + s * h)]
    return np.concatenate([fun(x, y) for x, y in pts])


def _flux_moments(p, h, gradn_fun):
    """<g, mu_a>_f on each local edge, g given per edge as a function of s."""
    xq, wq = basis.gauss(p + 4)
    MU = basis.lagrange(basis.gll_nodes(p), xq)
    out = []
    for f in range(4):
        g = gradn_fun(f, xq)
        out.append(h * np.einsum("q,q,qa->a", wq, g, MU))
    return np.concatenate(out)


@pytest.mark.parametrize("method", [el.HDG, el.SIPG_H])
@pytest.mark.parametrize("p", [1, 2, 3, 4])
def test_dtn_symmetric_psd_constants(method, p):
    ne = 16
    K, tau, h = _rand_elems(p, ne, 7 + p, method)
    S = el.element_dtn(p, K, np.full(ne, method), tau, h)
    for s in S:
        assert np.abs(s - s.T).max() <= 1e-12 * np.abs(s).max()
        ev = np.linalg.eigvalsh(0.5 * (s + s.T))
        assert ev.min() > -1e-11 * ev.max()
        # constant traces are annihilated (u=0, q=lambda=c solves the local problem)
        assert np.abs(s @ np.ones(len(s))).max() <= 1e-11 * np.abs(s).max()


@pytest.mark.parametrize("method", [el.HDG, el.SIPG_H, el.IIPG_H, el.NIPG_H])
@pytest.mark.parametrize("p", [1, 2, 3, 4])
def test_dtn_reproduces_linear_flux_closed_form(method, p):
    """For q = a + bx + cy (in every space, f = 0) the local solution is exact,
    so S_T lambda_q = <K grad q . n, mu>_f (closed form)."""
    ne = 6
    K, tau, h = _rand_elems(p, ne, 3 + p, method)
    S = el.element_dtn(p, K, np.full(ne, method), tau, h)
    b, c = 0.7, -1.3
    q = lambda x, y: 0.2 + b * x + c * y
    lam = _nodal_trace(p, h, q, 0.25, 0.5)
    normals = el.NORMALS
    for e in range(ne):
        mom = _flux_moments(p, h, lambda f, s: K[e] * (b * normals[f, 0] + c * normals[f, 1]) + 0 * s)
        assert np.allclose(S[e] @ lam, mom, atol=1e-11 * max(1.0, np.abs(mom).max()))


@pytest.mark.parametrize("method", [el.HDG, el.SIPG_H, el.IIPG_H, el.NIPG_H])
@pytest.mark.parametrize("p", [2, 3, 4])
def test_dtn_and_load_reproduce_quadratic(method, p):
    """q = x^2 + 2y^2 - xy, f = -K Lap q = -6K: S lambda_q - b_T = <K grad q.n, mu>."""
    ne = 4
    K, tau, h = _rand_elems(p, ne, 11 + p, method)
    x0, y0 = 0.125, 0.375
    meth = np.full(ne, method)
    S = el.element_dtn(p, K, meth, tau, h)
    q = lambda x, y: x * x + 2 * y * y - x * y
    gx = lambda x, y: 2 * x - y
    gy = lambda x, y: 4 * y - x
    lam = _nodal_trace(p, h, q, x0, y0)
    xq, _ = basis.gauss(p + 4)
    nq = len(xq)
    # the oracle's load ignores element position except through f samples
    f_qp = np.broadcast_to((-6.0 * K)[:, None, None], (ne, nq, nq)).copy()
    bT = el.element_rhs(p, K, meth, tau, h, f_qp)
    pts = [(lambda s: (x0 + s * h, y0 + 0 * s)), (lambda s: (x0 + h + 0 * s, y0 + s * h)),
           (lambda s: (x0 + s * h, y0 + h + 0 * s)), (lambda s: (x0 + 0 * s, y0 + s * h))]
    for e in range(ne):
        def gn(f, s):
            x, y = pts[f](s)
            return K[e] * (gx(x, y) * el.NORMALS[f, 0] + gy(x, y) * el.NORMALS[f, 1])
        mom = _flux_moments(p, h, gn)
        assert np.allclose(S[e] @ lam - bT[e], mom, atol=1e-11 * np.abs(mom).max())


@pytest.mark.parametrize("p", [1, 2, 3, 4])
def test_hdg_dtn_equals_staged_schur_elimination(p):
    """P3: the literal full (u, q) elimination equals the staged Schur form
    S = K W + t H - (K P + t E)^T (K G + t F)^-1 (K P + t E), t = tau h,
    G = Dx M^-1 Dx^T + ..., derived by eliminating u first."""
    R = el.ref(p)
    ne = 8
    K, tau, h = _rand_elems(p, ne, 5, el.HDG)
    S = el.element_dtn(p, K, np.zeros(ne, np.int8), tau, h)
    Mi = np.linalg.inv(R.M)
    # divergence form (integrated by parts) of HDG_local2 -- different algebra
    Dxd, Dyd = R.Fx - R.Dx.T, R.Fy - R.Dy.T
    G = Dxd @ Mi @ R.Dx.T + Dyd @ Mi @ R.Dy.T
    P = Dxd @ Mi @ R.Cx + Dyd @ Mi @ R.Cy
    W = R.Cx.T @ Mi @ R.Cx + R.Cy.T @ Mi @ R.Cy
    for e in range(ne):
        t = tau[e] * h
        Q = K[e] * G + t * R.F
        Rm = t * R.E + K[e] * P
        S0 = K[e] * W + t * R.H
        Sref = S0 - Rm.T @ np.linalg.solve(Q, Rm)
        assert np.allclose(S[e], Sref, atol=1e-12 * np.abs(Sref).max())


@pytest.mark.parametrize("method", [el.HDG, el.SIPG_H])
def test_dtn_scaling_laws(method):
    """P4/P6: S(aK, a tau, h) = a S(K, tau, h); S(K, tau, h) = S(K, tau h, 1);
    SIPG-H with tau = 10 p^2 K/h: S(K) = K S(1) (reading Q9)."""
    p = 3
    K = np.array([0.3, 2.0, 50.0])
    h = 1.0 / 16
    tau = 10 * p * p * K / h if method == el.SIPG_H else np.array([1.0, 3.0, 0.5])
    m = np.full(3, method)
    S = el.element_dtn(p, K, m, tau, h)
    S2 = el.element_dtn(p, 4.0 * K, m, 4.0 * tau, h)
    assert np.allclose(S2, 4.0 * S, atol=1e-11 * np.abs(S2).max())
    S3 = el.element_dtn(p, K, m, tau * h, 1.0)
    assert np.allclose(S3, S, atol=1e-12 * np.abs(S).max())
    if method == el.SIPG_H:
        S1 = el.element_dtn(p, np.ones(3), m, 10 * p * p / h * np.ones(3), h)
        assert np.allclose(S, K[:, None, None] * S1, atol=1e-11 * np.abs(S).max())


@pytest.mark.parametrize("method", [el.HDG, el.SIPG_H, el.IIPG_H, el.NIPG_H])
@pytest.mark.parametrize("p", [1, 3])
def test_local_conservation(method, p):
    """sum over dT of u_hat.n = int_T f for ANY lambda (test w = 1 in the
    local equation)."""
    ne = 5
    K, tau, h = _rand_elems(p, ne, 9, method)
    meth = np.full(ne, method)
    rng = np.random.default_rng(1)
    nq = p + 4
    f_qp = rng.uniform(-1, 1, (ne, nq, nq))
    S = el.element_dtn(p, K, meth, tau, h)
    b = el.element_rhs(p, K, meth, tau, h, f_qp)
    lam = rng.uniform(-1, 1, (ne, 4 * (p + 1)))
    flux = b - np.einsum("eij,ej->ei", S, lam)
    _, w = basis.gauss(nq)
    intf = h * h * np.einsum("y,x,eyx->e", w, w, f_qp)
    assert np.allclose(flux.sum(1), intf, atol=1e-12 * np.abs(intf).max())


# ---------------------------------------------------------------- IIPG-H / NIPG-H (Eq. IPG_H)
@pytest.mark.parametrize("method", [el.IIPG_H, el.NIPG_H])
@pytest.mark.parametrize("p", [1, 2, 3, 4])
def test_ipdg_dtn_nonsymmetric_with_constant_null_vectors(method, p):
    """Eq. IPG_H with s_f != 1 is not symmetric, but constants
    are both a right null vector (q = lambda = c solves the local problem) and a
    left one (test w = 1: the total flux is (f, 1), independent of lambda)."""
    ne = 12
    K, tau, h = _rand_elems(p, ne, 17 + p, method)
    S = el.element_dtn(p, K, np.full(ne, method), tau, h)
    one = np.ones(S.shape[1])
    for s in S:
        sc = np.abs(s).max()
        assert np.abs(s - s.T).max() > 1e-3 * sc
        assert np.abs(s @ one).max() <= 1e-11 * sc
        assert np.abs(one @ s).max() <= 1e-11 * sc


def _energy_terms(p, K, tau, h, method, lam):
    """q from the local solve (f = 0) and the quadratic forms of the energy
    identities: K (grad q, grad q)_T, tau ||q - lambda||^2_dT, K <grad q.n, q - lambda>_dT."""
    R = el.ref(p)
    q = el.recover_q(p, K, np.full(len(K), method), tau, h, lam)
    grad = K * np.einsum("ei,ij,ej->e", q, R.L, q)
    jump = tau * h * (np.einsum("ei,ij,ej->e", q, R.F, q) - 2 * np.einsum("ei,ia,ea->e", q, R.E, lam)
                      + np.einsum("ea,ab,eb->e", lam, R.H, lam))
    bnd = K * (np.einsum("ei,ij,ej->e", q, R.N, q) - np.einsum("ei,ia,ea->e", q, R.Nl, lam))
    return grad, jump, bnd


@pytest.mark.parametrize("p", [1, 2, 3, 4])
def test_nipg_energy_identity(p):
    """NIPG-H (s_f = -1), f = 0, test w = q in Eq. IPG_H: the s_f term cancels the
    consistency term, so lambda^T S_T lambda = K ||grad q||^2 + tau ||q - lambda||^2_dT
    (>= 0 for every tau > 0); a wrong s_f sign breaks it."""
    ne = 8
    K, tau, h = _rand_elems(p, ne, 23 + p, el.NIPG_H)
    tau = tau * np.geomspace(1e-3, 1.0, ne)       # any tau > 0
    S = el.element_dtn(p, K, np.full(ne, el.NIPG_H), tau, h)
    lam = np.random.default_rng(p).uniform(-1, 1, (ne, S.shape[1]))
    grad, jump, _ = _energy_terms(p, K, tau, h, el.NIPG_H, lam)
    lhs = np.einsum("ea,eab,eb->e", lam, S, lam)
    assert np.allclose(lhs, grad + jump, rtol=1e-10, atol=0)


@pytest.mark.parametrize("method,sf", [(el.IIPG_H, 0.0), (el.SIPG_H, 1.0)])
@pytest.mark.parametrize("p", [1, 3])
def test_ipdg_energy_identity(method, sf, p):
    """Eq. IPG_H tested with w = q (f = 0): lambda^T S_T lambda = K ||grad q||^2
    - (1 + s_f) K <grad q.n, q - lambda> + tau ||q - lambda||^2 (s_f = 0, 1)."""
    ne = 6
    K, tau, h = _rand_elems(p, ne, 31 + p, method)
    S = el.element_dtn(p, K, np.full(ne, method), tau, h)
    lam = np.random.default_rng(5 + p).uniform(-1, 1, (ne, S.shape[1]))
    grad, jump, bnd = _energy_terms(p, K, tau, h, method, lam)
    lhs = np.einsum("ea,eab,eb->e", lam, S, lam)
    rhs = grad - (1.0 + sf) * bnd + jump
    assert np.allclose(lhs, rhs, rtol=1e-9, atol=1e-10 * np.abs(grad).max())
