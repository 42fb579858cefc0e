"""Pins of the seed-point agglomeration oracle (oracle/agglomerate.py,
PAPER.md:491-498; readings A1-A3 in DESIGN.md section 3) against what does not
depend on it: scipy's graph shortest paths (brute force), the closed-form
Voronoi cells of a strip, the closed-form quadtree of a 2^m x 2^m grid, and
the invariants every correct agglomeration has."""
import numpy as np
import pytest
from scipy.sparse import coo_matrix
from scipy.sparse.csgraph import connected_components, shortest_path

from oracle import agglomerate as A
from workloads.unstructured import holed_quad_mesh, structured_quad_mesh


def _graph(ne, edge_elem):
    m = edge_elem[edge_elem[:, 1] >= 0]
    return coo_matrix((np.ones(len(m)), (m[:, 0], m[:, 1])), shape=(ne, ne)).tocsr()


@pytest.mark.parametrize("n,sx,sy,seed", [(12, 2, 2, 1), (20, 3, 2, 2), (24, 4, 2, 3001)])
def test_level1_is_graph_voronoi_by_scipy_shortest_paths(n, sx, sy, seed):
    """A1 against an independent library routine: unweighted all-source
    shortest paths from scipy, then argmin over (distance, seed index)."""
    m = holed_quad_mesh(n, holes=3, sx=sx, sy=sy, seed=seed)
    D = shortest_path(_graph(m.ne, m.edge_elem), directed=False, unweighted=True,
                      indices=m.seeds)                      # [nseed, ne]
    assert np.isfinite(D).all()
    want = np.lexsort((np.arange(len(m.seeds))[:, None].repeat(m.ne, 1), D), axis=0)[0]
    got = A.seed_agglomerate(m.ne, m.edge_elem, m.seeds)
    np.testing.assert_array_equal(got, want)


def test_level1_on_a_strip_is_nearest_seed_with_ties_to_the_lower_index():
    """1 x L strip: the dual graph is a path, d(t, s) = |t - s| (closed form)."""
    L = 23
    edge_elem = np.array([[t, t + 1] for t in range(L - 1)] + [[t, -1] for t in range(L)],
                         dtype=np.int32)
    seeds = [17, 3, 10, 20]
    got = A.seed_agglomerate(L, edge_elem, seeds)
    for t in range(L):
        d = [abs(t - s) for s in seeds]
        want = min(range(len(seeds)), key=lambda k: (d[k], k))
        assert got[t] == want
    seeds = [8, 2]                    # t = 5: d = 3 to both -> seed 0 (lower index)
    got = A.seed_agglomerate(L, edge_elem, seeds)
    assert got[5] == 0 and got[4] == 1 and got[6] == 0


@pytest.mark.parametrize("m", [2, 3, 4])
def test_quadrisection_of_a_square_grid_is_the_quadtree(m):
    """A2 closed form: one seed on a 2^m x 2^m grid without jitter; level k
    (k >= 2) id of element (i, j) = sum over the quadtree digits, east = x bit,
    north = y bit, most significant first.  A transposed key or swapped child
    digits breaks it."""
    n = 1 << m
    mesh = structured_quad_mesh(n, seeds=(5,))
    labels, skel = A.agglomerate_levels(mesh.ne, mesh.edge_elem, mesh.cx, mesh.cy, mesh.seeds,
                                        nlev=m + 3)
    # element numbering of the structured mesh: row by row
    i = np.arange(mesh.ne) % n
    j = np.arange(mesh.ne) // n
    assert (labels[0] == 0).all()
    for k in range(2, m + 2):
        want = np.zeros(mesh.ne, dtype=np.int64)
        for lvl in range(1, k):
            shift = m - lvl
            want = 4 * want + 2 * ((i >> shift) & 1) + ((j >> shift) & 1)
        np.testing.assert_array_equal(labels[k - 1], want)
    # one element per agglomerate at level m+1: the next split keeps it in child 0
    np.testing.assert_array_equal(labels[m + 1], 4 * labels[m])
    # level m+1 skeleton = every edge; level 1 skeleton = the boundary of the box
    assert skel[m].all()
    np.testing.assert_array_equal(skel[0], (mesh.edge_elem[:, 1] < 0).astype(np.uint8))


def test_split_sizes_connectivity_and_nested_skeletons():
    m = holed_quad_mesh(40, holes=6, sx=3, sy=2, seed=7)
    labels, skel = A.agglomerate_levels(m.ne, m.edge_elem, m.cx, m.cy, m.seeds, nlev=5)
    G = _graph(m.ne, m.edge_elem)
    # level-1 cells are connected (graph Voronoi cells with a consistent tie rule)
    for g in np.unique(labels[0]):
        idx = np.flatnonzero(labels[0] == g)
        nc, _ = connected_components(G[idx][:, idx], directed=False)
        assert nc == 1
    for k in range(labels.shape[0] - 1):
        par, ch = labels[k], labels[k + 1]
        np.testing.assert_array_equal(ch // 4, par)          # children refine parents
        for g in np.unique(par):
            msz = int((par == g).sum())
            h = [(msz + 1) // 2, msz // 2]
            want = sorted([(h[0] + 1) // 2, h[0] // 2, (h[1] + 1) // 2, h[1] // 2])
            got = sorted(int((ch == 4 * g + q).sum()) for q in range(4))
            assert got == want
        assert (skel[k] <= skel[k + 1]).all()                 # M_{k-1} inside M_{k,B}
    assert skel[:, m.edge_elem[:, 1] < 0].all()


def test_west_half_lies_left_of_east_half():
    """A2: every west element precedes every east element of its parent in (cx, cy, id)."""
    m = holed_quad_mesh(32, holes=4, sx=2, sy=2, seed=11)
    labels, _ = A.agglomerate_levels(m.ne, m.edge_elem, m.cx, m.cy, m.seeds, nlev=3)
    for g in np.unique(labels[0]):
        idx = np.flatnonzero(labels[0] == g)
        east = (labels[1][idx] // 2) % 2
        kx = [(m.cx[t], m.cy[t], t) for t in idx]
        assert max(k for k, e in zip(kx, east) if e == 0) < min(k for k, e in zip(kx, east) if e == 1)


def test_unreachable_element_raises():
    edge_elem = np.array([[0, 1], [2, -1], [0, -1], [1, -1]], dtype=np.int32)
    with pytest.raises(ValueError):
        A.seed_agglomerate(3, edge_elem, [0])


def test_macro_edges_of_the_quadtree_closed_form():
    """A4 on the 2^m grid with one seed: level 2 (four quadrants) has 4 interior
    macro-edges (W-E pairs (0,2), (1,3), S-N pairs (0,1), (2,3)) and 4 boundary
    ones; every macro-edge of level k is a union of level-(k+1) macro-edges."""
    n = 8
    mesh = structured_quad_mesh(n)
    labels, skel = A.agglomerate_levels(mesh.ne, mesh.edge_elem, mesh.cx, mesh.cy, mesh.seeds, 4)
    me, nme = A.macro_edges(labels[1], mesh.edge_elem)
    assert nme == 8
    np.testing.assert_array_equal(me >= 0, skel[1].astype(bool))
    a, b = mesh.edge_elem[:, 0], mesh.edge_elem[:, 1]
    pairs = sorted({(-1, int(labels[1][x])) if y < 0 else tuple(sorted((int(labels[1][x]), int(labels[1][y]))))
                    for x, y in zip(a, b) if y < 0 or labels[1][x] != labels[1][y]})
    assert pairs == [(-1, 0), (-1, 1), (-1, 2), (-1, 3), (0, 1), (0, 2), (1, 3), (2, 3)]
    for q in range(nme):      # a quadrant's share of dOmega: two sides; an interface: one
        assert (me == q).sum() == (n if pairs[q][0] < 0 else n // 2)
    me3, _ = A.macro_edges(labels[2], mesh.edge_elem)
    for q in range(nme):                           # nesting: children's macro-edges tile it
        sub = np.unique(me3[me == q])
        assert (sub >= 0).all()
        for r in sub:
            assert (me[me3 == r] == q).all()


def _params(mesh, labels, k):
    me, nme = A.macro_edges(labels[k], mesh.edge_elem)
    return me, nme, A.macro_edge_params(me, nme, mesh.edge_vert, mesh.vx, mesh.vy)


def test_macro_edge_parameter_of_the_quadtree_closed_form():
    """A5 on the unjittered 8 x 8 grid (one seed), level 2: each interior macro-edge is
    a straight 4-edge segment, s = distance to its start end / its length (exact in
    binary here); each quadrant's share of dOmega is an L of 8 edges from the end least
    in (x, y): s = arc length / 1."""
    n = 8
    mesh = structured_quad_mesh(n)
    labels, _ = A.agglomerate_levels(mesh.ne, mesh.edge_elem, mesh.cx, mesh.cy, mesh.seeds, 3)
    me, nme, P = _params(mesh, labels, 1)
    assert (P[me >= 0] >= 0).all()
    X, Y = mesh.vx, mesh.vy
    for q in range(nme):
        es = np.flatnonzero(me == q)
        verts = np.unique(mesh.edge_vert[es])
        deg = {v: int((mesh.edge_vert[es] == v).sum()) for v in verts}
        ends = sorted([v for v in verts if deg[v] == 1], key=lambda v: (X[v], Y[v], v))
        start, stop = ends
        corner = [v for v in verts if X[v] == 0.0 and Y[v] == 0.0 or X[v] == 1.0 and Y[v] == 0.0
                  or X[v] == 0.0 and Y[v] == 1.0 or X[v] == 1.0 and Y[v] == 1.0]
        for e in es:
            for c in range(2):
                v = mesh.edge_vert[e, c]
                if corner and len(es) == n:       # L-shaped boundary share (through a box corner)
                    cv = corner[0]
                    on_start_side = X[v] == X[cv] if X[start] == X[cv] else Y[v] == Y[cv]
                    d1 = lambda u, w: abs(X[u] - X[w]) + abs(Y[u] - Y[w])
                    want = d1(v, start) if on_start_side else d1(start, cv) + d1(v, cv)
                else:                              # straight segment
                    want = (abs(X[v] - X[start]) + abs(Y[v] - Y[start])) / \
                        (abs(X[stop] - X[start]) + abs(Y[stop] - Y[start]))
                assert P[e, c] == want, (q, e, c, P[e, c], want)


def test_macro_edge_parameter_invariants_on_holed_meshes():
    """A5 on jittered holed meshes: a parameterised macro-edge's s runs from 0 to 1,
    agrees bit for bit at every vertex its edges share, and each edge's s-increment
    is positive; a macro-edge is unparameterised exactly when it is not one open path
    (checked by scipy connected components and vertex degrees)."""
    mesh = holed_quad_mesh(48, holes=6, sx=3, sy=2, seed=21)
    labels, _ = A.agglomerate_levels(mesh.ne, mesh.edge_elem, mesh.cx, mesh.cy, mesh.seeds, 5)
    for k in range(4):
        me, nme, P = _params(mesh, labels, k)
        assert (P[me < 0] == -1).all()
        for q in range(nme):
            es = np.flatnonzero(me == q)
            ev = mesh.edge_vert[es]
            verts, inv = np.unique(ev, return_inverse=True)
            inv = inv.reshape(-1, 2)
            deg = np.bincount(inv.ravel(), minlength=len(verts))
            g = coo_matrix((np.ones(len(es)), (inv[:, 0], inv[:, 1])), shape=(len(verts),) * 2)
            ncomp, _ = connected_components(g, directed=False)
            is_path = ncomp == 1 and deg.max() <= 2 and (deg == 1).sum() == 2
            if not is_path:
                assert (P[es] == -1).all()
                continue
            assert (P[es] >= 0).all() and (P[es] <= 1).all()
            sv = {}
            for e in es:
                for c in range(2):
                    v = mesh.edge_vert[e, c]
                    assert sv.setdefault(v, P[e, c]) == P[e, c]
                assert P[e, 0] != P[e, 1]
            s_end = sorted(sv[v] for v, d in zip(verts, deg) if d == 1)
            assert s_end == [0.0, 1.0]


def test_macro_edge_around_a_hole_is_not_a_path():
    """One agglomerate holding a hole: its dOmega share is the outer loop plus the
    hole's loop -- not one open path, so it has no parameterisation (-1)."""
    mesh = holed_quad_mesh(16, holes=1, sx=1, sy=1, seed=5)
    labels, _ = A.agglomerate_levels(mesh.ne, mesh.edge_elem, mesh.cx, mesh.cy, mesh.seeds, 2)
    me, nme, P = _params(mesh, labels, 0)
    assert nme == 1 and (P == -1).all()


def test_macro_edge_parameter_is_arc_length_on_a_graded_line():
    """A5 with non-uniform fine edges: x graded as x^2 (no jitter); the horizontal level-2
    macro-edges on y = 1/2 are straight, so s = (x - x_start) / (x_stop - x_start)
    (to rounding).  A wrong length formula (e.g. a dropped sqrt) fails it."""
    mesh = structured_quad_mesh(8)
    mesh.vx = mesh.vx ** 2
    labels, _ = A.agglomerate_levels(mesh.ne, mesh.edge_elem, mesh.cx, mesh.cy, mesh.seeds, 3)
    me, nme, P = _params(mesh, labels, 1)
    X, Y = mesh.vx, mesh.vy
    checked = 0
    for q in range(nme):
        es = np.flatnonzero(me == q)
        verts = np.unique(mesh.edge_vert[es])
        if not (Y[verts] == 0.5).all():
            continue
        x0, x1 = X[verts].min(), X[verts].max()
        for e in es:
            for c in range(2):
                v = mesh.edge_vert[e, c]
                assert abs(P[e, c] - (X[v] - x0) / (x1 - x0)) <= 4e-16
                checked += 1
    assert checked == 2 * 8


@pytest.mark.parametrize("p", [1, 2, 4])
def test_macro_edge_transfer_reproduces_polynomials_in_arc_length(p):
    """A6: J is the P^p interpolation in s -- rows sum to 1, and the macro-edge
    coefficients q(t_j) of a degree-p polynomial q give q(s) at every fine node,
    s = s0 + (s1 - s0) xi_a (p = 1: the closed form [[1 - s0, s0], [1 - s1, s1]]);
    unparameterised edges get zero blocks."""
    from oracle.basis import gll_nodes
    mesh = holed_quad_mesh(32, holes=4, sx=2, sy=2, seed=13)
    labels, _ = A.agglomerate_levels(mesh.ne, mesh.edge_elem, mesh.cx, mesh.cy, mesh.seeds, 4)
    me, nme, P = _params(mesh, labels, 2)
    J = A.macro_edge_transfer(P, p)
    t = gll_nodes(p)
    rng = np.random.default_rng(p)
    coef = rng.standard_normal(p + 1)
    q = lambda x: np.polyval(coef, x)
    on = P[:, 0] >= 0
    assert on.sum() > 100 and (J[~on] == 0).all()
    np.testing.assert_allclose(J[on].sum(axis=2), 1.0, atol=1e-13)
    for e in np.flatnonzero(on):
        sa = P[e, 0] + (P[e, 1] - P[e, 0]) * t
        np.testing.assert_allclose(J[e] @ q(t), q(sa), atol=1e-12)
    # p = 1 closed form: J_e = [[1 - s0, s0], [1 - s1, s1]]
    if p == 1:
        e = np.flatnonzero(on)[0]
        np.testing.assert_allclose(J[e], [[1 - P[e, 0], P[e, 0]], [1 - P[e, 1], P[e, 1]]],
                                   atol=1e-15)
