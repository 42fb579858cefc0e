"""SURVEY.md 8(f) f4 on the GPU: seed-point agglomeration of an unstructured
quad mesh (mg_agglomerate_seeds; readings A1-A3) against
oracle/agglomerate.py, bit for bit (integer output): level labels and level
skeletons on holed, jittered meshes (the Example II stand-in, DESIGN.md
section 4), a 2^m grid, a strip, and the edge cases (one seed, every element a
seed, duplicate seeds, macro-edges (A4) their arc-length parameters (A5) and P^p transfer blocks (A6), levels past one element per agglomerate, a disconnected
mesh, bad ids)."""
import numpy as np
import pytest
import torch

from oracle import agglomerate as A
from workloads.unstructured import QuadMesh, holed_quad_mesh, structured_quad_mesh

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _built():
    from paper_1811_09909_b200 import build
    build.build()
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _gpu(m: QuadMesh, nlev: int):
    from paper_1811_09909_b200 import agglomerate_seeds
    d = torch.device("cuda:0")
    lab, sk, me, nme = agglomerate_seeds(torch.from_numpy(m.edge_elem).to(d).contiguous(),
                                torch.from_numpy(m.cx).to(d), torch.from_numpy(m.cy).to(d),
                                torch.from_numpy(m.seeds).to(d), nlev)
    return lab.cpu().numpy(), sk.cpu().numpy(), me.cpu().numpy(), nme


def _check(m: QuadMesh, nlev: int, params: bool = True):
    want_l, want_s = A.agglomerate_levels(m.ne, m.edge_elem, m.cx, m.cy, m.seeds, nlev)
    got_l, got_s, got_me, got_n = _gpu(m, nlev)
    np.testing.assert_array_equal(got_l, want_l)
    np.testing.assert_array_equal(got_s, want_s)
    for k in range(nlev - 1):
        want_me, want_n = A.macro_edges(want_l[k], m.edge_elem)
        np.testing.assert_array_equal(got_me[k], want_me)
        assert got_n[k] == want_n
        if params and m.edge_vert is not None:
            # A5: the same additions in the same order on both sides -> bit for bit
            want_p = A.macro_edge_params(want_me, want_n, m.edge_vert, m.vx, m.vy)
            got_p = _gpu_params(m, got_me[k], got_n[k])
            np.testing.assert_array_equal(got_p, want_p)
            if k == nlev - 2:   # A6 transfer blocks on the finest agglomerated level
                from paper_1811_09909_b200 import macro_edge_transfer
                for p in (1, 4):
                    J = macro_edge_transfer(torch.from_numpy(got_p).cuda().contiguous(), p)
                    # the two sides' GLL nodes come from different root finders (ulps)
                    np.testing.assert_allclose(J.cpu().numpy(), A.macro_edge_transfer(want_p, p),
                                               rtol=0, atol=1e-13)


def _gpu_params(m: QuadMesh, me: np.ndarray, nme: int):
    from paper_1811_09909_b200 import macro_edge_params
    d = torch.device("cuda:0")
    s = macro_edge_params(torch.from_numpy(me).to(d).contiguous(), nme,
                          torch.from_numpy(m.edge_vert).to(d).contiguous(),
                          torch.from_numpy(m.vx).to(d), torch.from_numpy(m.vy).to(d))
    return s.cpu().numpy()


# (n, holes, sx, sy, seed, nlev): Example II's setting is N = 7 levels from 7 or 4 seeds
# on a ~6700-element holed box; n = 96 gives ~8000 quads
CASES = [(24, 3, 2, 2, 1, 4), (64, 8, 4, 2, 3001, 6), (96, 8, 7, 1, 3002, 7),
         (96, 8, 2, 2, 3002, 7), (128, 10, 3, 3, 5, 8)]


@pytest.mark.parametrize("n,holes,sx,sy,seed,nlev", CASES)
def test_agglomeration_parity(n, holes, sx, sy, seed, nlev):
    _check(holed_quad_mesh(n, holes=holes, sx=sx, sy=sy, seed=seed), nlev)


def test_agglomeration_parity_large():
    """~250k elements (many BFS layer batches, 31k-element agglomerates at level 1)."""
    _check(holed_quad_mesh(512, holes=12, sx=4, sy=2, seed=9), 7, params=False)
    m = holed_quad_mesh(256, holes=10, sx=4, sy=2, seed=9)
    _check(m, 6)


def test_macro_edge_params_graded_line_and_bad_ids():
    from paper_1811_09909_b200 import MGError
    m = structured_quad_mesh(16)
    m.vx = m.vx ** 2
    _check(m, 4)
    lab, _ = A.agglomerate_levels(m.ne, m.edge_elem, m.cx, m.cy, m.seeds, 3)
    me, nme = A.macro_edges(lab[1], m.edge_elem)
    with pytest.raises(MGError, match="MG_ERR_ARG"):
        _gpu_params(m, me, nme - 1)                     # an id >= nmedge
    ev = m.edge_vert.copy()
    ev[0, 0] = len(m.vx)
    with pytest.raises(MGError, match="MG_ERR_ARG"):
        _gpu_params(QuadMesh(m.ne, m.cx, m.cy, m.edge_elem, m.seeds, ev, m.vx, m.vy), me, nme)


def test_quadtree_grid_and_levels_past_one_element():
    m = structured_quad_mesh(16, seeds=(37,))
    _check(m, 8)          # levels 6, 7: one element per agglomerate, empty siblings


def test_one_element_per_seed_and_duplicate_seeds():
    m = structured_quad_mesh(8)
    m.seeds = np.arange(m.ne, dtype=np.int32)[::-1].copy()
    _check(m, 3)
    m = holed_quad_mesh(32, holes=4, sx=2, sy=2, seed=4)
    m.seeds = np.array([m.seeds[0], m.seeds[1], m.seeds[0], m.seeds[2]], dtype=np.int32)
    _check(m, 4)


def test_strip_mesh():
    L = 301
    ee = np.array([[t, t + 1] for t in range(L - 1)] + [[t, -1] for t in range(L)], dtype=np.int32)
    m = QuadMesh(L, np.arange(L, dtype=np.float64), np.zeros(L), ee,
                 np.array([250, 3, 100, 101], dtype=np.int32))
    _check(m, 5)


def test_disconnected_mesh_and_bad_ids_fail_loudly():
    from paper_1811_09909_b200 import MGError
    m = holed_quad_mesh(16, holes=0, sx=1, sy=1, keep_all=True)
    ee = m.edge_elem.copy()
    # cut element 0 off: its interior edges become boundary edges of its neighbours
    cut = (ee[:, 0] == 0) & (ee[:, 1] >= 0)
    ee[cut, 0], ee[cut, 1] = ee[cut, 1], -1
    m2 = QuadMesh(m.ne, m.cx, m.cy, ee, np.array([m.ne - 1], dtype=np.int32))
    with pytest.raises(ValueError):
        A.seed_agglomerate(m2.ne, m2.edge_elem, m2.seeds)
    with pytest.raises(MGError, match="MG_ERR_SHAPE.*element 0"):
        _gpu(m2, 3)
    m3 = QuadMesh(m.ne, m.cx, m.cy, m.edge_elem, np.array([m.ne], dtype=np.int32))
    with pytest.raises(MGError, match="MG_ERR_ARG"):
        _gpu(m3, 3)
    ee4 = m.edge_elem.copy()
    ee4[3, 1] = m.ne
    with pytest.raises(MGError, match="MG_ERR_ARG"):
        _gpu(QuadMesh(m.ne, m.cx, m.cy, ee4, m.seeds), 3)
