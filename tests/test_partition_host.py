"""Host-side layout of the partitioned path (no GPU): the element blocks and
their local edge numbering (workloads.block_*) against the library's own plan
(include/mgdtn.h mg_partition_plan), and the invariants the halo protocol
relies on."""
import os

import numpy as np
import pytest

import workloads as W
from oracle import mesh

LIB = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                   "paper_1811_09909_b200", "libmgdtn.so")


@pytest.mark.parametrize("n,px,py", [(16, 2, 1), (16, 1, 2), (32, 2, 2), (32, 4, 2)])
def test_blocks_cover_the_mesh(n, px, py):
    """Every element belongs to exactly one block; every edge to one block, or to
    exactly two when it lies on a partition interface; the blocks' boundary edges
    that are not interfaces are exactly dOmega."""
    N = px * py
    cnt_e = np.zeros(n * n, int)
    cnt_edge = np.zeros(mesh.n_edges(n), int)
    for r in range(N):
        ox, oy, bx, by = W.block_of(n, px, py, r)
        jj, ii = np.divmod(np.arange(bx * by), bx)
        cnt_e[(oy + jj) * n + (ox + ii)] += 1
        cnt_edge[W.block_edge_ids(n, px, py, r)] += 1
    assert np.all(cnt_e == 1)
    assert np.all((cnt_edge >= 1) & (cnt_edge <= 2))
    shared = np.nonzero(cnt_edge == 2)[0]
    assert not np.any(mesh.boundary_edge_mask(n)[shared])
    # interface edges: (px-1) vertical lines of n edges + (py-1) horizontal lines of n edges
    assert len(shared) == (px - 1) * n + (py - 1) * n


def test_block_problem_slices_consistently():
    cfg = W.scaled_config(4, 32)
    pr = W.make_problem(cfg)
    px, py = 2, 2
    for r in range(4):
        bp = W.block_problem(pr, px, py, r)
        ox, oy, bx, by = W.block_of(cfg.n, px, py, r)
        for jl in (0, by - 1):
            for il in (0, bx - 1):
                g = (oy + jl) * cfg.n + (ox + il)
                l = jl * bx + il
                assert bp.K[l] == pr.K[g] and bp.tau[l] == pr.tau[g] and bp.method[l] == pr.method[g]
                assert np.array_equal(bp.f_qp[l], pr.f_qp[g])
        # g_D samples: a block side on dOmega carries the global samples, an interface zeros
        nq = pr.gD_qp.shape[1]
        assert bp.gD_qp.shape == (2 * bx + 2 * by, nq)
        bottom = bp.gD_qp[:bx]
        assert np.array_equal(bottom, pr.gD_qp[ox:ox + bx]) if oy == 0 else not bottom.any()


@pytest.mark.skipif(not os.path.exists(LIB), reason="libmgdtn.so not built")
@pytest.mark.parametrize("n,p,px,py,gne", [(32, 4, 2, 2, 16), (64, 2, 4, 2, 0), (16, 1, 2, 1, 4)])
def test_plan_matches_block_layout(n, p, px, py, gne):
    """The library's plan gives the same blocks as workloads.block_of on every
    partitioned level, replicates the levels from the gather level down, marks
    dOmega / interface sides consistently, and keeps local dims even where the
    next level is agglomerated locally."""
    from paper_1811_09909_b200 import Partition, partition_plan
    N = px * py
    for r in range(N):
        plan = partition_plan(n, n, p, Partition(r, N, px, py, gather_ne=gne))
        Lg = plan["gather_level"]
        assert Lg >= 1
        rx, ry = r % px, r // px
        dm = (int(ry == 0) << 0) | (int(rx == px - 1) << 1) | (int(ry == py - 1) << 2) | (int(rx == 0) << 3)
        for k, L in enumerate(plan["levels"], start=1):
            if k <= Lg:
                assert (L["nx"], L["ny"]) == (L["gnx"], L["gny"]) and L["imask"] == 0 and L["dmask"] == 15
            else:
                assert (L["ox"], L["oy"], L["nx"], L["ny"]) == W.block_of(L["gnx"], px, py, r)
                assert L["dmask"] == dm and L["imask"] == 15 & ~dm
                if k > Lg + 1:   # agglomerated locally into level k-1
                    assert L["nx"] % 2 == 0 and L["ny"] % 2 == 0
