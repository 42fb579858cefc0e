"""Seeded synthetic unstructured quadrilateral meshes for the seed-point
agglomeration.

The paper's Example II mesh (an 8-hole box of 6699 simplices)
is not in the container; this module stands in for it with a quad mesh of the
same character: a box with rectangular holes, an irregular element adjacency
near the holes and jittered vertices, so element centroids are not on a
lattice.  It holds NO arithmetic of the method: it only produces the mesh a
user hands to the agglomeration (element adjacency through shared edges,
element centroids) and the seed elements ("chosen based on the geometry of the
domain and the original fine mesh": the element nearest to
each point of a regular sx x sy lattice over the box).

Mesh description (shared with include/mgdtn.h, `mg_agglomerate_seeds`):
  ne elements, centroids cx[ne], cy[ne] (float64);
  nedge edges, edge_elem[nedge][2] (int32): the two elements sharing the edge,
  edge_elem[e][1] = -1 on the domain boundary (holes included); for the
  macro-edge parameterisation (`mg_macro_edge_params`) also edge_vert[nedge][2]
  (int32) the edge's end vertices and vx, vy[nvert] (float64) the vertex
  coordinates (grid vertex (a, b) has id b*(n+1)+a; unused ones included).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class QuadMesh:
    ne: int
    cx: np.ndarray          # [ne] float64
    cy: np.ndarray          # [ne] float64
    edge_elem: np.ndarray   # [nedge, 2] int32, second -1 on the boundary
    seeds: np.ndarray       # [nseed] int32 element ids
    edge_vert: np.ndarray = None   # [nedge, 2] int32 vertex ids of the edge's endpoints
    vx: np.ndarray = None          # [nvert] float64 vertex coordinates
    vy: np.ndarray = None

    @property
    def nedge(self) -> int:
        return int(self.edge_elem.shape[0])


def holed_quad_mesh(n: int, holes: int = 8, jitter: float = 0.3, sx: int = 4, sy: int = 2,
                    seed: int = 3001, keep_all: bool = False) -> QuadMesh:
    """n x n grid of the unit box minus `holes` random rectangular holes (each
    2..n/6 cells a side, seeded), interior vertices moved by up to `jitter` of a
    cell (uniform, seeded; the quads stay convex for jitter < 0.5).  Elements
    are numbered row by row over the kept cells; edges in order of first
    appearance over the elements' local edges (bottom, right, top, left).
    sx*sy seeds: the element with the nearest centroid to each lattice point
    ((a+0.5)/sx, (b+0.5)/sy), duplicates dropped."""
    rng = np.random.default_rng(seed)
    keep = np.ones((n, n), dtype=bool)
    if not keep_all:
        for _ in range(holes):
            w = int(rng.integers(2, max(3, n // 6 + 1)))
            h = int(rng.integers(2, max(3, n // 6 + 1)))
            i0 = int(rng.integers(1, max(2, n - w - 1)))
            j0 = int(rng.integers(1, max(2, n - h - 1)))
            keep[j0:j0 + h, i0:i0 + w] = False
    # jittered vertices (boundary of the box kept straight)
    vx = np.tile(np.arange(n + 1, dtype=np.float64), (n + 1, 1))
    vy = vx.T.copy()
    dx = rng.uniform(-jitter, jitter, size=(n + 1, n + 1))
    dy = rng.uniform(-jitter, jitter, size=(n + 1, n + 1))
    dx[:, 0] = dx[:, -1] = 0.0
    dy[0, :] = dy[-1, :] = 0.0
    vx = (vx + dx) / n
    vy = (vy + dy) / n
    eid = -np.ones((n, n), dtype=np.int64)
    cells = [(i, j) for j in range(n) for i in range(n) if keep[j, i]]
    for k, (i, j) in enumerate(cells):
        eid[j, i] = k
    ne = len(cells)
    cx = np.empty(ne)
    cy = np.empty(ne)
    edges: dict = {}
    order = []
    for k, (i, j) in enumerate(cells):
        corners = [(i, j), (i + 1, j), (i + 1, j + 1), (i, j + 1)]
        cx[k] = sum(vx[b, a] for a, b in corners) / 4.0
        cy[k] = sum(vy[b, a] for a, b in corners) / 4.0
        for f in range(4):
            a, b = corners[f], corners[(f + 1) % 4]
            key = (min(a, b), max(a, b))
            if key not in edges:
                edges[key] = [k, -1]
                order.append(key)
            else:
                edges[key][1] = k
    edge_elem = np.array([edges[key] for key in order], dtype=np.int32).reshape(-1, 2)
    edge_vert = np.array([[a[1] * (n + 1) + a[0], b[1] * (n + 1) + b[0]] for a, b in order],
                         dtype=np.int32).reshape(-1, 2)
    seeds = []
    for b in range(sy):
        for a in range(sx):
            px, py = (a + 0.5) / sx, (b + 0.5) / sy
            s = int(np.argmin((cx - px) ** 2 + (cy - py) ** 2))
            if s not in seeds:
                seeds.append(s)
    return QuadMesh(ne, cx, cy, edge_elem, np.array(seeds, dtype=np.int32), edge_vert,
                    vx.reshape(-1).copy(), vy.reshape(-1).copy())


def structured_quad_mesh(n: int, seeds=(0,)) -> QuadMesh:
    """Plain n x n grid (no holes, no jitter): the closed-form pin case."""
    m = holed_quad_mesh(n, holes=0, jitter=0.0, keep_all=True, sx=1, sy=1)
    m.seeds = np.array(seeds, dtype=np.int32)
    return m
