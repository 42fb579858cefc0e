"""Seed-point agglomeration of an unstructured quad mesh.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py): plain Python, one BFS per
seed, Python's sorted() per macro-element.  Shares nothing with the CUDA path.

PAPER.md:491-498 (section 3.1.2): "we first select a certain number of levels N
and seed points N_{T_1} ... Based on these selected seed points, we
agglomerate the elements in the finest mesh (k=N) to form N_{T_1}
macro-elements at level 1.  We then divide each macro-element in level 1 into
four approximately equal macro-elements to form level 2.  This process is
recursively repeated to create macro-elements in finer levels k=3,...,N-1."
PAPER.md:485-487: the level k-1 trace space lives on the boundary edges of the
level-k agglomerates ("first agglomerating the boundary edges of level k ...
then statically condensing out the interior edges").

The paper calls its procedure "ad hoc" and does not fix the rules; readings
(A1-A3):
  A1  level-1 agglomeration = graph Voronoi cells of the seeds on the element
      dual graph (elements adjacent through a shared edge): element t goes to
      the seed s minimising (hop distance d(t, s), s's index in the seed list).
  A2  "divide into four approximately equal": order the macro-element's
      elements by (cx, cy, element id); the first ceil(m/2) are the west half,
      the rest the east half; order each half by (cy, cx, element id); the
      first ceil(h/2) are its south quarter.  Child id = 4*parent + 2*east +
      north, so level k has N_{T_1} 4^{k-1} ids (some possibly empty).
  A3  an edge is on the level-k skeleton iff it lies on the domain boundary or
      its two elements have different level-k labels (k = 1..N-1); every edge
      is on the level-N (fine) skeleton.
  A4  PAPER.md:355-356: "each e in E_k is the intersection of two
      macro-elements in T_k": the level-k macro-edges are the non-empty sets
      {fine edges between agglomerates a < b} and {fine edges of agglomerate a
      on the domain boundary} (pair (-1, a)), numbered by the lexicographic
      order of their pairs; a fine edge off the level-k skeleton gets -1.
  A5  PAPER.md:360-372 (remark: macro-elements of no standard shape need "a
      parameterization of each macro-edge to define M_k"): a macro-edge whose
      fine edges form one simple open path is parameterised by arc length,
      s in [0, 1], from the end vertex that is least in (vx, vy, vertex id);
      s at a vertex = (sum of the lengths of the path's edges before it, added
      in path order) / (the path's total length, added in path order), edge
      length = sqrt(dx*dx + dy*dy).  A macro-edge that is not one open path
      (a closed loop, several pieces, a vertex shared by more than two of its
      edges) has no such parameterisation: its edges get s = -1.
"""
from __future__ import annotations

import math
from collections import deque

import numpy as np


def dual_adjacency(ne: int, edge_elem: np.ndarray):
    """Element neighbours through interior edges (PAPER.md:147-149 skeleton)."""
    adj = [[] for _ in range(ne)]
    for a, b in edge_elem.tolist():
        if b >= 0:
            adj[a].append(b)
            adj[b].append(a)
    return adj


def hop_distances(ne: int, adj, src: int) -> np.ndarray:
    """Breadth-first hop distance from element src (-1: unreachable)."""
    d = -np.ones(ne, dtype=np.int64)
    d[src] = 0
    q = deque([src])
    while q:
        t = q.popleft()
        for u in adj[t]:
            if d[u] < 0:
                d[u] = d[t] + 1
                q.append(u)
    return d


def seed_agglomerate(ne: int, edge_elem: np.ndarray, seeds) -> np.ndarray:
    """Level-1 labels (reading A1): argmin over seeds of (d(t, s), index)."""
    adj = dual_adjacency(ne, edge_elem)
    best = [None] * ne
    for k, s in enumerate(seeds):
        d = hop_distances(ne, adj, int(s))
        for t in range(ne):
            if d[t] >= 0 and (best[t] is None or (d[t], k) < best[t]):
                best[t] = (int(d[t]), k)
    if any(b is None for b in best):
        raise ValueError("element not reachable from any seed")
    return np.array([b[1] for b in best], dtype=np.int32)


def quadrisect(labels: np.ndarray, cx: np.ndarray, cy: np.ndarray) -> np.ndarray:
    """Next level's labels (reading A2)."""
    out = np.empty_like(labels)
    groups = {}
    for t, g in enumerate(labels.tolist()):
        groups.setdefault(g, []).append(t)
    for g, mem in groups.items():
        byx = sorted(mem, key=lambda t: (cx[t], cy[t], t))
        hx = (len(byx) + 1) // 2
        for east, half in ((0, byx[:hx]), (1, byx[hx:])):
            byy = sorted(half, key=lambda t: (cy[t], cx[t], t))
            hy = (len(byy) + 1) // 2
            for north, quarter in ((0, byy[:hy]), (1, byy[hy:])):
                for t in quarter:
                    out[t] = 4 * g + 2 * east + north
    return out


def skeleton(labels: np.ndarray, edge_elem: np.ndarray) -> np.ndarray:
    """1 where the edge is on the skeleton of the agglomerated level (A3)."""
    a = edge_elem[:, 0]
    b = edge_elem[:, 1]
    out = np.ones(len(a), dtype=np.uint8)
    inner = b >= 0
    out[inner] = (labels[a[inner]] != labels[b[inner]]).astype(np.uint8)
    return out


def macro_edges(labels: np.ndarray, edge_elem: np.ndarray):
    """Level macro-edge id of every fine edge (-1 off the skeleton) and the
    number of macro-edges (reading A4)."""
    pairs = []
    for a, b in edge_elem.tolist():
        if b < 0:
            pairs.append((-1, int(labels[a])))
        elif labels[a] != labels[b]:
            la, lb = int(labels[a]), int(labels[b])
            pairs.append((min(la, lb), max(la, lb)))
        else:
            pairs.append(None)
    ids = {q: k for k, q in enumerate(sorted({q for q in pairs if q is not None}))}
    return np.array([-1 if q is None else ids[q] for q in pairs], dtype=np.int32), len(ids)


def macro_edge_params(medge: np.ndarray, nmedge: int, edge_vert: np.ndarray, vx, vy):
    """s at each end vertex of every fine edge, [nedge, 2] (reading A5; -1 where the
    edge is off the skeleton or its macro-edge is not one open path)."""
    out = -np.ones((len(medge), 2))
    members = [[] for _ in range(nmedge)]
    for e, q in enumerate(medge.tolist()):
        if q >= 0:
            members[q].append(e)
    for q, es in enumerate(members):
        inc = {}                                  # vertex -> incident edges of q
        for e in es:
            for v in edge_vert[e].tolist():
                inc.setdefault(v, []).append(e)
        ends = [v for v, l in inc.items() if len(l) == 1]
        if any(len(l) > 2 for l in inc.values()) or len(ends) != 2:
            continue
        v = min(ends, key=lambda w: (vx[w], vy[w], w))
        path = []                                 # (edge, entry vertex, exit vertex)
        e = inc[v][0]
        while True:
            a, b = edge_vert[e].tolist()
            w = b if a == v else a
            path.append((e, v, w))
            nxt = [f for f in inc[w] if f != e]
            if not nxt:
                break
            v, e = w, nxt[0]
        if len(path) != len(es):                  # several pieces
            continue
        lengths = []
        for e, a, b in path:
            dx, dy = vx[b] - vx[a], vy[b] - vy[a]
            lengths.append(math.sqrt(dx * dx + dy * dy))
        total = 0.0
        for ln in lengths:
            total += ln
        cum = 0.0
        for (e, a, b), ln in zip(path, lengths):
            s0, cum = cum / total, cum + ln
            s1 = cum / total
            out[e, 0 if edge_vert[e][0] == a else 1] = s0
            out[e, 0 if edge_vert[e][0] == b else 1] = s1
    return out


def macro_edge_transfer(s: np.ndarray, p: int) -> np.ndarray:
    """J_e [nedge, p+1, p+1] (reading A6): row a = fine node, column j = macro-edge basis."""
    from oracle.basis import gll_nodes, lagrange
    t = gll_nodes(p)
    J = np.zeros((len(s), p + 1, p + 1))
    for e in range(len(s)):
        s0, s1 = s[e]
        if s0 < 0:
            continue
        J[e] = lagrange(t, s0 + (s1 - s0) * t)
    return J


def agglomerate_levels(ne, edge_elem, cx, cy, seeds, nlev: int):
    """Labels and skeleton flags of levels k = 1 .. nlev-1 (row k-1 each)."""
    if nlev < 2:
        raise ValueError("need at least two levels")
    lab = [seed_agglomerate(ne, edge_elem, seeds)]
    for _ in range(nlev - 2):
        lab.append(quadrisect(lab[-1], cx, cy))
    labels = np.stack(lab)
    skel = np.stack([skeleton(l, edge_elem) for l in lab])
    return labels, skel
