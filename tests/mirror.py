"""Mirror x -> 1 - x of a structured-mesh problem (test / tool helper, no method arithmetic):
element (i, j) -> (n-1-i, j); a horizontal edge keeps its row and its dofs run the other
way along +x (GLL nodes are symmetric, so the reversal is exact); a vertical edge moves to
column n - i with its dofs in place.  A problem and its mirror image are the same discrete
problem up to this relabelling, so solving both measures how far a converged solution moves
with the evaluation order alone."""
import numpy as np


def mirror_elements(a, n):
    """Per-element array (element e = j*n + i) of the mirrored mesh."""
    return np.asarray(a).reshape(n, n)[:, ::-1].reshape(-1).copy()


def mirror_trace_perm(n, k1):
    """Index array P with lam_mirrored[P] = lam: trace dof of the original mesh -> its
    position in the mirrored mesh's canonical numbering ([edges][k1], horizontal edges
    j*n + i first, then vertical edges nh + j*(n+1) + i)."""
    nh = n * (n + 1)
    P = np.empty((nh + (n + 1) * n, k1), dtype=np.int64)
    j, i = np.divmod(np.arange(nh), n)
    eh = j * n + (n - 1 - i)
    P[:nh] = eh[:, None] * k1 + (k1 - 1 - np.arange(k1))[None, :]
    j, i = np.divmod(np.arange((n + 1) * n), n + 1)
    ev = nh + j * (n + 1) + (n - i)
    P[nh:] = ev[:, None] * k1 + np.arange(k1)[None, :]
    return P.reshape(-1)
