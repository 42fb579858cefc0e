"""The oracle's element maps under the GPU's storage readings (test infrastructure,
numpy only; no CUDA code): R5, the constant-mode projection P S P with
P = I - 11^T/m (the exact DtN map annihilates constants, pin P2),
and R9, the average over the 8 symmetries of the square (the exact map of a uniform
square with scalar K commutes with them).  Both are orthogonal projections onto
subspaces that contain the exact map, so the projected map is never farther from
it (Frobenius norm) than the computed one: ||P(S - S*)P|| <= ||S - S*||.

At n >= 128 the per-V-cycle parity gate compares against the oracle run on these
projected maps: the oracle's own constant-mode rounding (|S 1| ~ 3e-15 |S|) is
amplified by the Galerkin coarse levels to ~2e-11 per V-cycle at n = 128
(tools/vcycle_floor.py, profiles/r02_vcycle_floor.jsonl), above the 1e-12 gate."""
import numpy as np


def d4_perms(p):
    """The 8 permutations of the local trace dofs (f, a) -> f*(p+1)+a induced by the
    symmetries of the unit square (edges bottom, right, top, left; global orientation)."""
    k = p + 1
    ends = {0: ((0, 0), (1, 0)), 1: ((1, 0), (1, 1)), 2: ((0, 1), (1, 1)), 3: ((0, 0), (0, 1))}
    out = []
    for g in range(8):
        def mp(x, y):
            X, Y = (y, x) if g & 4 else (x, y)
            return (1 - X if g & 1 else X, 1 - Y if g & 2 else Y)
        P = np.zeros(4 * k, int)
        for f in range(4):
            q0, q1 = mp(*ends[f][0]), mp(*ends[f][1])
            if q0[1] == q1[1]:
                fe, rev = (0 if q0[1] == 0 else 2), q0[0] > q1[0]
            else:
                fe, rev = (3 if q0[0] == 0 else 1), q0[1] > q1[1]
            for a in range(k):
                P[f * k + a] = fe * k + (p - a if rev else a)
        out.append(P)
    return out


def project_maps(S, p):
    m = S.shape[1]
    Pc = np.eye(m) - np.ones((m, m)) / m
    S = np.einsum("ab,ebc,cd->ead", Pc, S, Pc)
    return sum(S[:, P][:, :, P] for P in d4_perms(p)) / 8.0
