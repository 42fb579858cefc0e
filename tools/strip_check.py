#!/usr/bin/env python3
"""The single-pass strip apply (MGDTN_STRIP=R) against the two-pass apply: mg_apply
on every level must be bit-identical (same contributions, colour-0-
first sums); prints the result for R = 2, 4, 8 on config-2 / config-4 recipes."""
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
code = r'''
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[2])
import workloads as W
from paper_1811_09909_b200 import MGSolver, smoother_from_config
out = []
for ci, n in ((2, 256), (4, 128), (1, 128)):
    c = W.scaled_config(ci, n) if W.CONFIGS[ci].n != n else W.CONFIGS[ci]
    pr = W.make_problem(c)
    s = MGSolver(c.n, p=c.p)
    s.setup(pr.K, pr.method, pr.tau, smoother_from_config(c))
    for level in range(s.nlevels, 0, -1):
        x = torch.from_numpy(W.random_trace_vector(s.ndof(level), 7 + level))
        out.append(s.apply(level, x).cpu().numpy())
np.save(sys.argv[1], np.concatenate(out))
'''
res = {}
for R in ("0", "2", "4", "8"):
    env = dict(os.environ, MGDTN_STRIP=R)
    f = f"/tmp/strip_{R}.npy"
    subprocess.run([sys.executable, "-c", code, f, ROOT], check=True, env=env)
    res[R] = np.load(f)
for R in ("2", "4", "8"):
    d = np.abs(res[R] - res["0"])
    print(f"R={R}: max |diff| {d.max():.3e}  identical {bool((d == 0).all())}")
