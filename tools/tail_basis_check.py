#!/usr/bin/env python3
"""B_tail from the multi-column basis kernel vs the single-column one (must be
identical: same bodies, same order per column): prints max |diff| of one V-cycle
on config-2 / config-4 / config-1 setups.  MGDTN_TAIL_BASIS_NC selects the kernel."""
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
for ci, n in ((2, 64), (4, 64), (1, 32)):
    c = W.scaled_config(ci, n) if W.CONFIGS[ci].n != n else W.CONFIGS[ci]
    pr = W.make_problem(c)
    s = MGSolver(c.n, p=c.p)
    s.setup(pr.K, pr.method, pr.tau, smoother_from_config(c))
    r = torch.from_numpy(W.random_trace_vector(s.ndof(), 3))
    out.append(s.vcycle(r).cpu().numpy())
np.save(sys.argv[1], np.concatenate(out))
'''
res = []
for nc in ("1", "4"):
    env = dict(os.environ, MGDTN_TAIL_BASIS_NC=nc)
    f = f"/tmp/tb_{nc}.npy"
    subprocess.run([sys.executable, "-c", code, f, ROOT], check=True, env=env)
    res.append(np.load(f))
print("max |z_nc4 - z_nc1| =", float(abs(res[1] - res[0]).max()), "equal:", bool((res[0] == res[1]).all()))
