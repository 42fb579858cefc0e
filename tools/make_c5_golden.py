#!/usr/bin/env python3
"""Write tests/golden/c5_recipe_n<n>.json + .npy: the ORACLE's MG-PCG solve of the
config-5 recipe (HDG p=4, tau=1, K = 10^g with g a seeded Gaussian field of std 1.0 and
correlation length 32 ELEMENTS -- the full-size length, not scaled down --, f = 1,
u = 0 on dOmega, V(2,2) Chebyshev, rtol 1e-10) on an n x n mesh, the whole trace
solution stored.  Config 5 itself (4096^2, 168M trace dofs) is beyond the oracle's
memory; this is the largest size of its recipe the container solves.

The oracle runs under the GPU's readings: fine maps projected by R5 / R9
(tests/oracle_proj.py; both projections are onto subspaces holding the exact maps,
so they are no farther from them) and every coarse level built macro by macro and
projected onto S.1 = 0 (R10, oracle/multigrid.py galerkin="macro", project_levels=True).  Calls only
oracle/, workloads/ and that numpy projection -- no value comes from the CUDA path.

    python tools/make_c5_golden.py 512
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402

import workloads as W  # noqa: E402
from oracle import assembly, krylov, multigrid  # noqa: E402
from oracle_proj import project_maps  # noqa: E402


def main(n):
    c = W.config5_recipe(n)
    pr = W.make_problem(c)
    t0 = time.perf_counter()
    ts = assembly.TraceSystem(n, c.p, pr.K, pr.method, pr.tau, pr.f_qp, pr.f_const, pr.gD_qp)
    ts.S = project_maps(ts.S, c.p)
    ts.A_full = assembly.assemble_full(n, c.p, ts.S)
    ts.A = ts.A_full[ts.free][:, ts.free].tocsr()
    g_full = assembly.assemble_vector(n, c.p, ts.b)
    ts.g = g_full[ts.free] - ts.A_full[ts.free][:, ts.dir] @ ts.lam_D[ts.dir]
    H = multigrid.Hierarchy(ts.A, n, c.p, smoother=c.smoother, nu_pre=c.nu, nu_post=c.nu,
                            element_maps=ts.S, galerkin="macro", project_levels=True)
    res = krylov.pcg(ts.A, H.vcycle, ts.g, rtol=c.rtol, maxit=4000)
    t1 = time.perf_counter()
    lam = ts.to_full(res["x"])
    base = os.path.join(ROOT, "tests", "golden", f"c5_recipe_n{n}")
    np.save(base + ".npy", lam)
    lg = np.log10(pr.K)
    out = {
        "source": "tools/make_c5_golden.py (oracle/ under readings R5/R9/R10); config-5 recipe at n=%d, "
                  "ell = 32 elements" % n,
        "config": 5, "n": n, "p": c.p, "ell": c.extras["ell"], "iters": int(res["iters"]),
        "relres": float(res["relres"]), "true_relres": float(res["true_relres"]),
        "status": int(res["status"]), "log10K_min": float(lg.min()), "log10K_max": float(lg.max()),
        "lam_norm": float(np.linalg.norm(lam)), "ndof": int(len(lam)), "oracle_seconds": t1 - t0,
    }
    with open(base + ".json", "w") as f:
        json.dump(out, f)
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    for a in sys.argv[1:]:
        main(int(a))
