#!/usr/bin/env python3
"""Write tests/golden/c<k>_recipe_n<n>[_plain].json + .npy: the ORACLE's MG-PCG solve of
a heterogeneous config's recipe on an n x n mesh with the FULL-SIZE correlation length,
the whole trace solution stored:
  config 5 (W.config5_recipe): HDG p=4, tau=1, K = 10^g, g a seeded Gaussian field of std
    1.0 and correlation length 32 elements, f = 1, u = 0 on dOmega, V(2,2) Chebyshev.
    Config 5 itself (4096^2, 168M trace dofs) is beyond the oracle's memory.
  config 3 (W.config3_recipe): HDG p=2, tau=1, std 1.5, length 16 elements, clipped to a
    contrast of 1e6, V(3,3) block-Jacobi.  Config 3's own full-size oracle solve takes ~4 h.

The oracle runs under the GPU's readings: fine maps projected by R5 / R9
(tests/oracle_proj.py; both projections are onto subspaces holding the exact maps,
so they are no farther from them) and every coarse level built macro by macro and
projected onto S.1 = 0 (R10, oracle/multigrid.py galerkin="macro", project_levels=True).  Calls only
oracle/, workloads/ and that numpy projection -- no value comes from the CUDA path.

    python tools/make_recipe_golden.py 5 512
    python tools/make_recipe_golden.py 3 256 [--plain]

--plain: the oracle as it stands (no projections) -- with the readings' run at the same n
this measures how far the readings move the converged solution.
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


def main(idx, n, plain=False):
    c = W.config5_recipe(n) if idx == 5 else W.config3_recipe(n)
    pr = W.make_problem(c)
    t0 = time.perf_counter()
    ts = assembly.TraceSystem(n, c.p, pr.K, pr.method, pr.tau, pr.f_qp, pr.f_const, pr.gD_qp)
    if plain:
        H = multigrid.Hierarchy(ts.A, n, c.p, smoother=c.smoother, nu_pre=c.nu, nu_post=c.nu)
    else:
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
    base = os.path.join(ROOT, "tests", "golden", f"c{idx}_recipe_n{n}" + ("_plain" if plain else ""))
    np.save(base + ".npy", lam)
    lg = np.log10(pr.K)
    out = {
        "source": "tools/make_recipe_golden.py (oracle/%s); config-%d recipe at n=%d, ell = %g elements"
                  % ("" if plain else " under readings R5/R9/R10", idx, n, c.extras["ell"]),
        "config": idx, "n": n, "p": c.p, "ell": c.extras["ell"], "iters": int(res["iters"]),
        "relres": float(res["relres"]), "true_relres": float(res["true_relres"]),
        "status": int(res["status"]), "log10K_min": float(lg.min()), "log10K_max": float(lg.max()),
        "lam_norm": float(np.linalg.norm(lam)), "ndof": int(len(lam)), "oracle_seconds": t1 - t0,
    }
    with open(base + ".json", "w") as f:
        json.dump(out, f)
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    main(int(args[0]), int(args[1]), plain="--plain" in sys.argv)
