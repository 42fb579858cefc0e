#!/usr/bin/env python3
"""Write tests/golden/fullsize_oracle_c<k>.json: the ORACLE's MG-PCG solve of a
BASELINE.json config at its full size (iteration count, residual history,
||lambda||_2 and lambda at seeded sample dofs).  Calls only oracle/ and the
seeded input generators in workloads/ -- no value comes from the CUDA path.

    python tools/make_fullsize_golden.py 2 4 3
    python tools/make_fullsize_golden.py --r10 3     # -> fullsize_oracle_c3_r10.json

--r10: the oracle under the GPU's storage readings -- fine maps projected by R5 / R9
(tests/oracle_proj.py), every coarse level built macro by macro and projected onto
S.1 = 0 (R10, oracle/multigrid.py) -- i.e. the more accurate reference (each projection is
onto a subspace holding the exact maps).
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import workloads as W  # noqa: E402
from oracle import assembly, driver, krylov, multigrid  # noqa: E402

sys.path.insert(0, os.path.join(ROOT, "tests"))

NSAMPLE = 4096


def solve_r10(cfg, pr):
    from oracle_proj import project_maps
    ts = assembly.TraceSystem(cfg.n, cfg.p, pr.K, pr.method, pr.tau, pr.f_qp, pr.f_const, pr.gD_qp)
    ts.S = project_maps(ts.S, cfg.p)
    ts.A_full = assembly.assemble_full(cfg.n, cfg.p, ts.S)
    ts.A = ts.A_full[ts.free][:, ts.free].tocsr()
    g_full = assembly.assemble_vector(cfg.n, cfg.p, ts.b)
    ts.g = g_full[ts.free] - ts.A_full[ts.free][:, ts.dir] @ ts.lam_D[ts.dir]
    H = multigrid.Hierarchy(ts.A, cfg.n, cfg.p, smoother=cfg.smoother, nu_pre=cfg.nu, nu_post=cfg.nu,
                            element_maps=ts.S, galerkin="macro", project_levels=True)
    res = krylov.pcg(ts.A, H.vcycle, ts.g, rtol=cfg.rtol, maxit=4000)
    res["lam_full"] = ts.to_full(res["x"])
    return res


def main(idx, r10=False):
    cfg = W.CONFIGS[idx]
    pr = W.make_problem(cfg)
    t0 = time.perf_counter()
    res = solve_r10(cfg, pr) if r10 else driver.solve_problem(pr, maxit=4000)
    t1 = time.perf_counter()
    lam = res["lam_full"]
    rng = np.random.default_rng(3000 + idx)
    samp = np.sort(rng.choice(len(lam), size=min(NSAMPLE, len(lam)), replace=False))
    out = {
        "source": "tools/make_fullsize_golden.py (oracle/ only%s); config %d %s" % (
            ", readings R5/R9/R10" if r10 else "", idx, cfg.name),
        "config": idx, "n": cfg.n, "p": cfg.p, "iters": int(res["iters"]),
        "relres": float(res["relres"]) if "relres" in res else None,
        "true_relres": float(res["true_relres"]),
        "status": int(res["status"]),
        "hist": [float(v) for v in res.get("hist", [])],
        "lam_norm": float(np.linalg.norm(lam)), "ndof": int(len(lam)),
        "sample_idx": samp.tolist(), "sample_val": lam[samp].tolist(),
        "oracle_seconds": t1 - t0,
    }
    path = os.path.join(ROOT, "tests", "golden", f"fullsize_oracle_c{idx}{'_r10' if r10 else ''}.json")
    with open(path, "w") as f:
        json.dump(out, f)
    print(idx, cfg.name, "iters", out["iters"], "time %.1f s" % (t1 - t0), flush=True)


if __name__ == "__main__":
    r10 = "--r10" in sys.argv
    for a in sys.argv[1:]:
        if a != "--r10":
            main(int(a), r10)
