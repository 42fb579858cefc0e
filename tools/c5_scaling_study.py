#!/usr/bin/env python3
"""Oracle-only study of the config-5 recipe's PCG iteration count against the mesh
size (VERDICT r1 'what's weak' #4): is config 5's ~1220 iterations a property of
the method on this recipe (HDG tau = 1 at a ~1e9 K contrast) or of the build?
Runs oracle/ (never the CUDA path) on W.scaled_config(5, n) -- correlation length
scaled with n (the same field structure) -- and, with --unscaled, on the same
recipe with ell = 32 elements (the full-size correlation length in element units).

    python tools/c5_scaling_study.py 16 32 64 [--unscaled] > profiles/r02_c5_oracle_study.jsonl
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import workloads as W  # noqa: E402
from oracle import assembly, krylov, multigrid  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("ns", type=int, nargs="+")
    ap.add_argument("--unscaled", action="store_true")
    ap.add_argument("--maxit", type=int, default=4000)
    a = ap.parse_args()
    for n in a.ns:
        c = W.scaled_config(5, n)
        if a.unscaled:
            c.extras["ell"] = W.CONFIGS[5].extras["ell"]
        pr = W.make_problem(c)
        t0 = time.perf_counter()
        ts = assembly.TraceSystem(n, c.p, pr.K, pr.method, pr.tau, pr.f_qp, pr.f_const, pr.gD_qp)
        H = multigrid.Hierarchy(ts.A, n, c.p, smoother=c.smoother, nu_pre=c.nu, nu_post=c.nu)
        t1 = time.perf_counter()
        res = krylov.pcg(ts.A, H.vcycle, ts.g, rtol=c.rtol, maxit=a.maxit)
        t2 = time.perf_counter()
        lg = np.log10(pr.K)
        print(json.dumps({"n": n, "p": c.p, "ell": c.extras["ell"], "log10K_min": float(lg.min()),
                          "log10K_max": float(lg.max()), "iters": int(res["iters"]),
                          "status": int(res["status"]), "relres": float(res["relres"]),
                          "true_relres": float(res["true_relres"]), "setup_s": t1 - t0,
                          "solve_s": t2 - t1, "s_per_iter": (t2 - t1) / max(1, res["iters"]),
                          "trace_dofs": c.trace_dofs}), flush=True)


if __name__ == "__main__":
    main()
