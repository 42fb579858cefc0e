#!/usr/bin/env python3
"""Noise floor of the 1e-9 solution-parity gate.

Runs the ORACLE's MG-PCG solve of a config twice more with inputs perturbed
at rounding level -- (a) the right-hand side g scaled entrywise by
(1 + eps*u), u ~ U[-1,1]; (b) the element DtN maps scaled entrywise the same
way (symmetrically), i.e. what a different but valid FP64 operation order in
the setup produces -- and reports, against the committed golden
(tests/golden/fullsize_oracle_c<k>.json), the relative L2 change of lambda at
the golden's sample dofs and the iteration counts.  Calls only oracle/ and
workloads/.

    python tools/noise_floor.py 4  > profiles/r01_noise_floor_c4.json
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import workloads as W  # noqa: E402
from oracle import assembly, krylov, multigrid  # noqa: E402

EPS = np.finfo(np.float64).eps


def main(idx, which=("rhs", "operator")):
    cfg = W.CONFIGS[idx]
    pr = W.make_problem(cfg)
    gold = json.load(open(os.path.join(ROOT, "tests", "golden", f"fullsize_oracle_c{idx}.json")))
    samp = np.array(gold["sample_idx"])
    ref = np.array(gold["sample_val"])
    out = {"config": idx, "name": cfg.name, "golden_iters": gold["iters"], "runs": []}
    ts = assembly.TraceSystem(cfg.n, cfg.p, pr.K, pr.method, pr.tau, pr.f_qp, pr.f_const, pr.gD_qp)
    rng = np.random.default_rng(9000 + idx)

    def run(label, A, g):
        t0 = time.perf_counter()
        H = multigrid.Hierarchy(A, cfg.n, cfg.p, smoother=cfg.smoother, nu_pre=cfg.nu, nu_post=cfg.nu)
        res = krylov.pcg(A, H.vcycle, g, rtol=cfg.rtol, maxit=4000)
        lam = ts.to_full(res["x"])
        d = float(np.linalg.norm(lam[samp] - ref) / np.linalg.norm(ref))
        out["runs"].append({"perturbation": label, "iters": int(res["iters"]), "rel_diff_samples": d,
                            "seconds": time.perf_counter() - t0})
        print(label, res["iters"], d, flush=True, file=sys.stderr)

    # (a) rhs at rounding level
    g2 = ts.g * (1.0 + EPS * rng.uniform(-1, 1, ts.g.shape))
    if "rhs" in which:
        run("rhs (1 + eps u)", ts.A, g2)
    if "operator" not in which:
        print(json.dumps(out))
        return
    # (b) symmetric entrywise perturbation of the assembled operator at rounding level
    A = ts.A.tocoo()
    u = rng.uniform(-1, 1, A.nnz)
    key_lo = np.minimum(A.row, A.col).astype(np.int64) * A.shape[0] + np.maximum(A.row, A.col)
    _, inv = np.unique(key_lo, return_inverse=True)
    us = rng.uniform(-1, 1, inv.max() + 1)[inv]   # same factor for (i,j) and (j,i)
    del u
    import scipy.sparse as sp
    A2 = sp.csr_matrix((A.data * (1.0 + EPS * us), (A.row, A.col)), shape=A.shape)
    run("operator (1 + eps u), symmetric", A2, ts.g)
    print(json.dumps(out))


if __name__ == "__main__":
    main(int(sys.argv[1]), tuple(sys.argv[2].split(",")) if len(sys.argv) > 2 else ("rhs", "operator"))
