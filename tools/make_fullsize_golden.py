#!/usr/bin/env python3
"""Write tests/golden/fullsize_oracle_c<k>.json: the ORACLE's MG-PCG solve of a
BASELINE.json config at its full size (iteration count, residual history,
||lambda||_2 and lambda at seeded sample dofs).  Calls only oracle/ and the
seeded input generators in workloads/ -- no value comes from the CUDA path.

    python tools/make_fullsize_golden.py 2 4 3
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import workloads as W  # noqa: E402
from oracle import driver  # noqa: E402

NSAMPLE = 4096


def main(idx):
    cfg = W.CONFIGS[idx]
    pr = W.make_problem(cfg)
    t0 = time.perf_counter()
    res = driver.solve_problem(pr, maxit=4000)
    t1 = time.perf_counter()
    lam = res["lam_full"]
    rng = np.random.default_rng(3000 + idx)
    samp = np.sort(rng.choice(len(lam), size=min(NSAMPLE, len(lam)), replace=False))
    out = {
        "source": "tools/make_fullsize_golden.py (oracle/ only); config %d %s" % (idx, cfg.name),
        "config": idx, "n": cfg.n, "p": cfg.p, "iters": int(res["iters"]),
        "relres": float(res["relres"]) if "relres" in res else None,
        "true_relres": float(res["true_relres"]),
        "status": int(res["status"]),
        "hist": [float(v) for v in res.get("hist", [])],
        "lam_norm": float(np.linalg.norm(lam)), "ndof": int(len(lam)),
        "sample_idx": samp.tolist(), "sample_val": lam[samp].tolist(),
        "oracle_seconds": t1 - t0,
    }
    path = os.path.join(ROOT, "tests", "golden", f"fullsize_oracle_c{idx}.json")
    with open(path, "w") as f:
        json.dump(out, f)
    print(idx, cfg.name, "iters", out["iters"], "time %.1f s" % (t1 - t0), flush=True)


if __name__ == "__main__":
    for a in sys.argv[1:]:
        main(int(a))
