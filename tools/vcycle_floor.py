#!/usr/bin/env python3
"""Per-apply / per-V-cycle noise floor of the 1e-12 parity gate.

Runs the ORACLE only.  For a config's recipe at sub-mesh n it forms one V-cycle
z = B_N r (and one fine apply y = A x) three ways from the same element DtN maps:
  base -- the oracle's maps as computed (oracle/element.py);
  ulp  -- every map perturbed entrywise by (1 + eps u), u ~ U[-1,1] symmetric per
          element: what another valid FP64 operation order in the element solves
          produces (1 ulp per entry);
  proj -- the maps projected exactly as the GPU stores them: P S P with
          P = I - 11^T/m (reading R5) and the D4-orbit average (reading R9), written
          here in numpy from the group action (no CUDA code).
and reports the relative L2 difference of each against base.  A GPU / oracle gap at
or below the 'ulp' floor is the oracle's own rounding, not a GPU error.

    python tools/vcycle_floor.py 2:64,2:128,2:256,5:64,5:128 > profiles/r02_vcycle_floor.jsonl

The last three columns compare evaluation orders of the hierarchy itself: global vs per-macro
Galerkin product (both FP64, same maps), per-macro without vs with reading R10, and R10 with
the Schur complement by solve vs explicit inverse -- the reproducibility of a V-cycle with
and without the per-level constant-mode projection.
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import workloads as W  # noqa: E402
from oracle import assembly, multigrid  # noqa: E402

sys.path.insert(0, os.path.join(ROOT, "tests"))
from oracle_proj import project_maps  # noqa: E402

EPS = np.finfo(np.float64).eps


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def main(spec):
    for item in spec.split(","):
        ci, n = map(int, item.split(":"))
        c = W.scaled_config(ci, n) if W.CONFIGS[ci].n != n else W.CONFIGS[ci]
        pr = W.make_problem(c, with_f=False)
        ts = assembly.TraceSystem(n, c.p, pr.K, pr.method, pr.tau, None, 1.0)
        rng = np.random.default_rng(7000 + ci)
        r = W.random_trace_vector(ts.ndof, 600)[ts.free]
        x = W.random_trace_vector(ts.ndof, c.seed_vec + 1)[ts.free]
        U = rng.uniform(-1, 1, ts.S.shape)
        U = 0.5 * (U + U.transpose(0, 2, 1))
        out = {"config": ci, "n": n, "p": c.p}
        res = {}
        for label, S in (("base", ts.S), ("ulp", ts.S * (1.0 + EPS * U)), ("proj", project_maps(ts.S, c.p))):
            A = assembly.assemble_full(n, c.p, S)[ts.free][:, ts.free].tocsr()
            H = multigrid.Hierarchy(A, n, c.p, smoother=c.smoother, nu_pre=c.nu, nu_post=c.nu)
            res[label] = (A @ x, H.vcycle(r))
        for label in ("ulp", "proj"):
            out[f"apply_{label}"] = rel(res[label][0], res["base"][0])
            out[f"vcycle_{label}"] = rel(res[label][1], res["base"][1])
        # two valid FP64 evaluation orders of the same hierarchy on the projected maps:
        # the global sparse Galerkin product vs macro by macro (Prop. DtN), each without and
        # with R10 (every coarse level projected onto S.1 = 0), and R10 with the Schur
        # complement through an explicit inverse instead of a solve
        Sp = project_maps(ts.S, c.p)
        A = assembly.assemble_full(n, c.p, Sp)[ts.free][:, ts.free].tocsr()
        kw = dict(smoother=c.smoother, nu_pre=c.nu, nu_post=c.nu)
        z = {
            "global": multigrid.Hierarchy(A, n, c.p, **kw).vcycle(r),
            "macro": multigrid.Hierarchy(A, n, c.p, **kw, element_maps=Sp, galerkin="macro").vcycle(r),
            "macro_r10": multigrid.Hierarchy(A, n, c.p, **kw, element_maps=Sp, galerkin="macro",
                                             project_levels=True).vcycle(r),
            "macro_r10_inv": multigrid.Hierarchy(A, n, c.p, **kw, element_maps=Sp, galerkin="macro",
                                                 project_levels=True, schur_inv=True).vcycle(r),
        }
        out["vcycle_global_vs_macro"] = rel(z["macro"], z["global"])
        out["vcycle_macro_vs_macro_r10"] = rel(z["macro_r10"], z["macro"])
        out["vcycle_r10_solve_vs_inv"] = rel(z["macro_r10_inv"], z["macro_r10"])
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "2:64,2:128,5:64")
