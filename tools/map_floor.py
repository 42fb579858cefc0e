#!/usr/bin/env python3
"""Where the GPU / oracle gap of a converged config-3 solution comes from: solve the recipe
at size n on the GPU (a) with its own element maps and (b) with the ORACLE's element maps
(projected by readings R5 / R9, tests/oracle_proj.py) injected through
mg_debug_set_element_dtn + MG_OPT_KEEP_FINE_MAPS, so that the rest of the setup and the
whole solve run on the GPU from identical maps; compare both with the whole-vector oracle
golden under the readings (tests/golden/c3_recipe_n<n>.npy) and report the element maps'
own difference.  No value flows from the GPU into the oracle.

    python tools/map_floor.py --n 512
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads as W  # noqa: E402


def main(n, idx):
    from oracle import assembly
    from oracle_proj import project_maps
    from paper_1811_09909_b200 import MGSolver, smoother_from_config
    c = W.config3_recipe(n) if idx == 3 else W.config5_recipe(n)
    pr = W.make_problem(c)
    t0 = time.perf_counter()
    ts = assembly.TraceSystem(n, c.p, pr.K, pr.method, pr.tau, pr.f_qp, pr.f_const, pr.gD_qp)
    So = project_maps(ts.S, c.p)
    t1 = time.perf_counter()
    gold = np.load(os.path.join(ROOT, "tests", "golden", f"c{idx}_recipe_n{n}.npy"))
    out = {"config": idx, "n": n, "oracle_maps_s": t1 - t0}
    s = MGSolver(n, p=c.p)
    sm = smoother_from_config(c)
    s.setup(pr.K, pr.method, pr.tau, sm)
    N = s.nlevels
    Sg = s.element_dtn(N).cpu().numpy()
    d = np.abs(Sg - So).max(axis=(1, 2)) / np.abs(So).max(axis=(1, 2))
    lk = np.log10(pr.K)
    out["maps_rel_max"] = float(d.max())
    out["maps_rel_median"] = float(np.median(d))
    out["maps_rel_max_by_log10K"] = {f"{a:+.0f}..{a + 1:+.0f}": float(d[(lk >= a) & (lk < a + 1)].max())
                                     for a in range(-3, 3) if np.any((lk >= a) & (lk < a + 1))}
    g, lam_bc = s.assemble_rhs(pr.f_qp, pr.f_const, pr.gD_qp)
    lam, info = s.pcg_solve(g, rtol=c.rtol, maxit=4000)
    own = (lam + lam_bc).cpu().numpy()
    s.set_option(s.OPT_KEEP_FINE_MAPS, 1)
    s.set_element_dtn(N, torch.from_numpy(So))
    s.setup(pr.K, pr.method, pr.tau, sm)
    Si = s.element_dtn(N).cpu().numpy()
    out["injected_maps_rel_max"] = float((np.abs(Si - So).max(axis=(1, 2)) / np.abs(So).max(axis=(1, 2))).max())
    g2, lam_bc2 = s.assemble_rhs(pr.f_qp, pr.f_const, pr.gD_qp)
    lam2, info2 = s.pcg_solve(g2, rtol=c.rtol, maxit=4000)
    inj = (lam2 + lam_bc2).cpu().numpy()
    rel = lambda a, b: float(np.linalg.norm(a - b) / np.linalg.norm(b))
    out.update({"iters_own": info["iters"], "iters_injected": info2["iters"],
                "own_vs_oracle": rel(own, gold), "injected_vs_oracle": rel(inj, gold),
                "own_vs_injected": rel(own, inj)})
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=256)
    ap.add_argument("--config", type=int, default=3)
    a = ap.parse_args()
    main(a.n, a.config)
