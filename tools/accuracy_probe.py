#!/usr/bin/env python3
"""Accuracy of the GPU element DtN maps, the fine apply and one V-cycle against
the oracle on a config (sampled elements / full vectors where the oracle can),
to see how far inside the 1e-12 per-operator gate the GPU is.

    python tools/accuracy_probe.py --config 4 [--n 128]"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads as W  # noqa: E402
from oracle import assembly, multigrid  # noqa: E402
from oracle import element as el  # noqa: E402
from paper_1811_09909_b200 import MGSolver, smoother_from_config  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--n", type=int, default=128)
    a = ap.parse_args()
    cfg = W.scaled_config(a.config, a.n)
    pr = W.make_problem(cfg)
    s = MGSolver(cfg.n, p=cfg.p)
    s.setup(pr.K, pr.method, pr.tau, smoother_from_config(cfg))
    S = s.element_dtn(s.nlevels).cpu().numpy()
    So = el.element_dtn(cfg.p, pr.K, pr.method, pr.tau, 1.0 / cfg.n)
    per = np.abs(S - So).max(axis=(1, 2)) / np.abs(So).max(axis=(1, 2))
    ts = assembly.TraceSystem(cfg.n, cfg.p, pr.K, pr.method, pr.tau, pr.f_qp, pr.f_const, pr.gD_qp)
    H = multigrid.Hierarchy(ts.A, cfg.n, cfg.p, smoother=cfg.smoother, nu_pre=cfg.nu, nu_post=cfg.nu)
    x = W.random_trace_vector(s.ndof(), 11)
    y = s.apply(s.nlevels, torch.from_numpy(x)).cpu().numpy()[ts.free]
    yo = ts.A @ x[ts.free]
    z = s.vcycle(torch.from_numpy(x)).cpu().numpy()[ts.free]
    zo = H.vcycle(x[ts.free])
    out = {"config": cfg.name, "n": cfg.n,
           "elem_dtn_rel_max": float(per.max()), "elem_dtn_rel_median": float(np.median(per)),
           "apply_rel": float(np.linalg.norm(y - yo) / np.linalg.norm(yo)),
           "vcycle_rel": float(np.linalg.norm(z - zo) / np.linalg.norm(zo))}
    # every level: apply vs the oracle hierarchy's assembled Galerkin operator
    for k in range(s.nlevels - 1, 0, -1):
        Lo = H.levels[s.nlevels - k]
        xk = W.random_trace_vector(s.ndof(k), 20 + k)
        yk = s.apply(k, torch.from_numpy(xk)).cpu().numpy()[Lo.free]
        yok = Lo.A @ xk[Lo.free]
        out[f"lev{k}_apply_rel"] = float(np.linalg.norm(yk - yok) / np.linalg.norm(yok))
    print(json.dumps(out))


if __name__ == "__main__":
    main()
