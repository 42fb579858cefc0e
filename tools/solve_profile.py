#!/usr/bin/env python3
"""One setup + rhs + PCG solve of a config inside NVTX ranges, for per-kernel
device times under ncu with warm caches:

  ncu --nvtx --nvtx-include "mg/" --cache-control none --clock-control none \
      --metrics gpu__time_duration.sum --csv --log-file out.csv \
      python tools/solve_profile.py --config 2

Prints the CUDA-event time of each phase when run without ncu."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_1811_09909_b200 import MGSolver, smoother_from_config  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--eager", action="store_true", help="no CUDA graphs (per-kernel profiling)")
    ap.add_argument("--maxit", type=int, default=4000, help="PCG iteration cap (short per-iteration profiles)")
    ap.add_argument("--warm", type=int, default=2)
    ap.add_argument("--opt", action="append", default=[], help="KEY=VALUE for mg_set_option (repeatable)")
    ap.add_argument("--sweep", type=int, default=0, help="mg_set_option MG_OPT_SWEEP (-1 off, 0 auto, 1 force)")
    a = ap.parse_args()
    cfg = W.CONFIGS[a.config]
    pr = W.make_problem(cfg)
    dev = torch.device("cuda", 0)
    st = torch.cuda.Stream(dev)
    K = torch.from_numpy(pr.K).to(dev)
    meth = torch.from_numpy(pr.method).to(dev)
    tau = torch.from_numpy(pr.tau).to(dev)
    fq = None if pr.f_qp is None else torch.from_numpy(pr.f_qp).to(dev)
    gD = None if pr.gD_qp is None else torch.from_numpy(pr.gD_qp).to(dev)
    sm = smoother_from_config(cfg)
    with torch.cuda.stream(st):
        s = MGSolver(cfg.n, p=cfg.p, device=dev, stream=st)
        if a.eager:
            s.use_graphs(False)
        if a.sweep:
            s.set_option(s.OPT_SWEEP, a.sweep)
        for kv in a.opt:
            k, v = kv.split("=")
            s.set_option(int(k), int(v))
        for _ in range(a.warm):   # warm-up (graph capture, lazy attributes)
            s.setup(K, meth, tau, sm)
            g, _ = s.assemble_rhs(fq, pr.f_const, gD)
            s.pcg_solve(g, rtol=cfg.rtol, maxit=a.maxit)
        torch.cuda.synchronize()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        torch.cuda.nvtx.range_push("mg")
        ev[0].record(st)
        torch.cuda.nvtx.range_push("setup")
        s.setup(K, meth, tau, sm)
        torch.cuda.nvtx.range_pop()
        ev[1].record(st)
        torch.cuda.nvtx.range_push("rhs")
        g, _ = s.assemble_rhs(fq, pr.f_const, gD)
        torch.cuda.nvtx.range_pop()
        ev[2].record(st)
        torch.cuda.nvtx.range_push("solve")
        lam, info = s.pcg_solve(g, rtol=cfg.rtol, maxit=a.maxit)
        torch.cuda.nvtx.range_pop()
        ev[3].record(st)
        torch.cuda.nvtx.range_pop()
        torch.cuda.synchronize()
    print(json.dumps({"config": cfg.name, "setup_ms": ev[0].elapsed_time(ev[1]),
                      "rhs_ms": ev[1].elapsed_time(ev[2]), "solve_ms": ev[2].elapsed_time(ev[3]),
                      "iters": info["iters"], "launches": s.last_launch_count()}))


if __name__ == "__main__":
    main()
