#!/usr/bin/env python3
"""One warm mg_setup_dtn of a config inside an NVTX range "setup" (for ncu launch
lists of the setup phase) and its CUDA-event time:
    python tools/setup_probe.py --config 2 [--reps 5]"""
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
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    cfg = W.CONFIGS[a.config]
    pr = W.make_problem(cfg, with_f=False)
    dev = torch.device("cuda", 0)
    st = torch.cuda.Stream(dev)
    K = torch.from_numpy(pr.K).to(dev)
    m = torch.from_numpy(pr.method).to(dev)
    tau = torch.from_numpy(pr.tau).to(dev)
    ts = []
    with torch.cuda.stream(st):
        s = MGSolver(cfg.n, p=cfg.p, device=dev, stream=st)
        sm = smoother_from_config(cfg)
        s.setup(K, m, tau, sm)
        for k in range(a.reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record(st)
            if k == a.reps - 1:
                torch.cuda.nvtx.range_push("setup")
            s.setup(K, m, tau, sm)
            if k == a.reps - 1:
                torch.cuda.nvtx.range_pop()
            e1.record(st)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
    print(json.dumps({"config": cfg.name, "setup_ms": ts}))


if __name__ == "__main__":
    main()
