#!/usr/bin/env python3
"""Time mg_apply on one level of a config in isolation (CUDA events on the
library stream, L2 flushed before each rep), for A/B of apply kernels and for
ncu captures:  python tools/apply_probe.py --config 2 [--level N] [--reps 20]"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_1811_09909_b200 import MGSolver, smoother_from_config  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--n", type=int, default=0)
    ap.add_argument("--level", type=int, default=0, help="0 = finest")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--no-flush", action="store_true")
    ap.add_argument("--op", default="apply", choices=["apply", "smooth"],
                    help="smooth: one fine smoothing step through mg_smooth (apply + D^-1 epilogue, "
                         "plus mg_smooth's two masked input copies and one output copy)")
    ap.add_argument("--opt", action="append", default=[], help="KEY=VALUE for mg_set_option (repeatable)")
    ap.add_argument("--sweep", type=int, default=0, help="mg_set_option MG_OPT_SWEEP")
    ap.add_argument("--steps", type=int, default=1, help="smoothing steps per probe (--op smooth)")
    ap.add_argument("--scheme", default="config", choices=["config", "nipg", "iipg", "tiles"],
                    help="nonsymmetric context with IIPG-H / NIPG-H elements (full-storage apply)")
    a = ap.parse_args()
    cfg = W.CONFIGS[a.config] if not a.n else W.scaled_config(a.config, a.n)
    ns = a.scheme != "config"
    pr = W.nonsymmetric_problem(cfg, a.scheme) if ns else W.make_problem(cfg, with_f=False)
    dev = torch.device("cuda", 0)
    st = torch.cuda.Stream(dev)
    with torch.cuda.stream(st):
        s = MGSolver(cfg.n, p=cfg.p, device=dev, stream=st, nonsymmetric=ns)
        sm = smoother_from_config(cfg)
        if ns:
            sm.kind = 0
        s.setup(pr.K, pr.method, pr.tau, sm)
        if a.sweep:
            s.set_option(s.OPT_SWEEP, a.sweep)
        for kv in a.opt:
            k, v = kv.split("=")
            s.set_option(int(k), int(v))
        lev = a.level or s.nlevels
        nd = s.ndof(lev)
        x = torch.rand(nd, dtype=torch.float64, device=dev)
        y = torch.empty_like(x)
        flush = torch.empty(256 << 18, dtype=torch.float32, device=dev)
        ts = []
        for k in range(a.reps + 3):
            if not a.no_flush:
                flush.fill_(float(k))
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            torch.cuda.nvtx.range_push("probe")
            if a.op == "apply":
                s.apply(lev, x, y)
            else:
                s.smooth(lev, x, y, a.steps)
            torch.cuda.nvtx.range_pop()
            e1.record(st)
            torch.cuda.synchronize()
            if k >= 3:
                ts.append(e0.elapsed_time(e1) * 1e3)
    info = s.level_info(lev)
    ne = info["nx"] * info["ny"]
    m = 4 * (info["p"] + 1)
    alg = ne * 8 * (m * m if ns else m * (m + 1) // 2) + 16 * nd
    t = float(np.median(ts))
    print(json.dumps({"config": cfg.name, "level": lev, "p": info["p"], "ne": ne, "us_median": t,
                      "us_min": float(np.min(ts)), "alg_bytes": alg, "GBps": alg / t / 1e3,
                      "apply": os.environ.get("MGDTN_APPLY", "tma"), "op": a.op,
                      "scheme": a.scheme}))


if __name__ == "__main__":
    main()
