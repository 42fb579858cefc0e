#!/usr/bin/env python3
"""Benchmark: fine trace DoFs/s of the whole MG-PCG hot path (BASELINE.json
metric), one JSON line on rank 0.

A step = one pass of the whole hot path over one synthetic problem with its
inputs (K, method, tau, f samples) already resident in HBM: batched element
DtN setup + p/h hierarchy + smoother setup (mg_setup_dtn), right-hand side
(mg_assemble_rhs) and the MG-preconditioned CG solve to 1e-10 (mg_pcg_solve).
value = trace DoFs (all edges x (p+1), as BASELINE.json counts them) of all
ranks / max-over-ranks device time per step.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl reference]

--impl reference times the CPU oracle (oracle/, plain numpy/scipy FP64) on a
bounded sample of the same workload (the reference arm of this tier).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import workloads as W  # noqa: E402

L2_FLUSH_BYTES = 256 << 20


def _peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


def _dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


class ClockSampler:
    """SM clocks and throttle reasons sampled DURING the timed region (NVML,
    every 10 ms, in a background thread; falls back to nothing if NVML is
    unavailable)."""

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.rows = []
        self._stop = None
        self._th = None

    def start(self):
        import threading
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.idx)
            self.smax = float(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))
        except Exception:
            return
        bits = {"hw_slowdown": pynvml.nvmlClocksEventReasonHwSlowdown,
                "hw_thermal_slowdown": pynvml.nvmlClocksEventReasonHwThermalSlowdown,
                "sw_thermal_slowdown": pynvml.nvmlClocksEventReasonSwThermalSlowdown,
                "sw_power_cap": pynvml.nvmlClocksEventReasonSwPowerCap}
        self._stop = threading.Event()

        def run():
            while not self._stop.is_set():
                try:
                    sm = float(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
                    rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                    self.rows.append((sm, [k for k, v in bits.items() if rs & v]))
                except Exception:
                    pass
                self._stop.wait(0.01)

        self._th = threading.Thread(target=run, daemon=True)
        self._th.start()

    def stop(self):
        if self._th is None:
            return None
        self._stop.set()
        self._th.join(timeout=2)
        if not self.rows:
            return None
        sm = [r[0] for r in self.rows]
        reasons = sorted({k for r in self.rows for k in r[1]})
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": self.smax, "reasons": reasons,
                "samples": len(self.rows), "source": "NVML every 10 ms during the timed steps"}


def cpu_threads():
    try:
        from threadpoolctl import threadpool_info
        info = threadpool_info()
        return max([i.get("num_threads", 1) for i in info] + [1])
    except Exception:
        return os.cpu_count() or 1


# measured oracle wall time (s) of one setup + rhs + PCG solve of a config's recipe at
# sub-mesh n (tools/c5_scaling_study.py, profiles/r02_c5_oracle_study.jsonl); the config-5
# recipe's iteration count grows with n (32 / 114 / 217 at n = 16 / 32 / 64)
# (8-core container, 2 BLAS threads; the box host measured 2-3x faster): the heterogeneous
# recipes' iteration counts grow with n, so the config-2 scaling estimate does not hold there
ORACLE_SECONDS = {3: {32: 1.5, 64: 8.8, 128: 54.0},
                  4: {64: 3.0, 128: 13.5, 256: 69.9},
                  5: {16: 0.3, 32: 2.1, 64: 11.5, 128: 150.0}}


def oracle_sample_n(cfg, budget_s: float) -> int:
    """Largest power-of-two sub-mesh (<= cfg.n) the oracle finishes in ~budget_s
    (calibrated: config-2 recipe at n=256 takes ~20 s on an 8-core host; config 5 from
    its measured table)."""
    if cfg.index in ORACLE_SECONDS:
        tab = ORACLE_SECONDS[cfg.index]
        fit = [n for n, t in tab.items() if t <= budget_s and n <= cfg.n]
        return max(fit) if fit else min(tab)
    n = cfg.n
    est = 20.0 * (n / 256.0) ** 2 * ((cfg.p + 1) / 5.0) ** 3
    while n > 16 and est > budget_s:
        n //= 2
        est /= 4.0
    return n


def run_oracle_step(cfg):
    from oracle import driver
    pr = W.make_problem(cfg)
    t0 = time.perf_counter()
    res = driver.solve_problem(pr)
    t1 = time.perf_counter()
    return t1 - t0, res["iters"]


def reference_arm(args, cfg):
    rank, world, _ = _dist_env()
    if rank != 0:
        return 0
    per_step = 180.0 / max(1, args.steps + args.warmup)
    ns = oracle_sample_n(cfg, per_step)
    sc = W.scaled_config(cfg.index, ns) if ns != cfg.n else cfg
    for _ in range(args.warmup):
        run_oracle_step(sc)
    times, its = [], []
    for _ in range(args.steps):
        t, it = run_oracle_step(sc)
        times.append(t)
        its.append(it)
    tstep = float(np.mean(times))
    value = sc.trace_dofs / tstep
    sample = (f"oracle setup+rhs+PCG on the config-{cfg.index} recipe at n={ns} "
              f"({sc.trace_dofs} trace dofs, {its[-1]} PCG iterations) per step")
    line = {
        "impl": "reference", "metric": "fine trace DoFs/s in MG-PCG solve to 1e-10", "value": value,
        "unit": "trace DoF/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": tstep * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": {"workload": cfg.name, "n": cfg.n, "p": cfg.p, "sample_n": ns},
        "cpu_baseline": {"value": value, "unit": "trace DoF/s", "cores": cpu_threads(), "kind": "oracle",
                         "sample": sample},
        "e2e": {"value": value, "unit": "trace DoF/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def bytes_per_iteration(s, sm, ns=False, krylov="pcg"):
    """Modelled algorithmic bytes of one solver iteration (SURVEY 8(d) "per PCG
    iteration"): what the method must move, each operand once per use.
      per apply on level l: S_T (packed m(m+1)/2 or, nonsymmetric, m^2 doubles per
        element) + 16 B per trace dof (x read, y written);
      per smoothing step: an apply + D_e^-1 (packed, k1(k1+1)/2 doubles per edge) +
        r read and e read/written (24 B/dof; Chebyshev d read/written +16 B/dof);
      per non-coarsest level and V-cycle: nu_pre + nu_post smoothing steps (the first
        pre-step from e = 0 has no apply), one residual apply (+8 B/dof for r), the
        transfers (restriction reads the residual, prolongation reads / writes e:
        24 B/dof);
      per Krylov iteration: one fine apply + ~6 fine vector passes (PCG x, r, p, z
        updates and dots; GMRES: its Gram-Schmidt passes are counted at 2 per basis
        vector by the caller's iteration count, approximated here by 6)."""
    NORB = {1: 7, 2: 14, 3: 22, 4: 33}
    NCS = {1: 2, 2: 4, 3: 6, 4: 9}
    tot = 0
    nl = s.nlevels
    fine_p = s.level_info(nl)["p"]
    for level in range(nl, 1, -1):
        li = s.level_info(level)
        ne, p, ndof = li["nx"] * li["ny"], li["p"], li["ndof"]
        m, k1 = 4 * (p + 1), p + 1
        # D4-orbit storage (reading R9) on the finest level and its p-coarsened level
        orb = not ns and (level == nl or (level == nl - 1 and fine_p > 1))
        npk = m * m if ns else NORB[p] if orb else m * (m + 1) // 2
        S = 8 * ne * npk
        apply_b = S + 16 * ndof
        nedge = ndof // k1
        D = 8 * nedge * (NCS[p] if orb else k1 * (k1 + 1) // 2)
        steps = sm.nu_pre + sm.nu_post
        if getattr(sm, "nu_doubling", 0):
            steps *= 2 ** (nl - level)
        vec = 24 + (16 if sm.kind == 1 else 0)
        tot += steps * (apply_b + D + vec * ndof) - (apply_b if sm.nu_pre > 0 else 0)
        tot += apply_b + 8 * ndof + 24 * ndof
    fine = s.level_info(nl)
    m = 4 * (fine["p"] + 1)
    npk = m * m if ns else NORB[fine["p"]]
    tot += 8 * fine["nx"] * fine["ny"] * npk + 16 * fine["ndof"] + 6 * 8 * fine["ndof"]
    return tot


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=5,
                    help="BASELINE.json config index (1-5); default 5, the largest single-GPU config "
                         "and the north star's scaling run (one problem on every N: strong scaling)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-graphs", action="store_true")
    ap.add_argument("--smoother", default="config", choices=["config", "bj", "cheb", "lusgs"],
                    help="override the config's smoother (lusgs: SURVEY 8(f) f3)")
    ap.add_argument("--scheme", default="config", choices=["config", "nipg", "iipg", "tiles"],
                    help="SURVEY 8(f) f2: the config's recipe with IIPG-H / NIPG-H elements "
                         "(workloads.nonsymmetric_problem), a MG_BUILD_NONSYMMETRIC context, "
                         "block-Jacobi and left-preconditioned GMRES (one GPU)")
    args = ap.parse_args()
    _, world0, _ = _dist_env()
    cfg = W.CONFIGS[args.config]
    if args.impl == "reference":
        return reference_arm(args, cfg)
    ns = args.scheme != "config"
    if ns and world0 > 1:
        ap.error("--scheme nipg / iipg / tiles runs on one GPU")

    import torch
    import torch.distributed as dist
    from paper_1811_09909_b200 import MGSolver, Partition, nccl_unique_id, smoother_from_config

    rank, world, local = _dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    part = None
    if world > 1:
        # one global problem sharded in element blocks over px x py ranks:
        # NCCL halo sums of interface edges, all-reduced PCG scalars, gathered coarse levels
        dist.init_process_group("nccl", device_id=dev)
        px = {2: 2, 4: 2, 8: 4, 16: 4}.get(world, world)
        py = world // px
        obj = [nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        part = Partition(rank, world, px, py, nccl_id=obj[0])

    # ---- inputs resident in HBM (N > 1: this rank's element block of the one problem)
    pr = W.nonsymmetric_problem(cfg, args.scheme) if ns else W.make_problem(cfg)
    if part is not None:
        pr = W.block_problem(pr, part.px, part.py, rank)
    K = torch.from_numpy(pr.K).to(dev)
    meth = torch.from_numpy(pr.method).to(dev)
    tau = torch.from_numpy(pr.tau).to(dev)
    fq = None if pr.f_qp is None else torch.from_numpy(pr.f_qp).to(dev)
    gD = None if pr.gD_qp is None else torch.from_numpy(pr.gD_qp).to(dev)
    stream = torch.cuda.Stream(dev)
    with torch.cuda.stream(stream):
        s = MGSolver(cfg.n, p=cfg.p, device=dev, stream=stream, partition=part, nonsymmetric=ns)
    if args.no_graphs:
        s.use_graphs(False)
    sm = smoother_from_config(cfg)
    if args.smoother != "config":
        sm.kind = {"bj": 0, "cheb": 1, "lusgs": 2}[args.smoother]
    if ns:
        sm.kind = 0   # block-Jacobi: Chebyshev needs a real spectrum, PCG a symmetric A

    def solve(g):
        if ns:
            return s.gmres_solve(g, tol=cfg.rtol, maxit=400)
        return s.pcg_solve(g, rtol=cfg.rtol, maxit=4000)
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device=dev)
    st = {"phase": []}

    def step(ev=None):
        # ev: 4 events (step start, after setup, after rhs, step end) of a timed step;
        # the phase split comes from the timed steps themselves
        if ev is not None:
            ev[0].record(stream)
        s.setup(K, meth, tau, sm)
        if ev is not None:
            ev[1].record(stream)
        g, lam_bc = s.assemble_rhs(fq, pr.f_const, gD)
        if ev is not None:
            ev[2].record(stream)
        lam, info = solve(g)
        if ev is not None:
            ev[3].record(stream)
        st["info"] = info
        st["g"], st["lam"] = g, lam
        return lam

    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            step()
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        clocks = ClockSampler(local)
        clocks.start()
        ev = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(args.steps)]
        launches0 = s.total_launch_count()
        for k in range(args.steps):
            flush.fill_(float(k))                     # evict L2 between steps (outside the window)
            step(ev[k])
        torch.cuda.synchronize(dev)
        launches = s.total_launch_count() - launches0
        ck = clocks.stop()
        t_ms = sum(e[0].elapsed_time(e[3]) for e in ev)
        t_setup = float(np.mean([e[0].elapsed_time(e[1]) for e in ev]))
        t_rhs = float(np.mean([e[1].elapsed_time(e[2]) for e in ev]))
        t_solve = float(np.mean([e[2].elapsed_time(e[3]) for e in ev]))
        if world > 1:
            tt = torch.tensor([t_ms], dtype=torch.float64, device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            t_ms = float(tt.item())
            dist.barrier()
    ms_per_step = t_ms / args.steps
    info = st["info"]
    converged = info["status"] == "converged" and info["relres"] <= cfg.rtol
    # the true residual of the last timed solve, ||g - A lambda|| / ||g|| (the stopping test
    # is on the recursive residual; on ill-conditioned systems the two
    # part after many iterations), through the row-validated apply; one GPU only
    true_relres = None
    if world == 1 and not ns:
        with torch.cuda.stream(stream):
            Al = s.apply(s.nlevels, st["lam"])
            true_relres = float(torch.linalg.norm(st["g"] - Al) / torch.linalg.norm(st["g"]))
    # one global problem on all ranks (strong scaling) when partitioned; a solve that did
    # not reach rtol gives no throughput
    value = cfg.trace_dofs / (ms_per_step * 1e-3) if converged else None

    # ---- phase breakdown + dominant-kernel roofline (fine-level apply, 2 colour passes)
    with torch.cuda.stream(stream):
        def timed(fn, reps, warm=1):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            for _ in range(warm):   # lazy module loading / first-launch attributes stay untimed
                fn()
            tot = 0.0
            for _ in range(reps):
                flush.fill_(1.0)
                a.record(stream)
                fn()
                b.record(stream)
                torch.cuda.synchronize(dev)
                tot += a.elapsed_time(b)
            return tot / reps
        x = torch.rand(s.ndof(), dtype=torch.float64, device=dev)
        y = torch.empty_like(x)
        N = s.nlevels
        t_apply = timed(lambda: s.apply(N, x, y), 20, warm=3)
    ne = cfg.n * cfg.n // world      # this rank's elements
    m = 4 * (cfg.p + 1)
    npk = m * m if ns else m * (m + 1) // 2
    ndof = s.ndof()
    # the element maps as stored (orbit values, reading R9; ns: full) + x + y
    norb = {1: 7, 2: 14, 3: 22, 4: 33}[cfg.p]
    alg_bytes = ne * 8 * (npk if ns else norb) + 16 * ndof
    peaks = _peaks()
    peak = peaks.get("hbm_gbs", 6650.0)
    achieved = alg_bytes / (t_apply * 1e-3) / 1e9
    bpi = bytes_per_iteration(s, sm, ns)
    t_iter = t_solve / max(1, info["iters"])
    solve_roof = {"bytes_per_iter": int(bpi), "ms_per_iter": t_iter,
                  "achieved_gbs": bpi / (t_iter * 1e-3) / 1e9,
                  "frac": bpi / (t_iter * 1e-3) / 1e9 / peaks.get("hbm_gbs", 6650.0),
                  "model": "bench.bytes_per_iteration (SURVEY 8(d) per-iteration byte model)"}
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        traffic = json.load(open(tpath)).get(cfg.name)

    # ---- end to end through the C ABI with HOST buffers (h2d inputs, d2h solution);
    # collective on a partition (every rank solves its block), rank 0 reports
    e2e = None
    if ns:   # no mg_solve_host for GMRES: the same public calls with the copies in the region
        Kh = torch.from_numpy(pr.K).pin_memory()
        mh = torch.from_numpy(pr.method).pin_memory()
        th = torch.from_numpy(pr.tau).pin_memory()
        fh = None if pr.f_qp is None else torch.from_numpy(pr.f_qp).pin_memory()
        gh = None if pr.gD_qp is None else torch.from_numpy(pr.gD_qp).pin_memory()
        out = torch.empty(ndof, dtype=torch.float64).pin_memory()

        def host_step():
            Kd, md, td = (Kh.to(dev, non_blocking=True), mh.to(dev, non_blocking=True),
                          th.to(dev, non_blocking=True))
            fd = None if fh is None else fh.to(dev, non_blocking=True)
            gd = None if gh is None else gh.to(dev, non_blocking=True)
            s.setup(Kd, md, td, sm)
            g2, lbc = s.assemble_rhs(fd, pr.f_const, gd)
            lam2, _ = solve(g2)
            out.copy_(lam2 + lbc, non_blocking=True)
            torch.cuda.synchronize(dev)
        with torch.cuda.stream(stream):
            host_step()
            te = []
            for _ in range(max(1, min(args.steps, 3))):
                flush.fill_(2.0)
                torch.cuda.synchronize(dev)
                t0 = time.perf_counter()
                host_step()
                te.append(time.perf_counter() - t0)
        h2d = 8 * ne * 2 + ne + (0 if fh is None else 8 * fh.numel()) + (0 if gh is None else 8 * gh.numel())
        e2e = {"value": cfg.trace_dofs / float(np.mean(te)), "unit": "trace DoF/s",
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(8 * ndof)}
    else:
        Kh = torch.from_numpy(pr.K).pin_memory()
        mh = torch.from_numpy(pr.method).pin_memory()
        th = torch.from_numpy(pr.tau).pin_memory()
        fh = None if pr.f_qp is None else torch.from_numpy(pr.f_qp).pin_memory()
        gh = None if pr.gD_qp is None else torch.from_numpy(pr.gD_qp).pin_memory()
        out = torch.empty(ndof, dtype=torch.float64).pin_memory()
        # long solves (config 5: ~50 s each) are timed once, without a warm-up call: every
        # graph and the staging buffer already exist from the timed steps / bind_staging
        long_solve = t_solve > 5000.0
        with torch.cuda.stream(stream):
            s.bind_staging(fh is not None, gh is not None)
            if not long_solve:
                s.solve_host(Kh, mh, th, fh, pr.f_const, gh, sm, cfg.rtol, 4000, out=out.numpy())
            te = []
            for _ in range(1 if long_solve else max(1, min(args.steps, 3))):
                flush.fill_(2.0)
                torch.cuda.synchronize(dev)
                if world > 1:
                    dist.barrier()
                t0 = time.perf_counter()
                s.solve_host(Kh, mh, th, fh, pr.f_const, gh, sm, cfg.rtol, 4000, out=out.numpy())
                te.append(time.perf_counter() - t0)
            if world > 1:   # the slowest rank's wall time
                tt = torch.tensor([float(np.mean(te))], dtype=torch.float64, device=dev)
                dist.all_reduce(tt, op=dist.ReduceOp.MAX)
                te = [float(tt.item())]
        h2d = 8 * ne * 2 + ne + (0 if fh is None else 8 * fh.numel()) + (0 if gh is None else 8 * gh.numel())
        e2e = {"value": cfg.trace_dofs / float(np.mean(te)), "unit": "trace DoF/s",
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(8 * ndof)}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and not ns:
        n_smp = oracle_sample_n(cfg, 30.0)
        sc = W.scaled_config(cfg.index, n_smp) if n_smp != cfg.n else cfg
        t, its = run_oracle_step(sc)
        cpu = {"value": sc.trace_dofs / t, "unit": "trace DoF/s", "cores": cpu_threads(), "kind": "oracle",
               "sample": f"one oracle setup+rhs+PCG solve of the config-{cfg.index} recipe at n={n_smp} "
                         f"({sc.trace_dofs} trace dofs, {its} iterations, {t:.1f} s)"}

    if rank == 0:
        line = {
            "metric": ("fine trace DoFs/s in MG-GMRES solve to 1e-10" if ns
                       else "fine trace DoFs/s in MG-PCG solve to 1e-10"),
            "value": value, "unit": "trace DoF/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "strong" if world > 1 else "weak",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": cfg.name + ("" if not ns else f"+{args.scheme}"),
                       "n": cfg.n, "p": cfg.p, "trace_dofs": cfg.trace_dofs,
                       "smoother": ["block-jacobi", "chebyshev", "lu-sgs"][sm.kind], "nu": cfg.nu,
                       "rtol": cfg.rtol,
                       "parallelism": f"elem-blocks{part.px}x{part.py}" if part else "1gpu",
                       "l2": "256 MiB flush between steps (outside the per-step event window)",
                       "step": "setup_dtn + assemble_rhs + " + ("gmres_solve" if ns else "pcg_solve")},
            "iters": info["iters"], "solve_status": info["status"], "relres": info["relres"],
            "true_relres": true_relres,
            **({} if converged else {"invalid": "the solve did not reach rtol: no throughput"}),
            "phases_ms": {"setup": t_setup, "rhs": t_rhs, "solve": t_solve, "fine_apply": t_apply,
                          "source": "CUDA events inside the timed steps (mean); fine_apply: 20 "
                                    "mg_apply calls after an L2 flush"},
            "solve_only_dofs_per_s": cfg.trace_dofs / (t_solve * 1e-3),
            "gpu_launches": int(launches),
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "kernel": ("k_apply_seg<p,*,*,NSYM> full-storage" if ns else "k_apply_orb<p,*>")
                                   + " fine-level colour passes (mg_apply, both colours)",
                         "alg_bytes_model": ("8*m*m" if ns else "8*NORB (D4 orbit values, reading R9)")
                                            + " per element + 16 B per trace dof (x read, y written)",
                         "alg_bytes_per_apply": alg_bytes,
                         "peak_source": "MEASURED_PEAKS.json hbm_gbs (burst copy)" if "hbm_gbs" in peaks
                         else "fallback 6650 GB/s (B200_PROFILING.md)"},
            "solve_roofline": solve_roof,
            "clocks": ck, "e2e": e2e, "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
