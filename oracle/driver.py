"""End-to-end oracle solve: trace system -> hierarchy -> MG-PCG (north star).

Mirrors the C-ABI sequence mg_build_hierarchy / mg_setup_dtn /
mg_assemble_rhs / mg_pcg_solve on plain numpy data.
"""
from __future__ import annotations

import time

import numpy as np

from .assembly import TraceSystem
from .krylov import pcg
from .multigrid import Hierarchy


def setup(n, p, K, method, tau, f_qp=None, f_const=0.0, gD_qp=None, smoother=0, nu=2,
          n_h_levels=0, **kw):
    ts = TraceSystem(n, p, K, method, tau, f_qp, f_const, gD_qp)
    H = Hierarchy(ts.A, n, p, n_h_levels=n_h_levels, smoother=smoother, nu_pre=nu, nu_post=nu, **kw)
    return ts, H


def solve(n, p, K, method, tau, f_qp=None, f_const=0.0, gD_qp=None, smoother=0, nu=2,
          rtol=1e-10, maxit=2000, n_h_levels=0, **kw):
    t0 = time.perf_counter()
    ts, H = setup(n, p, K, method, tau, f_qp, f_const, gD_qp, smoother, nu, n_h_levels, **kw)
    t1 = time.perf_counter()
    res = pcg(ts.A, H.vcycle, ts.g, rtol=rtol, maxit=maxit)
    t2 = time.perf_counter()
    res["lam_full"] = ts.to_full(res["x"])
    res["t_setup"], res["t_solve"] = t1 - t0, t2 - t1
    res["ts"], res["H"] = ts, H
    return res


def solve_problem(prob, **kw):
    c = prob.cfg
    return solve(c.n, c.p, prob.K, prob.method, prob.tau, prob.f_qp, prob.f_const, prob.gD_qp,
                 smoother=c.smoother, nu=c.nu, rtol=c.rtol, **kw)
