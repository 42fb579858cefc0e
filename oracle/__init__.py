"""CPU FP64 oracle for the DtN-based geometric multigrid of arXiv:1811.09909.

TEST INFRASTRUCTURE ONLY.  Only `tests/`, `__graft_entry__.smoke()` and the
`cpu_baseline` / `--impl reference` legs of `bench.py` may import or execute
anything under `oracle/`.  The product path (`paper_1811_09909_b200`, the
C-ABI library `libmgdtn.so`) never imports it, and this package never imports
the product path.  The two share no code; only `workloads/` (seeded input
generators, no method arithmetic) feeds both.

The oracle is plain, slow and literal: numpy / scipy in float64, each
function citing the PAPER.md passage it follows.  Where the paper is silent
it takes SURVEY.md 8(c)'s reading (listed in DESIGN.md, "Readings").

Modules
  basis      GLL nodes, Gauss quadrature, 1D Lagrange bases        (Q2)
  element    reference-element matrices, HDG / SIPG-H local solves (Eqs. HDG,
             HDG_flux, SIPG_H; static condensation PAPER.md:305-316)
  mesh       structured numbering
  assembly   trace system A lambda = g (Eq. 3.1), strong Dirichlet data (Q4)
  multigrid  p/h hierarchy, transfers, smoothers, Algorithm 1 V-cycle
  krylov     PCG (north star), GMRES and MG-as-solver (PAPER.md:937-939,
             1008-1018)

Parity pins: every function here is pinned by a `-m "not gpu"` test in
tests/test_oracle_*.py against closed forms, invariants, brute force or the
paper's printed iteration counts (tests/golden/).  Functions with no such
pin: none known; the PCG iteration counts of the five configs are pinned
only GPU-vs-oracle (the paper has no PCG) and qualitatively by P14.
"""
