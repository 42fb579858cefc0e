/*
 * mgdtn.h -- C ABI of the B200-native DtN geometric multigrid for hybridized
 * high-order finite elements (Wildey, Muralikrishnan, Bui-Thanh,
 * arXiv:1811.09909, "Unified geometric multigrid algorithm for hybridized
 * high-order finite element methods").
 *
 * The library solves the trace (skeleton) system  A lambda = g  (PAPER.md:321-325,
 * Eq. `trace_linear_system`) of  -div(K grad q) = f,  q = g_D on dOmega
 * (Eq. `primal_elliptic`) on a structured nx x ny mesh of
 * squares, with CG preconditioned by one multigrid V-cycle (Algorithm 1,
 * PAPER.md:941-963) whose coarse operators and transfers are built only from
 * the fine-scale element DtN maps.
 *
 * Conventions (all functions):
 *   - Return an int status: MG_OK (0) or a negative MG_ERR_*; never abort,
 *     never throw across the ABI.  mg_last_error() gives a message,
 *     mg_last_error_index() the offending element / edge (or -1).
 *   - Array arguments are DEVICE pointers owned by the caller and borrowed
 *     for the duration of the call, unless the name ends in _host.
 *   - All device work is issued on the ctx stream (mg_build_hierarchy's
 *     `cuda_stream`, a cudaStream_t or NULL = legacy default stream).
 *     mg_apply / mg_vcycle / mg_assemble_rhs are asynchronous; mg_setup_dtn
 *     synchronises once at its end (to report local-solve errors); the solvers
 *     and the *_host calls synchronise the stream.
 *   - The library allocates no device memory: everything lives in one
 *     caller-allocated workspace (mg_workspace_bytes / mg_bind_workspace)
 *     that must stay alive until mg_destroy.
 *
 * Numbering (layout contract of every trace vector):
 *   element (i,j), 0<=i<nx, 0<=j<ny: id = j*nx + i
 *   horizontal edge H(i,j), 0<=i<nx, 0<=j<=ny: id = j*nx + i
 *   vertical   edge V(i,j), 0<=i<=nx, 0<=j<ny: id = nx*(ny+1) + j*(nx+1) + i
 *   trace dof (edge e, node a) = e*(p_k+1) + a; nodes are the GLL points of the
 *   edge in its global orientation (+x for horizontal, +y for vertical).
 *   A level-k vector has nedges_k*(p_k+1) doubles; entries on dOmega are
 *   Dirichlet: ignored on input and written as 0 by mg_apply / mg_vcycle /
 *   mg_pcg_solve (the Dirichlet values themselves come from mg_assemble_rhs).
 *
 * Levels use the paper's numbering: level N (= mg_num_levels) is the finest
 * (order p); if p > 1 level N-1 is the P1 space on the same mesh (p-coarsening,
 * PAPER.md:383-407); below that each level agglomerates 2x2 macro-elements
 * down to level 1 (a 2x2 macro mesh, 8 dofs, unless
 * n_h_levels stops earlier).  Level 1 is solved directly.
 */
#ifndef MGDTN_H
#define MGDTN_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (errors are negative) ---- */
enum {
  MG_OK = 0,
  MG_ERR_ARG = -1,              /* bad argument (NULL, out of range) */
  MG_ERR_SHAPE = -2,            /* mesh not coarsenable / sizes inconsistent */
  MG_ERR_SINGULAR_LOCAL = -3,   /* a local (element) solve broke down */
  MG_ERR_NOT_SPD = -4,          /* Cholesky of a local block / edge block / A_1 failed */
  MG_ERR_CUDA = -5,             /* CUDA runtime error (message has the CUDA string) */
  MG_ERR_NCCL = -6,             /* multi-GPU communicator (NCCL / loopback) error */
  MG_ERR_STATE = -7,            /* call order violated (e.g. solve before setup) */
  MG_ERR_WORKSPACE = -8,        /* workspace missing, too small or misaligned */
  MG_ERR_UNSUPPORTED = -9       /* valid request this build does not implement */
};

/* ---- solve outcomes (not errors; SPEC krylov "returns a status, never panics") ---- */
enum { MG_CONVERGED = 0, MG_MAXIT = 1, MG_DIVERGED = 2, MG_BREAKDOWN = 3 };

/* ---- hybridized method per element ---- */
enum { MG_HDG = 0,      /* Eqs. HDG, HDG_flux */
       MG_SIPG_H = 1,   /* Eq. SIPG_H, s_f = 1 */
       MG_IIPG_H = 2,   /* Eq. IPG_H, s_f = 0: nonsymmetric */
       MG_NIPG_H = 3 }; /* Eq. IPG_H, s_f = -1: nonsymmetric */

/* ---- mg_build_hierarchy_ex flags ---- */
enum { MG_BUILD_NONSYMMETRIC = 1 };  /* A may be nonsymmetric (MG_IIPG_H / MG_NIPG_H elements):
                                        element maps stored full (m*m doubles instead of
                                        m(m+1)/2), local / edge / macro / coarsest blocks by
                                        LU, restriction by Eq. 3.5 (Q_{k-1} != I_k^T).
                                        Accepts every method code.  Solvers: mg_mg_solve and
                                        mg_gmres_solve (mg_pcg_solve / mg_solve_host return
                                        MG_ERR_UNSUPPORTED: PCG needs a symmetric A).
                                        Smoother: block-Jacobi only.  One GPU only. */

/* ---- smoothers ---- */
enum { MG_SMOOTH_BLOCK_JACOBI = 0,  /* edge blocks, e += omega D_B^-1 (r - A e) */
       MG_SMOOTH_CHEBYSHEV = 1,     /* Chebyshev on D_B^-1 A over [lmax/ratio, lmax] */
       MG_SMOOTH_LUSGS = 2 };       /* LU-SGS on edge blocks: forward
                                       block Gauss-Seidel over 4 edge colours (H even / odd
                                       rows, V even / odd columns), then backward; one
                                       "step" = both sweeps.  One GPU only. */

/* Structured mesh of nx x ny squares of side h with lower-left corner (x0,y0).
 * nx and ny must be even and divisible by 2^(number of h-levels). */
typedef struct {
  int32_t nx, ny;
  double x0, y0, h;
} mg_quad_mesh;

/* Element-block partition for multi-GPU runs (NULL or
 * nranks == 1 selects the single-GPU path).  One rank per GPU; rank
 * r = ry*px + rx holds the global elements [rx*nx/px, (rx+1)*nx/px) x
 * [ry*ny/py, (ry+1)*ny/py) of every level down to the gather level and the
 * whole of every coarser level.  On a rank, mg_quad_mesh stays the GLOBAL mesh;
 * every element array (K, method, tau, f samples) is the rank's block in local
 * element order (local id = jl*(nx/px) + il), every trace vector is the block's
 * local edge numbering (the header's numbering on the nx/px x ny/py block), and
 * interface edges are held by both ranks with identical values; g_D samples are
 * the block's 2*(nx/px)+2*(ny/py) boundary edges (interface ones ignored).
 * Dots count an interface edge once (the rank below / to the left owns it).
 *   nccl_id:   128 bytes from mg_get_nccl_unique_id on rank 0, the same on every
 *              rank (the caller broadcasts it, e.g. torch.distributed)
 *   gather_ne: replicate levels with <= gather_ne global elements (0: 16384)
 *   loopback:  NULL, or a hub from mg_loopback_create (nranks virtual ranks in one
 *              process on one GPU, each driven by its own host thread -- tests) */
typedef struct {
  int32_t rank, nranks, px, py;
  const uint8_t* nccl_id;
  int32_t gather_ne;
  void* loopback;
} mg_partition;

/* NCCL unique id (rank 0), MG_ERR_NCCL if libnccl.so.2 cannot be loaded. */
int mg_get_nccl_unique_id(uint8_t out[128]);
/* Loopback communicator hub for nranks virtual ranks on one GPU (tests). */
void* mg_loopback_create(int32_t nranks);
void mg_loopback_destroy(void* hub);
/* A virtual rank failed: every rank waiting in a loopback collective returns MG_ERR_NCCL. */
void mg_loopback_abort(void* hub);

/* Host-only partition plan (no device work; for checking the decomposition):
 * nlevels, the paper-numbered level of the first replicated level (0: none)
 * and, per level k = 1..nlevels, info[8*(k-1) ..] = {nx, ny, ox, oy, gnx, gny,
 * dmask, imask}: this rank's block dims, its element offset in the global
 * level, the global level dims, the sides on dOmega and the partition-interface
 * sides (bit f: 0 bottom, 1 right, 2 top, 3 left). */
int mg_partition_plan(const mg_quad_mesh* mesh, int32_t p, int32_t n_h_levels,
                      const mg_partition* part, int32_t max_levels, int32_t* nlevels,
                      int32_t* gather_level, int32_t* info);
/* Global edge ids (in halo-message order) of interface side `side` of a level's
 * block: the neighbour's matching side must list the same ids in the same order.
 * global_edges may be NULL (count only). */
int mg_partition_side_edges(const mg_quad_mesh* mesh, int32_t p, int32_t n_h_levels,
                            const mg_partition* part, int32_t level, int32_t side,
                            int64_t* global_edges, int32_t* count);

/* Smoother configuration.  V(nu_pre, nu_post); the Chebyshev "steps" are the
 * polynomial degree.  lambda_max of D_B^-1 A_k is estimated per level by
 * `lmax_iters` power iterations from v_i = 1 + (i mod 7)/7 (i = global dof
 * id), Rayleigh quotient in the D_B inner product, times `lmax_safety`
 * (SURVEY.md 8(c) Q11).  omega applies to block-Jacobi only (paper: 1). */
typedef struct {
  int32_t kind;
  int32_t nu_pre, nu_post;      /* 0 <= nu <= 8 */
  double omega;                 /* block-Jacobi damping, default 1 */
  double cheb_ratio;            /* lambda_min = lambda_max / ratio, default 30 */
  int32_t lmax_iters;           /* default 20 */
  double lmax_safety;           /* default 1.05 */
  int32_t nu_doubling;          /* 1: nu steps on the finest level, x 2 per coarser level
                                   (beta_0 = beta_1 = 2; block-Jacobi
                                   only); 0: V(nu_pre, nu_post) on every level (configs) */
} mg_smoother_cfg;

/* Build the level structure (host only; no device work).  p in 1..4.
 * n_h_levels = 0 coarsens until the macro mesh is 2 x 2 (or until a side
 * becomes odd).  With a partition (nranks > 1) it also creates the communicator
 * (collective: every rank calls it).  Errors: MG_ERR_ARG, MG_ERR_SHAPE,
 * MG_ERR_NCCL.  On a partitioned ctx every call that launches work is
 * collective (all ranks call it in the same order). */
int mg_build_hierarchy(const mg_quad_mesh* mesh, int32_t p, int32_t n_h_levels,
                       const mg_partition* part, void* cuda_stream, void** out_ctx);
/* The same with flags (MG_BUILD_NONSYMMETRIC; 0 = mg_build_hierarchy).  A
 * nonsymmetric build with a partition (nranks > 1) returns MG_ERR_UNSUPPORTED. */
int mg_build_hierarchy_ex(const mg_quad_mesh* mesh, int32_t p, int32_t n_h_levels,
                          const mg_partition* part, int32_t flags, void* cuda_stream,
                          void** out_ctx);

/* Bytes of device workspace the ctx needs (256-byte aligned pointer). */
int mg_workspace_bytes(const void* ctx, size_t* bytes);

/* Bind the caller-allocated device workspace (kept alive until mg_destroy). */
int mg_bind_workspace(void* ctx, void* dev_ptr, size_t bytes);

/* Batched element-local setup and the whole hierarchy (PAPER.md:305-316,
 * 572-811, 1050-1067):
 *   per element: local static condensation -> DtN map S_T (FP64),
 *   p-coarsening S_T^(1) = J_p^T S_T J_p (Eq. ANm1),
 *   per 2x2 agglomerate: A_II^-1, P_M = -A_II^-1 A_IB J, coarse DtN (Eq. Akm1),
 *   edge-block diagonals D_e^-1, Chebyshev lambda_max, coarsest A_1^-1.
 * K[ne] > 0 (scalar permeability per element), method[ne] in {MG_HDG,
 * MG_SIPG_H} (any of the four codes on a MG_BUILD_NONSYMMETRIC ctx; an IIPG-H /
 * NIPG-H code on a symmetric ctx is MG_ERR_ARG), tau[ne] > 0 (stabilisation of the element's own flux,
 * Eq. HDG_flux / IPDG_flux), all device arrays in element-id order.
 * Errors: MG_ERR_NOT_SPD / MG_ERR_SINGULAR_LOCAL (nonsymmetric context: a
 * vanishing LU pivot) with the element / edge / macro index, MG_ERR_ARG for
 * invalid K, tau or method (checked on the device; reported by this call). */
int mg_setup_dtn(void* ctx, const double* K, const int8_t* method, const double* tau,
                 const mg_smoother_cfg* smoother);

/* Right-hand side of the trace system and the Dirichlet trace values.
 * f_qp: [ne][nq][nq] samples of f at the tensor Gauss-Legendre points of each
 *   element (nq = p+4 per direction, point order [qy][qx]), or NULL -> f = f_const.
 * gD_qp: [2*nx+2*ny][nq] samples of g_D on the boundary edges (order: bottom
 *   H(i,0) i=0..nx-1, top H(i,ny), left V(0,j) j=0..ny-1, right V(nx,j); nq
 *   Gauss points along the edge's global orientation), or NULL -> g_D = 0.
 * Outputs (device, ndof_N doubles each):
 *   g: sum_T G_T^T b_T - A_FD lambda_D on free dofs, 0 on dOmega;
 *   lambda_bc: per-edge L2 projection of g_D on dOmega (reading Q4), 0 elsewhere
 *   (may be NULL).  The full trace solution is lambda_free + lambda_bc. */
int mg_assemble_rhs(void* ctx, const double* f_qp, double f_const, const double* gD_qp,
                    double* g, double* lambda_bc);

/* y = A_level x (level in 1..N), x, y device [ndof_level], x != y. */
int mg_apply(void* ctx, int32_t level, const double* x, double* y);

/* z = B_N r: one V-cycle of Algorithm 1 with the step-3 local correction
 * from e = 0.  r, z device [ndof_N]. */
int mg_vcycle(void* ctx, const double* r, double* z);

/* Per-operator entry points (for parity checks of single steps):
 *   mg_smooth:        e <- nsteps smoother iterations on A_level e = r (in place)
 *   mg_local_correct: e += T_k res  (Eq. 3.11; level must have a coarser h-level)
 *   mg_restrict:      rc = Q_{k-1} res  (Eqs. 3.5/3.6, full formula)
 *   mg_prolong:       e += I_k ec       (Eqs. 3.3/3.4)
 * level = k (the finer of the two levels for restrict/prolong). */
int mg_smooth(void* ctx, int32_t level, const double* r, double* e, int32_t nsteps);
int mg_local_correct(void* ctx, int32_t level, const double* res, double* e);
int mg_restrict(void* ctx, int32_t level, const double* res, double* rc);
int mg_prolong(void* ctx, int32_t level, const double* ec, double* e);

/* MG-preconditioned CG on A lambda = g from lambda_0 = 0 (north star).
 * Stops when ||r_k||_2 <= rtol ||g||_2 (recursive residual, free dofs;
 * PAPER.md:1012-1015 normalisation) or after maxit iterations.
 * g, lambda: device [ndof_N].  Host outputs (may be NULL): iters, relres
 * (recursive), solve_status (MG_CONVERGED / MG_MAXIT / MG_DIVERGED /
 * MG_BREAKDOWN), resid_hist [maxit+1].  Synchronises the stream. */
int mg_pcg_solve(void* ctx, const double* g, double* lambda, double rtol, int32_t maxit,
                 int32_t* iters, double* relres, int32_t* solve_status, double* resid_hist);

/* The paper's own Krylov setting, host-driven loops of
 * library kernels, lambda_0 = 0, stopping on the TRUE residual
 * ||g - A lambda|| <= tol ||g||:
 *   mg_mg_solve:    MG as a solver, lambda += B_N (g - A lambda)
 *   mg_gmres_solve: full GMRES left-preconditioned by B_N,
 *                   modified Gram-Schmidt; basis: caller-owned device scratch of
 *                   (maxit + 1) * ndof_N doubles.
 * resid_hist (host, may be NULL): [maxit + 1] relative residuals. */
int mg_mg_solve(void* ctx, const double* g, double* lambda, double tol, int32_t maxit,
                int32_t* iters, double* relres, int32_t* solve_status, double* resid_hist);
int mg_gmres_solve(void* ctx, const double* g, double* lambda, double tol, int32_t maxit,
                   double* basis, int32_t* iters, double* relres, int32_t* solve_status,
                   double* resid_hist);

/* The whole user call with HOST buffers: copy K/method/tau/f/g_D to the
 * device, setup, rhs, PCG, copy the full trace solution (free + Dirichlet)
 * back.  lambda_host [ndof_N].  f_qp_host / gD_qp_host may be NULL. */
int mg_solve_host(void* ctx, const double* K_host, const int8_t* method_host,
                  const double* tau_host, const double* f_qp_host, double f_const,
                  const double* gD_qp_host, const mg_smoother_cfg* smoother, double rtol,
                  int32_t maxit, double* lambda_host, int32_t* iters, double* relres,
                  int32_t* solve_status);

/* Device staging for mg_solve_host (inputs + outputs of one call):
 * bytes for K, tau, method, g, lambda and, if requested, the f / g_D samples. */
int mg_staging_bytes(const void* ctx, int32_t with_f, int32_t with_gD, size_t* bytes);
int mg_bind_staging(void* ctx, void* dev_ptr, size_t bytes);

/* Volume recovery (element by element):
 * q_T from the element's full trace (free solution + Dirichlet values,
 * lambda + lambda_bc of mg_assemble_rhs) and the same f as mg_assemble_rhs:
 *   q_T = Q^-1 (R lambda_T + f_w)  (the local solve of Eqs. HDG / SIPG_H).
 * lambda_full: device [ndof_N]; q_out: device [ne][(p+1)^2], GLL nodal coefficients
 * of Q^p (node b*(p+1)+a, a along x), element-id order.  If q_exact_qp (device
 * [ne][nq][nq], nq = p+4, the f_qp sampling grid) is given and l2_err (host) is
 * not NULL, *l2_err = ||q_T - q_exact||_{L2(Omega)} by that quadrature (all ranks'
 * elements on a partition).  Synchronises when l2_err is requested. */
int mg_recover_volume(void* ctx, const double* lambda_full, const double* f_qp, double f_const,
                      double* q_out, const double* q_exact_qp, double* l2_err);

/* Introspection. */
int mg_num_levels(const void* ctx, int32_t* nlevels);
int mg_level_info(const void* ctx, int32_t level, int32_t* nx, int32_t* ny, int32_t* p,
                  int64_t* ndof);
/* Element DtN maps of a level as dense [ne][m][m] (m = 4(p_k+1)), element-id
 * order (dst device).  mg_debug_set_element_dtn overwrites them (test hook;
 * the symmetric part's upper triangle is what is stored). */
int mg_copy_element_dtn(const void* ctx, int32_t level, double* dst);
/* Element DtN maps of selected elements of a level (full-size parity sampling):
 * elems: device int64 [n] element ids (j*nx+i), dst: device [n][m][m]. */
int mg_gather_element_dtn(const void* ctx, int32_t level, const int64_t* elems, int64_t n,
                          double* dst);
int mg_debug_set_element_dtn(void* ctx, int32_t level, const double* src);
/* Chebyshev lambda_max estimate of a level (host out; 0 if not Chebyshev). */
int mg_level_lambda_max(const void* ctx, int32_t level, double* lam);
/* Number of kernel launches issued by the last mg_pcg_solve (timing claims). */
int mg_last_launch_count(const void* ctx, int64_t* launches);
/* Kernel launches issued through this ctx since it was built. */
int mg_total_launch_count(const void* ctx, int64_t* launches);
/* 1 (default): replay each PCG iteration as two captured CUDA graphs; 0: eager launches. */
int mg_set_use_graphs(void* ctx, int32_t on);

/* Debug / invariant mode: checks a set-up hierarchy on the device and fills
 * report[4] (host): [0] max over every level's element maps of ||S_T 1||_inf / max|S_T| (the
 * exact DtN maps annihilate constants; readings R5 / R10 make it rounding-
 * level), [1] the number of NaN / Inf entries in the maps, edge-block inverses, orbit records
 * and the coarsest inverse, [2] the relative L2 difference between the two-colour apply and
 * an independent atomicAdd scatter apply on the finest level (-1: not run, partitioned or
 * nonsymmetric contexts), [3] 0.  MG_ERR_STATE (with mg_last_error) if [0] > 1e-12, [1] > 0
 * or [2] > 1e-13; synchronises the stream. */
int mg_check_invariants(void* ctx, double* report);

/* Execution options of a context (no effect on the arithmetic each kernel performs;
 * they select which kernel / how many CTAs run it, so that tests can drive every code
 * path at small sizes).  Drops the captured graphs.  MG_ERR_ARG for an unknown key.
 *   MG_OPT_SWEEP          0 (default): the single-pass streamed smoothing kernel on the
 *                         orbit levels large enough for it; 1: wherever its geometry allows
 *                         (one GPU, nx % 64 == 0); -1: never (two-colour passes).
 *   MG_OPT_APPLY_GRID_CAP 0 (default): the tuned grid; n > 0: at most n CTAs per apply pass
 *                         (each CTA then walks many chunks: ring wrap-around at small n).
 *   MG_OPT_COMM_TIMEOUT_MS partitioned contexts: every host wait polls NCCL's asynchronous
 *                         error state and gives up after this many ms (default 300000),
 *                         aborting the communicator and returning MG_ERR_NCCL.
 *   MG_OPT_GATHER_NE      packed P1 levels (one-GPU or replicated) with at most this many
 *                         elements run the apply / residual / smoothing step as one
 *                         gather-form pass (default 65536; 0: never).  Bitwise the same
 *                         results as the pair of colour passes.
 *   MG_OPT_KEEP_FINE_MAPS 1: mg_setup_dtn keeps the finest level's element maps as
 *                         mg_debug_set_element_dtn wrote them (no local solves) and builds
 *                         the rest of the hierarchy from them -- a test hook that runs the
 *                         whole setup and solve on another implementation's element maps;
 *                         0 (default): mg_setup_dtn computes them. */
enum { MG_OPT_SWEEP = 1, MG_OPT_APPLY_GRID_CAP = 2, MG_OPT_COMM_TIMEOUT_MS = 3,
       MG_OPT_GATHER_NE = 4, MG_OPT_KEEP_FINE_MAPS = 5 };
int mg_set_option(void* ctx, int32_t key, int64_t value);

/* ---- Seed-point agglomeration of an unstructured quad mesh ----
 * PAPER.md:491-498 (section 3.1.2): N levels, N_T1 seed points; the fine
 * elements (level N) are agglomerated around the seeds into N_T1 level-1
 * macro-elements, then every level-k macro-element is divided into four
 * approximately equal ones to form level k+1, k = 1 .. N-2.  PAPER.md:485-487:
 * the level-(k-1) traces live on the boundary edges of the level-k agglomerates.
 * Readings (A1-A3): level 1 = graph Voronoi cells of the
 * seeds on the element dual graph (hop distance, ties to the lower seed index);
 * the four-way split = west / east halves by rank under (cx, cy, id), the first
 * ceil(m/2) west, then south / north by rank under (cy, cx, id) inside each half,
 * child id 4*parent + 2*east + north; an edge is on the level-k skeleton iff it
 * is on the domain boundary or its two elements differ in level-k label.
 *   ne, nedge      elements and edges of the fine mesh (ne < 2^31)
 *   edge_elem      DEVICE int32 [nedge][2]: the two elements of the edge,
 *                  [e][1] = -1 on the domain boundary
 *   cx, cy         DEVICE float64 [ne]: element centroids (the split's keys)
 *   seeds          DEVICE int32 [nseed]: seed elements (duplicates: lower index wins)
 *   nlev           N >= 2; outputs levels 1 .. N-1 (nseed * 4^(N-2) < 2^31)
 *   labels         DEVICE int32 [(nlev-1)][ne] (caller-owned): row k-1 = level-k id
 *   skel           DEVICE uint8 [(nlev-1)][nedge] (caller-owned): row k-1 = level-k skeleton
 *   medge          DEVICE int32 [(nlev-1)][nedge] or NULL: row k-1 = the fine edge's level-k
 *                  macro-edge id, -1 off the skeleton (reading A4: a
 *                  macro-edge is the intersection of two agglomerates, or an agglomerate's
 *                  share of the domain boundary = pair (-1, a); ids in lexicographic
 *                  order of the pairs (lo, hi))
 *   nmedge         HOST int64 [nlev-1] (required with medge): macro-edges per level
 *   stream         cudaStream_t (NULL: legacy default); returns after it synchronises.
 * Scratch (keys, member lists) is allocated with cudaMallocAsync on `stream`
 * and freed before return: a setup-time call, once per mesh.  Errors: MG_ERR_ARG
 * (NULL pointer, sizes, a seed or edge element id out of range), MG_ERR_SHAPE with
 * *bad_index = the lowest element no seed reaches (disconnected mesh),
 * MG_ERR_CUDA.  bad_index may be NULL; it is -1 unless MG_ERR_SHAPE. */
int mg_agglomerate_seeds(int64_t ne, int64_t nedge, const int32_t* edge_elem, const double* cx,
                         const double* cy, int32_t nseed, const int32_t* seeds, int32_t nlev,
                         int32_t* labels, uint8_t* skel, int32_t* medge, int64_t* nmedge,
                         void* stream, int64_t* bad_index);

/* Arc-length parameterisation of one level's macro-edges (
 * macro-elements of no standard shape need "a parameterization
 * of each macro-edge to define M_k"; reading A5).  A macro-edge
 * whose fine edges form one simple open path gets s in [0, 1] at every vertex: the
 * lengths sqrt(dx*dx + dy*dy) of the path's edges before the vertex, added in path
 * order from the end vertex least in (vx, vy, vertex id), divided by the path's
 * length (added in the same order).  Any other macro-edge (a closed loop, several
 * pieces, a vertex shared by more than two of its edges) gets s = -1, as do the
 * fine edges off the level's skeleton.
 *   medge          DEVICE int32 [nedge]: one level's macro-edge ids (a row of
 *                  mg_agglomerate_seeds' medge), -1 off the skeleton, < nmedge
 *   edge_vert      DEVICE int32 [nedge][2]: the fine edge's end vertices, < nvert
 *   vx, vy         DEVICE float64 [nvert]: vertex coordinates
 *   s              DEVICE float64 [nedge][2] (caller-owned): s at edge_vert[e][0], [1]
 *   stream         cudaStream_t; returns after it synchronises.  Scratch: cudaMallocAsync.
 * Errors: MG_ERR_ARG (NULL, sizes, a vertex or macro-edge id out of range), MG_ERR_CUDA. */
int mg_macro_edge_params(int64_t nedge, const int32_t* medge, int64_t nmedge,
                         const int32_t* edge_vert, int64_t nvert, const double* vx,
                         const double* vy, double* s, void* stream);

/* P^p transfer blocks of the parameterised macro-edges (reading A6,
 * DESIGN.md section 3): the level's trace space on a macro-edge is P^p in its arc
 * length s with the GLL nodal basis on [0, 1]; fine node a of fine edge e (GLL node
 * t_a from edge_vert[e][0] to [1]) sits at s = s0 + (s1 - s0) t_a, so the injection
 * M_{k-1} -> M_k on that edge is J_e[a][j] = l_j(s).
 *   s      DEVICE float64 [nedge][2]: mg_macro_edge_params' output (s0 < 0: zero block)
 *   p      1 .. 7
 *   J      DEVICE float64 [nedge][p+1][p+1] (caller-owned), row a, column j
 *   stream cudaStream_t; returns after it synchronises.
 * Errors: MG_ERR_ARG (NULL, sizes, p), MG_ERR_CUDA. */
int mg_macro_edge_transfer(int64_t nedge, const double* s, int32_t p, double* J, void* stream);

const char* mg_last_error(const void* ctx);
int64_t mg_last_error_index(const void* ctx);
void mg_destroy(void* ctx);

#ifdef __cplusplus
}
#endif
#endif /* MGDTN_H */
