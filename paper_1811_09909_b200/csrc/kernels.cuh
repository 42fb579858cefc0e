// Device data layout, indexing helpers and kernel launchers (sm_100a, FP64).
//
// Element DtN maps of a level are stored packed-symmetric (upper triangle,
// row-major, npk = m(m+1)/2 entries, m = 4(p+1)) -- or, in a context built for
// the nonsymmetric schemes IIPG-H / NIPG-H (LevelDev::ns), in full row-major
// storage (npk = m*m, entry kk = a*m + b) -- and element-interleaved in
// chunks of 32 same-colour elements:
//     S[((colour*nchunk + chunk)*npk + kk)*32 + lane]
// so that one warp-wide load of entry kk of 32 consecutive elements is one
// contiguous 256-byte segment.  Colour = (i+j) mod 2 (checkerboard: elements of
// one colour share no edge), index within the colour s = j*(nx/2) + (i>>1),
// chunk = s/32, lane = s%32.
#pragma once
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

namespace mgdtn {

constexpr int MAX_NU = 8;      // max smoothing steps per side
constexpr int MAX_K1 = 5;      // p <= 4

// smoothing update modes of the colour-1 apply pass
enum ApplyMode : int {
  AM_W0 = 0,      // pass 0: y[e] = (S_T x_T)[e]
  AM_APPLY = 1,   // pass 1: y[e] += (S_T x_T)[e]  (+ optional dot x.y)
  AM_RESID = 2,   // pass 1: w[e] = r[e] - (w[e] + (S_T x_T)[e])
  AM_SMOOTH = 3,  // pass 1: d = c1 d + c2 Dinv (r - A x)_e ; x[e] += d  (in place)
  AM_DINV = 4,    // pass 1: y[e] = (A x)_e ; x[e] = Dinv (A x)_e (in place; power iteration)
  AM_GSC = 5,     // pass 1, LU-SGS colour sweep: on edges of colour `step` only,
                  // x[e] += omega Dinv (r - A x)_e (in place; segmented-ring kernel only)
  AM_RESPR = 6,   // pass 1 (orbit levels): res_e = r - A x, then the p-restriction
                  // rc_e = J_p^T res_e (+ the coarse level's first smoothing step); res
                  // itself is not stored (PRArgs)
  AM_W0P = 7,     // pass 0 (orbit levels) with the p-prolongation folded in: x_e += J_p ec_e
                  // on the element's edges as they are gathered, stored back, then y = S x
  AM_W0U = 8,     // pass 0 (orbit fine level, PCG) with the direction update folded in:
                  // p_e = z_e + beta p_e (k_pcg_pupdate's arithmetic; z = PRArgs::ec,
                  // beta = PRArgs::coef[4]) as the edges are gathered, stored back, y = S p
  AM_W0H = 9      // pass 0 (P1 orbit level, one GPU) with the h-prolongation folded in:
                  // x_e += (I_k ec)_e (prolong_edge_term; ec = PRArgs::ec, P_M = PRArgs::Jp)
                  // as the edges are gathered, stored back, then y = S x
};

// Flag in the `step` argument of the orbit-level smoothing passes (k_apply_orb / orb2,
// AM_SMOOTH): Chebyshev step 1 after a first step from e = 0, whose direction d_0 equals
// the iterate x_1 bit for bit (0 + d_0 = d_0): d is read from x (no second stream; the
// first step then need not store d at all).
constexpr int STEP_D_FROM_X = 1 << 8;
// ... and the last Chebyshev step of a pre- or post-smoothing sweep: its direction is never
// read (the next step of the V-cycle is a restriction, or the V-cycle ends, and every sweep
// starts with a step 0 that reads no d), so it is not stored.
constexpr int STEP_NO_D_STORE = 1 << 9;

// AM_RESPR: the p-coarse level's restriction target (bodies.cuh p_restrict_body)
struct PRArgs {
  const double* Jp;     // K1 x 2 (row a: the two P1 coefficients of dof a)
  double* rc;           // coarse residual (2 per edge)
  double* ec;           // fuse: coarse first smoothing step e = c2 D^-1 rc
  double* dc;           // fuse, Chebyshev: its direction d = e
  const double* Dso;    // coarse P1 orbit level's D_e^-1 orbits (SoA, stride nedge)
  const double* coef;   // coarse smoothing coefficients (coef[1] = c2 of step 0)
  int64_t nedge;
  int fuse, smoother;
};

// LU-SGS colour of local edge f of element (i,j): horizontal edges of even / odd
// rows 0 / 1, vertical edges of even / odd columns 2 / 3 (an element's four edges
// have four different colours, so one colour's edges share no element)
__host__ __device__ __forceinline__ int gs_colour(int i, int j, int f) {
  return f == 0 ? (j & 1) : f == 2 ? ((j + 1) & 1) : f == 3 ? 2 + (i & 1) : 2 + ((i + 1) & 1);
}

struct LevelDev {
  int nx, ny, p, k1, m, npk;
  int ns;                  // 1: nonsymmetric operator (full S_T storage, LU factors; Eq. IPG_H)
  int64_t ne, nedge, ndof;
  int nchunk;              // chunks of 32 per colour
  double* S;               // interleaved packed DtN
  double* Dinv;            // SoA [k1*k1][nedge]: entry (a,b) of edge e at (a*k1+b)*nedge + e
  double* Dc;              // the same blocks in colour-1 element-chunk order, packed upper
                           // triangle: Dc[((chunk*ndi + f*nde + pk(a,b))*32 + lane] for edge f
                           // of colour-1 slot 32*chunk+lane (every free edge has exactly one
                           // colour-1 element); streamed with S_T by the smoothing applies
  int ndi;                 // 4 * k1*(k1+1)/2
  double* coef;            // [2*MAX_NU] smoothing coefficients (c1_j, c2_j), device
  int smoother;            // 0 BJ, 1 Chebyshev (d vector used)
  // D4-orbit storage (d4.cuh, reading R9): set on the levels whose element maps are all
  // D4-invariant (the finest level and its p-coarsened P1 level, symmetric contexts)
  int orb;                 // 1: the apply streams So / Dco (k_apply_orb)
  double* So;              // [2][nchunk][NORB][32] orbit values of the element maps
  double* Dco;             // [nchunk][4][NCS][32] D_e^-1 orbits, colour-1 element order
  double* Dso;             // [NCS][nedge] D_e^-1 orbits, SoA (edge-parallel kernels)
  const int* clist;        // non-null: an orbit-level pass covers only these chunks (ncl of them)
  int ncl;
  int sweep;               // mg_set_option MG_OPT_SWEEP: 0 auto, 1 wherever possible, -1 never
  int gather;              // one-pass gather-form apply (k_apply_gather; plan_gather)
  int grid_cap;            // mg_set_option MG_OPT_APPLY_GRID_CAP: max CTAs per apply pass (0: none)
  // partitioned levels (multi-GPU): local sides 0 bottom, 1 right, 2 top, 3 left
  int dmask;               // sides on the global boundary dOmega (Dirichlet); 15 on one GPU
  int imask;               // sides that are partition interfaces (15 & ~dmask on a rank, or 0)
  int ox, oy, gnx, gny;    // this block's element offset in the global level and the global
                           // level's dims (0, 0, nx, ny on one GPU)
};

// global edge id of local edge e of a level block (power-iteration start vector)
__host__ __device__ __forceinline__ int64_t global_edge(const LevelDev& L, int64_t e) {
  const int64_t nh = (int64_t)L.nx * (L.ny + 1);
  if (e < nh) {
    const int j = (int)(e / L.nx), i = (int)(e - (int64_t)j * L.nx);
    return (int64_t)(L.oy + j) * L.gnx + (L.ox + i);
  }
  const int64_t r = e - nh;
  const int j = (int)(r / (L.nx + 1)), i = (int)(r - (int64_t)j * (L.nx + 1));
  return (int64_t)L.gnx * (L.gny + 1) + (int64_t)(L.oy + j) * (L.gnx + 1) + (L.ox + i);
}

// non-owned interface sides: an interface edge is counted in dot products by
// one rank only, the one below / to the left of it
__host__ __device__ __forceinline__ int nonowned_mask(int imask) { return imask & 9; }

// ---------------------------------------------------------------- indexing
__host__ __device__ __forceinline__ int64_t hedge(int nx, int i, int j) {
  return (int64_t)j * nx + i;
}
__host__ __device__ __forceinline__ int64_t vedge(int nx, int ny, int i, int j) {
  return (int64_t)nx * (ny + 1) + (int64_t)j * (nx + 1) + i;
}
__host__ __device__ __forceinline__ int pk_index(int i, int j, int m) {  // i <= j
  return i * (2 * m - i + 1) / 2 + (j - i);
}
// storage index of entry (a, b) of an element map: packed upper triangle, or
// row-major when the level is nonsymmetric
__host__ __device__ __forceinline__ int s_index(int a, int b, int m, int ns) {
  if (ns) return a * m + b;
  return a <= b ? pk_index(a, b, m) : pk_index(b, a, m);
}
__host__ __device__ __forceinline__ int64_t s_offset(int nchunk, int npk, int colour, int64_t s,
                                                     int kk) {
  int64_t chunk = s >> 5;
  int lane = (int)(s & 31);
  return (((int64_t)colour * nchunk + chunk) * npk + kk) * 32 + lane;
}
// element (i,j) -> (colour, s)
__host__ __device__ __forceinline__ void elem_slot(int nx, int i, int j, int& colour,
                                                   int64_t& s) {
  colour = (i + j) & 1;
  s = (int64_t)j * (nx >> 1) + (i >> 1);
}
// (colour, s) -> element (i,j)
// (32-bit unsigned division: every slot / edge / dof index of a level is < 2^32)
__host__ __device__ __forceinline__ void slot_elem(int nx, int colour, int64_t s, int& i,
                                                   int& j) {
  const unsigned nxh = (unsigned)(nx >> 1), su = (unsigned)s;
  j = (int)(su / nxh);
  i = 2 * (int)(su - (unsigned)j * nxh) + ((j + colour) & 1);
}
// the 4 edges {bottom, right, top, left} of element (i,j) and their dOmega flags
// (dmask: which local mesh sides lie on dOmega; the others are partition interfaces)
__host__ __device__ __forceinline__ void elem_edges(int nx, int ny, int i, int j, int64_t e[4],
                                                    bool bd[4], int dmask = 15) {
  e[0] = hedge(nx, i, j);
  e[1] = vedge(nx, ny, i + 1, j);
  e[2] = hedge(nx, i, j + 1);
  e[3] = vedge(nx, ny, i, j);
  bd[0] = (j == 0) && (dmask & 1);
  bd[1] = (i == nx - 1) && (dmask & 2);
  bd[2] = (j == ny - 1) && (dmask & 4);
  bd[3] = (i == 0) && (dmask & 8);
}
// interface bits of element (i,j): bit f set if its edge f lies on a partition interface
__host__ __device__ __forceinline__ int elem_itf(int nx, int ny, int i, int j, int imask) {
  if (!imask) return 0;
  return ((j == 0) ? (imask & 1) : 0) | ((i == nx - 1) ? (imask & 2) : 0) |
         ((j == ny - 1) ? (imask & 4) : 0) | ((i == 0) ? (imask & 8) : 0);
}
// local side of edge e: -1 if not on the local mesh boundary, else 0 bottom, 1 right, 2 top, 3 left
__host__ __device__ __forceinline__ int edge_side(int nx, int ny, int64_t e) {
  const unsigned nh = (unsigned)nx * (unsigned)(ny + 1), eu = (unsigned)e;
  if (eu < nh) {
    const unsigned j = eu / (unsigned)nx;
    return j == 0 ? 0 : j == (unsigned)ny ? 2 : -1;
  }
  const unsigned i = (eu - nh) % (unsigned)(nx + 1);
  return i == 0 ? 3 : i == (unsigned)nx ? 1 : -1;
}
// edge id -> is it on dOmega
__host__ __device__ __forceinline__ bool edge_on_boundary(int nx, int ny, int64_t e,
                                                          int dmask = 15) {
  const int sd = edge_side(nx, ny, e);
  return sd >= 0 && ((dmask >> sd) & 1);
}
// edge id -> counted by this rank in global dot products (not a non-owned interface edge)
__host__ __device__ __forceinline__ bool edge_counted(int nx, int ny, int64_t e, int nomask) {
  if (!nomask) return true;
  const int sd = edge_side(nx, ny, e);
  return sd < 0 || !((nomask >> sd) & 1);
}
// interface edges of side f in their order along the side (the neighbour rank's
// matching side lists the same global edges in the same order)
__host__ __device__ __forceinline__ int side_len(int nx, int ny, int f) {
  return (f == 0 || f == 2) ? nx : ny;
}
__host__ __device__ __forceinline__ int64_t side_edge(int nx, int ny, int f, int q) {
  return f == 0 ? hedge(nx, q, 0) : f == 2 ? hedge(nx, q, ny) : f == 3 ? vedge(nx, ny, 0, q)
                                                                      : vedge(nx, ny, nx, q);
}

// ---------------------------------------------------------------- device error slot
struct DevError {
  int code;        // 0 = none, else MG_ERR_*
  int pad;
  long long index; // element / edge index
};
__device__ __forceinline__ void report_error(DevError* err, int code, long long index) {
  if (atomicCAS(&err->code, 0, code) == 0) err->index = index;
}

// explicit inverse of an SPD k x k block (row-major) by Cholesky; false if not SPD
__host__ __device__ __forceinline__ bool chol_inverse(const double* D, int K1, double* inv) {
  double Lc[MAX_K1 * MAX_K1];
  bool ok = true;
  for (int j = 0; j < K1; ++j) {
    double d = D[j * K1 + j];
    for (int k = 0; k < j; ++k) d -= Lc[j * K1 + k] * Lc[j * K1 + k];
    if (!(d > 0.0)) {
      ok = false;
      d = 1e-300;
    }
    d = sqrt(d);
    Lc[j * K1 + j] = d;
    for (int i = j + 1; i < K1; ++i) {
      double s = D[i * K1 + j];
      for (int k = 0; k < j; ++k) s -= Lc[i * K1 + k] * Lc[j * K1 + k];
      Lc[i * K1 + j] = s / d;
    }
  }
  for (int c = 0; c < K1; ++c) {
    double v[MAX_K1];
    for (int a = 0; a < K1; ++a) {
      double s = (a == c) ? 1.0 : 0.0;
      for (int k = 0; k < a; ++k) s -= Lc[a * K1 + k] * v[k];
      v[a] = s / Lc[a * K1 + a];
    }
    for (int a = K1 - 1; a >= 0; --a) {
      double s = v[a];
      for (int k = a + 1; k < K1; ++k) s -= Lc[k * K1 + a] * v[k];
      v[a] = s / Lc[a * K1 + a];
    }
    for (int a = 0; a < K1; ++a) inv[a * K1 + c] = v[a];
  }
  return ok;
}

// explicit inverse of a general k x k block (row-major) by Gauss-Jordan elimination
// with partial pivoting (the nonsymmetric schemes' edge / macro / coarsest blocks);
// false if a pivot vanishes
__host__ __device__ __forceinline__ bool gj_inverse(const double* D, int n, double* inv, double* A) {
  // A: n*n scratch
  for (int q = 0; q < n * n; ++q) {
    A[q] = D[q];
    inv[q] = (q / n == q % n) ? 1.0 : 0.0;
  }
  bool ok = true;
  for (int k = 0; k < n; ++k) {
    int piv = k;
    double best = fabs(A[k * n + k]);
    for (int r = k + 1; r < n; ++r)
      if (fabs(A[r * n + k]) > best) {
        best = fabs(A[r * n + k]);
        piv = r;
      }
    if (!(best > 0.0)) {
      ok = false;
      A[k * n + k] = 1e-300;
      piv = k;
    }
    if (piv != k)
      for (int c = 0; c < n; ++c) {
        double t = A[k * n + c];
        A[k * n + c] = A[piv * n + c];
        A[piv * n + c] = t;
        t = inv[k * n + c];
        inv[k * n + c] = inv[piv * n + c];
        inv[piv * n + c] = t;
      }
    const double dinv = 1.0 / A[k * n + k];
    for (int c = 0; c < n; ++c) {
      A[k * n + c] *= dinv;
      inv[k * n + c] *= dinv;
    }
    for (int r = 0; r < n; ++r) {
      if (r == k) continue;
      const double f = A[r * n + k];
      if (f == 0.0) continue;
      for (int c = 0; c < n; ++c) {
        A[r * n + c] -= f * A[k * n + c];
        inv[r * n + c] -= f * inv[k * n + c];
      }
    }
  }
  return ok;
}

// reference tables on the device (one set per p)
struct RefDev {
  int p, k1, nv, m, nqf;
  const double *G, *F, *P, *E, *W, *H, *LN, *Nl, *fq, *ew, *H1inv, *Jp;
  const double *Lv, *Nv;   // volume stiffness L and <grad phi_j.n, phi_i>_dT (IPDG with s_f != 1)
  // pencil tables per method (refelem.h RefTables::Pencil): [0] HDG, [1] SIPG-H
  const double *plam[2], *pmu[2], *pAt[2], *pBk[2], *pfq[2];
  const double *pTt[2], *vq, *wq;   // volume recovery (refelem.h)
};

// ---------------------------------------------------------------- programmatic dependent launch
// Every solve-path kernel is launched with programmatic stream serialization
// and starts with pdl_enter(): it may be scheduled while its predecessor is
// still running (hiding the launch latency of the long chain of small V-cycle
// kernels) but waits for the predecessor's completion and memory flush before
// touching any data.  In a kernel launched without the attribute both are no-ops.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
// No explicit griddepcontrol.launch_dependents: the dependent grid is released when this
// grid exits (the implicit trigger).  Triggering at kernel entry let the next kernel's
// CTAs take SM slots and spin for the whole of a long pass; measured (round 2, solve
// time, trigger at entry -> at exit): config 2 6.03 -> 5.71 ms, config 3 3389 -> 3127 ms,
// config 4 150 -> 116 ms, config 5 (30 iterations) 1417 -> 1163 ms.  What PDL still buys:
// the launch of the dependent and its pre-wait prologue (the element-data TMA prefetch of
// the apply kernels) overlap the primary's drain.
__device__ __forceinline__ void pdl_trigger() {}
__device__ __forceinline__ void pdl_enter() {
  pdl_wait();
  pdl_trigger();
}

bool pdl_enabled();   // MGDTN_PDL=0 turns programmatic dependent launch off (A/B)

template <typename... KArgs, typename... Args>
inline void launch_ex(void (*kern)(KArgs...), int grid, int block, size_t smem, bool pdl,
                      cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = (pdl && pdl_enabled()) ? 1 : 0;
  cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

// ---------------------------------------------------------------- launchers
// all launchers return the number of kernels launched (for launch counting)
// pdl: programmatic dependent launch; the S_T prefetch then starts before the
// previous kernel finishes, so the previous kernel must not write this level's S_T.
int launch_apply(const LevelDev& L, int colour, int mode, const double* x, double* y,
                 const double* r, double* d, int step, double* partials, bool pdl,
                 cudaStream_t st);
int apply_grid(const LevelDev& L);   // blocks of an AM_APPLY colour pass (partials length)
int apply_grid_mode(const LevelDev& L, int mode);   // blocks of a colour pass in `mode`
// whole apply: the colour-0 pass (AM_W0) then the colour-1 pass in `mode`
int launch_apply2(const LevelDev& L, int mode, const double* x, double* y, const double* r,
                  double* d, int step, double* partials, bool pdl, cudaStream_t st);
int apply2_grid(const LevelDev& L, int mode);  // blocks of launch_apply2 (partials length)
// residual + p-restriction in the pair of colour passes of an orbit level (AM_RESPR);
// y is scratch for the colour-0 partial sums
// colour-0 pass with the p-prolongation x += J_p ec folded in (AM_W0P): afterwards x
// holds the prolonged iterate on every edge (each edge has one colour-0 element) and y
// the colour-0 partial sums of A x, as after p_prolong + the colour-0 pass
int launch_w0_prolong(const LevelDev& F, const double* Jp, const double* ec, double* x, double* y,
                      cudaStream_t st);
// colour-0 pass of the PCG apply with p = z + beta p folded in (AM_W0U; scal[4] = beta):
// afterwards p holds the new direction on every edge and y the colour-0 partial sums of
// A p, as after k_pcg_pupdate + the colour-0 pass; -1 if F is not a one-GPU orbit level
int launch_w0_update(const LevelDev& F, const double* z, const double* scal, double* p, double* y,
                     cudaStream_t st);
// colour-0 pass with the h-prolongation e += I_k ec folded in (AM_W0H): afterwards x holds
// the prolonged iterate on every edge and y the colour-0 partial sums, as after
// k_prolong_edges + the colour-0 pass; -1 unless F is a one-GPU P1 orbit level
int launch_w0_hprolong(const LevelDev& F, const double* ec, const double* Pm, double* x, double* y,
                       cudaStream_t st);
int launch_resid_prestrict(const LevelDev& F, const LevelDev& C, const double* Jp, const double* x,
                           double* y, const double* r, double* rc, bool fuse, double* ec,
                           double* dc, cudaStream_t st);
// single-pass tiled apply on a one-GPU orbit level (k_tile.cu): AM_APPLY (y = A x, dot
// x.y into partials if given), AM_RESID (y = r - A x), AM_SMOOTH (xo = x + d, out of place)
bool tile_level(const LevelDev& L);
bool gather_level(const LevelDev& L);
int launch_apply_gather(const LevelDev& L, int mode, const double* x, double* y, const double* r,
                        double* d, double* xo, int step, cudaStream_t st);
int apply_tile_grid(const LevelDev& L);
int launch_apply_tile(const LevelDev& L, int mode, const double* x, double* y, const double* r,
                      double* d, double* xo, int step, double* partials, cudaStream_t st);

int launch_local_dtn(const LevelDev& L, const RefDev& R, double h, const double* K,
                     const int8_t* method, const double* tau, DevError* err, cudaStream_t st);
int launch_local_rhs(const LevelDev& L, const RefDev& R, double h, const double* K,
                     const int8_t* method, const double* tau, const double* f_qp,
                     double f_const, const double* lamD, double* g, DevError* err,
                     cudaStream_t st);
int launch_dirichlet(const LevelDev& L, const RefDev& R, const double* gD_qp, double* lamD,
                     cudaStream_t st);
// volume recovery q_T from the full trace and, if qex_qp, the
// per-block partial sums of ||q - q_exact||^2 over the elements (partials[grid])
int launch_recover(const LevelDev& L, const RefDev& R, double h, const double* K,
                   const int8_t* method, const double* tau, const double* lam,
                   const double* f_qp, double f_const, double* q_out, const double* qex_qp,
                   double* partials, int* grid_out, cudaStream_t st);
int launch_p_coarsen(const LevelDev& F, const LevelDev& C, const double* Jp, cudaStream_t st);
// Rm: the restriction's macro matrix of a nonsymmetric level (k_setup.cu), else unused
int launch_agglomerate(const LevelDev& F, const LevelDev& C, double* KIIinv, double* Pm,
                       DevError* err, cudaStream_t st, double* dense_out = nullptr,
                       double* Rm = nullptr);
// nonsymmetric context (k_local_ns.cu): the same three element-local operations
int launch_local_dtn_ns(const LevelDev& L, const RefDev& R, double h, const double* K,
                        const int8_t* method, const double* tau, DevError* err, int project,
                        cudaStream_t st);
int launch_local_rhs_ns(const LevelDev& L, const RefDev& R, double h, const double* K,
                        const int8_t* method, const double* tau, const double* f_qp,
                        double f_const, const double* lamD, double* g, cudaStream_t st);
int launch_recover_ns(const LevelDev& L, const RefDev& R, double h, const double* K,
                      const int8_t* method, const double* tau, const double* lam,
                      const double* f_qp, double f_const, double* q_out, const double* qex_qp,
                      double* partials, int* grid_out, cudaStream_t st);
int launch_edge_blocks(const LevelDev& L, DevError* err, cudaStream_t st);
int launch_dinv_pack(const LevelDev& L, cudaStream_t st);   // Dinv (SoA) -> Dc (or Dso / Dco)
// orbit storage of a D4-invariant level (R9): the packed maps are replaced by their orbit
// averages (in place) and the orbit values written to So
int launch_orbit_pack(const LevelDev& L, cudaStream_t st);
// invariant checks (k_debug.cu, mg_check_invariants): out[0] = max ||S_T 1|| / max|S_T|,
// out[1] += non-finite entries; an atomicAdd scatter apply (y zero on entry)
int launch_check_maps(const LevelDev& L, double* out, cudaStream_t st);
int launch_check_finite(const double* v, int64_t n, double* out, cudaStream_t st);
int launch_apply_atomic(const LevelDev& L, const double* x, double* y, cudaStream_t st);
// R10: P S P (P = I - 11^T/8) on every map of a symmetric p = 1 level (k_setup.cu)
int launch_project_const(const LevelDev& L, cudaStream_t st);
int launch_dense_to_packed(const LevelDev& L, const double* src, cudaStream_t st);
int launch_packed_to_dense(const LevelDev& L, double* dst, cudaStream_t st);
int launch_gather_dense(const LevelDev& L, const int64_t* elems, int64_t n, double* dst,
                        cudaStream_t st);

// MG transfer / smoothing kernels
int launch_smooth_first(const LevelDev& L, const double* r, double* e, double* d,
                        cudaStream_t st);
int launch_lc_restrict(const LevelDev& F, const double* res, double* e, const double* KIIinv,
                       const double* Pm, double* cbuf, bool do_lc, bool do_restrict,
                       cudaStream_t st);
int launch_restrict_edges(const LevelDev& F, const LevelDev& C, const double* res,
                          const double* cbuf, double* rc, bool fuse_first, double* ec,
                          double* dc, cudaStream_t st);
int launch_prolong_macro(const LevelDev& F, const LevelDev& C, const double* ec,
                         const double* Pm, double* e, cudaStream_t st);
int launch_p_restrict(const LevelDev& F, const LevelDev& C, const double* Jp,
                      const double* res, double* rc, bool fuse_first, double* ec, double* dc,
                      cudaStream_t st);
int launch_p_prolong(const LevelDev& F, const double* Jp, const double* ec, double* e,
                     cudaStream_t st);
int launch_coarse_assemble_factor(const LevelDev& L, const int* fpos, int nf, double* A1,
                                  double* A1inv, DevError* err, cudaStream_t st);
int launch_coarse_solve(const LevelDev& L, const int* fidx, int nf, const double* A1inv,
                        const double* r, double* e, cudaStream_t st);

// vectors / reductions (grid-stride, deterministic two-stage reductions)
int vec_grid(int64_t n);
// L (optional): skip the non-owned partition-interface dofs of that level
int launch_dot(const double* a, const double* b, int64_t n, double* partials, int grid,
               cudaStream_t st, const LevelDev* L = nullptr);
int launch_scalar_op(double* scal, int src, int dst, int op, cudaStream_t st);
// out[slot] = sum(partials[0:n]); then op: 0 none, 1 alpha = s[0]/sum (breakdown check),
// 2 beta = sum/s[0] and s[0] = sum
int launch_reduce(const double* partials, int n, double* scal, int slot, int op,
                  DevError* err, cudaStream_t st);
int launch_pcg_update(double* x, double* r, const double* p, const double* ap,
                      const double* scal, int64_t n, double* partials, int grid,
                      cudaStream_t st, const LevelDev* L = nullptr);
int launch_pcg_pupdate(double* p, const double* z, const double* scal, int64_t n,
                       cudaStream_t st);
// the update fused with the next V-cycle's first smoothing step on an orbit fine level
// (e = c2 D_e^-1 r, d = e); partials[grid] of ||r||^2
int launch_pcg_update_sf(const LevelDev& L, double* x, double* r, const double* p,
                         const double* ap, const double* scal, double* partials, int grid,
                         double* e, double* d, cudaStream_t st);
int launch_pcg_init(int* istate, double* scal, double rtol, int maxit, cudaStream_t st);
int launch_pcg_check(const double* scal, int* istate, double* hist, int hist_cap,
                     cudaGraphConditionalHandle h, cudaStream_t st);
int launch_pow_init(const LevelDev& L, double* v, cudaStream_t st);
int launch_edge_dinv(const LevelDev& L, const double* y, double* u, double* partials,
                     int grid, cudaStream_t st);
int launch_scale_by_norm(double* v, const double* u, int64_t n, const double* scal, int slot,
                         cudaStream_t st);
int launch_lmax_finish(const double* scal, double safety, double ratio, int nu_max,
                       double* lam_out, double* coef, cudaStream_t st);
int launch_set_bj_coef(double omega, double* coef, cudaStream_t st);
int launch_copy(double* dst, const double* src, int64_t n, cudaStream_t st);
int launch_zero(double* dst, int64_t n, cudaStream_t st);
int launch_copy_masked(const LevelDev& L, double* dst, const double* src, cudaStream_t st);
int launch_add(double* dst, const double* src, int64_t n, cudaStream_t st);
int launch_axpy_dev(const double* coef, double sign, const double* x, double* y, int64_t n,
                    cudaStream_t st);   // y += sign * coef[0] * x (device coefficient)
int launch_scale_rsqrt(const double* ss, double* v, int64_t n, cudaStream_t st);
int launch_combine(double* x, const double* V, int64_t n, const double* y, int m,
                   cudaStream_t st);   // x = sum_i y[i] V_i
int launch_axpby(double a, const double* x, double b, const double* y, double* z, int64_t n,
                 cudaStream_t st);   // z = a x + b y

// ---------------------------------------------------------------- partitioned levels (k_part.cu)
int itf_stride(const LevelDev& L);     // doubles per side in a halo buffer
int eblk_stride(const LevelDev& L);    // doubles per side in an edge-block halo buffer
__host__ __device__ int64_t itf_edges(const LevelDev& L);
int itf_blocks();                      // partial-sum slots of launch_itf_epilogue
int launch_itf_pack(const LevelDev& L, const double* y, double* send, cudaStream_t st);
int launch_itf_epilogue(const LevelDev& L, int mode, double* x, double* y, const double* r,
                        double* d, int step, const double* recv, double* partials,
                        cudaStream_t st);
int launch_restrict_halo_pack(const LevelDev& C, const double* cbuf, double* send,
                              cudaStream_t st);
int launch_restrict_halo_finish(const LevelDev& C, double* rc, const double* send,
                                const double* recv, bool fuse, double* ec, double* dc,
                                cudaStream_t st);
int launch_eblk_pack(const LevelDev& L, double* send, cudaStream_t st);
int launch_eblk_finish(const LevelDev& L, const double* recv, DevError* err, cudaStream_t st);
int launch_gather_vec(const LevelDev& G, int bx, int by, int px, int py, int64_t ndof_loc,
                      const double* all, double* out, cudaStream_t st);
int launch_scatter_vec(const LevelDev& Lc, int ox, int oy, int nxg, int nyg, const double* glob,
                       double* loc, cudaStream_t st);
int launch_gather_S(const LevelDev& G, int bx, int by, int px, const double* dense,
                    cudaStream_t st);

}  // namespace mgdtn
