// V-cycle transfer / smoothing kernels and PCG vector kernels.
//
// Transfers: p-level I_N = J_N, Q_{N-1} = J_N^T (per
// edge); h-levels I_k = [P_M ; J], Q_{k-1} = [P_M^T , J^T] with
// P_M = -A_II^-1 A_IB J per macro.  Local correction T_k = [A_II^-1 0; 0 0]
// (Eq. 3.11) per macro.  Reductions are deterministic two-stage trees.
#include <cstdlib>

#include "bodies.cuh"
#include "d4.cuh"

namespace mgdtn {

bool pdl_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = std::getenv("MGDTN_PDL");
    v = (e && std::atoi(e) == 0) ? 0 : 1;
  }
  return v == 1;
}

static inline int cap_grid(int64_t work, int threads, int cap) {
  int64_t g = (work + threads - 1) / threads;
  if (g < 1) g = 1;
  return (int)(g < cap ? g : cap);
}

#define GTID ((int64_t)blockIdx.x * blockDim.x + threadIdx.x)
#define GNT ((int64_t)gridDim.x * blockDim.x)

// ---------------------------------------------------------------- V-cycle operations (bodies.cuh)
__global__ void k_smooth_first(LevelDev L, const double* __restrict__ r, double* e, double* d) {
  pdl_enter();
  smooth_first_body(L, r, e, d, GTID, GNT);
}

// the same step as a pass over the colour-1 elements (every free edge has exactly
// one): D_e^-1 from the packed, chunk-interleaved Dc (coalesced, 40% fewer bytes
// than the SoA blocks at p=4).  Single-GPU levels only (a partition-interface edge
// may have no local colour-1 element).
template <int K1>
__global__ void k_smooth_first_dc(LevelDev L, const double* __restrict__ r, double* e, double* d) {
  pdl_enter();
  constexpr int NDE = K1 * (K1 + 1) / 2;
  const double c2 = L.coef[1];
  const unsigned nec = (unsigned)(L.ne >> 1);
  // work item = (edge f of the colour-1 element at slot s), f-major: a warp covers 32
  // consecutive slots of one local edge, so every Dc row load is 256 contiguous bytes
  for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < 4 * (int64_t)nec;
       w += (int64_t)gridDim.x * blockDim.x) {
    const int f = (int)((unsigned)w / nec);
    const int64_t s = (int64_t)((unsigned)w - (unsigned)f * nec);
    int i, j;
    slot_elem(L.nx, 1, s, i, j);
    int64_t ed[4];
    bool bd[4];
    elem_edges(L.nx, L.ny, i, j, ed, bd, L.dmask);
    if (bd[f]) continue;
    const double* Dp = L.Dc + ((s >> 5) * L.ndi + f * NDE) * 32 + (s & 31);
    double rv[K1];
#pragma unroll
    for (int a = 0; a < K1; ++a) rv[a] = __ldg(r + ed[f] * K1 + a);
#pragma unroll
    for (int a = 0; a < K1; ++a) {
      double c = 0.0;
#pragma unroll
      for (int b = 0; b < K1; ++b) {
        const int lo = a < b ? a : b, hi = a < b ? b : a;
        c = fma(__ldg(Dp + (int64_t)(lo * (2 * K1 - lo + 1) / 2 + (hi - lo)) * 32), rv[b], c);
      }
      const double v = c2 * c;
      e[ed[f] * K1 + a] = v;
      if (L.smoother == 1) d[ed[f] * K1 + a] = v;
    }
  }
}

// the same step on an orbit-stored level (R9): edge-parallel, D_e^-1 from its
// centrosymmetric orbits Dso (SoA, coalesced), r / e / d as contiguous per-edge rows
template <int P>
__global__ void __launch_bounds__(128) k_smooth_first_orb(LevelDev L, const double* __restrict__ r,
                                                         double* e, double* d) {
  pdl_enter();
  using D = D4<P>;
  constexpr int K1 = P + 1, EB = 128;
  // 128 edges per block: r staged through shared memory (coalesced loads / stores)
  __shared__ double sr[EB * K1];
  const double c2 = L.coef[1];
  const int t = threadIdx.x;
  for (int64_t e0 = (int64_t)blockIdx.x * EB; e0 < L.nedge; e0 += (int64_t)gridDim.x * EB) {
    const int ne = (int)(L.nedge - e0 < EB ? L.nedge - e0 : EB);
    const int64_t off = e0 * K1;
    for (int q = t; q < ne * K1; q += EB) sr[q] = __ldg(r + off + q);
    __syncthreads();
    double ev[K1];
#pragma unroll
    for (int a = 0; a < K1; ++a) ev[a] = 0.0;
    if (t < ne && !edge_on_boundary(L.nx, L.ny, e0 + t, L.dmask)) {
      double dv[D::NCS];
#pragma unroll
      for (int o = 0; o < D::NCS; ++o) dv[o] = __ldg(L.Dso + (int64_t)o * L.nedge + e0 + t);
#pragma unroll
      for (int a = 0; a < K1; ++a) {
        double c = 0.0;
#pragma unroll
        for (int b = 0; b < K1; ++b) c = fma(dv[D::cs(D::pe(a, b))], sr[t * K1 + b], c);
        ev[a] = c2 * c;
      }
    }
    // (each thread reads and rewrites only its own edge's row of sr)
    if (t < ne) {
#pragma unroll
      for (int a = 0; a < K1; ++a) sr[t * K1 + a] = ev[a];
    }
    __syncthreads();
    for (int q = t; q < ne * K1; q += EB) {
      e[off + q] = sr[q];
      if (L.smoother == 1) d[off + q] = sr[q];
    }
    __syncthreads();
  }
}

int launch_smooth_first(const LevelDev& L, const double* r, double* e, double* d,
                        cudaStream_t st) {
  if (L.orb) {
    const int g = cap_grid(L.nedge, 128, 148 * 8);
    switch (L.k1) {
      case 2: launch_ex(k_smooth_first_orb<1>, g, 128, 0, true, st, L, r, e, d); return 1;
      case 3: launch_ex(k_smooth_first_orb<2>, g, 128, 0, true, st, L, r, e, d); return 1;
      case 4: launch_ex(k_smooth_first_orb<3>, g, 128, 0, true, st, L, r, e, d); return 1;
      default: launch_ex(k_smooth_first_orb<4>, g, 128, 0, true, st, L, r, e, d); return 1;
    }
  }
  if (L.imask == 0 && L.Dc != nullptr) {
    const int g = cap_grid(2 * L.ne, 128, 148 * 16);
    switch (L.k1) {
      case 2: launch_ex(k_smooth_first_dc<2>, g, 128, 0, true, st, L, r, e, d); return 1;
      case 3: launch_ex(k_smooth_first_dc<3>, g, 128, 0, true, st, L, r, e, d); return 1;
      case 4: launch_ex(k_smooth_first_dc<4>, g, 128, 0, true, st, L, r, e, d); return 1;
      default: launch_ex(k_smooth_first_dc<5>, g, 128, 0, true, st, L, r, e, d); return 1;
    }
  }
  launch_ex(k_smooth_first, cap_grid(L.nedge, 128, 148 * 8), 128, 0, true, st, L, r, e, d);
  return 1;
}

__global__ void k_lc_restrict(LevelDev F, const double* __restrict__ res, double* e,
                              const double* __restrict__ KIIinv, const double* __restrict__ Pm,
                              double* cbuf, int do_lc, int do_restrict) {
  pdl_enter();
  lc_restrict_body(F, res, e, KIIinv, Pm, cbuf, do_lc, do_restrict, GTID, GNT);
}

int launch_lc_restrict(const LevelDev& F, const double* res, double* e, const double* KIIinv,
                       const double* Pm, double* cbuf, bool do_lc, bool do_restrict,
                       cudaStream_t st) {
  int64_t nmac = (int64_t)(F.nx / 2) * (F.ny / 2);
  launch_ex(k_lc_restrict, cap_grid(8 * nmac, 128, 148 * 8), 128, 0, true, st, F, res, e, KIIinv, Pm, cbuf,
                                                              do_lc, do_restrict);
  return 1;
}

__global__ void k_restrict_edges(LevelDev F, LevelDev C, const double* __restrict__ res,
                                 const double* __restrict__ cbuf, double* rc, int fuse,
                                 double* ec, double* dc) {
  pdl_enter();
  restrict_edges_body(F, C, res, cbuf, rc, fuse, ec, dc, GTID, GNT);
}

int launch_restrict_edges(const LevelDev& F, const LevelDev& C, const double* res,
                          const double* cbuf, double* rc, bool fuse_first, double* ec,
                          double* dc, cudaStream_t st) {
  launch_ex(k_restrict_edges, cap_grid(C.nedge, 128, 148 * 8), 128, 0, true, st, F, C, res, cbuf, rc,
                                                                    fuse_first, ec, dc);
  return 1;
}

// Prolongation e += I_k e_c (Eqs. 3.3 / 3.4, bodies.cuh prolong_macro_body) gathered per fine edge (one thread per fine edge, one 16-byte
// read-modify-write of its two dofs, consecutive threads on consecutive edges): a
// macro-interior edge ie[k] takes rows 2k, 2k+1 of P_M e_c(M); an edge on a macro-edge
// takes its half of J e_c (f0: (c0, cm), f1: (cm, c1)).  Every fine dof gets the one
// term prolong_macro_body adds to it, in the same arithmetic, and the top / right
// interface macro-edges are covered too (no k_prolong_itf).
__global__ void __launch_bounds__(128) k_prolong_edges(LevelDev F, LevelDev C,
                                                       const double* __restrict__ ec,
                                                       const double* __restrict__ Pm, double* e) {
  pdl_enter();
  const int nx = F.nx, nxc = C.nx, nyc = C.ny;
  for (int64_t E = GTID; E < F.nedge; E += GNT) {
    bool skip;
    const double2 v = prolong_edge_term(nx, F.ny, nxc, nyc, C.dmask, ec, Pm, E, skip);
    if (skip) continue;
    double2* ep = reinterpret_cast<double2*>(e) + E;
    double2 o = *ep;
    o.x += v.x;
    o.y += v.y;
    *ep = o;
  }
}

// (agglomerated levels are P1: two dofs per edge on both sides)
int launch_prolong_macro(const LevelDev& F, const LevelDev& C, const double* ec,
                         const double* Pm, double* e, cudaStream_t st) {
  launch_ex(k_prolong_edges, cap_grid(F.nedge, 128, 148 * 16), 128, 0, true, st, F, C, ec, Pm, e);
  return 1;
}

__global__ void k_p_restrict(LevelDev F, LevelDev C, const double* __restrict__ Jp,
                             const double* __restrict__ res, double* rc, int fuse, double* ec,
                             double* dc) {
  pdl_enter();
  p_restrict_body(F, C, Jp, res, rc, fuse, ec, dc, GTID, GNT);
}

int launch_p_restrict(const LevelDev& F, const LevelDev& C, const double* Jp,
                      const double* res, double* rc, bool fuse_first, double* ec, double* dc,
                      cudaStream_t st) {
  launch_ex(k_p_restrict, cap_grid(F.nedge, 128, 148 * 8), 128, 0, true, st, F, C, Jp, res, rc, fuse_first,
                                                                ec, dc);
  return 1;
}

__global__ void k_p_prolong(LevelDev F, const double* __restrict__ Jp,
                            const double* __restrict__ ec, double* e) {
  pdl_enter();
  p_prolong_body(F, Jp, ec, e, GTID, GNT);
}

// the same per edge with the fine rows staged through shared memory (128 edges per
// block, coalesced loads and stores)
template <int K1>
__global__ void __launch_bounds__(128) k_p_prolong_st(LevelDev F, const double* __restrict__ Jp,
                                                      const double* __restrict__ ec, double* e) {
  pdl_enter();
  constexpr int EB = 128;
  __shared__ double se[EB * K1];
  double j0[K1], j1[K1];
#pragma unroll
  for (int a = 0; a < K1; ++a) {
    j0[a] = __ldg(Jp + a * 2);
    j1[a] = __ldg(Jp + a * 2 + 1);
  }
  const int t = threadIdx.x;
  for (int64_t e0 = (int64_t)blockIdx.x * EB; e0 < F.nedge; e0 += (int64_t)gridDim.x * EB) {
    const int ne = (int)(F.nedge - e0 < EB ? F.nedge - e0 : EB);
    const int64_t off = e0 * K1;
    for (int q = t; q < ne * K1; q += EB) se[q] = e[off + q];
    __syncthreads();
    if (t < ne && !edge_on_boundary(F.nx, F.ny, e0 + t, F.dmask)) {
      const double2 c = reinterpret_cast<const double2*>(ec)[e0 + t];
#pragma unroll
      for (int a = 0; a < K1; ++a) se[t * K1 + a] += fma(j0[a], c.x, j1[a] * c.y);
    }
    __syncthreads();
    for (int q = t; q < ne * K1; q += EB) e[off + q] = se[q];
    __syncthreads();
  }
}

int launch_p_prolong(const LevelDev& F, const double* Jp, const double* ec, double* e,
                     cudaStream_t st) {
  const int g = cap_grid(F.nedge, 128, 148 * 8);
  switch (F.k1) {
    case 3: launch_ex(k_p_prolong_st<3>, g, 128, 0, true, st, F, Jp, ec, e); return 1;
    case 4: launch_ex(k_p_prolong_st<4>, g, 128, 0, true, st, F, Jp, ec, e); return 1;
    case 5: launch_ex(k_p_prolong_st<5>, g, 128, 0, true, st, F, Jp, ec, e); return 1;
    default: launch_ex(k_p_prolong, g, 128, 0, true, st, F, Jp, ec, e); return 1;
  }
}

// ---------------------------------------------------------------- reductions
__device__ __forceinline__ double block_sum(double v) {
  __shared__ double red[32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  const int nw = blockDim.x >> 5;
  double t = 0.0;
  if (w == 0) {
    t = lane < nw ? red[lane] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  }
  return t;  // valid in thread 0
}

int vec_grid(int64_t n) { return cap_grid(n, 256, 148 * 4); }

// OwnMask: dofs of non-owned partition-interface edges are skipped, so a global
// dot product counts every duplicated dof once (nomask == 0: single GPU)
struct OwnMask {
  int nx, ny, k1, nomask;
};
static OwnMask own_mask(const LevelDev* L) {
  return L ? OwnMask{L->nx, L->ny, L->k1, nonowned_mask(L->imask)} : OwnMask{1, 1, 1, 0};
}
__device__ __forceinline__ bool counted(const OwnMask& o, int64_t i) {
  return !o.nomask || edge_counted(o.nx, o.ny, (unsigned)i / (unsigned)o.k1, o.nomask);
}

__global__ void k_dot(const double* __restrict__ a, const double* __restrict__ b, int64_t n,
                      double* partials, OwnMask om) {
  pdl_enter();
  double s = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    if (counted(om, i)) s = fma(a[i], b[i], s);
  s = block_sum(s);
  if (threadIdx.x == 0) partials[blockIdx.x] = s;
}

int launch_dot(const double* a, const double* b, int64_t n, double* partials, int grid,
               cudaStream_t st, const LevelDev* L) {
  launch_ex(k_dot, grid, 256, 0, true, st, a, b, n, partials, own_mask(L));
  return 1;
}

// scal layout (PCG): [0] rz, [1] pAp, [2] rr, [3] alpha, [4] beta, [5] gg, [6..] misc
__global__ void k_reduce(const double* __restrict__ partials, int n, double* scal, int slot,
                         int op) {
  pdl_enter();
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) s += partials[i];
  s = block_sum(s);
  if (threadIdx.x == 0) {
    if (op == 1) {          // alpha = rz / pAp; pAp <= 0 is a breakdown (checked by
                            // k_pcg_check): alpha = 0 keeps x unchanged
      scal[3] = s > 0.0 ? scal[0] / s : 0.0;
    } else if (op == 2) {   // beta = rz_new / rz_old, then rz = rz_new
      scal[4] = s / scal[0];
    }
    scal[slot] = s;
  }
}

int launch_reduce(const double* partials, int n, double* scal, int slot, int op, DevError* err,
                  cudaStream_t st) {
  (void)err;
  launch_ex(k_reduce, 1, 1024, 0, true, st, partials, n, scal, slot, op);
  return 1;
}

__global__ void k_pcg_update(double* x, double* r, const double* __restrict__ p,
                             const double* __restrict__ ap, const double* __restrict__ scal,
                             int64_t n, double* partials, OwnMask om) {
  pdl_enter();
  const double alpha = scal[3];
  double s = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    x[i] = fma(alpha, p[i], x[i]);
    const double ri = fma(-alpha, ap[i], r[i]);
    r[i] = ri;
    if (counted(om, i)) s = fma(ri, ri, s);
  }
  s = block_sum(s);
  if (threadIdx.x == 0) partials[blockIdx.x] = s;
}

int launch_pcg_update(double* x, double* r, const double* p, const double* ap,
                      const double* scal, int64_t n, double* partials, int grid,
                      cudaStream_t st, const LevelDev* L) {
  launch_ex(k_pcg_update, grid, 256, 0, true, st, x, r, p, ap, scal, n, partials, own_mask(L));
  return 1;
}

// The PCG update fused with the next V-cycle's first smoothing step (reading R2: from
// e = 0 the first step needs no apply, e = c2 D_e^-1 r): thread per fine edge, x += alpha p,
// r -= alpha Ap, ||r||^2 partials, and on the orbit level e = c2 D_e^-1 r (d = e for
// Chebyshev) from the centrosymmetric D_e^-1 orbits -- r is not read a second time by a
// separate first-step kernel.  After the last iteration the e / d it wrote are unused.
template <int P>
__global__ void __launch_bounds__(128) k_pcg_update_sf(LevelDev L, double* x, double* r,
                                                      const double* __restrict__ p,
                                                      const double* __restrict__ ap,
                                                      const double* __restrict__ scal,
                                                      double* partials, OwnMask om, double* e,
                                                      double* d) {
  pdl_enter();
  using D = D4<P>;
  constexpr int K1 = P + 1, EB = 128;
  // a block's 128 edges are 128*K1 contiguous doubles of every vector: staged through
  // shared memory so that global loads and stores are fully coalesced (a thread's own
  // edge block sits K1 doubles after its neighbour's)
  __shared__ double sx[EB * K1], sr[EB * K1], sp[EB * K1], sa[EB * K1];
  const double alpha = scal[3];
  const double c2 = L.coef[1];
  const int t = threadIdx.x;
  double s = 0.0;
  for (int64_t e0 = (int64_t)blockIdx.x * EB; e0 < L.nedge; e0 += (int64_t)gridDim.x * EB) {
    const int ne = (int)(L.nedge - e0 < EB ? L.nedge - e0 : EB);
    const int64_t off = e0 * K1;
    for (int q = t; q < ne * K1; q += EB) {
      sx[q] = x[off + q];
      sr[q] = r[off + q];
      sp[q] = p[off + q];
      sa[q] = ap[off + q];
    }
    __syncthreads();
    if (t < ne) {
      const int64_t ed = e0 + t;
      const bool cnt = counted(om, ed * K1);
      double rv[K1];
#pragma unroll
      for (int a = 0; a < K1; ++a) {
        sx[t * K1 + a] = fma(alpha, sp[t * K1 + a], sx[t * K1 + a]);
        rv[a] = fma(-alpha, sa[t * K1 + a], sr[t * K1 + a]);
        sr[t * K1 + a] = rv[a];
        if (cnt) s = fma(rv[a], rv[a], s);
      }
      double ev[K1];
#pragma unroll
      for (int a = 0; a < K1; ++a) ev[a] = 0.0;
      if (!edge_on_boundary(L.nx, L.ny, ed, L.dmask)) {
        double dv[D::NCS];
#pragma unroll
        for (int o = 0; o < D::NCS; ++o) dv[o] = __ldg(L.Dso + (int64_t)o * L.nedge + ed);
#pragma unroll
        for (int a = 0; a < K1; ++a) {
          double c = 0.0;
#pragma unroll
          for (int b = 0; b < K1; ++b) c = fma(dv[D::cs(D::pe(a, b))], rv[b], c);
          ev[a] = c2 * c;
        }
      }
#pragma unroll
      for (int a = 0; a < K1; ++a) sp[t * K1 + a] = ev[a];   // e (and d = e)
    }
    __syncthreads();
    for (int q = t; q < ne * K1; q += EB) {
      x[off + q] = sx[q];
      r[off + q] = sr[q];
      e[off + q] = sp[q];
      if (L.smoother == 1 && d) d[off + q] = sp[q];   // (d null: read from e, STEP_D_FROM_X)
    }
    __syncthreads();
  }
  s = block_sum(s);
  if (threadIdx.x == 0) partials[blockIdx.x] = s;
}

int launch_pcg_update_sf(const LevelDev& L, double* x, double* r, const double* p,
                         const double* ap, const double* scal, double* partials, int grid,
                         double* e, double* d, cudaStream_t st) {
  const int threads = 128;
  switch (L.p) {
    case 1: launch_ex(k_pcg_update_sf<1>, grid, threads, 0, true, st, L, x, r, p, ap, scal, partials, own_mask(&L), e, d); break;
    case 2: launch_ex(k_pcg_update_sf<2>, grid, threads, 0, true, st, L, x, r, p, ap, scal, partials, own_mask(&L), e, d); break;
    case 3: launch_ex(k_pcg_update_sf<3>, grid, threads, 0, true, st, L, x, r, p, ap, scal, partials, own_mask(&L), e, d); break;
    default: launch_ex(k_pcg_update_sf<4>, grid, threads, 0, true, st, L, x, r, p, ap, scal, partials, own_mask(&L), e, d); break;
  }
  return 1;
}

// scalar op of k_reduce on an already reduced (all-reduced) value scal[src]:
// op 1: alpha = scal[0] / s; op 2: beta = s / scal[0]; then scal[dst] = s
__global__ void k_scalar_op(double* scal, int src, int dst, int op) {
  pdl_enter();
  if (threadIdx.x == 0) {
    const double s = scal[src];
    if (op == 1) scal[3] = s > 0.0 ? scal[0] / s : 0.0;
    else if (op == 2) scal[4] = s / scal[0];
    scal[dst] = s;
  }
}

int launch_scalar_op(double* scal, int src, int dst, int op, cudaStream_t st) {
  launch_ex(k_scalar_op, 1, 32, 0, true, st, scal, src, dst, op);
  return 1;
}

__global__ void k_pcg_pupdate(double* p, const double* __restrict__ z,
                              const double* __restrict__ scal, int64_t n) {
  pdl_enter();
  const double beta = scal[4];
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    p[i] = fma(beta, p[i], z[i]);
}

int launch_pcg_pupdate(double* p, const double* z, const double* scal, int64_t n,
                       cudaStream_t st) {
  launch_ex(k_pcg_pupdate, vec_grid(n), 256, 0, true, st, p, z, scal, n);
  return 1;
}

// ---------------------------------------------------------------- device-side PCG control
// istate: [0] iteration count, [1] solve status, [2] maxit.  scal[9] = rtol.
// The whole solve is one CUDA graph whose loop is a conditional WHILE node:
// this kernel ends every iteration (PAPER.md:1012-1015 normalisation
// ||r_k|| / ||g||) and decides whether the body runs again -- no host round
// trip per iteration.  Status codes match include/mgdtn.h.
__global__ void k_pcg_init(int* istate, double* scal, double rtol, int maxit) {
  pdl_enter();
  istate[0] = 0;
  istate[1] = 1;   // MG_MAXIT until decided
  istate[2] = maxit;
  scal[9] = rtol;
}

int launch_pcg_init(int* istate, double* scal, double rtol, int maxit, cudaStream_t st) {
  launch_ex(k_pcg_init, 1, 1, 0, true, st, istate, scal, rtol, maxit);
  return 1;
}

__global__ void k_pcg_check(const double* __restrict__ scal, int* istate, double* hist,
                            int hist_cap, cudaGraphConditionalHandle h) {
  pdl_enter();
  const double gg = scal[5];
  int cont = 0;
  if (!(gg > 0.0)) {   // g = 0 -> lambda = 0 in 0 iterations
    istate[0] = 0;
    istate[1] = 0;
    if (hist_cap > 0) hist[0] = 0.0;
  } else {
    const int it = istate[0] + 1;
    istate[0] = it;
    if (it == 1 && hist_cap > 0) hist[0] = 1.0;
    const double pAp = scal[1], rr = scal[2], rtol = scal[9];
    const double rel = sqrt(rr / gg);
    if (it < hist_cap) hist[it] = rel;
    int status = 1;               // MG_MAXIT
    if (!(pAp > 0.0) || !isfinite(rr)) status = 3;        // MG_BREAKDOWN
    else if (rel <= rtol) status = 0;                      // MG_CONVERGED
    else if (rel > 1e6) status = 2;                        // MG_DIVERGED
    else if (it < istate[2]) cont = 1;
    istate[1] = status;
  }
  cudaGraphSetConditional(h, cont);
}

int launch_pcg_check(const double* scal, int* istate, double* hist, int hist_cap,
                     cudaGraphConditionalHandle h, cudaStream_t st) {
  launch_ex(k_pcg_check, 1, 1, 0, true, st, scal, istate, hist, hist_cap, h);
  return 1;
}

// ---------------------------------------------------------------- lambda_max (Q11)
__global__ void k_pow_init(LevelDev L, double* v) {
  pdl_enter(); pow_init_body(L, v, GTID, GNT); }

int launch_pow_init(const LevelDev& L, double* v, cudaStream_t st) {
  launch_ex(k_pow_init, vec_grid(L.ndof), 256, 0, true, st, L, v);
  return 1;
}

// u = Dinv y per edge; partials[2*b] = sum u.u, partials[2*b+1] = sum u.y
__global__ void k_edge_dinv(LevelDev L, const double* __restrict__ y, double* u,
                            double* partials) {
  pdl_enter();
  const int K1 = L.k1;
  double s_uu = 0.0, s_uy = 0.0;
  for (int64_t ed = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; ed < L.nedge;
       ed += (int64_t)gridDim.x * blockDim.x) {
    if (edge_on_boundary(L.nx, L.ny, ed, L.dmask)) {
      for (int a = 0; a < K1; ++a) u[ed * K1 + a] = 0.0;
      continue;
    }
    const double* Di = L.Dinv + ed;
    for (int a = 0; a < K1; ++a) {
      double c = 0.0;
      for (int b = 0; b < K1; ++b) c = fma(Di[(a * K1 + b) * L.nedge], y[ed * K1 + b], c);
      u[ed * K1 + a] = c;
      s_uu = fma(c, c, s_uu);
      s_uy = fma(c, y[ed * K1 + a], s_uy);
    }
  }
  double a = block_sum(s_uu);
  if (threadIdx.x == 0) partials[blockIdx.x] = a;
  double b = block_sum(s_uy);
  if (threadIdx.x == 0) partials[gridDim.x + blockIdx.x] = b;
}

int launch_edge_dinv(const LevelDev& L, const double* y, double* u, double* partials,
                     int grid, cudaStream_t st) {
  launch_ex(k_edge_dinv, grid, 256, 0, true, st, L, y, u, partials);
  return 1;
}

__global__ void k_scale_by_norm(double* v, const double* __restrict__ u, int64_t n,
                                const double* __restrict__ scal, int slot) {
  pdl_enter();
  const double inv = 1.0 / sqrt(scal[slot]);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    v[i] = u[i] * inv;
}

int launch_scale_by_norm(double* v, const double* u, int64_t n, const double* scal, int slot,
                         cudaStream_t st) {
  launch_ex(k_scale_by_norm, vec_grid(n), 256, 0, true, st, v, u, n, scal, slot);
  return 1;
}

__global__ void k_lmax_finish(const double* __restrict__ scal, double safety, double ratio,
                              int nu_max, double* lam_out, double* coef) {
  pdl_enter();
  lmax_finish_body(scal[8], scal[7], safety, ratio, nu_max, lam_out, coef);
}

int launch_lmax_finish(const double* scal, double safety, double ratio, int nu_max,
                       double* lam_out, double* coef, cudaStream_t st) {
  launch_ex(k_lmax_finish, 1, 1, 0, true, st, scal, safety, ratio, nu_max, lam_out, coef);
  return 1;
}

__global__ void k_set_bj_coef(double omega, double* coef) {
  pdl_enter();
  int k = threadIdx.x;
  if (k < MAX_NU) {
    coef[2 * k] = 0.0;
    coef[2 * k + 1] = omega;
  }
}

int launch_set_bj_coef(double omega, double* coef, cudaStream_t st) {
  launch_ex(k_set_bj_coef, 1, 32, 0, true, st, omega, coef);
  return 1;
}

__global__ void k_copy(double* dst, const double* __restrict__ src, int64_t n) {
  pdl_enter();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

int launch_copy(double* dst, const double* src, int64_t n, cudaStream_t st) {
  launch_ex(k_copy, vec_grid(n), 256, 0, true, st, dst, src, n);
  return 1;
}

__global__ void k_zero(double* dst, int64_t n) {
  pdl_enter();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = 0.0;
}

int launch_zero(double* dst, int64_t n, cudaStream_t st) {
  launch_ex(k_zero, vec_grid(n), 256, 0, true, st, dst, n);
  return 1;
}

// dst = src with the dOmega (Dirichlet) entries set to 0 (inputs are ignored there)
__global__ void k_copy_masked(LevelDev L, double* dst, const double* __restrict__ src) {
  pdl_enter();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < L.ndof;
       i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = edge_on_boundary(L.nx, L.ny, (unsigned)i / (unsigned)L.k1, L.dmask) ? 0.0 : src[i];
}

int launch_copy_masked(const LevelDev& L, double* dst, const double* src, cudaStream_t st) {
  launch_ex(k_copy_masked, vec_grid(L.ndof), 256, 0, true, st, L, dst, src);
  return 1;
}

__global__ void k_add(double* dst, const double* __restrict__ src, int64_t n) {
  pdl_enter();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    dst[i] += src[i];
}

int launch_add(double* dst, const double* src, int64_t n, cudaStream_t st) {
  launch_ex(k_add, vec_grid(n), 256, 0, true, st, dst, src, n);
  return 1;
}

// z = a x + b y (host scalars; the host-driven Krylov drivers)
__global__ void k_axpby(double a, const double* __restrict__ x, double b, const double* y,
                        double* z, int64_t n) {
  pdl_enter();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    z[i] = fma(a, x[i], b * y[i]);
}

int launch_axpby(double a, const double* x, double b, const double* y, double* z, int64_t n,
                 cudaStream_t st) {
  launch_ex(k_axpby, vec_grid(n), 256, 0, true, st, a, x, b, y, z, n);
  return 1;
}

// ---------------------------------------------------------------- GMRES helpers (gmres_impl)
// modified Gram-Schmidt with device-resident coefficients: the Hessenberg column
// never round-trips through the host inside an Arnoldi step.  The arithmetic is
// the host-coefficient version's (k_axpby with b = 1, then (1/||v||) v).
__global__ void k_axpy_dev(const double* __restrict__ coef, double sign,
                           const double* __restrict__ x, double* y, int64_t n) {
  pdl_enter();
  const double a = sign * coef[0];
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    y[i] = fma(a, x[i], y[i]);
}
int launch_axpy_dev(const double* coef, double sign, const double* x, double* y, int64_t n,
                    cudaStream_t st) {
  launch_ex(k_axpy_dev, vec_grid(n), 256, 0, true, st, coef, sign, x, y, n);
  return 1;
}

// v <- v / sqrt(ss[0]) (no-op when ss[0] <= 0: the Krylov space is exhausted)
__global__ void k_scale_rsqrt(const double* __restrict__ ss, double* v, int64_t n) {
  pdl_enter();
  const double s = ss[0];
  if (!(s > 0.0)) return;
  const double a = 1.0 / sqrt(s);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    v[i] = a * v[i];
}
int launch_scale_rsqrt(const double* ss, double* v, int64_t n, cudaStream_t st) {
  launch_ex(k_scale_rsqrt, vec_grid(n), 256, 0, true, st, ss, v, n);
  return 1;
}

// x = sum_{i < m} y[i] V[i*n ..] (in order i = 0, 1, ..: the sequential axpy's rounding)
__global__ void k_combine(double* x, const double* __restrict__ V, int64_t n,
                          const double* __restrict__ y, int m) {
  pdl_enter();
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int i = 0; i < m; ++i) acc = fma(y[i], V[(int64_t)i * n + t], acc);
    x[t] = acc;
  }
}
int launch_combine(double* x, const double* V, int64_t n, const double* y, int m,
                   cudaStream_t st) {
  launch_ex(k_combine, vec_grid(n), 256, 0, true, st, x, V, n, y, m);
  return 1;
}

}  // namespace mgdtn
