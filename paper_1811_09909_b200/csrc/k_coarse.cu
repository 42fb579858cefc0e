// Coarse tail of the V-cycle (Algorithm 1) as ONE launch.
//
// Below ~64x64 macro-elements a level's work is a few microseconds of L2
// traffic, but Algorithm 1 needs ~11 dependent steps per level (smoothing
// passes, residual, local correction, restriction, prolongation), each of
// which costs a kernel launch.  k_coarse_tail runs every remaining level --
// down-sweep, the coarsest direct solve B_1 = A_1^-1 and
// the up-sweep -- inside one thread-block cluster whose CTAs are separated by
// hardware cluster barriers (barrier.cluster arrive.release / wait.acquire)
// instead of kernel boundaries.  The operations are the same device bodies as
// the standalone kernels (bodies.cuh), in the same order, so results are
// identical to the launch-per-step V-cycle up to nothing (same arithmetic,
// same summation order per output).
#include <cooperative_groups.h>

#include <cstdlib>

#include "bodies.cuh"
#include "tail.h"

namespace cg = cooperative_groups;

namespace mgdtn {

constexpr int TAIL_TPB = 512;

// Shared-memory vectors (single-CTA tail, P.smem_doubles > 0): every level
// vector of the tail (r, e, w, d and the restriction buffer) lives in shared
// memory for the whole V-cycle tail, so the ~11 dependent steps per level pay
// shared-memory instead of L2 latency on every vector access; the bodies take
// generic pointers and run unchanged.  Only the top tail level's r (and, when
// its first smoothing step was fused upstream, e and d) come in from global
// memory, and only its e goes back out.  The read-only level matrices stay in
// global memory (L1-cached).
template <bool BASIS>
__device__ __forceinline__ void k_coarse_tail_t(const TailParams& G,
                                                             const int* __restrict__ tfidx, int nfb,
                                                             double* Bt) {
  pdl_enter();
  cg::cluster_group cl = cg::this_cluster();
  const int64_t t0 = (int64_t)cl.block_rank() * TAIL_TPB + threadIdx.x;
  const int64_t nt = (int64_t)cl.num_blocks() * TAIL_TPB;
  // one CTA: a CTA barrier keeps the (small, L1-resident) level data in L1;
  // a cluster barrier's acquire invalidates it
  const bool single = cl.num_blocks() == 1;
  auto sync = [&]() {
    if (single) __syncthreads();
    else cl.sync();
  };
  extern __shared__ __align__(16) double tail_smem[];
  __shared__ TailParams SP;
  const bool use_smem = single && G.smem_doubles > 0;
  if (use_smem) {
    if (threadIdx.x == 0) {
      SP = G;
      double* q = tail_smem;
      for (int k = 0; k < G.nlev; ++k) {
        TailLevel& L = SP.lev[k];
        const int64_t n = L.d.ndof;
        L.r = q; q += n;
        L.e = q; q += n;
        L.w = q; q += n;
        L.dv = q; q += n;
        if (k < G.nlev - 1) {
          L.cbuf = q;
          q += (int64_t)(L.d.nx / 2) * (L.d.ny / 2) * 8;
        }
      }
    }
    for (int64_t i = threadIdx.x; i < G.smem_doubles; i += TAIL_TPB) tail_smem[i] = 0.0;
    __syncthreads();
    const TailLevel& T = G.lev[0];
    const TailLevel& S0 = SP.lev[0];
    if (BASIS) {   // r = unit vector on free dof tfidx[blockIdx.x]; e starts at 0
      if (threadIdx.x == 0) {
        S0.r[tfidx[blockIdx.x]] = 1.0;
        SP.first_fused = 0;
      }
    } else {
      const bool fused = G.first_fused != 0 && G.nu_pre > 0;
      for (int64_t i = threadIdx.x; i < T.d.ndof; i += TAIL_TPB) {
        S0.r[i] = T.r[i];
        if (fused) {
          S0.e[i] = T.e[i];
          S0.dv[i] = T.dv[i];
        }
      }
    }
    __syncthreads();
  }
  const TailParams& P = use_smem ? SP : G;
  const int nlev = P.nlev;
  // ---- down-sweep: pre-smoothing, residual, step 3 + restriction
  // smoothing steps of tail level li (beta = 2 doubling per coarser level); the
  // coefficient slot is clamped to MAX_NU-1 (block-Jacobi's are step-invariant)
  auto nu_of = [&](int nu, int li) { return P.nu_doubling ? nu << li : nu; };
  auto cs = [](int s) { return s < MAX_NU ? s : MAX_NU - 1; };
  for (int li = 0; li < nlev - 1; ++li) {
    const TailLevel& L = P.lev[li];
    const TailLevel& C = P.lev[li + 1];
    const int nu_pre = nu_of(P.nu_pre, li);
    int s0 = 0;
    if (nu_pre > 0) {
      const bool first_done = li == 0 ? P.first_fused != 0 : true;
      if (!first_done) {
        smooth_first_body(L.d, L.r, L.e, L.dv, t0, nt);
        sync();
      }
      s0 = 1;
    } else {
      zero_body(L.e, L.d.ndof, t0, nt);
      sync();
    }
    for (int s = s0; s < nu_pre; ++s) {
      apply_pass_body<1, AM_W0, false>(L.d, 0, L.e, L.w, nullptr, nullptr, 0, t0, nt);
      sync();
      apply_pass_body<1, AM_SMOOTH, false>(L.d, 1, L.e, L.w, L.r, L.dv, cs(s), t0, nt);
      sync();
    }
    apply_pass_body<1, AM_W0, false>(L.d, 0, L.e, L.w, nullptr, nullptr, 0, t0, nt);
    sync();
    apply_pass_body<1, AM_RESID, false>(L.d, 1, L.e, L.w, L.r, nullptr, 0, t0, nt);
    sync();
    lc_restrict_body(L.d, L.w, L.e, L.KIIinv, L.Pm, L.cbuf, 1, 1, t0, nt);
    sync();
    const int fuse = (li + 1 < nlev - 1) && nu_of(P.nu_pre, li + 1) > 0;
    restrict_edges_body(L.d, C.d, L.w, L.cbuf, C.r, fuse, C.e, C.dv, t0, nt);
    sync();
  }
  // ---- coarsest: B_1 = A_1^-1
  {
    const TailLevel& B = P.lev[nlev - 1];
    coarse_solve_body(P.fidx, P.nf, P.A1inv, B.r, B.e, t0, nt);
    sync();
  }
  // ---- up-sweep: prolongation (step 4) and post-smoothing
  for (int li = nlev - 2; li >= 0; --li) {
    const TailLevel& L = P.lev[li];
    const TailLevel& C = P.lev[li + 1];
    prolong_macro_body(L.d, C.d, C.e, L.Pm, L.e, t0, nt);
    sync();
    for (int s = 0; s < nu_of(P.nu_post, li); ++s) {
      apply_pass_body<1, AM_W0, false>(L.d, 0, L.e, L.w, nullptr, nullptr, 0, t0, nt);
      sync();
      apply_pass_body<1, AM_SMOOTH, false>(L.d, 1, L.e, L.w, L.r, L.dv, cs(s), t0, nt);
      sync();
    }
  }
  if (BASIS) {   // column blockIdx.x of B_tail
    for (int i = threadIdx.x; i < nfb; i += TAIL_TPB)
      Bt[(int64_t)i * nfb + blockIdx.x] = SP.lev[0].e[tfidx[i]];
  } else if (use_smem) {   // the top tail level's correction goes back to global memory
    const int64_t n = G.lev[0].d.ndof;
    for (int64_t i = threadIdx.x; i < n; i += TAIL_TPB) G.lev[0].e[i] = SP.lev[0].e[i];
  }
}

__global__ void __launch_bounds__(TAIL_TPB, 1) k_coarse_tail(const __grid_constant__ TailParams G) {
  k_coarse_tail_t<false>(G, nullptr, 0, nullptr);
}
__global__ void __launch_bounds__(TAIL_TPB, 1) k_tail_basis(const __grid_constant__ TailParams G,
                                                            const int* __restrict__ tfidx, int nfb,
                                                            double* Bt) {
  k_coarse_tail_t<true>(G, tfidx, nfb, Bt);
}

// e = B_tail r on the free dofs of the top tail level: one CTA per row, each
// thread a strided slice of the row (coalesced, one memory round trip), fixed
// warp-shuffle + shared-memory tree (deterministic)
constexpr int TD_THREADS = 256;
__global__ void __launch_bounds__(TD_THREADS) k_tail_dense(const int* __restrict__ tfidx, int nf,
                                                           const double* __restrict__ Bt,
                                                           const double* __restrict__ r,
                                                           double* e) {
  __shared__ double red[TD_THREADS / 32];
  pdl_enter();
  const int row = blockIdx.x;
  const double* b = Bt + (int64_t)row * nf;
  double acc = 0.0;
  for (int j = threadIdx.x; j < nf; j += TD_THREADS) acc = fma(__ldg(b + j), __ldg(r + tfidx[j]), acc);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < TD_THREADS / 32; ++w) s += red[w];
    e[tfidx[row]] = s;
  }
}

int launch_tail_dense(const int* tfidx, int nf, const double* Bt, const double* r, double* e,
                      cudaStream_t st) {
  launch_ex(k_tail_dense, nf, TD_THREADS, 0, true, st, tfidx, nf, Bt, r, e);
  return 1;
}

// B_tail with NC columns per CTA: thread group g (TAIL_TPB / NC threads) runs the tail
// V-cycle of column blockIdx.x * NC + g on its own shared-memory copy of the tail
// vectors; the groups share every CTA barrier and the (L1-resident) level matrices.
// The single-column kernel leaves 3/4 of its threads idle on the 16x16 top level
// (128 elements per colour pass); NC = 4 fills them.  Same bodies, same order per
// column as k_coarse_tail_t<true>.
template <int NC>
__global__ void __launch_bounds__(TAIL_TPB, 1)
    k_tail_basis_mc(const __grid_constant__ TailParams P, const int* __restrict__ tfidx, int nfb,
                    double* Bt) {
  extern __shared__ __align__(16) double tail_smem[];
  constexpr int NG = TAIL_TPB / NC;
  const int g = threadIdx.x / NG, tg = threadIdx.x - g * NG;
  const int col = blockIdx.x * NC + g;
  const int nlev = P.nlev;
  double* base = tail_smem + (int64_t)g * P.smem_doubles;
  // per-level vector offsets of the k_coarse_tail_t shared-memory layout
  double *vr[MAX_TAIL], *ve[MAX_TAIL], *vw[MAX_TAIL], *vd[MAX_TAIL], *vc[MAX_TAIL];
  {
    double* q = base;
    for (int k = 0; k < nlev; ++k) {
      const int64_t n = P.lev[k].d.ndof;
      vr[k] = q; q += n;
      ve[k] = q; q += n;
      vw[k] = q; q += n;
      vd[k] = q; q += n;
      vc[k] = q;
      if (k < nlev - 1) q += (int64_t)(P.lev[k].d.nx / 2) * (P.lev[k].d.ny / 2) * 8;
    }
  }
  for (int64_t i = threadIdx.x; i < (int64_t)NC * P.smem_doubles; i += TAIL_TPB) tail_smem[i] = 0.0;
  __syncthreads();
  if (tg == 0 && col < nfb) vr[0][tfidx[col]] = 1.0;
  __syncthreads();
  auto nu_of = [&](int nu, int li) { return P.nu_doubling ? nu << li : nu; };
  auto cs = [](int s) { return s < MAX_NU ? s : MAX_NU - 1; };
  for (int li = 0; li < nlev - 1; ++li) {
    const TailLevel& L = P.lev[li];
    const TailLevel& C = P.lev[li + 1];
    const int nu_pre = nu_of(P.nu_pre, li);
    int s0 = 0;
    if (nu_pre > 0) {
      if (li == 0) {   // below the top level the restriction did the first step (fuse)
        smooth_first_body(L.d, vr[li], ve[li], vd[li], tg, NG);
        __syncthreads();
      }
      s0 = 1;
    } else {
      zero_body(ve[li], L.d.ndof, tg, NG);
      __syncthreads();
    }
    for (int s = s0; s < nu_pre; ++s) {
      apply_pass_body<1, AM_W0, false>(L.d, 0, ve[li], vw[li], nullptr, nullptr, 0, tg, NG);
      __syncthreads();
      apply_pass_body<1, AM_SMOOTH, false>(L.d, 1, ve[li], vw[li], vr[li], vd[li], cs(s), tg, NG);
      __syncthreads();
    }
    apply_pass_body<1, AM_W0, false>(L.d, 0, ve[li], vw[li], nullptr, nullptr, 0, tg, NG);
    __syncthreads();
    apply_pass_body<1, AM_RESID, false>(L.d, 1, ve[li], vw[li], vr[li], nullptr, 0, tg, NG);
    __syncthreads();
    lc_restrict_body(L.d, vw[li], ve[li], L.KIIinv, L.Pm, vc[li], 1, 1, tg, NG);
    __syncthreads();
    const int fuse = (li + 1 < nlev - 1) && nu_of(P.nu_pre, li + 1) > 0;
    restrict_edges_body(L.d, C.d, vw[li], vc[li], vr[li + 1], fuse, ve[li + 1], vd[li + 1], tg, NG);
    __syncthreads();
    (void)C;
  }
  coarse_solve_body(P.fidx, P.nf, P.A1inv, vr[nlev - 1], ve[nlev - 1], tg, NG);
  __syncthreads();
  for (int li = nlev - 2; li >= 0; --li) {
    const TailLevel& L = P.lev[li];
    const TailLevel& C = P.lev[li + 1];
    prolong_macro_body(L.d, C.d, ve[li + 1], L.Pm, ve[li], tg, NG);
    __syncthreads();
    for (int s = 0; s < nu_of(P.nu_post, li); ++s) {
      apply_pass_body<1, AM_W0, false>(L.d, 0, ve[li], vw[li], nullptr, nullptr, 0, tg, NG);
      __syncthreads();
      apply_pass_body<1, AM_SMOOTH, false>(L.d, 1, ve[li], vw[li], vr[li], vd[li], cs(s), tg, NG);
      __syncthreads();
    }
  }
  if (col < nfb)
    for (int i = tg; i < nfb; i += NG) Bt[(int64_t)i * nfb + col] = ve[0][tfidx[i]];
}

int launch_tail_basis(const TailParams& P, const int* tfidx, int nf, double* Bt, cudaStream_t st) {
  const size_t smem1 = (size_t)P.smem_doubles * sizeof(double);
  static int mc = -1;   // MGDTN_TAIL_BASIS_NC: columns per CTA (1 = the single-column kernel)
  if (mc < 0) {
    const char* e = std::getenv("MGDTN_TAIL_BASIS_NC");
    mc = e ? std::atoi(e) : 4;
  }
  int nc = mc;
  while (nc > 1 && (size_t)nc * smem1 > 220 * 1024) nc /= 2;
  if (nc >= 4 || nc == 2) {
    const size_t smem = (size_t)nc * smem1;
    auto kern = nc >= 4 ? k_tail_basis_mc<4> : k_tail_basis_mc<2>;
    if (nc >= 4) nc = 4;
    static size_t attr4 = 0, attr2 = 0;
    size_t& attr = nc == 4 ? attr4 : attr2;
    if (smem > attr) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      attr = smem;
    }
    kern<<<(nf + nc - 1) / nc, TAIL_TPB, smem, st>>>(P, tfidx, nf, Bt);
    return 1;
  }
  static size_t attr = 0;
  if (smem1 > attr) {
    cudaFuncSetAttribute(k_tail_basis, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem1);
    attr = smem1;
  }
  k_tail_basis<<<nf, TAIL_TPB, smem1, st>>>(P, tfidx, nf, Bt);
  return 1;
}

// deterministic cluster-wide sum: CTA sums (fixed shuffle tree) -> part[rank]
// -> every thread adds part[0..ncta) in order
__device__ double cluster_sum(cg::cluster_group& cl, double v, double* part) {
  __shared__ double red[TAIL_TPB / 32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < TAIL_TPB / 32; ++w) s += red[w];
    part[cl.block_rank()] = s;
  }
  if (cl.num_blocks() == 1) __syncthreads();
  else cl.sync();
  double s = 0.0;
  for (unsigned b = 0; b < cl.num_blocks(); ++b) s += part[b];
  if (cl.num_blocks() == 1) __syncthreads();   // part / red reusable afterwards
  else cl.sync();
  return s;
}

// Chebyshev lambda_max of D_B^-1 A_k (Q11) for every tail level except the
// coarsest: power iteration v <- D^-1 A v (AM_DINV epilogue, in place), then
// lambda = safety * v.Av / v.Dv and the Chebyshev coefficients.  The levels'
// iterations are independent: one cluster per level, all running concurrently,
// each with its own reduction scratch part[li * cluster size ..].
__global__ void __launch_bounds__(TAIL_TPB, 1)
    k_tail_lmax(const __grid_constant__ TailParams P, int iters, double safety, double ratio,
                int nu_max, double* part_all) {
  cg::cluster_group cl = cg::this_cluster();
  const int64_t t0 = (int64_t)cl.block_rank() * TAIL_TPB + threadIdx.x;
  const int64_t nt = (int64_t)cl.num_blocks() * TAIL_TPB;
  const bool single = cl.num_blocks() == 1;
  auto sync = [&]() {
    if (single) __syncthreads();
    else cl.sync();
  };
  {
    const int li = (int)(blockIdx.x / cl.num_blocks());
    if (li >= P.nlev - 1) return;
    double* part = part_all + (int64_t)li * cl.num_blocks();
    const TailLevel& L = P.lev[li];
    pow_init_body(L.d, L.e, t0, nt);
    sync();
    double vDv_t = 0.0;
    for (int it = 0; it < iters; ++it) {
      apply_pass_body<1, AM_W0, false>(L.d, 0, L.e, L.w, nullptr, nullptr, 0, t0, nt);
      sync();
      vDv_t = apply_pass_body<1, AM_DINV, false, true>(L.d, 1, L.e, L.w, nullptr, nullptr, 0, t0, nt);
      sync();
    }
    const double vDv = cluster_sum(cl, vDv_t, part);
    apply_pass_body<1, AM_W0, false>(L.d, 0, L.e, L.w, nullptr, nullptr, 0, t0, nt);
    sync();
    const double vAv_t =
        apply_pass_body<1, AM_APPLY, false, true>(L.d, 1, L.e, L.w, nullptr, nullptr, 0, t0, nt);
    const double vAv = cluster_sum(cl, vAv_t, part);
    if (t0 == 0) lmax_finish_body(vAv, vDv, safety, ratio, nu_max, L.lam, L.d.coef);
    sync();
  }
}

int tail_cluster_size() {
  static int cs = 0;
  if (cs == 0) {
    const char* e = std::getenv("MGDTN_TAIL_CLUSTER");
    int want = e ? std::atoi(e) : 1;
    if (want != 1 && want != 2 && want != 4 && want != 8 && want != 16) want = 1;
    if (want > 8) {
      if (cudaFuncSetAttribute(k_coarse_tail, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) !=
          cudaSuccess) {
        cudaGetLastError();
        want = 8;
      }
    }
    // make sure a cluster of this size can be resident
    while (want > 1) {
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3(want);
      cfg.blockDim = dim3(TAIL_TPB);
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = want;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      int ncl = 0;
      if (cudaOccupancyMaxActiveClusters(&ncl, k_coarse_tail, &cfg) == cudaSuccess && ncl > 0) break;
      cudaGetLastError();
      want /= 2;
    }
    cs = want;
  }
  return cs;
}

int launch_tail_lmax(const TailParams& P, int iters, double safety, double ratio, int nu_max,
                     double* part, cudaStream_t st) {
  const int cs = tail_cluster_size();
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(cs * (P.nlev > 1 ? P.nlev - 1 : 1));   // one cluster per level
  cfg.blockDim = dim3(TAIL_TPB);
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cs;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  if (cs > 8) cudaFuncSetAttribute(k_tail_lmax, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchKernelEx(&cfg, k_tail_lmax, P, iters, safety, ratio, nu_max, part);
  return 1;
}

int launch_coarse_tail(const TailParams& P, cudaStream_t st) {
  const int cs = tail_cluster_size();
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(cs);
  cfg.blockDim = dim3(TAIL_TPB);
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cs;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  if (cs == 1 && P.smem_doubles > 0) {
    const size_t smem = (size_t)P.smem_doubles * sizeof(double);
    static size_t attr = 0;
    if (smem > attr) {
      cudaFuncSetAttribute(k_coarse_tail, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      attr = smem;
    }
    cfg.dynamicSmemBytes = smem;
  }
  cudaLaunchKernelEx(&cfg, k_coarse_tail, P);
  return 1;
}

}  // namespace mgdtn
