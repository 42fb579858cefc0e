// Trace-operator apply y = A_k x = sum_T G_T^T S_T G_T x (PAPER.md:305-325,
// 330-344: A is the sum of the element DtN maps) with a conflict-free
// 2-colour scatter: colour-0 elements write their edge outputs, colour-1
// elements (which share no edge with each other) read-modify-write them and
// run the fused epilogue (residual, smoothing update, dot product).
//
// Three kernels, all thread-per-element with persistent one-warp CTAs that each
// own every gridDim-th chunk of 32 same-colour elements and stream the chunks'
// element data into a shared-memory ring with cp.async.bulk (TMA bulk copy) +
// mbarrier complete_tx, independently of the thread count:
//
//   k_apply_orb  -- levels stored by D4 orbit (d4.cuh, reading R9): the finest
//                   level and its p-coarsened P1 level.  One chunk is NORB*256
//                   bytes (8.4 KB at p = 4 against 53.8 KB packed); the colour-1
//                   smoothing / power-iteration / LU-SGS passes read the
//                   centrosymmetric D_e^-1 orbits (4*NCS values per element) in
//                   the epilogue.  The matvec reads each orbit value once from
//                   shared memory (the compiler keeps it in a register for all
//                   the entries of its orbit).
//   k_apply_tma  -- packed-symmetric levels (the agglomerated P1 levels), whole
//                   chunk per stage, the next chunk's x gather issued before the
//                   current matvec.
//   k_apply_seg  -- packed levels in the modes that also stream D_e^-1, and the
//                   nonsymmetric context's full row-major maps: the chunk cut into
//                   segments circulating through a many-slot ring.
//
// All are launched with programmatic dependent launch inside the solve: the
// element-data prefetch (immutable during a solve) overlaps the previous
// kernel's tail; griddepcontrol.wait precedes every x / y access.
#include <cstdlib>
#include <cstring>

#include "bodies.cuh"
#include "d4.cuh"

namespace mgdtn {

// ---------------------------------------------------------------- PTX helpers (TMA bulk + mbarrier)
__device__ __forceinline__ uint64_t evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void tma_bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                             uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1], %2, [%3], %4;" ::"r"(smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}

// ---------------------------------------------------------------- orbit-storage apply (R9)
// Chunk records: So[((colour*nchunk + chunk)*NORB + o)*32 + lane] (orbit values of the
// 32 elements of the chunk), Dco[((chunk*4 + f)*NCS + o)*32 + lane] (D_e^-1 orbit o of
// edge f of colour-1 slot 32*chunk + lane; 0 on dOmega).  A stage holds one chunk's So
// record; the epilogue reads its Dco values straight from global memory (one 256-byte
// segment per warp and value), edge by edge, so that nothing but x and y_T is live
// across the matvec and the CTA's shared-memory footprint stays small enough for
// 8 resident CTAs per SM.
template <int P>
struct OrbCfg {
  using D = D4<P>;
  static constexpr int STAGE_BYTES = D::NORB * 256;
  static constexpr int NST = 3;                                // stages per CTA
  static constexpr int CPS = P == 4 ? 8 : P == 3 ? 10 : 12;    // CTAs per SM (regs / smem)
};

// Epilogue of one element, in two phases (the semantics of bodies.cuh epi_load /
// epi_store): every value it reads -- y, r, d and the D_e^-1 orbits of its 4 edges --
// is loaded first, so that the loads of all edges are in flight together (x / y / d may
// alias, so a load placed after a store could not be hoisted above it), then each
// edge is finished and stored.
template <int P, int MODE, bool DOT, int F0 = 0, int NF = 4>
__device__ __forceinline__ void orb_epilogue(const LevelDev& L, const int64_t ed[4],
                                             const bool bd[4], int itf, int gsm,
                                             const double* xv, const double* yv, const double* x,
                                             double* y, const double* __restrict__ r, double* d,
                                             const double* __restrict__ Dp, int step, double c1,
                                             double c2, double& dot, const PRArgs& pr,
                                             const double* din = nullptr, bool dst = true) {
  using D = D4<P>;
  constexpr int K1 = P + 1, M = 4 * K1, NCS = D::NCS;
  constexpr bool HASD = MODE == AM_SMOOTH || MODE == AM_DINV || MODE == AM_GSC;
  if (MODE == AM_W0 || MODE == AM_W0P || MODE == AM_W0U || MODE == AM_W0H) {
#pragma unroll
    for (int f = F0; f < F0 + NF; ++f) {
      double v[K1];
#pragma unroll
      for (int a = 0; a < K1; ++a) v[a] = bd[f] ? 0.0 : yv[f * K1 + a];
      st_edge<K1>(y + ed[f] * K1, v);
      // W0P / W0U: the prolonged iterate / new direction goes back to x (dOmega rows stay
      // untouched)
      if ((MODE == AM_W0P || MODE == AM_W0U || MODE == AM_W0H) && !bd[f])
        st_edge<K1>(const_cast<double*>(x) + ed[f] * K1, xv + f * K1);
    }
    return;
  }
  // an edge is "live" if its epilogue reads anything: not on dOmega, not a partition
  // interface edge (partial sum only), and (LU-SGS) of the swept colour
  bool live[4];
#pragma unroll
  for (int f = F0; f < F0 + NF; ++f)
    live[f] = !bd[f] && !((itf >> f) & 1) && (MODE != AM_GSC || ((gsm >> f) & 1));
  constexpr bool RZ = MODE == AM_SMOOTH && DOT;   // r . x_new: r kept past the load phase
  double t[M], dd[M], dv[HASD ? 4 * NCS : 1], rk[RZ ? M : 1];
#pragma unroll
  for (int f = F0; f < F0 + NF; ++f) {
    const int64_t base = ed[f] * K1;
    double yo[K1], rv[K1];
#pragma unroll
    for (int a = 0; a < K1; ++a) {
      yo[a] = rv[a] = 0.0;
      dd[f * K1 + a] = 0.0;
    }
    if (live[f]) {
      ld_edge<K1>(y + base, yo);
      if (MODE != AM_APPLY && MODE != AM_DINV) ld_edge<K1>(r + base, rv);
      // (din: d read from x, STEP_D_FROM_X)
      if (MODE == AM_SMOOTH && L.smoother == 1 && step > 0)
        ld_edge<K1>((din ? din : d) + base, dd + f * K1);
    }
#pragma unroll
    for (int a = 0; a < K1; ++a) {
      t[f * K1 + a] = (MODE == AM_APPLY || MODE == AM_DINV) ? yo[a] : rv[a] - yo[a];
      if (RZ) rk[RZ ? f * K1 + a : 0] = rv[a];
    }
    if (HASD) {
#pragma unroll
      for (int o = 0; o < NCS; ++o) dv[f * NCS + o] = live[f] ? __ldg(Dp + (f * NCS + o) * 32) : 0.0;
    }
  }
  double* xo = const_cast<double*>(x);
#pragma unroll
  for (int f = F0; f < F0 + NF; ++f) {
    const int64_t base = ed[f] * K1;
    const double* xf = xv + f * K1;
    const double* yf = yv + f * K1;
    double dnv[K1], xnv[K1];
    if (bd[f]) {   // dOmega: y = 0 (APPLY / RESID / DINV); SMOOTH / GSC leave x untouched
      if (MODE == AM_APPLY || MODE == AM_RESID || MODE == AM_DINV) {
#pragma unroll
        for (int a = 0; a < K1; ++a) y[base + a] = 0.0;
      }
      continue;
    }
    if ((itf >> f) & 1) {   // partition interface: partial sum, finished after the halo
#pragma unroll
      for (int a = 0; a < K1; ++a) y[base + a] = yf[a];
      continue;
    }
    if (!live[f]) continue;   // LU-SGS: another colour's edge
    if (MODE == AM_APPLY) {
      double v[K1];
#pragma unroll
      for (int a = 0; a < K1; ++a) {
        v[a] = t[f * K1 + a] + yf[a];
        if (DOT) dot = fma(xf[a], v[a], dot);
      }
      st_edge<K1>(y + base, v);
      continue;
    }
    if (MODE == AM_RESID) {
      double v[K1];
#pragma unroll
      for (int a = 0; a < K1; ++a) v[a] = t[f * K1 + a] - yf[a];
      st_edge<K1>(y + base, v);
      continue;
    }
    if (MODE == AM_RESPR) {   // p_restrict_body's arithmetic on this edge's residual
      double v0 = 0.0, v1 = 0.0;
#pragma unroll
      for (int a = 0; a < K1; ++a) {
        const double rs = t[f * K1 + a] - yf[a];
        v0 = fma(__ldg(pr.Jp + a * 2), rs, v0);
        v1 = fma(__ldg(pr.Jp + a * 2 + 1), rs, v1);
      }
      const int64_t E = ed[f];
      reinterpret_cast<double2*>(pr.rc)[E] = make_double2(v0, v1);
      if (pr.fuse) {
        // the coarse P1 orbit level's D_e^-1 (k_dinv_orb: its full SoA blocks hold exactly
        // these centrosymmetric orbit values, so this is p_restrict_body's arithmetic)
        using D1 = D4<1>;
        const double* Do = pr.Dso + E;
        const int64_t sd = pr.nedge;
        const double c2c = __ldg(pr.coef + 1);
        const double q00 = __ldg(Do + D1::cs(D1::pe(0, 0)) * sd), q01 = __ldg(Do + D1::cs(D1::pe(0, 1)) * sd);
        const double q10 = __ldg(Do + D1::cs(D1::pe(1, 0)) * sd), q11 = __ldg(Do + D1::cs(D1::pe(1, 1)) * sd);
        double e0 = c2c * (q00 * v0 + q01 * v1);
        double e1 = c2c * (q10 * v0 + q11 * v1);
        reinterpret_cast<double2*>(pr.ec)[E] = make_double2(e0, e1);
        if (pr.smoother == 1 && pr.dc) reinterpret_cast<double2*>(pr.dc)[E] = make_double2(e0, e1);
      }
      continue;
    }
    double res[K1];
#pragma unroll
    for (int a = 0; a < K1; ++a) {
      if (MODE == AM_DINV) {
        res[a] = t[f * K1 + a] + yf[a];   // (A x)_e
        y[base + a] = res[a];
      } else {
        res[a] = t[f * K1 + a] - yf[a];   // (r - A x)_e
      }
    }
#pragma unroll
    for (int a = 0; a < K1; ++a) {
      double cc = 0.0;
#pragma unroll
      for (int bq = 0; bq < K1; ++bq)
        cc = fma(dv[HASD ? f * NCS + D::cs(D::pe(a, bq)) : 0], res[bq], cc);
      if (MODE == AM_DINV) {
        xo[base + a] = cc;
        if (DOT) dot = fma(cc, res[a], dot);
      } else if (MODE == AM_GSC) {
        xo[base + a] = fma(c2, cc, xf[a]);
      } else {
        double dn = c2 * cc;
        if (L.smoother == 1 && step > 0) dn = fma(c1, dd[f * K1 + a], dn);
        dnv[a] = dn;
        xnv[a] = xf[a] + dn;
        if (RZ) dot = fma(rk[RZ ? f * K1 + a : 0], xnv[a], dot);   // r . x_new
      }
    }
    if (MODE == AM_SMOOTH) {
      if (L.smoother == 1 && dst) st_edge<K1>(d + base, dnv);
      st_edge<K1>(xo + base, xnv);
    }
  }
}

template <int P, int MODE, bool DOT>
__global__ void __launch_bounds__(32) k_apply_orb(const LevelDev L, int colour, const double* x,
                                                  double* y, const double* __restrict__ r,
                                                  double* d, int step,
                                                  double* __restrict__ partials, int early,
                                                  const PRArgs pr) {
  using D = D4<P>;
  using C = OrbCfg<P>;
  constexpr int K1 = P + 1, M = 4 * K1, NORB = D::NORB, NCS = D::NCS, NST = C::NST;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t bars[NST];
  double* stage_buf = reinterpret_cast<double*>(smem_raw);
  const int lane = threadIdx.x;
  const int64_t nec = L.ne >> 1;
  const int nchunk = L.nchunk;
  const double* Sbase = L.So + (int64_t)colour * nchunk * NORB * 32;
  const uint64_t pol = evict_first_policy();
  const int G = (int)gridDim.x, b = (int)blockIdx.x;
  // L.clist: this launch covers only the listed chunks (the partitioned levels' split
  // colour-1 pass: interface chunks first, then the rest while the halo is exchanged)
  const int ntot = L.clist ? L.ncl : nchunk;
  const int nmine = b < ntot ? (ntot - 1 - b) / G + 1 : 0;
  auto chunk_at = [&](int k) -> int64_t {
    const int q = b + k * G;
    return L.clist ? (int64_t)__ldg(L.clist + q) : (int64_t)q;
  };
  if (lane == 0) {
#pragma unroll
    for (int s = 0; s < NST; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  __syncwarp();
  auto issue = [&](int k) {   // lane 0: chunk of position k into stage k % NST
    const int s = k % NST;
    const int64_t c = chunk_at(k);
    mbar_expect_tx(&bars[s], (uint32_t)C::STAGE_BYTES);
    tma_bulk_g2s(stage_buf + (size_t)s * NORB * 32, Sbase + c * NORB * 32, C::STAGE_BYTES,
                 &bars[s], pol);
  };
  if (early) {   // element data are immutable during a solve: prefetch before the wait
    if (lane == 0)
      for (int k = 0; k < NST && k < nmine; ++k) issue(k);
    pdl_trigger();
    pdl_wait();
  } else {
    pdl_wait();
    if (lane == 0)
      for (int k = 0; k < NST && k < nmine; ++k) issue(k);
    pdl_trigger();
  }
  const double* din = (step & STEP_D_FROM_X) ? x : nullptr;
  const bool dst = !(step & STEP_NO_D_STORE);
  step &= STEP_D_FROM_X - 1;
  double c1 = 0.0, c2 = 0.0;
  if (MODE == AM_SMOOTH) {
    c1 = L.coef[2 * step];
    c2 = L.coef[2 * step + 1];
  } else if (MODE == AM_GSC) {
    c2 = L.coef[1];   // omega (block-Jacobi coefficients)
  }
  const double beta = MODE == AM_W0U ? pr.coef[4] : 0.0;   // (after the dependency wait)
  double dot = 0.0;
  // software pipeline: the x gather of chunk k+1 is issued before the matvec of chunk k
  // (x of a same-colour element is never written by another same-colour element)
  int64_t edn[4] = {0, 0, 0, 0};
  bool bdn[4] = {true, true, true, true};
  int itfn = 0, ein = 0, ejn = 0;
  double xn[M];
  auto prefetch = [&](int k) {
#pragma unroll
    for (int a = 0; a < M; ++a) xn[a] = 0.0;
    itfn = 0;
#pragma unroll
    for (int f = 0; f < 4; ++f) {
      edn[f] = 0;
      bdn[f] = true;
    }
    if (k >= nmine) return;
    const int64_t s = chunk_at(k) * 32 + lane;
    if (s < nec) {
      slot_elem(L.nx, colour, s, ein, ejn);
      elem_edges(L.nx, L.ny, ein, ejn, edn, bdn, L.dmask);
      itfn = elem_itf(L.nx, L.ny, ein, ejn, L.imask);
      gather_x<K1>(x, edn, bdn, xn);
      if (MODE == AM_W0P) {   // x_e + J_p ec_e (p_prolong_body's arithmetic)
#pragma unroll
        for (int f = 0; f < 4; ++f) {
          if (bdn[f]) continue;
          const double2 cc = __ldg(reinterpret_cast<const double2*>(pr.ec) + edn[f]);
#pragma unroll
          for (int a = 0; a < K1; ++a)
            xn[f * K1 + a] += fma(__ldg(pr.Jp + a * 2), cc.x, __ldg(pr.Jp + a * 2 + 1) * cc.y);
        }
      }
      if (MODE == AM_W0H) {   // x_e + (I_k ec)_e (k_prolong_edges' arithmetic)
#pragma unroll
        for (int f = 0; f < 4; ++f) {
          if (bdn[f]) continue;
          bool skip;
          const double2 v = prolong_edge_term(L.nx, L.ny, L.nx >> 1, L.ny >> 1, L.dmask, pr.ec,
                                              pr.Jp, edn[f], skip);
          if (skip) continue;
          xn[f * K1] += v.x;
          xn[f * K1 + 1] += v.y;
        }
      }
      if (MODE == AM_W0U) {   // p_e = z_e + beta p_e (k_pcg_pupdate's arithmetic)
#pragma unroll
        for (int f = 0; f < 4; ++f) {
          if (bdn[f]) continue;
          double zv[K1];
          ld_edge<K1>(pr.ec + edn[f] * K1, zv);
#pragma unroll
          for (int a = 0; a < K1; ++a) xn[f * K1 + a] = fma(beta, xn[f * K1 + a], zv[a]);
        }
      }
    }
  };
  prefetch(0);
  for (int k = 0; k < nmine; ++k) {
    const int64_t c = chunk_at(k);
    const int64_t s = c * 32 + lane;
    const bool act = s < nec;
    int64_t ed[4];
    bool bd[4];
    const int itf = itfn, ei = ein, ej = ejn;
    double xv[M], yv[M];
#pragma unroll
    for (int f = 0; f < 4; ++f) {
      ed[f] = edn[f];
      bd[f] = bdn[f];
    }
#pragma unroll
    for (int a = 0; a < M; ++a) {
      xv[a] = xn[a];
      yv[a] = 0.0;
    }
    prefetch(k + 1);
    const int st = k % NST;
    mbar_wait(&bars[st], (uint32_t)((k / NST) & 1));
    const double* Sp = stage_buf + (size_t)st * NORB * 32 + lane;
#pragma unroll
    for (int a = 0; a < M; ++a) {
#pragma unroll
      for (int bb = a; bb < M; ++bb) {
        const double sv = Sp[D::orb(D::pk(a, bb)) * 32];
        yv[a] = fma(sv, xv[bb], yv[a]);
        if (bb != a) yv[bb] = fma(sv, xv[a], yv[bb]);
      }
    }
    __syncwarp();
    if (lane == 0 && k + NST < nmine) {
      fence_proxy_async();
      issue(k + NST);
    }
    if (act) {
      int gsm = 0;
      if (MODE == AM_GSC) {
#pragma unroll
        for (int f = 0; f < 4; ++f) gsm |= (gs_colour(ei, ej, f) == step) << f;
      }
      const double* Dp = L.Dco + c * 4 * NCS * 32 + lane;
      if (MODE == AM_SMOOTH || MODE == AM_GSC) {   // two edges at a time (registers)
        orb_epilogue<P, MODE, DOT, 0, 2>(L, ed, bd, itf, gsm, xv, yv, x, y, r, d, Dp, step, c1, c2, dot, pr, din, dst);
        orb_epilogue<P, MODE, DOT, 2, 2>(L, ed, bd, itf, gsm, xv, yv, x, y, r, d, Dp, step, c1, c2, dot, pr, din, dst);
      } else {
        orb_epilogue<P, MODE, DOT>(L, ed, bd, itf, gsm, xv, yv, x, y, r, d, Dp, step, c1, c2, dot, pr);
      }
    }
  }
  if (DOT) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
    if (lane == 0) partials[blockIdx.x] = dot;
  }
}

// Two-warp variant of the colour-1 smoothing pass (k_apply_orb2): both warps of a CTA work on the
// same chunk, warp w computing the rows of edges 2w, 2w+1 (each row summed over all
// columns in increasing order, i.e. bitwise the rows of the symmetric loop above) and
// running the epilogue of those two edges.  Half the accumulators and half the epilogue
// per thread (228 instead of 255 registers; still 8 warps per SM), and the two warps'
// epilogue loads overlap each other's row sums (the one-warp pass sits at 2 warps per
// scheduler, 87 % of cycles with no eligible warp; profiles/r02_orb2.txt).
template <int P, int MODE, bool DOT, int W>
__device__ __forceinline__ void orb2_rows(const double* Sp, const double* xv, double* yv) {
  using D = D4<P>;
  constexpr int K1 = P + 1, M = 4 * K1;
#pragma unroll
  for (int a = 2 * W * K1; a < 2 * W * K1 + 2 * K1; ++a) {
    double acc = 0.0;
#pragma unroll
    for (int b = 0; b < M; ++b) {
      const int lo = a < b ? a : b, hi = a < b ? b : a;
      acc = fma(Sp[D::orb(D::pk(lo, hi)) * 32], xv[b], acc);
    }
    yv[a] = acc;
  }
}

#ifndef ORB2_MINB
#define ORB2_MINB 4
#endif
template <int P, int MODE, bool DOT>
__global__ void __launch_bounds__(64, ORB2_MINB) k_apply_orb2(const LevelDev L, int colour, const double* x,
                                                   double* y, const double* __restrict__ r,
                                                   double* d, int step,
                                                   double* __restrict__ partials, int early,
                                                   const PRArgs pr) {
  using D = D4<P>;
  using C = OrbCfg<P>;
  constexpr int K1 = P + 1, M = 4 * K1, NORB = D::NORB, NCS = D::NCS, NST = C::NST;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t bars[NST];
  __shared__ double dsum[2];
  double* stage_buf = reinterpret_cast<double*>(smem_raw);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t nec = L.ne >> 1;
  const int nchunk = L.nchunk;
  const double* Sbase = L.So + (int64_t)colour * nchunk * NORB * 32;
  const uint64_t pol = evict_first_policy();
  const int G = (int)gridDim.x, b = (int)blockIdx.x;
  const int nmine = b < nchunk ? (nchunk - 1 - b) / G + 1 : 0;
  if (threadIdx.x == 0) {
#pragma unroll
    for (int s = 0; s < NST; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  auto issue = [&](int k) {   // thread 0: chunk b + k*G into stage k % NST
    const int s = k % NST;
    const int64_t c = b + (int64_t)k * G;
    mbar_expect_tx(&bars[s], (uint32_t)C::STAGE_BYTES);
    tma_bulk_g2s(stage_buf + (size_t)s * NORB * 32, Sbase + c * NORB * 32, C::STAGE_BYTES,
                 &bars[s], pol);
  };
  if (early) {
    if (threadIdx.x == 0)
      for (int k = 0; k < NST && k < nmine; ++k) issue(k);
    pdl_trigger();
    pdl_wait();
  } else {
    pdl_wait();
    if (threadIdx.x == 0)
      for (int k = 0; k < NST && k < nmine; ++k) issue(k);
    pdl_trigger();
  }
  const double* din = (step & STEP_D_FROM_X) ? x : nullptr;
  const bool dst = !(step & STEP_NO_D_STORE);
  step &= STEP_D_FROM_X - 1;
  double c1 = 0.0, c2 = 0.0;
  if (MODE == AM_SMOOTH) {
    c1 = L.coef[2 * step];
    c2 = L.coef[2 * step + 1];
  }
  double dot = 0.0;
  int64_t edn[4] = {0, 0, 0, 0};
  bool bdn[4] = {true, true, true, true};
  double xn[M];
  auto prefetch = [&](int k) {
#pragma unroll
    for (int a = 0; a < M; ++a) xn[a] = 0.0;
#pragma unroll
    for (int f = 0; f < 4; ++f) {
      edn[f] = 0;
      bdn[f] = true;
    }
    if (k >= nmine) return;
    const int64_t s = (b + (int64_t)k * G) * 32 + lane;
    if (s < nec) {
      int ei, ej;
      slot_elem(L.nx, colour, s, ei, ej);
      elem_edges(L.nx, L.ny, ei, ej, edn, bdn, L.dmask);
      gather_x<K1>(x, edn, bdn, xn);
    }
  };
  prefetch(0);
  for (int k = 0; k < nmine; ++k) {
    const int64_t c = b + (int64_t)k * G;
    const bool act = c * 32 + lane < nec;
    int64_t ed[4];
    bool bd[4];
    double xv[M], yv[M];
#pragma unroll
    for (int f = 0; f < 4; ++f) {
      ed[f] = edn[f];
      bd[f] = bdn[f];
    }
#pragma unroll
    for (int a = 0; a < M; ++a) {
      xv[a] = xn[a];
      yv[a] = 0.0;
    }
    prefetch(k + 1);
    const int st = k % NST;
    mbar_wait(&bars[st], (uint32_t)((k / NST) & 1));
    const double* Sp = stage_buf + (size_t)st * NORB * 32 + lane;
    if (w == 0) orb2_rows<P, MODE, DOT, 0>(Sp, xv, yv);
    else orb2_rows<P, MODE, DOT, 1>(Sp, xv, yv);
    __syncthreads();   // both warps are done with stage st
    if (threadIdx.x == 0 && k + NST < nmine) {
      fence_proxy_async();
      issue(k + NST);
    }
    if (act) {
      const double* Dp = L.Dco + c * 4 * NCS * 32 + lane;
      if (w == 0)
        orb_epilogue<P, MODE, DOT, 0, 2>(L, ed, bd, 0, 0, xv, yv, x, y, r, d, Dp, step, c1, c2, dot, pr, din, dst);
      else
        orb_epilogue<P, MODE, DOT, 2, 2>(L, ed, bd, 0, 0, xv, yv, x, y, r, d, Dp, step, c1, c2, dot, pr, din, dst);
    }
  }
  if (DOT) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
    if (lane == 0) dsum[w] = dot;
    __syncthreads();
    if (threadIdx.x == 0) partials[blockIdx.x] = dsum[0] + dsum[1];
  }
}

// ---------------------------------------------------------------- whole-chunk TMA apply (packed levels)
template <int P>
struct TmaCfg {
  static constexpr int K1 = P + 1, M = 4 * K1, NPK = M * (M + 1) / 2;
  static constexpr int CHUNK_BYTES = NPK * 32 * 8;
  // stages per one-warp CTA and CTAs per SM (measured sweep, profiles/r01_tma_sweep.jsonl)
  static constexpr int NST = P == 1 ? 4 : 2;
  static constexpr int CPS = P == 4 ? 2 : P == 3 ? 3 : P == 2 ? 4 : 6;
};

template <int P, int MODE, bool DOT, int NST>
__global__ void __launch_bounds__(32) k_apply_tma(const LevelDev L, int colour, const double* x,
                                                  double* y, const double* __restrict__ r,
                                                  double* d, int step,
                                                  double* __restrict__ partials, int early) {
  using C = TmaCfg<P>;
  constexpr int K1 = C::K1, M = C::M, NPK = C::NPK;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t bars[NST];
  double* stage_buf = reinterpret_cast<double*>(smem_raw);
  const int lane = threadIdx.x;
  const int64_t nec = L.ne >> 1;
  const int nchunk = (int)((nec + 31) >> 5);
  const double* Sbase = L.S + (int64_t)colour * L.nchunk * NPK * 32;
  const uint64_t pol = evict_first_policy();
  const int G = (int)gridDim.x, b = (int)blockIdx.x;
  const int nmine = b < nchunk ? (nchunk - 1 - b) / G + 1 : 0;
  if (lane == 0) {
#pragma unroll
    for (int s = 0; s < NST; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  __syncwarp();
  auto issue = [&](int k) {   // lane 0: chunk of position k into stage k % NST
    const int s = k % NST;
    const int64_t c = (int64_t)b + (int64_t)k * G;
    mbar_expect_tx(&bars[s], C::CHUNK_BYTES);
    tma_bulk_g2s(stage_buf + (size_t)s * NPK * 32, Sbase + c * NPK * 32, C::CHUNK_BYTES, &bars[s],
                 pol);
  };
  if (early) {   // S_T is immutable during a solve: prefetch before the dependency wait
    if (lane == 0)
      for (int k = 0; k < NST && k < nmine; ++k) issue(k);
    pdl_trigger();
    pdl_wait();
  } else {
    pdl_wait();
    if (lane == 0)
      for (int k = 0; k < NST && k < nmine; ++k) issue(k);
    pdl_trigger();
  }
  double c1 = 0.0, c2 = 0.0;
  if (MODE == AM_SMOOTH) {
    c1 = L.coef[2 * step];
    c2 = L.coef[2 * step + 1];
  }
  double dot = 0.0;
  int64_t edn[4] = {0, 0, 0, 0};
  bool bdn[4] = {true, true, true, true};
  int itfn = 0;
  double xn[M];
  auto prefetch = [&](int k) {
#pragma unroll
    for (int a = 0; a < M; ++a) xn[a] = 0.0;
    itfn = 0;
#pragma unroll
    for (int f = 0; f < 4; ++f) {
      edn[f] = 0;
      bdn[f] = true;
    }
    if (k >= nmine) return;
    const int64_t s = ((int64_t)b + (int64_t)k * G) * 32 + lane;
    if (s < nec) {
      int i, j;
      slot_elem(L.nx, colour, s, i, j);
      elem_edges(L.nx, L.ny, i, j, edn, bdn, L.dmask);
      itfn = elem_itf(L.nx, L.ny, i, j, L.imask);
      gather_x<K1>(x, edn, bdn, xn);
    }
  };
  prefetch(0);
  for (int k = 0; k < nmine; ++k) {
    const int64_t s = ((int64_t)b + (int64_t)k * G) * 32 + lane;
    const bool act = s < nec;
    int64_t ed[4];
    bool bd[4];
    const int itf = itfn;
    double xv[M], yv[M], t[M], dd[M];
#pragma unroll
    for (int f = 0; f < 4; ++f) {
      ed[f] = edn[f];
      bd[f] = bdn[f];
    }
#pragma unroll
    for (int a = 0; a < M; ++a) {
      xv[a] = xn[a];
      yv[a] = 0.0;
      t[a] = 0.0;
      dd[a] = 0.0;
    }
    if (act) epi_load<K1, MODE>(L, ed, bd, y, r, d, t, dd, itf);   // needed after the matvec only
    prefetch(k + 1);
    const int st = k % NST;
    mbar_wait(&bars[st], (uint32_t)((k / NST) & 1));
    const double* Sp = stage_buf + (size_t)st * NPK * 32 + lane;
#pragma unroll
    for (int a = 0; a < M; ++a) {
#pragma unroll
      for (int bb = a; bb < M; ++bb) {
        const int kk = a * (2 * M - a + 1) / 2 + (bb - a);
        const double sv = Sp[kk * 32];
        yv[a] = fma(sv, xv[bb], yv[a]);
        if (bb != a) yv[bb] = fma(sv, xv[a], yv[bb]);
      }
    }
    __syncwarp();
    if (lane == 0 && k + NST < nmine) {
      fence_proxy_async();
      issue(k + NST);
    }
    if (act) epi_store<K1, MODE, DOT>(L, ed, bd, xv, yv, t, dd, x, y, d, step, c1, c2, dot, itf);
  }
  if (DOT) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
    if (lane == 0) partials[blockIdx.x] = dot;
  }
}

// ---------------------------------------------------------------- segmented-ring apply (packed levels)
// Same thread-per-element work as k_apply_tma, but the CTA's S_T stream (and,
// in the smoothing modes, the colour-1 elements' packed D_e^-1 blocks, see
// LevelDev::Dc) is cut into segments of SEGR rows (SEGR * 256 bytes) that
// circulate through an NSLOT-slot shared-memory ring, each slot with its own
// mbarrier.  A slot is refilled with the segment NSLOT ahead as soon as the
// warp has consumed it.
// NSYM: a nonsymmetric context's full row-major maps (npk = m*m, Eq. IPG_H); the
// epilogue then takes D_e^-1 from the SoA blocks (epi_store), not from the ring.
template <int P, bool NSYM = false>
struct SegCfg {
  static constexpr int K1 = P + 1, M = 4 * K1, NPK = NSYM ? M * M : M * (M + 1) / 2;
  static constexpr int NDE = K1 * (K1 + 1) / 2;   // packed D_e^-1 entries per edge
  static constexpr int NDI = 4 * NDE;             // per colour-1 element
  static constexpr int SEGR = NSYM ? (P == 4 ? 25 : 16)
                                   : (P == 4 ? 30 : P == 3 ? 17 : P == 2 ? 13 : 12);   // rows | NPK
  static constexpr int NSEG_S = NPK / SEGR;
  static constexpr int NSEG_D = (NDI + SEGR - 1) / SEGR;
  static constexpr int SEG_BYTES = SEGR * 32 * 8;
  static constexpr int NSLOT = NSYM ? (P == 4 ? 16 : P == 3 ? 16 : P == 2 ? 12 : 8)
                                    : (P == 4 ? 14 : P == 3 ? 16 : P == 2 ? 12 : 8);
  static constexpr int CPS = P == 4 ? 2 : P == 3 ? 3 : P == 2 ? 4 : 6;
  static_assert(NPK % SEGR == 0, "segment rows must divide the packed matrix");
};

template <int P, int MODE, bool DOT, bool NSYM = false>
__global__ void __launch_bounds__(32) k_apply_seg(const LevelDev L, int colour, const double* x,
                                                  double* y, const double* __restrict__ r,
                                                  double* d, int step,
                                                  double* __restrict__ partials, int early) {
  using C = SegCfg<P, NSYM>;
  constexpr int K1 = C::K1, M = C::M, NPK = C::NPK, SEGR = C::SEGR, NSLOT = C::NSLOT;
  constexpr bool HASD =
      !NSYM && (MODE == AM_SMOOTH || MODE == AM_DINV || MODE == AM_GSC);   // + D_e^-1
  constexpr int NS = C::NSEG_S + (HASD ? C::NSEG_D : 0);          // segments per chunk
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t bars[NSLOT];
  double* ring = reinterpret_cast<double*>(smem_raw);
  const int lane = threadIdx.x;
  const int64_t nec = L.ne >> 1;
  const int nchunk = L.nchunk;
  const double* Sbase = L.S + (int64_t)colour * nchunk * NPK * 32;
  const uint64_t pol = evict_first_policy();
  const int G = (int)gridDim.x, b = (int)blockIdx.x;
  const int nmine = b < nchunk ? (nchunk - 1 - b) / G + 1 : 0;
  const int total = nmine * NS;
  if (lane == 0) {
#pragma unroll
    for (int s = 0; s < NSLOT; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  __syncwarp();
  auto issue = [&](int g) {   // lane 0: global segment g of this CTA into slot g % NSLOT
    const int k = g / NS, q = g - k * NS;
    const int64_t c = (int64_t)b + (int64_t)k * G;
    const double* src;
    int rows = SEGR;
    if (q < C::NSEG_S) {
      src = Sbase + (c * NPK + q * SEGR) * 32;
    } else {
      const int r0 = (q - C::NSEG_S) * SEGR;
      rows = C::NDI - r0 < SEGR ? C::NDI - r0 : SEGR;
      src = L.Dc + (c * C::NDI + r0) * 32;
    }
    const int s = g % NSLOT;
    mbar_expect_tx(&bars[s], (uint32_t)(rows * 256));
    tma_bulk_g2s(ring + (size_t)s * SEGR * 32, src, (uint32_t)(rows * 256), &bars[s], pol);
  };
  auto wait_seg = [&](int g) -> const double* {
    const int s = g % NSLOT;
    mbar_wait(&bars[s], (uint32_t)((g / NSLOT) & 1));
    return ring + (size_t)s * SEGR * 32 + lane;
  };
  auto release = [&](int g) {   // the warp is done with segment g: refill its slot
    __syncwarp();
    if (lane == 0 && g + NSLOT < total) {
      fence_proxy_async();
      issue(g + NSLOT);
    }
  };
  if (early) {   // S_T / D_e^-1 are immutable during a solve: prefetch before the dependency wait
    if (lane == 0)
      for (int g = 0; g < NSLOT && g < total; ++g) issue(g);
    pdl_trigger();
    pdl_wait();
  } else {
    pdl_wait();
    if (lane == 0)
      for (int g = 0; g < NSLOT && g < total; ++g) issue(g);
    pdl_trigger();
  }
  double c1 = 0.0, c2 = 0.0;
  if (MODE == AM_SMOOTH) {
    c1 = L.coef[2 * step];
    c2 = L.coef[2 * step + 1];
  } else if (MODE == AM_GSC) {
    c2 = L.coef[1];   // omega (block-Jacobi coefficients)
  }
  double dot = 0.0;
  for (int k = 0; k < nmine; ++k) {
    const int64_t c = (int64_t)b + (int64_t)k * G;
    const int64_t s = c * 32 + lane;
    const bool act = s < nec;
    int64_t ed[4] = {0, 0, 0, 0};
    bool bd[4] = {true, true, true, true};
    int itf = 0;
    double xv[M], yv[M], t[M], dd[M];
#pragma unroll
    for (int a = 0; a < M; ++a) {
      xv[a] = 0.0;
      yv[a] = 0.0;
      t[a] = 0.0;
      dd[a] = 0.0;
    }
    int ei = 0, ej = 0;
    if (act) {   // every global read of the element, independent of the ring: overlaps the wait
      slot_elem(L.nx, colour, s, ei, ej);
      elem_edges(L.nx, L.ny, ei, ej, ed, bd, L.dmask);
      itf = elem_itf(L.nx, L.ny, ei, ej, L.imask);
      gather_x<K1>(x, ed, bd, xv);
      epi_load<K1, MODE == AM_GSC ? AM_RESID : MODE>(L, ed, bd, y, r, d, t, dd, itf);
    }
    const int g0 = k * NS;
    const double* Sp = nullptr;
    if (NSYM) {
#pragma unroll
      for (int a = 0; a < M; ++a) {
#pragma unroll
        for (int bb = 0; bb < M; ++bb) {
          const int kk = a * M + bb;
          if (kk % SEGR == 0) Sp = wait_seg(g0 + kk / SEGR);
          yv[a] = fma(Sp[(kk % SEGR) * 32], xv[bb], yv[a]);
          if (kk % SEGR == SEGR - 1) release(g0 + kk / SEGR);
        }
      }
    } else {
#pragma unroll
      for (int a = 0; a < M; ++a) {
#pragma unroll
        for (int bb = a; bb < M; ++bb) {
          const int kk = a * (2 * M - a + 1) / 2 + (bb - a);
          if (kk % SEGR == 0) Sp = wait_seg(g0 + kk / SEGR);
          const double sv = Sp[(kk % SEGR) * 32];
          yv[a] = fma(sv, xv[bb], yv[a]);
          if (bb != a) yv[bb] = fma(sv, xv[a], yv[bb]);
          if (kk % SEGR == SEGR - 1) release(g0 + kk / SEGR);
        }
      }
    }
    if (!HASD) {
      if (act) epi_store<K1, MODE, DOT>(L, ed, bd, xv, yv, t, dd, x, y, d, step, c1, c2, dot, itf);
      continue;
    } else {
      // smoothing / power-iteration epilogue with D_e^-1 from the ring (packed upper
      // triangle per edge, rows f*NDE + pk(a,b) of the colour-1 element's record)
      const double* Dp[C::NSEG_D];
#pragma unroll
      for (int q = 0; q < C::NSEG_D; ++q) Dp[q] = wait_seg(g0 + C::NSEG_S + q);
      auto dinv = [&](int f, int a, int bq) {
        const int lo = a < bq ? a : bq, hi = a < bq ? bq : a;
        const int row = f * C::NDE + lo * (2 * K1 - lo + 1) / 2 + (hi - lo);
        return Dp[row / SEGR][(row % SEGR) * 32];
      };
      if (act) {
        double* xo = const_cast<double*>(x);
#pragma unroll
        for (int f = 0; f < 4; ++f) {
          const int64_t base = ed[f] * K1;
          if (bd[f]) {
            if (MODE == AM_DINV) {
#pragma unroll
              for (int a = 0; a < K1; ++a) y[base + a] = 0.0;
            }
            continue;
          }
          if ((itf >> f) & 1) {   // partition interface: partial sum, finished after the halo
#pragma unroll
            for (int a = 0; a < K1; ++a) y[base + a] = yv[f * K1 + a];
            continue;
          }
          if (MODE == AM_GSC && gs_colour(ei, ej, f) != step) continue;   // other colours: untouched
          double res[K1];
#pragma unroll
          for (int a = 0; a < K1; ++a) {
            if (MODE == AM_DINV) {
              res[a] = t[f * K1 + a] + yv[f * K1 + a];   // (A x)_e
              y[base + a] = res[a];
            } else {
              res[a] = t[f * K1 + a] - yv[f * K1 + a];   // (r - A x)_e
            }
          }
#pragma unroll
          for (int a = 0; a < K1; ++a) {
            double cc = 0.0;
#pragma unroll
            for (int bq = 0; bq < K1; ++bq) cc = fma(dinv(f, a, bq), res[bq], cc);
            if (MODE == AM_DINV) {
              xo[base + a] = cc;
              if (DOT) dot = fma(cc, res[a], dot);
            } else if (MODE == AM_GSC) {
              xo[base + a] = fma(c2, cc, xv[f * K1 + a]);
            } else {
              double dn = c2 * cc;
              if (L.smoother == 1) {
                if (step > 0) dn = fma(c1, dd[f * K1 + a], dn);
                d[base + a] = dn;
              }
              xo[base + a] = xv[f * K1 + a] + dn;
            }
          }
        }
      }
#pragma unroll
      for (int q = 0; q < C::NSEG_D; ++q) release(g0 + C::NSEG_S + q);
    }
  }
  if (DOT) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
    if (lane == 0) partials[blockIdx.x] = dot;
  }
}

// ---------------------------------------------------------------- host side
static int num_sms() {
  static int v = 0;
  if (v == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    if (v <= 0) v = 148;
  }
  return v;
}

static constexpr bool mode_has_dinv(int mode) {
  return mode == AM_SMOOTH || mode == AM_DINV || mode == AM_GSC;
}
// Packed levels: the segmented ring for the passes that stream D_e^-1 and for every
// pass at p = 2 (config 3 solve 4.37 -> 3.98 s, profiles/r01_seg_pmask.jsonl); the
// whole-chunk kernel otherwise (config 2: 33.8 vs 37.9 us per apply).
static bool use_seg(int mode, int p) { return mode_has_dinv(mode) || p == 2; }

// resident CTAs per SM of an instantiation at its dynamic shared memory (occupancy
// calculator, cached per instantiation; also sets the smem attribute)
template <typename Kern>
static int resident(Kern k, size_t smem) {
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int nb = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k, 32, smem);
  return nb > 0 ? nb : 1;
}
template <int P, int MODE, bool DOT>
static int orb_resident() {
  static int v = 0;
  if (v == 0) v = resident(k_apply_orb<P, MODE, DOT>, (size_t)OrbCfg<P>::NST * OrbCfg<P>::STAGE_BYTES);
  return v;
}
template <int P, int MODE, bool DOT>
static int seg_resident() {
  static int v = 0;
  if (v == 0) v = resident(k_apply_seg<P, MODE, DOT>, (size_t)SegCfg<P>::NSLOT * SegCfg<P>::SEG_BYTES);
  return v;
}
template <int P, int MODE, bool DOT>
static int seg_ns_resident() {
  static int v = 0;
  using C = SegCfg<P, true>;
  if (v == 0) v = resident(k_apply_seg<P, MODE, DOT, true>, (size_t)C::NSLOT * C::SEG_BYTES);
  return v;
}
template <int P, int MODE, bool DOT>
static int tma_resident() {
  static int v = 0;
  if (v == 0)
    v = resident(k_apply_tma<P, MODE, DOT, TmaCfg<P>::NST>,
                 (size_t)TmaCfg<P>::NST * TmaCfg<P>::CHUNK_BYTES);
  return v;
}

// grid of at most gmax persistent CTAs over n chunks with the work spread evenly:
// k = ceil(n / gmax) chunks per CTA, ceil(n / k) CTAs (every CTA gets k or k-1)
static int balanced_grid(int64_t n, int64_t gmax) {
  if (n <= 0) return 1;
  if (gmax < 1) gmax = 1;
  const int64_t k = (n + gmax - 1) / gmax;
  return (int)((n + k - 1) / k);
}

// two-warp colour-1 smoothing pass (k_apply_orb2): one-GPU orbit levels at p = 4.
// Config 5: 2.32-2.62 vs 2.48-2.89 ms per pass, solve 883 vs 902 ms / 30 iterations; the
// other colour-1 modes (APPLY + DOT 1.53 vs 1.24 ms, RESPR 2.46 vs 2.14 ms) and p = 3
// (config 4: 95.9 vs 94.4 ms) measured slower (profiles/r02_orb2.txt)
static bool orb2_on(const LevelDev& L, int mode) {
  return L.orb && L.p == 4 && !L.imask && !L.clist && mode == AM_SMOOTH;
}
template <int P, int MODE, bool DOT>
static int orb2_resident() {
  static int v = 0;
  if (v == 0) v = resident(k_apply_orb2<P, MODE, DOT>, (size_t)OrbCfg<P>::NST * OrbCfg<P>::STAGE_BYTES);
  return v;
}
template <int P>
static int orb2_cps(int) {
  if constexpr (P != 4) return 1;
  else return orb2_resident<P, AM_SMOOTH, false>();
}

// CTAs per SM of a pass: the configured count, capped by what is resident
template <int P>
static int cps_of(const LevelDev& L, int mode) {
  const bool hd = mode_has_dinv(mode);
  if (orb2_on(L, mode)) return orb2_cps<P>(mode);
  if (L.orb) {
    const int res = hd ? orb_resident<P, AM_SMOOTH, false>() : orb_resident<P, AM_APPLY, true>();
    return OrbCfg<P>::CPS < res ? OrbCfg<P>::CPS : res;
  }
  if (L.ns) {
    const int res = seg_ns_resident<P, AM_W0, false>();
    return SegCfg<P, true>::CPS < res ? SegCfg<P, true>::CPS : res;
  }
  if (use_seg(mode, P)) {
    const int res = seg_resident<P, AM_W0, false>();
    return SegCfg<P>::CPS < res ? SegCfg<P>::CPS : res;
  }
  const int res = tma_resident<P, AM_W0, false>();
  return TmaCfg<P>::CPS < res ? TmaCfg<P>::CPS : res;
}

int apply_grid(const LevelDev& L) { return apply_grid_mode(L, AM_APPLY); }

int apply_grid_mode(const LevelDev& L, int mode) {
  const int64_t nchunk = L.clist ? (int64_t)L.ncl : (L.ne / 2 + 31) / 32;
  int cps;
  switch (L.p) {
    case 1: cps = cps_of<1>(L, mode); break;
    case 2: cps = cps_of<2>(L, mode); break;
    case 3: cps = cps_of<3>(L, mode); break;
    default: cps = cps_of<4>(L, mode); break;
  }
  int64_t gmax = (int64_t)num_sms() * cps;
  if (L.grid_cap > 0 && gmax > L.grid_cap) gmax = L.grid_cap;
  return balanced_grid(nchunk, gmax);
}

template <int P, int MODE, bool DOT>
static void launch_one(const LevelDev& L, int colour, const double* x, double* y, const double* r,
                       double* d, int step, double* partials, int grid, bool pdl,
                       cudaStream_t st) {
  if constexpr (MODE == AM_SMOOTH && DOT) {
    // r . x_new of a smoothing pass (the PCG's r.z in the V-cycle's last fine step): one-GPU
    // orbit levels only (k_apply_orb2 at p = 4, k_apply_orb otherwise)
    const int early = pdl ? 1 : 0;
    if (!L.orb || L.ns || colour != 1) return;
    if constexpr (P == 4) {
      if (orb2_on(L, MODE)) {
        orb2_resident<P, MODE, DOT>();
        launch_ex(k_apply_orb2<P, MODE, DOT>, grid, 64,
                  (size_t)OrbCfg<P>::NST * OrbCfg<P>::STAGE_BYTES, pdl, st, L, colour, x, y, r, d,
                  step, partials, early, PRArgs{});
        return;
      }
    }
    orb_resident<P, MODE, DOT>();
    launch_ex(k_apply_orb<P, MODE, DOT>, grid, 32, (size_t)OrbCfg<P>::NST * OrbCfg<P>::STAGE_BYTES,
              pdl, st, L, colour, x, y, r, d, step, partials, early, PRArgs{});
  } else {
  const int early = pdl ? 1 : 0;
  if (L.ns) {   // nonsymmetric context: full-storage apply (no LU-SGS / power iteration there)
    if (MODE == AM_GSC || MODE == AM_DINV) return;
    using C = SegCfg<P, true>;
    seg_ns_resident<P, MODE, DOT>();   // sets the dynamic smem attribute once
    launch_ex(k_apply_seg<P, MODE, DOT, true>, grid, 32, (size_t)C::NSLOT * C::SEG_BYTES, pdl, st,
              L, colour, x, y, r, d, step, partials, early);
    return;
  }
  if (L.orb) {
    if constexpr (P == 4 && MODE == AM_SMOOTH) {
      if (colour == 1 && orb2_on(L, MODE)) {
        orb2_resident<P, MODE, DOT>();
        launch_ex(k_apply_orb2<P, MODE, DOT>, grid, 64,
                  (size_t)OrbCfg<P>::NST * OrbCfg<P>::STAGE_BYTES, pdl, st, L, colour, x, y, r, d,
                  step, partials, early, PRArgs{});
        return;
      }
    }
    orb_resident<P, MODE, DOT>();
    launch_ex(k_apply_orb<P, MODE, DOT>, grid, 32, (size_t)OrbCfg<P>::NST * OrbCfg<P>::STAGE_BYTES,
              pdl, st, L, colour, x, y, r, d, step, partials, early, PRArgs{});
    return;
  }
  if (MODE == AM_GSC || use_seg(MODE, P)) {
    seg_resident<P, MODE, DOT>();
    launch_ex(k_apply_seg<P, MODE, DOT>, grid, 32, (size_t)SegCfg<P>::NSLOT * SegCfg<P>::SEG_BYTES,
              pdl, st, L, colour, x, y, r, d, step, partials, early);
    return;
  }
  tma_resident<P, MODE, DOT>();
  launch_ex(k_apply_tma<P, MODE, DOT, TmaCfg<P>::NST>, grid, 32,
            (size_t)TmaCfg<P>::NST * TmaCfg<P>::CHUNK_BYTES, pdl, st, L, colour, x, y, r, d, step,
            partials, early);
  }
}

template <int P>
static void dispatch_apply(const LevelDev& L, int colour, int mode, const double* x, double* y,
                           const double* r, double* d, int step, double* partials, int grid,
                           bool pdl, cudaStream_t st) {
  switch (mode) {
    case AM_W0:
      launch_one<P, AM_W0, false>(L, colour, x, y, r, d, step, partials, grid, pdl, st);
      break;
    case AM_APPLY:
      if (partials)
        launch_one<P, AM_APPLY, true>(L, colour, x, y, r, d, step, partials, grid, pdl, st);
      else
        launch_one<P, AM_APPLY, false>(L, colour, x, y, r, d, step, partials, grid, pdl, st);
      break;
    case AM_RESID:
      launch_one<P, AM_RESID, false>(L, colour, x, y, r, d, step, partials, grid, pdl, st);
      break;
    case AM_DINV:
      if (partials)
        launch_one<P, AM_DINV, true>(L, colour, x, y, r, d, step, partials, grid, pdl, st);
      else
        launch_one<P, AM_DINV, false>(L, colour, x, y, r, d, step, partials, grid, pdl, st);
      break;
    case AM_GSC:
      launch_one<P, AM_GSC, false>(L, colour, x, y, r, d, step, partials, grid, pdl, st);
      break;
    default:
      if (partials && L.orb)   // (r . x_new: the PCG's r.z in the V-cycle's last fine step)
        launch_one<P, AM_SMOOTH, true>(L, colour, x, y, r, d, step, partials, grid, pdl, st);
      else
        launch_one<P, AM_SMOOTH, false>(L, colour, x, y, r, d, step, partials, grid, pdl, st);
      break;
  }
}

int launch_apply(const LevelDev& L, int colour, int mode, const double* x, double* y,
                 const double* r, double* d, int step, double* partials, bool pdl,
                 cudaStream_t st) {
  const int grid = apply_grid_mode(L, mode);
  switch (L.p) {
    case 1: dispatch_apply<1>(L, colour, mode, x, y, r, d, step, partials, grid, pdl, st); break;
    case 2: dispatch_apply<2>(L, colour, mode, x, y, r, d, step, partials, grid, pdl, st); break;
    case 3: dispatch_apply<3>(L, colour, mode, x, y, r, d, step, partials, grid, pdl, st); break;
    default: dispatch_apply<4>(L, colour, mode, x, y, r, d, step, partials, grid, pdl, st); break;
  }
  return 1;
}

int apply2_grid(const LevelDev& L, int mode) { return apply_grid_mode(L, mode); }

template <int P>
static void launch_w0p(const LevelDev& F, const double* x, double* y, const PRArgs& pr,
                       cudaStream_t st) {
  const int grid = apply_grid_mode(F, AM_W0);
  orb_resident<P, AM_W0P, false>();
  launch_ex(k_apply_orb<P, AM_W0P, false>, grid, 32,
            (size_t)OrbCfg<P>::NST * OrbCfg<P>::STAGE_BYTES, true, st, F, 0, x, y,
            (const double*)nullptr, (double*)nullptr, 0, (double*)nullptr, 1, pr);
}

int launch_w0_prolong(const LevelDev& F, const double* Jp, const double* ec, double* x, double* y,
                      cudaStream_t st) {
  if (!F.orb || F.imask || F.p < 2) return -1;
  PRArgs pr{};
  pr.Jp = Jp;
  pr.ec = const_cast<double*>(ec);
  switch (F.p) {
    case 2: launch_w0p<2>(F, x, y, pr, st); break;
    case 3: launch_w0p<3>(F, x, y, pr, st); break;
    default: launch_w0p<4>(F, x, y, pr, st); break;
  }
  return 1;
}

template <int P>
static void launch_w0u(const LevelDev& F, const double* x, double* y, const PRArgs& pr,
                       cudaStream_t st) {
  const int grid = apply_grid_mode(F, AM_W0);
  orb_resident<P, AM_W0U, false>();
  launch_ex(k_apply_orb<P, AM_W0U, false>, grid, 32,
            (size_t)OrbCfg<P>::NST * OrbCfg<P>::STAGE_BYTES, true, st, F, 0, x, y,
            (const double*)nullptr, (double*)nullptr, 0, (double*)nullptr, 1, pr);
}

int launch_w0_hprolong(const LevelDev& F, const double* ec, const double* Pm, double* x, double* y,
                       cudaStream_t st) {
  if (!F.orb || F.imask || F.clist || F.p != 1 || (F.nx & 1) || (F.ny & 1)) return -1;
  PRArgs pr{};
  pr.ec = const_cast<double*>(ec);
  pr.Jp = Pm;
  const int grid = apply_grid_mode(F, AM_W0);
  orb_resident<1, AM_W0H, false>();
  launch_ex(k_apply_orb<1, AM_W0H, false>, grid, 32,
            (size_t)OrbCfg<1>::NST * OrbCfg<1>::STAGE_BYTES, true, st, F, 0, x, y,
            (const double*)nullptr, (double*)nullptr, 0, (double*)nullptr, 1, pr);
  return 1;
}

int launch_w0_update(const LevelDev& F, const double* z, const double* scal, double* p, double* y,
                     cudaStream_t st) {
  if (!F.orb || F.imask || F.clist) return -1;
  PRArgs pr{};
  pr.ec = const_cast<double*>(z);
  pr.coef = scal;
  switch (F.p) {
    case 1: launch_w0u<1>(F, p, y, pr, st); break;
    case 2: launch_w0u<2>(F, p, y, pr, st); break;
    case 3: launch_w0u<3>(F, p, y, pr, st); break;
    default: launch_w0u<4>(F, p, y, pr, st); break;
  }
  return 1;
}

// residual + p-restriction (AM_RESPR): colour-0 pass, then the colour-1 pass whose
// epilogue restricts each edge's residual instead of storing it
template <int P>
static void launch_respr(const LevelDev& F, const double* x, double* y, const double* r,
                         const PRArgs& pr, cudaStream_t st) {
  const int grid = apply_grid_mode(F, AM_RESPR);
  orb_resident<P, AM_RESPR, false>();
  launch_ex(k_apply_orb<P, AM_RESPR, false>, grid, 32,
            (size_t)OrbCfg<P>::NST * OrbCfg<P>::STAGE_BYTES, true, st, F, 1, x, y, r,
            (double*)nullptr, 0, (double*)nullptr, 1, pr);
}

int launch_resid_prestrict(const LevelDev& F, const LevelDev& C, const double* Jp, const double* x,
                           double* y, const double* r, double* rc, bool fuse, double* ec,
                           double* dc, cudaStream_t st) {
  if (!F.orb || F.imask || F.p < 2) return -1;
  if (!C.orb || C.p != 1 || !C.Dso) return -1;
  PRArgs pr{Jp, rc, ec, dc, C.Dso, C.coef, C.nedge, fuse ? 1 : 0, C.smoother};
  int n = launch_apply(F, 0, AM_W0, x, y, nullptr, nullptr, 0, nullptr, true, st);
  switch (F.p) {
    case 2: launch_respr<2>(F, x, y, r, pr, st); break;
    case 3: launch_respr<3>(F, x, y, r, pr, st); break;
    default: launch_respr<4>(F, x, y, r, pr, st); break;
  }
  return n + 1;
}

// ---------------------------------------------------------------- gather-form apply (small P1 levels)
// One pass, thread per edge: an interior edge's output is the sum of the two rows of
// S_T x_T that belong to it, one from each adjacent element, so no two threads write
// the same value and the colour-0 / colour-1 pair of passes (two dependent launches)
// becomes one.  Each row is accumulated in increasing column order from 0 and the two
// rows are combined in the colour-0-then-colour-1 order of the pair of passes (APPLY:
// y0 + y1; RESID / SMOOTH: (r - y0) - y1), so the results are bitwise those of the pair.
// The smoothing update is written out of place (xo): the pair updates x in place only
// because a colour-1 element owns its edges, which a per-edge thread does not.
// Packed symmetric P1 maps (the agglomerated levels), one-GPU / replicated levels
// (every domain-side edge on dOmega).
template <int MODE>
__global__ void __launch_bounds__(128) k_apply_gather(const LevelDev L, const double* x, double* y,
                                                      const double* __restrict__ r, double* d,
                                                      double* xo, int step) {
  pdl_enter();
  constexpr int K1 = 2, M = 8;
  const int nx = L.nx, ny = L.ny;
  const int64_t nh = (int64_t)nx * (ny + 1);
  double c1 = 0.0, c2 = 0.0;
  if (MODE == AM_SMOOTH) {
    c1 = L.coef[2 * step];
    c2 = L.coef[2 * step + 1];
  }
  for (int64_t E = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; E < L.nedge;
       E += (int64_t)gridDim.x * blockDim.x) {
    int i, j;
    bool bnd;
    int ti[2], tj[2], tf[2];   // the two adjacent elements and this edge's side in each
    if (E < nh) {
      j = (int)((unsigned)E / (unsigned)nx);
      i = (int)E - j * nx;
      bnd = j == 0 || j == ny;
      ti[0] = i; tj[0] = j - 1; tf[0] = 2;   // below: its top edge
      ti[1] = i; tj[1] = j;     tf[1] = 0;   // above: its bottom edge
    } else {
      const int64_t q = E - nh;
      j = (int)((unsigned)q / (unsigned)(nx + 1));
      i = (int)q - j * (nx + 1);
      bnd = i == 0 || i == nx;
      ti[0] = i - 1; tj[0] = j; tf[0] = 1;   // left: its right edge
      ti[1] = i;     tj[1] = j; tf[1] = 3;   // right: its left edge
    }
    const double2 xe = reinterpret_cast<const double2*>(x)[E];
    if (bnd) {   // dOmega: y = 0 (APPLY / RESID); the smoothed iterate keeps x
      if (MODE == AM_SMOOTH) reinterpret_cast<double2*>(xo)[E] = xe;
      else reinterpret_cast<double2*>(y)[E] = make_double2(0.0, 0.0);
      continue;
    }
    double yc[2][K1];   // [colour][row]
    int64_t s1 = 0;     // colour-1 slot and its side of this edge (D_e^-1 record)
    int f1 = 0;
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      int colour;
      int64_t s;
      elem_slot(nx, ti[k], tj[k], colour, s);
      if (colour) {
        s1 = s;
        f1 = tf[k];
      }
      int64_t ed[4];
      bool bd[4];
      elem_edges(nx, ny, ti[k], tj[k], ed, bd, L.dmask);
      double xv[M];
      gather_x<K1>(x, ed, bd, xv);
      const double* Sp = L.S + s_offset(L.nchunk, L.npk, colour, s, 0);
#pragma unroll
      for (int a = 0; a < K1; ++a) {
        const int ra = tf[k] * K1 + a;
        double acc = 0.0;
#pragma unroll
        for (int b = 0; b < M; ++b) acc = fma(__ldg(Sp + (int64_t)s_index(ra, b, M, 0) * 32), xv[b], acc);
        yc[colour][a] = acc;
      }
    }
    if (MODE == AM_APPLY) {
      reinterpret_cast<double2*>(y)[E] = make_double2(yc[0][0] + yc[1][0], yc[0][1] + yc[1][1]);
      continue;
    }
    const double2 rv = __ldg(reinterpret_cast<const double2*>(r) + E);
    const double res0 = (rv.x - yc[0][0]) - yc[1][0], res1 = (rv.y - yc[0][1]) - yc[1][1];
    if (MODE == AM_RESID) {
      reinterpret_cast<double2*>(y)[E] = make_double2(res0, res1);
      continue;
    }
    // D_e^-1 as the pair's colour-1 pass reads it: the packed upper triangle of the
    // colour-1 element's record (LevelDev::Dc; rows f*3 + {00, 01, 11})
    const double* Dr = L.Dc + ((s1 >> 5) * 12 + f1 * 3) * 32 + (s1 & 31);
    const double D00 = __ldg(Dr), D01 = __ldg(Dr + 32), D11 = __ldg(Dr + 64);
    double dd[2] = {0.0, 0.0};
    if (L.smoother == 1 && step > 0) {
      const double2 t = reinterpret_cast<const double2*>(d)[E];
      dd[0] = t.x;
      dd[1] = t.y;
    }
    double dn[2];
    dn[0] = c2 * fma(D01, res1, fma(D00, res0, 0.0));
    dn[1] = c2 * fma(D11, res1, fma(D01, res0, 0.0));
    if (L.smoother == 1 && step > 0) {
      dn[0] = fma(c1, dd[0], dn[0]);
      dn[1] = fma(c1, dd[1], dn[1]);
    }
    if (L.smoother == 1) reinterpret_cast<double2*>(d)[E] = make_double2(dn[0], dn[1]);
    reinterpret_cast<double2*>(xo)[E] = make_double2(xe.x + dn[0], xe.y + dn[1]);
  }
}

bool gather_level(const LevelDev& L) {
  return L.gather && !L.orb && !L.ns && L.p == 1 && L.imask == 0 && L.dmask == 15 && L.Dc;
}

int launch_apply_gather(const LevelDev& L, int mode, const double* x, double* y, const double* r,
                        double* d, double* xo, int step, cudaStream_t st) {
  const int64_t nb = (L.nedge + 127) / 128, cap = (int64_t)num_sms() * 16;
  const int g = (int)(nb < 1 ? 1 : nb < cap ? nb : cap);
  switch (mode) {
    case AM_APPLY: launch_ex(k_apply_gather<AM_APPLY>, g, 128, 0, true, st, L, x, y, r, d, xo, step); break;
    case AM_RESID: launch_ex(k_apply_gather<AM_RESID>, g, 128, 0, true, st, L, x, y, r, d, xo, step); break;
    case AM_SMOOTH: launch_ex(k_apply_gather<AM_SMOOTH>, g, 128, 0, true, st, L, x, y, r, d, xo, step); break;
    default: return -1;
  }
  return 1;
}

int launch_apply2(const LevelDev& L, int mode, const double* x, double* y, const double* r,
                  double* d, int step, double* partials, bool pdl, cudaStream_t st) {
  int n = launch_apply(L, 0, AM_W0, x, y, nullptr, nullptr, 0, nullptr, pdl, st);
  return n + launch_apply(L, 1, mode, x, y, r, d, step, partials, pdl, st);
}

}  // namespace mgdtn
