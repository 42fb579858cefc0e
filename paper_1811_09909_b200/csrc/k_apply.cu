// Trace-operator apply y = A_k x = sum_T G_T^T S_T G_T x (PAPER.md:305-325,
// 330-344: A is the sum of the element DtN maps) with a conflict-free
// 2-colour scatter: colour-0 elements write their edge outputs, colour-1
// elements (which share no edge with each other) read-modify-write them and
// run the fused epilogue (residual, smoothing update, dot product).
//
// HBM-bound: 8*npk bytes of packed S_T per element against 2*m*m flops.
//
// k_apply_tma (default): persistent one-warp CTAs.  Each CTA owns every
// gridDim-th chunk of 32 same-colour elements and streams the chunks' packed
// S_T (npk*256 contiguous bytes, kernels.cuh layout) into an NST-stage
// shared-memory ring with cp.async.bulk (TMA bulk copy) + mbarrier
// complete_tx, so that NST chunks (~100 KB per CTA, ~200 KB per SM) are in
// flight independently of the thread count.  Lane l computes element
// 32*chunk + l from shared memory (conflict-free: entry kk of the 32 lanes is
// 256 contiguous bytes).  Launched with programmatic dependent launch inside
// the solve: the S_T prefetch (S_T is immutable during a solve) overlaps the
// previous kernel's tail; griddepcontrol.wait precedes every x / y access.
//
// k_apply_ldg: the first version (thread per element, direct L1-bypassing
// loads), kept for A/B measurement (MGDTN_APPLY=ldg).
#include <cstdlib>
#include <cstring>
#include <type_traits>

#include "bodies.cuh"

namespace mgdtn {

__device__ __forceinline__ uint64_t evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

// L2 policy of a level's operator stream: fraction `keep` evict_last (stays resident
// across the many applies of a solve), the rest evict_first
__device__ __forceinline__ uint64_t stream_policy(float keep) {
  if (!(keep > 0.0f)) return evict_first_policy();
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.L2::evict_first.b64 %0, %1;"
               : "=l"(pol)
               : "f"(keep > 1.0f ? 1.0f : keep));
  return pol;
}

__device__ __forceinline__ double ld_stream(const double* p, uint64_t pol) {
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;"
               : "=d"(v)
               : "l"(p), "l"(pol));
  return v;
}

// ---------------------------------------------------------------- PTX helpers (TMA bulk + mbarrier + PDL)
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

// ---------------------------------------------------------------- TMA-pipelined apply
template <int P>
struct TmaCfg {
  static constexpr int K1 = P + 1, M = 4 * K1, NPK = M * (M + 1) / 2;
  static constexpr int CHUNK_BYTES = NPK * 32 * 8;
  // stages per one-warp CTA and CTAs per SM (measured sweep, profiles/r01_tma_sweep.jsonl):
  // more resident warps hide the x-gather / y read-modify-write latency better
  // than deeper per-CTA rings
  static constexpr int NST = P == 4 ? 2 : P == 3 ? 2 : P == 2 ? 2 : 4;
  static constexpr int CPS = P == 4 ? 2 : P == 3 ? 3 : P == 2 ? 4 : 6;
};

// tick != nullptr: dynamic chunk scheduling (MGDTN_GRID=dyn).  The CTA's first NST
// chunks are static (blockIdx.x + k*gridDim.x, prefetched before the PDL wait); every
// later chunk is a ticket tick[0]++ (+ NST*gridDim.x) taken when its stage frees up, so
// the SMs that stream faster take more chunks.  Tickets are taken only after the PDL
// wait (the previous launch on this level / colour, which used the same counter, has
// then completed), and the last CTA to exit resets the counter for the next launch.
template <int P, int MODE, bool DOT, int NST, bool XPF = true>
__global__ void __launch_bounds__(32) k_apply_tma(const LevelDev L, int colour, const double* x,
                                                  double* y, const double* __restrict__ r,
                                                  double* d, int step,
                                                  double* __restrict__ partials, int early,
                                                  unsigned* tick) {
  using C = TmaCfg<P>;
  constexpr int K1 = C::K1, M = C::M, NPK = C::NPK;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t bars[NST];
  __shared__ int cid[NST];   // chunk in each stage (-1: none)
  double* stage_buf = reinterpret_cast<double*>(smem_raw);
  const int lane = threadIdx.x;
  const int64_t nec = L.ne >> 1;
  const int nchunk = (int)((nec + 31) >> 5);
  const double* Sbase = L.S + (int64_t)colour * L.nchunk * NPK * 32;
  const uint64_t pol = stream_policy(colour == 0 && L.l2keep0 ? 1.0f : L.l2keep);
  // static chunks of this CTA: c_k = blockIdx.x + k * gridDim.x
  const int nmine_static =
      (int)blockIdx.x < nchunk ? (nchunk - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
  const int nmine = tick ? 0x7fffffff : nmine_static;   // dynamic: until a ticket runs out
  if (lane == 0) {
#pragma unroll
    for (int s = 0; s < NST; ++s) {
      mbar_init(&bars[s], 1);
      cid[s] = s < nmine_static ? (int)blockIdx.x + s * (int)gridDim.x : -1;
    }
    fence_mbar_init();
  }
  __syncwarp();
  auto chunk_of = [&](int k) -> int {   // chunk processed at position k (-1: done)
    if (tick) return cid[k % NST];
    return k < nmine_static ? (int)blockIdx.x + k * (int)gridDim.x : -1;
  };
  auto issue = [&](int k) {   // lane 0: chunk of position k into stage k % NST
    const int s = k % NST;
    int c;
    if (tick && k >= NST) {
      const unsigned t = atomicAdd(tick, 1u) + (unsigned)(NST * gridDim.x);
      c = t < (unsigned)nchunk ? (int)t : -1;
      cid[s] = c;
    } else {
      c = chunk_of(k);
    }
    if (c < 0) return;
    mbar_expect_tx(&bars[s], C::CHUNK_BYTES);
    tma_bulk_g2s(stage_buf + (size_t)s * NPK * 32, Sbase + (int64_t)c * NPK * 32, C::CHUNK_BYTES,
                 &bars[s], pol);
  };
  if (early) {   // S_T is immutable during a solve: prefetch before the dependency wait
    if (lane == 0)
      for (int k = 0; k < NST && k < nmine_static; ++k) issue(k);
    pdl_trigger();
    pdl_wait();
  } else {
    pdl_wait();
    if (lane == 0)
      for (int k = 0; k < NST && k < nmine_static; ++k) issue(k);
    pdl_trigger();
  }
  double c1 = 0.0, c2 = 0.0;
  if (MODE == AM_SMOOTH) {
    c1 = L.coef[2 * step];
    c2 = L.coef[2 * step + 1];
  }
  double dot = 0.0;
  // software pipeline over the CTA's chunks: the x gather of chunk k+1 is issued
  // before the matvec of chunk k (x of a same-colour element is never written by
  // another same-colour element, so the early read is exact in every mode)
  int64_t edn[4] = {0, 0, 0, 0};
  bool bdn[4] = {true, true, true, true};
  int itfn = 0;
  double xn[M];
  auto prefetch = [&](int k) {
#pragma unroll
    for (int a = 0; a < M; ++a) xn[a] = 0.0;
    const int ck = chunk_of(k);
    const int64_t s = (int64_t)ck * 32 + lane;
    if (ck >= 0 && s < nec) {
      int i, j;
      slot_elem(L.nx, colour, s, i, j);
      elem_edges(L.nx, L.ny, i, j, edn, bdn, L.dmask);
      itfn = elem_itf(L.nx, L.ny, i, j, L.imask);
      gather_x<K1>(x, edn, bdn, xn);
    } else {
      itfn = 0;
#pragma unroll
      for (int f = 0; f < 4; ++f) {
        edn[f] = 0;
        bdn[f] = true;
      }
    }
  };
  prefetch(0);
  for (int k = 0; k < nmine; ++k) {
    const int c = chunk_of(k);
    if (c < 0) break;
    const int64_t s = (int64_t)c * 32 + lane;
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
    if (L.probe == 1) {   // measurement probe: the S_T stream alone (no gather, math, stores)
      const int st = k % NST;
      mbar_wait(&bars[st], (uint32_t)((k / NST) & 1));
      __syncwarp();
      if (lane == 0 && k + NST < nmine) {
        fence_proxy_async();
        issue(k + NST);
      }
      __syncwarp();
      continue;
    }
    if (act) epi_load<K1, MODE>(L, ed, bd, y, r, d, t, dd, itf);   // needed after the matvec only
    if (XPF) prefetch(k + 1);
    const int st = k % NST;
    mbar_wait(&bars[st], (uint32_t)((k / NST) & 1));
    const double* Sp = stage_buf + (size_t)st * NPK * 32 + lane;
#pragma unroll
    for (int a = 0; a < M; ++a) {
#pragma unroll
      for (int b = a; b < M; ++b) {
        const int kk = a * (2 * M - a + 1) / 2 + (b - a);
        const double sv = Sp[kk * 32];
        yv[a] = fma(sv, xv[b], yv[a]);
        if (b != a) yv[b] = fma(sv, xv[a], yv[b]);
      }
    }
    __syncwarp();
    if (lane == 0 && k + NST < nmine) {
      fence_proxy_async();
      issue(k + NST);
    }
    __syncwarp();   // cid of position k + NST visible to the prefetch below
    if (act) epi_store<K1, MODE, DOT>(L, ed, bd, xv, yv, t, dd, x, y, d, step, c1, c2, dot, itf);
    if (!XPF) prefetch(k + 1);
  }
  if (DOT) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
    if (lane == 0) partials[blockIdx.x] = dot;
  }
  if (tick && lane == 0) {   // last CTA out resets the ticket counter for the next launch
    __threadfence();
    if (atomicAdd(tick + 1, 1u) == gridDim.x - 1u) {
      atomicExch(tick, 0u);
      atomicExch(tick + 1, 0u);
    }
  }
}

// ---------------------------------------------------------------- two-warp TMA apply
// k_apply_tma with TWO warps per CTA sharing the chunk ring: warp w computes the
// packed rows a in [A0*w, A0 + w*(M-A0)) of every element of the chunk (A0 splits the
// npk entries in halves), so each warp issues half the FMA chain; the partial
// sums of the other warp's two edges go through shared memory, and warp w runs
// the epilogue of edges {2w, 2w+1}.  Same math, same per-entry FMA order within
// each row; the two halves are added once (y = y_w0 + y_w1).
template <int M>
struct RowSplit {   // smallest A0 with sum_{a<A0} (M - a) >= npk / 2
  static constexpr int NPK = M * (M + 1) / 2;
  static constexpr int calc() {
    int acc = 0;
    for (int a = 0; a < M; ++a) {
      acc += M - a;
      if (2 * acc >= NPK) return a + 1;
    }
    return M;
  }
  static constexpr int A0 = calc();
};

template <int P, int MODE, bool DOT, int NST>
__global__ void __launch_bounds__(64) k_apply_tma2(const LevelDev L, int colour, const double* x,
                                                   double* y, const double* __restrict__ r,
                                                   double* d, int step,
                                                   double* __restrict__ partials, int early) {
  using C = TmaCfg<P>;
  constexpr int K1 = C::K1, M = C::M, NPK = C::NPK, A0 = RowSplit<M>::A0, HK = 2 * K1;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t bars[NST];
  __shared__ double xch[2][K1][32];   // one edge's partial sums handed to the other warp
  __shared__ double dred[2];
  double* stage_buf = reinterpret_cast<double*>(smem_raw);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t nec = L.ne >> 1;
  const int nchunk = (int)((nec + 31) >> 5);
  const double* Sbase = L.S + (int64_t)colour * L.nchunk * NPK * 32;
  const uint64_t pol = stream_policy(colour == 0 && L.l2keep0 ? 1.0f : L.l2keep);
  const int nmine = (int)blockIdx.x < nchunk ? (nchunk - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
  if (threadIdx.x == 0) {
#pragma unroll
    for (int s = 0; s < NST; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  auto issue = [&](int k) {
    const int c = (int)blockIdx.x + k * (int)gridDim.x;
    const int s = k % NST;
    mbar_expect_tx(&bars[s], C::CHUNK_BYTES);
    tma_bulk_g2s(stage_buf + (size_t)s * NPK * 32, Sbase + (int64_t)c * NPK * 32, C::CHUNK_BYTES,
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
  double dot = 0.0;
  for (int k = 0; k < nmine; ++k) {
    const int c = (int)blockIdx.x + k * (int)gridDim.x;
    const int64_t s = (int64_t)c * 32 + lane;
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
    if (act) {
      int i, j;
      slot_elem(L.nx, colour, s, i, j);
      elem_edges(L.nx, L.ny, i, j, ed, bd, L.dmask);
      itf = elem_itf(L.nx, L.ny, i, j, L.imask);
      gather_x<K1>(x, ed, bd, xv);
      if (wid == 0) epi_load<K1, MODE, true, 3>(L, ed, bd, y, r, d, t, dd, itf);
      else epi_load<K1, MODE, true, 12>(L, ed, bd, y, r, d, t, dd, itf);
    }
    const int st = k % NST;
    mbar_wait(&bars[st], (uint32_t)((k / NST) & 1));
    const double* Sp = stage_buf + (size_t)st * NPK * 32 + lane;
    if (wid == 0) {
#pragma unroll
      for (int a = 0; a < A0; ++a) {
#pragma unroll
        for (int b = a; b < M; ++b) {
          const int kk = a * (2 * M - a + 1) / 2 + (b - a);
          const double sv = Sp[kk * 32];
          yv[a] = fma(sv, xv[b], yv[a]);
          if (b != a) yv[b] = fma(sv, xv[a], yv[b]);
        }
      }
    } else {
#pragma unroll
      for (int a = A0; a < M; ++a) {
#pragma unroll
        for (int b = a; b < M; ++b) {
          const int kk = a * (2 * M - a + 1) / 2 + (b - a);
          const double sv = Sp[kk * 32];
          yv[a] = fma(sv, xv[b], yv[a]);
          if (b != a) yv[b] = fma(sv, xv[a], yv[b]);
        }
      }
    }
    // hand the other warp's two edges over, one edge per round (warp 0 owns edges
    // 0,1 = outputs [0,HK)); the first barrier also frees the stage for the refill
#pragma unroll
    for (int hr = 0; hr < 2; ++hr) {
#pragma unroll
      for (int q = 0; q < K1; ++q) xch[wid][q][lane] = yv[(wid == 0 ? HK : 0) + hr * K1 + q];
      __syncthreads();
      if (hr == 0 && threadIdx.x == 0 && k + NST < nmine) {
        fence_proxy_async();
        issue(k + NST);
      }
#pragma unroll
      for (int q = 0; q < K1; ++q) {
        const int o = (wid == 0 ? 0 : HK) + hr * K1 + q;
        yv[o] = yv[o] + xch[wid ^ 1][q][lane];
      }
      __syncthreads();
    }
    if (act) {
      if (wid == 0) epi_store<K1, MODE, DOT, 3>(L, ed, bd, xv, yv, t, dd, x, y, d, step, 0.0, 0.0, dot, itf);
      else epi_store<K1, MODE, DOT, 12>(L, ed, bd, xv, yv, t, dd, x, y, d, step, 0.0, 0.0, dot, itf);
    }
  }
  if (DOT) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
    if (lane == 0) dred[wid] = dot;
    __syncthreads();
    if (threadIdx.x == 0) partials[blockIdx.x] = dred[0] + dred[1];
  }
}

// ---------------------------------------------------------------- segmented-ring apply (default)
// Same thread-per-element work as k_apply_tma, but the CTA's S_T stream (and,
// in the smoothing modes, the colour-1 elements' packed D_e^-1 blocks, see
// LevelDev::Dc) is cut into segments of SEGR rows (SEGR * 256 bytes) that
// circulate through an NSLOT-slot shared-memory ring, each slot with its own
// mbarrier.  A slot is refilled with the segment NSLOT ahead as soon as the
// warp has consumed it, so ~NSLOT-1 segments (~100 KB per CTA, ~200 KB per SM)
// are always in flight -- twice the whole-chunk double buffer of k_apply_tma,
// whose in-flight bytes drop to one chunk while the other is being consumed
// (ncu: k_apply_tma at config 2 stalls on the stage wait and reaches 44% of
// DRAM peak).
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
                                    : (P == 4 ? 14 : P == 3 ? 16 : P == 2 ? 16 : 12);
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
  const uint64_t pol = stream_policy(colour == 0 && L.l2keep0 ? 1.0f : L.l2keep);
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

// ---------------------------------------------------------------- fused two-colour apply
// One launch for the whole apply.  Each CTA streams its colour-0 chunks, then
// its colour-1 chunks, through ONE TMA ring, so the colour-1 S_T prefetch
// overlaps the colour-0 tail and the launch boundary between the passes
// disappears.  A colour-1 element reads y on its 4 edges, which its colour-0
// neighbours wrote, and (AM_SMOOTH / AM_DINV) overwrites x there, which they
// read: the passes are separated by one grid barrier (arrive: release atomic;
// wait: acquire spin on the generation L.sync[0]; the last CTA to arrive resets
// the count L.sync[1] and advances the generation).  MGDTN_FUSED=2 selects the
// per-chunk-flag variant instead (colour-1 chunk [s0,s1] waits only for the
// colour-0 chunks holding [s0-1,s1+1] u [s0-nx/2,s1-nx/2] u [s0+nx/2,s1+nx/2]):
// it overlaps the passes but adds two dependent L2 round trips to every
// colour-1 chunk, which measured slower (profiles/r01_fused_probe.jsonl).
// Forward progress: CTAs wait only after all of their own colour-0 chunks are
// done, colour-0 work never waits, and the grid never exceeds one resident
// wave (launch_fused_t clamps it with the occupancy calculator).  The
// generation is read after griddepcontrol.wait, i.e. after the previous launch
// on this level has completed.
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u32(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void wait_range(const unsigned* fl, int64_t slo, int64_t shi,
                                           int64_t nec, unsigned gen, int lane) {
  if (slo < 0) slo = 0;
  if (shi > nec - 1) shi = nec - 1;
  if (shi < slo) return;
  for (int64_t q = (slo >> 5) + lane; q <= (shi >> 5); q += 32) {
    while (ld_acquire_u32(fl + q) != gen) __nanosleep(32);
  }
}

// pre-wait epilogue loads of a colour-1 element (no colour-0 output involved):
// RESID / SMOOTH: t = r; SMOOTH (Chebyshev): dd = d
template <int K1, int MODE>
__device__ __forceinline__ void epi_load_r(const LevelDev& L, const int64_t ed[4], const bool bd[4],
                                           const double* __restrict__ r, const double* d,
                                           double* t, double* dd) {
#pragma unroll
  for (int f = 0; f < 4; ++f) {
    const int64_t base = ed[f] * K1;
#pragma unroll
    for (int a = 0; a < K1; ++a) {
      if (MODE == AM_RESID || MODE == AM_SMOOTH) t[f * K1 + a] = bd[f] ? 0.0 : __ldg(r + base + a);
      if (MODE == AM_SMOOTH) dd[f * K1 + a] = (bd[f] || L.smoother != 1) ? 0.0 : d[base + a];
    }
  }
}
// post-wait: the colour-0 partial sums (APPLY / DINV: t = y; RESID / SMOOTH: t = r - y)
template <int K1, int MODE>
__device__ __forceinline__ void epi_load_y(const int64_t ed[4], const bool bd[4], const double* y,
                                           double* t) {
#pragma unroll
  for (int f = 0; f < 4; ++f) {
    const int64_t base = ed[f] * K1;
#pragma unroll
    for (int a = 0; a < K1; ++a) {
      const double yo = bd[f] ? 0.0 : y[base + a];
      if (MODE == AM_APPLY || MODE == AM_DINV) t[f * K1 + a] = yo;
      else t[f * K1 + a] -= yo;
    }
  }
}

template <int P, int MODE, bool DOT, int NST, bool FLAGS>
__global__ void __launch_bounds__(32) k_apply_fused(const LevelDev L, const double* x, double* y,
                                                    const double* __restrict__ r, double* d,
                                                    int step, double* __restrict__ partials,
                                                    int early) {
  using C = TmaCfg<P>;
  constexpr int K1 = C::K1, M = C::M, NPK = C::NPK;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t bars[NST];
  double* stage_buf = reinterpret_cast<double*>(smem_raw);
  const int lane = threadIdx.x;
  const int64_t nec = L.ne >> 1;
  const int nchunk = L.nchunk;
  const int64_t nxh = L.nx >> 1;
  const uint64_t pol = stream_policy(L.l2keep);
  const int G = (int)gridDim.x, b = (int)blockIdx.x;
  const int nmine0 = b < nchunk ? (nchunk - 1 - b) / G + 1 : 0;   // same count for colour 1
  const int nitems = 2 * nmine0;
  unsigned* flags = L.sync + 2;   // FLAGS variant: per colour-0 chunk
  if (lane == 0) {
#pragma unroll
    for (int s = 0; s < NST; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  __syncwarp();
  auto issue = [&](int k) {   // lane 0: item k of this CTA into stage k % NST
    const int colour = k < nmine0 ? 0 : 1;
    const int c = b + (k - colour * nmine0) * G;
    const int s = k % NST;
    mbar_expect_tx(&bars[s], C::CHUNK_BYTES);
    tma_bulk_g2s(stage_buf + (size_t)s * NPK * 32,
                 L.S + ((int64_t)colour * nchunk + c) * NPK * 32, C::CHUNK_BYTES, &bars[s], pol);
  };
  if (early) {   // S_T is immutable during a solve: prefetch before the dependency wait
    if (lane == 0)
      for (int k = 0; k < NST && k < nitems; ++k) issue(k);
    pdl_trigger();
    pdl_wait();
  } else {
    pdl_wait();
    if (lane == 0)
      for (int k = 0; k < NST && k < nitems; ++k) issue(k);
    pdl_trigger();
  }
  const unsigned gen = *reinterpret_cast<volatile unsigned*>(L.sync) + 1u;
  double c1 = 0.0, c2 = 0.0;
  if (MODE == AM_SMOOTH) {
    c1 = L.coef[2 * step];
    c2 = L.coef[2 * step + 1];
  }
  double dot = 0.0;
  for (int k = 0; k < nitems; ++k) {
    const int colour = k < nmine0 ? 0 : 1;
    const int c = b + (k - colour * nmine0) * G;
    const int64_t s = (int64_t)c * 32 + lane;
    const bool act = s < nec;
    int64_t ed[4] = {0, 0, 0, 0};
    bool bd[4] = {true, true, true, true};
    double xv[M], yv[M], t[M], dd[M];
#pragma unroll
    for (int a = 0; a < M; ++a) {
      xv[a] = 0.0;
      yv[a] = 0.0;
      t[a] = 0.0;
      dd[a] = 0.0;
    }
    if (!FLAGS && k == nmine0) {   // grid barrier between the colour passes
      __syncwarp();
      if (lane == 0) {   // one poller per CTA (not 32): the flag's L2 line stays uncontended
        __threadfence();
        if (atomicAdd(L.sync + 1, 1u) == (unsigned)G - 1u) {
          L.sync[1] = 0u;
          __threadfence();
          st_release_u32(L.sync, gen);
        }
        while (ld_acquire_u32(L.sync) != gen) __nanosleep(100);
      }
      __syncwarp();
    }
    if (L.probe == 1) {   // measurement probe: the S_T stream alone
      const int st = k % NST;
      mbar_wait(&bars[st], (uint32_t)((k / NST) & 1));
      __syncwarp();
      if (lane == 0 && k + NST < nitems) {
        fence_proxy_async();
        issue(k + NST);
      }
      continue;
    }
    if (act) {
      int i, j;
      slot_elem(L.nx, colour, s, i, j);
      elem_edges(L.nx, L.ny, i, j, ed, bd, L.dmask);
      gather_x<K1>(x, ed, bd, xv);
      if (colour == 1) {
        if (FLAGS) epi_load_r<K1, MODE>(L, ed, bd, r, d, t, dd);
        else epi_load<K1, MODE>(L, ed, bd, y, r, d, t, dd);
      }
    }
    if (FLAGS && colour == 1) {
      const int64_t s0 = (int64_t)c * 32, s1 = s0 + 31;
      wait_range(flags, s0 - 1, s1 + 1, nec, gen, lane);
      wait_range(flags, s0 - nxh, s1 - nxh, nec, gen, lane);
      wait_range(flags, s0 + nxh, s1 + nxh, nec, gen, lane);
      __syncwarp();
      if (act) epi_load_y<K1, MODE>(ed, bd, y, t);
    }
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
    if (lane == 0 && k + NST < nitems) {
      fence_proxy_async();
      issue(k + NST);
    }
    if (colour == 0) {
      if (act) epi_store<K1, AM_W0, false>(L, ed, bd, xv, yv, t, dd, x, y, d, step, c1, c2, dot);
      if (FLAGS) {
        __syncwarp();
        if (lane == 0) {
          __threadfence();
          st_release_u32(flags + c, gen);
        }
      }
    } else if (act) {
      epi_store<K1, MODE, DOT>(L, ed, bd, xv, yv, t, dd, x, y, d, step, c1, c2, dot);
    }
  }
  if (DOT) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
    if (lane == 0) partials[blockIdx.x] = dot;
  }
  if (FLAGS && lane == 0) {   // the last CTA out advances the generation for the next launch
    __threadfence();
    if (atomicAdd(L.sync + 1, 1u) == (unsigned)G - 1u) {
      L.sync[1] = 0u;
      __threadfence();
      *reinterpret_cast<volatile unsigned*>(L.sync) = gen;
    }
  }
}

// ---------------------------------------------------------------- direct-load apply
// A/B variant of the packed apply, and THE apply of a nonsymmetric context (NS:
// full row-major S_T, Eq. IPG_H with s_f != 1): thread per element, the 32 lanes
// of a warp read one entry of 32 consecutive elements as one 256-byte segment.
template <int P, int MODE, bool DOT, bool NS = false>
__global__ void __launch_bounds__(128) k_apply_ldg(const LevelDev L, int colour,
                                                   const double* x, double* y,
                                                   const double* __restrict__ r, double* d,
                                                   int step, double* __restrict__ partials,
                                                   int early) {
  (void)early;
  constexpr int K1 = P + 1;
  constexpr int M = 4 * K1;
  constexpr int NPK = NS ? M * M : M * (M + 1) / 2;
  const int64_t nec = L.ne >> 1;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const uint64_t pol = stream_policy(colour == 0 && L.l2keep0 ? 1.0f : L.l2keep);
  pdl_wait();
  pdl_trigger();
  double c1 = 0.0, c2 = 0.0;
  if (MODE == AM_SMOOTH) {
    c1 = L.coef[2 * step];
    c2 = L.coef[2 * step + 1];
  }
  double dot = 0.0;
  for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < nec; s += stride) {
    int i, j;
    slot_elem(L.nx, colour, s, i, j);
    int64_t ed[4];
    bool bd[4];
    elem_edges(L.nx, L.ny, i, j, ed, bd, L.dmask);
    const int itf = elem_itf(L.nx, L.ny, i, j, L.imask);
    double xv[M], yv[M], t[M], dd[M];
    gather_x<K1>(x, ed, bd, xv);
    epi_load<K1, MODE>(L, ed, bd, y, r, d, t, dd, itf);
#pragma unroll
    for (int a = 0; a < M; ++a) yv[a] = 0.0;
    const double* Sp = L.S + ((((int64_t)colour * L.nchunk + (s >> 5)) * NPK) << 5) + (s & 31);
    if (NS) {
#pragma unroll
      for (int a = 0; a < M; ++a)
#pragma unroll
        for (int b = 0; b < M; ++b) yv[a] = fma(ld_stream(Sp + ((a * M + b) << 5), pol), xv[b], yv[a]);
    } else {
#pragma unroll
      for (int a = 0; a < M; ++a) {
#pragma unroll
        for (int b = a; b < M; ++b) {
          const int kk = a * (2 * M - a + 1) / 2 + (b - a);
          const double sv = ld_stream(Sp + (kk << 5), pol);
          yv[a] = fma(sv, xv[b], yv[a]);
          if (b != a) yv[b] = fma(sv, xv[a], yv[b]);
        }
      }
    }
    epi_store<K1, MODE, DOT>(L, ed, bd, xv, yv, t, dd, x, y, d, step, c1, c2, dot, itf);
  }
  if (DOT) {
    __shared__ double red[4];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = dot;
    __syncthreads();
    if (threadIdx.x == 0) partials[blockIdx.x] = (red[0] + red[1]) + (red[2] + red[3]);
  }
}

// ---------------------------------------------------------------- single-pass strip apply
// y = A x (AM_APPLY, optional dot) or w = r - A e (AM_RESID) in ONE pass over S_T
// (MGDTN_STRIP=1, one GPU, nx % 64 == 0, ny % R == 0).  A CTA (one warp) owns tiles of
// 64 columns x R rows; for each row it streams the row's colour-0 chunk, then its
// colour-1 chunk (32 elements each, the S_T chunk layout), through the same TMA ring as
// k_apply_tma.  Lane l holds the elements of columns x0+2l (A) and x0+2l+1 (B), so every
// edge inside the tile is completed in registers: the A|B edge in-lane, the edge left
// of A with the B contribution of lane l-1 (shuffle), a bottom edge with the top
// contribution carried from the previous row.  Tile-perimeter edges leave their two
// partial sums (by the colour of the contributing element) in pc0 / pc1, finished by
// k_strip_fixup.  Every sum is taken colour 0 first, as in the two-pass apply (colour 0
// writes, colour 1 adds), so y is bit-identical to it (the dot's summation order differs).
template <int P, int MODE, bool DOT, int RR>
__global__ void __launch_bounds__(32) k_apply_strip(const LevelDev L, const double* x, double* y,
                                                    const double* __restrict__ r,
                                                    double* __restrict__ partials, int early) {
  using C = TmaCfg<P>;
  constexpr int K1 = C::K1, M = C::M, NPK = C::NPK, NST = 2, TW = 64;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t bars[NST];
  double* stage_buf = reinterpret_cast<double*>(smem_raw);
  const int lane = threadIdx.x;
  const int nx = L.nx, ny = L.ny, nxh = nx >> 1;
  const int ntx = nx / TW, ntiles = ntx * (ny / RR);
  const int nmine = (int)blockIdx.x < ntiles ? (ntiles - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
  const int npos = nmine * 2 * RR;
  const uint64_t pol = stream_policy(L.l2keep);
  if (lane == 0) {
#pragma unroll
    for (int st = 0; st < NST; ++st) mbar_init(&bars[st], 1);
    fence_mbar_init();
  }
  __syncwarp();
  auto issue = [&](int pos) {   // lane 0
    const int tile = (int)blockIdx.x + (pos / (2 * RR)) * (int)gridDim.x;
    const int kk = pos % (2 * RR);
    const int x0 = (tile % ntx) * TW, y0 = (tile / ntx) * RR;
    const int j = y0 + (kk >> 1), c = kk & 1;
    const int64_t q = ((int64_t)j * nxh + (x0 >> 1)) >> 5;
    const int st = pos % NST;
    mbar_expect_tx(&bars[st], C::CHUNK_BYTES);
    tma_bulk_g2s(stage_buf + (size_t)st * NPK * 32, L.S + (((int64_t)c * L.nchunk + q) * NPK) * 32,
                 C::CHUNK_BYTES, &bars[st], pol);
  };
  if (early) {
    if (lane == 0)
      for (int pos = 0; pos < NST && pos < npos; ++pos) issue(pos);
    pdl_trigger();
    pdl_wait();
  } else {
    pdl_wait();
    if (lane == 0)
      for (int pos = 0; pos < NST && pos < npos; ++pos) issue(pos);
    pdl_trigger();
  }
  double dot = 0.0;
  // epilogue of a completed edge: c0 / c1 = the colour-0 / colour-1 element's part
  auto finish = [&](int64_t g, const double* c0, const double* c1) {
#pragma unroll
    for (int a = 0; a < K1; ++a) {
      double v;
      if (MODE == AM_RESID) v = (__ldg(r + g * K1 + a) - c0[a]) - c1[a];
      else v = c0[a] + c1[a];
      y[g * K1 + a] = v;
      if (DOT) dot = fma(x[g * K1 + a], v, dot);
    }
  };
  auto zero = [&](int64_t g) {
#pragma unroll
    for (int a = 0; a < K1; ++a) y[g * K1 + a] = 0.0;
  };
  auto partial = [&](int64_t g, int colour, const double* v) {
    double* dst = colour ? L.pc1 : L.pc0;
#pragma unroll
    for (int a = 0; a < K1; ++a) dst[g * K1 + a] = v[a];
  };
  // x of the element at position q (software pipeline: gathered one position ahead,
  // so the gather's latency overlaps the previous matvec)
  auto gather_at = [&](int q, double* xo) {
    if (q >= npos) return;
    const int tile = (int)blockIdx.x + (q / (2 * RR)) * (int)gridDim.x;
    const int kk = q % (2 * RR);
    const int j = (tile / ntx) * RR + (kk >> 1), c = kk & 1;
    const int i = (tile % ntx) * TW + 2 * lane + ((c + j) & 1);
    int64_t ed[4];
    bool bd[4];
    elem_edges(nx, ny, i, j, ed, bd, 15);
    gather_x<K1>(x, ed, bd, xo);
  };
  double xn[M];
  gather_at(0, xn);
  int pos = 0;
  for (int k = 0; k < nmine; ++k) {
    const int tile = (int)blockIdx.x + k * (int)gridDim.x;
    const int x0 = (tile % ntx) * TW, y0 = (tile / ntx) * RR;
    const int cA = x0 + 2 * lane, cB = cA + 1;
    double carA[K1], carB[K1];   // tops of the previous row's A / B elements
    for (int rj = 0; rj < RR; ++rj) {
      const int j = y0 + rj;
      double A[M], B[M];   // edge contributions of the elements in columns cA / cB
#pragma unroll
      for (int c = 0; c < 2; ++c, ++pos) {
        const int d = (c + j) & 1;   // colour c sits in column x0 + 2l + d
        double xv[M], yv[M];
#pragma unroll
        for (int a = 0; a < M; ++a) xv[a] = xn[a];
        gather_at(pos + 1, xn);
        const int st = pos % NST;
        mbar_wait(&bars[st], (uint32_t)((pos / NST) & 1));
        const double* Sp = stage_buf + (size_t)st * NPK * 32 + lane;
#pragma unroll
        for (int a = 0; a < M; ++a) yv[a] = 0.0;
#pragma unroll
        for (int a = 0; a < M; ++a) {
#pragma unroll
          for (int b = a; b < M; ++b) {
            const int kk = a * (2 * M - a + 1) / 2 + (b - a);
            const double sv = Sp[kk * 32];
            yv[a] = fma(sv, xv[b], yv[a]);
            if (b != a) yv[b] = fma(sv, xv[a], yv[b]);
          }
        }
        __syncwarp();
        if (lane == 0 && pos + NST < npos) {
          fence_proxy_async();
          issue(pos + NST);
        }
        if (d == 0) {
#pragma unroll
          for (int a = 0; a < M; ++a) A[a] = yv[a];
        } else {
#pragma unroll
          for (int a = 0; a < M; ++a) B[a] = yv[a];
        }
      }
      const int colA = j & 1, colB = colA ^ 1;   // colours of the A / B elements
      // local edge f of an element: 0 bottom, 1 right, 2 top, 3 left (K1 values each)
      // (1) A|B edge V(cB, j)
      {
        const int64_t g = vedge(nx, ny, cB, j);
        if (colA == 0) finish(g, A + 1 * K1, B + 3 * K1);
        else finish(g, B + 3 * K1, A + 1 * K1);
      }
      // (2) left edge of A, V(cA, j): B.right of lane l - 1
      {
        double lb[K1];
#pragma unroll
        for (int a = 0; a < K1; ++a) lb[a] = __shfl_up_sync(0xffffffffu, B[1 * K1 + a], 1);
        const int64_t g = vedge(nx, ny, cA, j);
        if (lane > 0) {
          if (colA == 0) finish(g, A + 3 * K1, lb);
          else finish(g, lb, A + 3 * K1);
        } else if (x0 == 0) {
          zero(g);
        } else {
          partial(g, colA, A + 3 * K1);
        }
      }
      // (3) right edge of the strip, V(x0 + 64, j): lane 31's B.right
      if (lane == 31) {
        const int64_t g = vedge(nx, ny, cB + 1, j);
        if (cB + 1 == nx) zero(g);
        else partial(g, colB, B + 1 * K1);
      }
      // (4) bottoms H(cA, j), H(cB, j) with the carried tops of row j - 1
      {
        const int64_t gA = hedge(nx, cA, j), gB = hedge(nx, cB, j);
        if (rj > 0) {
          if (colA == 0) {
            finish(gA, A + 0 * K1, carA);
            finish(gB, carB, B + 0 * K1);
          } else {
            finish(gA, carA, A + 0 * K1);
            finish(gB, B + 0 * K1, carB);
          }
        } else if (j == 0) {
          zero(gA);
          zero(gB);
        } else {
          partial(gA, colA, A + 0 * K1);
          partial(gB, colB, B + 0 * K1);
        }
      }
#pragma unroll
      for (int a = 0; a < K1; ++a) {
        carA[a] = A[2 * K1 + a];
        carB[a] = B[2 * K1 + a];
      }
    }
    // tops of the tile's last row, H(cA, y0 + R), H(cB, y0 + R)
    {
      const int jt = y0 + RR;
      const int64_t gA = hedge(nx, cA, jt), gB = hedge(nx, cB, jt);
      const int colA = (jt - 1) & 1;   // colour of the row-(jt-1) element in column cA
      if (jt == ny) {
        zero(gA);
        zero(gB);
      } else {
        partial(gA, colA, carA);
        partial(gB, colA ^ 1, carB);
      }
    }
  }
  if (DOT) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
    if (lane == 0) partials[blockIdx.x] = dot;
  }
}

// perimeter edges of the strip tiles: horizontal tile boundaries j = R t (0 < j < ny),
// vertical ones i = 64 t (0 < i < nx); y = c0 + c1 (AM_RESID: (r - c0) - c1)
template <int MODE, bool DOT>
__global__ void __launch_bounds__(256) k_strip_fixup(const LevelDev L, const double* x, double* y,
                                                     const double* __restrict__ r,
                                                     double* __restrict__ partials) {
  pdl_enter();
  const int nx = L.nx, ny = L.ny, R = L.strip_r, K1 = L.k1;
  const int64_t nh = (int64_t)(ny / R - 1) * nx, nv = (int64_t)(nx / 64 - 1) * ny;
  double dot = 0.0;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < nh + nv;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t g;
    if (t < nh) {
      const int jb = (int)(t / nx + 1) * R, i = (int)(t % nx);
      g = hedge(nx, i, jb);
    } else {
      const int64_t u = t - nh;
      const int ib = (int)(u / ny + 1) * 64, j = (int)(u % ny);
      g = vedge(nx, ny, ib, j);
    }
    for (int a = 0; a < K1; ++a) {
      const double c0 = L.pc0[g * K1 + a], c1 = L.pc1[g * K1 + a];
      const double v = MODE == AM_RESID ? (__ldg(r + g * K1 + a) - c0) - c1 : c0 + c1;
      y[g * K1 + a] = v;
      if (DOT) dot = fma(x[g * K1 + a], v, dot);
    }
  }
  if (DOT) {
    __shared__ double red[8];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = dot;
    __syncthreads();
    if (threadIdx.x == 0) {
      double s = 0.0;
      for (int w = 0; w < 8; ++w) s += red[w];
      partials[blockIdx.x] = s;
    }
  }
}

static int strip_fixup_grid(const LevelDev& L) {
  const int64_t n = (int64_t)(L.ny / L.strip_r - 1) * L.nx + (int64_t)(L.nx / 64 - 1) * L.ny;
  const int64_t g = (n + 255) / 256;
  return (int)(g < 148 ? (g > 0 ? g : 1) : 148);
}
static int strip_grid(const LevelDev& L) {
  const int ntiles = (L.nx / 64) * (L.ny / L.strip_r);
  const int g = 148 * 2;
  return ntiles < g ? ntiles : g;
}
static bool strip_ok(const LevelDev& L, int mode) {
  return L.strip_r > 0 && (mode == AM_APPLY || mode == AM_RESID) && L.pc0 && L.pc1 &&
         !L.ns && L.imask == 0 && L.dmask == 15 && L.nx % 64 == 0 && L.ny % L.strip_r == 0 &&
         L.ny / L.strip_r >= 1;
}

template <int P, int MODE, bool DOT>
static void launch_strip_t(const LevelDev& L, const double* x, double* y, const double* r,
                           double* partials, bool pdl, cudaStream_t st) {
  const size_t smem = (size_t)2 * TmaCfg<P>::CHUNK_BYTES;
  const int grid = strip_grid(L);
  double* pf = partials ? partials + grid : nullptr;
  switch (L.strip_r) {
#define STRIP_CASE(RV)                                                                        \
    case RV: {                                                                                \
      static bool attr = false;                                                               \
      if (!attr) {                                                                            \
        cudaFuncSetAttribute(k_apply_strip<P, MODE, DOT, RV>,                                 \
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);         \
        attr = true;                                                                          \
      }                                                                                       \
      launch_ex(k_apply_strip<P, MODE, DOT, RV>, grid, 32, smem, pdl, st, L, x, y, r,         \
                partials, pdl ? 1 : 0);                                                       \
      break;                                                                                  \
    }
    STRIP_CASE(2)
    STRIP_CASE(4)
    default: STRIP_CASE(8)
#undef STRIP_CASE
  }
  launch_ex(k_strip_fixup<MODE, DOT>, strip_fixup_grid(L), 256, 0, true, st, L, x, y, r, pf);
}

template <int P>
static void launch_strip_p(const LevelDev& L, int mode, const double* x, double* y,
                           const double* r, double* partials, bool pdl, cudaStream_t st) {
  if (mode == AM_RESID) launch_strip_t<P, AM_RESID, false>(L, x, y, r, nullptr, pdl, st);
  else if (partials) launch_strip_t<P, AM_APPLY, true>(L, x, y, r, partials, pdl, st);
  else launch_strip_t<P, AM_APPLY, false>(L, x, y, r, nullptr, pdl, st);
}

// ---------------------------------------------------------------- LU-SGS colour sweep, edge rows only
// One LU-SGS colour sweep (reading F3) needs (r - A x)_e on the
// edges of ONE colour only, and every element has exactly one edge of each colour:
// each element forms just the K1 rows of S_T x_T belonging to that edge (K1*M of
// its m(m+1)/2 packed entries, 100 of 210 at p = 4) with plain coalesced loads (the
// 32 lanes of a warp share the edge's local index within a mesh row).  Pass 0
// (colour-0 elements) writes the partial sums y_e; pass 1 (colour-1 elements) adds
// its own, x_e += omega D_e^-1 (r_e - y_e).  Each row is accumulated in increasing
// column order, the order of the whole-matrix packed loop; D_e^-1 comes from the SoA
// blocks (the masked apply reads their packed upper triangle), so the two agree to
// rounding.  Measured slower than the TMA-streamed masked apply at config 2 (38.7 vs
// 34.9 ms LU-SGS solve): off by default, MGDTN_GS=rows selects it.
template <int P, int PASS>
__global__ void __launch_bounds__(128) k_gs_rows(const LevelDev L, int gcol, double* x, double* y,
                                                 const double* __restrict__ r) {
  constexpr int K1 = P + 1, M = 4 * K1, NPK = M * (M + 1) / 2;
  pdl_enter();
  const int colour = PASS;
  const int64_t nec = L.ne >> 1;
  const uint64_t pol = stream_policy(L.l2keep);
  const double om = L.coef[1];
  for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < nec;
       s += (int64_t)gridDim.x * blockDim.x) {
    int i, j;
    slot_elem(L.nx, colour, s, i, j);
    int64_t ed[4];
    bool bd[4];
    elem_edges(L.nx, L.ny, i, j, ed, bd, L.dmask);
    int fc = 0;
#pragma unroll
    for (int f = 1; f < 4; ++f)
      if (gs_colour(i, j, f) == gcol) fc = f;
    if (bd[fc]) continue;
    double xv[M];
    gather_x<K1>(x, ed, bd, xv);
    const double* Sp = L.S + ((((int64_t)colour * L.nchunk + (s >> 5)) * NPK) << 5) + (s & 31);
    double yv[K1];
    auto rows = [&](auto F) {
      constexpr int f = decltype(F)::value;
#pragma unroll
      for (int al = 0; al < K1; ++al) {
        const int a = f * K1 + al;
        double acc = 0.0;
#pragma unroll
        for (int b = 0; b < M; ++b) {
          const int kk = b < a ? b * (2 * M - b + 1) / 2 + (a - b) : a * (2 * M - a + 1) / 2 + (b - a);
          acc = fma(ld_stream(Sp + ((int64_t)kk << 5), pol), xv[b], acc);
        }
        yv[al] = acc;
      }
    };
    switch (fc) {
      case 0: rows(std::integral_constant<int, 0>{}); break;
      case 1: rows(std::integral_constant<int, 1>{}); break;
      case 2: rows(std::integral_constant<int, 2>{}); break;
      default: rows(std::integral_constant<int, 3>{}); break;
    }
    const int64_t base = ed[fc] * K1;
    if (PASS == 0) {
#pragma unroll
      for (int al = 0; al < K1; ++al) y[base + al] = yv[al];
    } else {
      double res[K1];
#pragma unroll
      for (int al = 0; al < K1; ++al) res[al] = (__ldg(r + base + al) - y[base + al]) - yv[al];
      const double* Di = L.Dinv + ed[fc];
#pragma unroll
      for (int al = 0; al < K1; ++al) {
        double c = 0.0;
#pragma unroll
        for (int b = 0; b < K1; ++b) c = fma(__ldg(Di + (al * K1 + b) * L.nedge), res[b], c);
        x[base + al] = fma(om, c, xv[fc * K1 + al]);
      }
    }
  }
}

static bool gs_full() {   // MGDTN_GS=rows: the edge-row sweep (A/B); default the masked apply
  static int v = -1;
  if (v < 0) {
    const char* e = std::getenv("MGDTN_GS");
    v = (e && std::strcmp(e, "rows") == 0) ? 0 : 1;
  }
  return v == 1;
}

int launch_gs_sweep(const LevelDev& L, int gcol, double* x, double* y, const double* r,
                    cudaStream_t st) {
  if (gs_full() || L.ns || L.imask) return -1;   // caller uses the masked full apply
  const int64_t nec = L.ne / 2;
  int64_t g = (nec + 127) / 128;
  const int grid = (int)(g < 148 * 8 ? (g > 0 ? g : 1) : 148 * 8);
#define GS_LAUNCH(PP)                                                                     \
  launch_ex(k_gs_rows<PP, 0>, grid, 128, 0, true, st, L, gcol, x, y, r);                 \
  launch_ex(k_gs_rows<PP, 1>, grid, 128, 0, true, st, L, gcol, x, y, r);
  switch (L.p) {
    case 1: GS_LAUNCH(1) break;
    case 2: GS_LAUNCH(2) break;
    case 3: GS_LAUNCH(3) break;
    default: GS_LAUNCH(4) break;
  }
#undef GS_LAUNCH
  return 2;
}

// ---------------------------------------------------------------- host side
// apply kernel: MGDTN_APPLY = auto (default: seg for the smoothing / power-iteration
// passes, which stream D_e^-1 too, tma for the others; profiles/r01_seg_probe.jsonl)
// | seg | tma | ldg  (A/B)
static int apply_impl() {
  static int v = -1;
  if (v < 0) {
    const char* e = std::getenv("MGDTN_APPLY");
    v = !e ? 0 : std::strcmp(e, "ldg") == 0 ? 1 : std::strcmp(e, "tma") == 0 ? 2
             : std::strcmp(e, "seg") == 0 ? 3 : 0;
  }
  return v;
}
static bool use_ldg() { return apply_impl() == 1; }
static bool mode_has_dinv(int mode) {
  return mode == AM_SMOOTH || mode == AM_DINV || mode == AM_GSC;
}
// MGDTN_SEG_PMASK: bit p set -> "auto" uses the segmented ring for EVERY pass at order p
// (default bit 2: at p = 2 it beats the whole-chunk kernel for the plain passes too,
// config 3 solve 4.37 -> 3.98 s; at p = 1, 3 and 4 it loses, profiles/r01_seg_pmask.jsonl)
static int seg_pmask() {
  static int v = -1;
  if (v < 0) {
    const char* e = std::getenv("MGDTN_SEG_PMASK");
    v = e ? std::atoi(e) : (1 << 2);
  }
  return v;
}
static bool use_seg(int mode, int p) {
  return apply_impl() == 3 ||
         (apply_impl() == 0 && (mode_has_dinv(mode) || ((seg_pmask() >> p) & 1)));
}

static int env_int(const char* name, int dflt) {
  const char* e = std::getenv(name);
  return e ? std::atoi(e) : dflt;
}
static int tma_cps(int p) {   // CTAs per SM (tuning knob MGDTN_TMA_CPS, 0 = per-p default)
  static int v = -1;
  if (v < 0) v = env_int("MGDTN_TMA_CPS", 0);
  if (v > 0) return v;
  return p == 4 ? TmaCfg<4>::CPS : p == 3 ? TmaCfg<3>::CPS : p == 2 ? TmaCfg<2>::CPS : TmaCfg<1>::CPS;
}
static int tma_nst() {   // stages per CTA (tuning knob MGDTN_TMA_NST, 0 = per-p default)
  static int v = -1;
  if (v < 0) v = env_int("MGDTN_TMA_NST", 0);
  return v;
}

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

// resident CTAs per SM of a segmented-ring instantiation (occupancy calculator, cached)
template <int P, int MODE, bool DOT>
static int seg_resident() {
  static int v = 0;
  if (v == 0) {
    const size_t smem = (size_t)SegCfg<P>::NSLOT * SegCfg<P>::SEG_BYTES;
    cudaFuncSetAttribute(k_apply_seg<P, MODE, DOT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    int nb = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_apply_seg<P, MODE, DOT>, 32, smem);
    v = nb > 0 ? nb : 1;
  }
  return v;
}

static int seg_cps(int p) {   // CTAs per SM (tuning knob MGDTN_SEG_CPS, 0 = per-p default)
  static int v = -1;
  if (v < 0) v = env_int("MGDTN_SEG_CPS", 0);
  int c = v > 0 ? v : p == 4 ? SegCfg<4>::CPS : p == 3 ? SegCfg<3>::CPS : p == 2 ? SegCfg<2>::CPS
                                                                                   : SegCfg<1>::CPS;
  const int res = p == 4 ? seg_resident<4, AM_W0, false>() : p == 3 ? seg_resident<3, AM_W0, false>()
                  : p == 2 ? seg_resident<2, AM_W0, false>() : seg_resident<1, AM_W0, false>();
  return c < res ? c : res;
}

template <int P, int MODE, bool DOT>
static void launch_seg(const LevelDev& L, int colour, const double* x, double* y, const double* r,
                       double* d, int step, double* partials, int grid, bool pdl,
                       cudaStream_t st) {
  const size_t smem = (size_t)SegCfg<P>::NSLOT * SegCfg<P>::SEG_BYTES;
  seg_resident<P, MODE, DOT>();   // sets the dynamic smem attribute once
  launch_ex(k_apply_seg<P, MODE, DOT>, grid, 32, smem, pdl, st, L, colour, x, y, r, d, step,
            partials, pdl ? 1 : 0);
}

// MGDTN_GRID: how the whole-chunk TMA apply spreads a colour's chunks over its CTAs
//   bal (default) -- balanced_grid: every CTA the same number of chunks
//   full          -- 148 x CTAs-per-SM CTAs, chunk c to CTA c mod grid (per-SM balance
//                    when the CTAs land round-robin on the SMs)
//   dyn           -- full grid, first NST chunks static, then tickets (dynamic)
static int grid_mode() {
  static int v = -1;
  if (v < 0) {
    const char* e = std::getenv("MGDTN_GRID");
    v = !e ? 0 : std::strcmp(e, "full") == 0 ? 1 : std::strcmp(e, "dyn") == 0 ? 2 : 0;
  }
  return v;
}
// the ticket counter pair of a level / colour (LevelDev::sync tail, mgdtn.cu layout)
static unsigned* ticket_of(const LevelDev& L, int colour) {
  if (grid_mode() != 2 || L.sync == nullptr) return nullptr;
  return L.sync + 2 + L.nchunk + 2 * colour;
}

// nonsymmetric context's apply: MGDTN_NS_APPLY = seg (default, full-storage segmented
// ring) | ldg (thread per element, direct loads; A/B)
static bool ns_use_ldg() {
  static int v = -1;
  if (v < 0) {
    const char* e = std::getenv("MGDTN_NS_APPLY");
    v = (e && std::strcmp(e, "ldg") == 0) ? 1 : 0;
  }
  return v == 1;
}
template <int P, int MODE, bool DOT>
static int seg_ns_resident() {
  static int v = 0;
  if (v == 0) {
    using C = SegCfg<P, true>;
    const size_t smem = (size_t)C::NSLOT * C::SEG_BYTES;
    cudaFuncSetAttribute(k_apply_seg<P, MODE, DOT, true>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int nb = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_apply_seg<P, MODE, DOT, true>, 32, smem);
    v = nb > 0 ? nb : 1;
  }
  return v;
}
static int seg_ns_cps(int p) {
  const int c = p == 4 ? SegCfg<4, true>::CPS : p == 3 ? SegCfg<3, true>::CPS
                : p == 2 ? SegCfg<2, true>::CPS : SegCfg<1, true>::CPS;
  const int res = p == 4 ? seg_ns_resident<4, AM_W0, false>() : p == 3 ? seg_ns_resident<3, AM_W0, false>()
                  : p == 2 ? seg_ns_resident<2, AM_W0, false>() : seg_ns_resident<1, AM_W0, false>();
  return c < res ? c : res;
}

// grid of at most gmax persistent CTAs over n chunks with the work spread evenly:
// k = ceil(n / gmax) chunks per CTA, ceil(n / k) CTAs (every CTA gets k or k-1)
static int balanced_grid(int64_t n, int64_t gmax) {
  if (n <= 0) return 1;
  if (gmax < 1) gmax = 1;
  const int64_t k = (n + gmax - 1) / gmax;
  return (int)((n + k - 1) / k);
}

int apply_grid(const LevelDev& L) { return apply_grid_mode(L, AM_APPLY); }

int apply_grid_mode(const LevelDev& L, int mode) {
  const int64_t nec = L.ne / 2;
  if (L.ns && !ns_use_ldg() && !use_ldg())
    return balanced_grid((nec + 31) / 32, (int64_t)num_sms() * seg_ns_cps(L.p));
  if (use_ldg() || L.ns) {
    int64_t g = (nec + 127) / 128;
    const int64_t gmax = 148 * 8;
    return (int)(g < gmax ? (g > 0 ? g : 1) : gmax);
  }
  const int64_t nchunk = (nec + 31) / 32;
  if (use_seg(mode, L.p)) return balanced_grid(nchunk, (int64_t)num_sms() * seg_cps(L.p));
  if (grid_mode() != 0) {
    const int64_t g = (int64_t)num_sms() * tma_cps(L.p);
    return (int)(nchunk < g ? (nchunk > 0 ? nchunk : 1) : g);
  }
  return balanced_grid(nchunk, 148 * tma_cps(L.p));
}

static bool use_xpf() {   // MGDTN_XPF=0: no x-gather prefetch of the next chunk (A/B)
  static int v = -1;
  if (v < 0) v = env_int("MGDTN_XPF", 1);
  return v != 0;
}

template <int P, int MODE, bool DOT, int NST, bool XPF>
static void launch_tma_x(const LevelDev& L, int colour, const double* x, double* y,
                         const double* r, double* d, int step, double* partials, int grid,
                         bool pdl, cudaStream_t st) {
  const size_t smem = (size_t)NST * TmaCfg<P>::CHUNK_BYTES;
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(k_apply_tma<P, MODE, DOT, NST, XPF>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr_set = true;
  }
  launch_ex(k_apply_tma<P, MODE, DOT, NST, XPF>, grid, 32, smem, pdl, st, L, colour, x, y, r, d,
            step, partials, pdl ? 1 : 0, ticket_of(L, colour));
}

static bool use_tma2() {   // MGDTN_TMA2=1: two warps per CTA (A/B; measured slower)
  static int v = -1;
  if (v < 0) v = env_int("MGDTN_TMA2", 0);
  return v != 0;
}

template <int P, int MODE, bool DOT, int NST>
static void launch_tma(const LevelDev& L, int colour, const double* x, double* y, const double* r,
                       double* d, int step, double* partials, int grid, bool pdl,
                       cudaStream_t st) {
  if (use_tma2() && MODE != AM_SMOOTH && MODE != AM_DINV) {
    const size_t smem = (size_t)NST * TmaCfg<P>::CHUNK_BYTES;
    static bool attr_set = false;
    if (!attr_set) {
      cudaFuncSetAttribute(k_apply_tma2<P, MODE, DOT, NST>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      attr_set = true;
    }
    launch_ex(k_apply_tma2<P, MODE, DOT, NST>, grid, 64, smem, pdl, st, L, colour, x, y, r, d,
              step, partials, pdl ? 1 : 0);
    return;
  }
  if (use_xpf())
    launch_tma_x<P, MODE, DOT, NST, true>(L, colour, x, y, r, d, step, partials, grid, pdl, st);
  else
    launch_tma_x<P, MODE, DOT, NST, false>(L, colour, x, y, r, d, step, partials, grid, pdl, st);
}

template <int P, int MODE, bool DOT>
static void launch_one(const LevelDev& L, int colour, const double* x, double* y, const double* r,
                       double* d, int step, double* partials, int grid, bool pdl,
                       cudaStream_t st) {
  if (L.ns) {   // nonsymmetric context: full-storage apply (no LU-SGS / power iteration there)
    if (MODE == AM_GSC || MODE == AM_DINV) return;
    if (ns_use_ldg() || use_ldg()) {
      launch_ex(k_apply_ldg<P, MODE, DOT, true>, grid, 128, 0, pdl, st, L, colour, x, y, r, d,
                step, partials, 0);
    } else {
      using C = SegCfg<P, true>;
      seg_ns_resident<P, MODE, DOT>();   // sets the dynamic smem attribute once
      launch_ex(k_apply_seg<P, MODE, DOT, true>, grid, 32, (size_t)C::NSLOT * C::SEG_BYTES, pdl,
                st, L, colour, x, y, r, d, step, partials, pdl ? 1 : 0);
    }
    return;
  }
  if (MODE == AM_GSC) {   // colour sweeps exist in the segmented-ring kernel only
    launch_seg<P, AM_GSC, false>(L, colour, x, y, r, d, step, partials, grid, pdl, st);
    return;
  }
  if (use_ldg()) {
    launch_ex(k_apply_ldg<P, MODE, DOT>, grid, 128, 0, pdl, st, L, colour, x, y, r, d, step,
             partials, 0);
    return;
  }
  if (use_seg(MODE, P)) {
    launch_seg<P, MODE, DOT>(L, colour, x, y, r, d, step, partials, grid, pdl, st);
    return;
  }
  using C = TmaCfg<P>;
  int nst = tma_nst();
  if (nst <= 0 || nst * C::CHUNK_BYTES > 220 * 1024) nst = C::NST;
  switch (nst) {   // tuning knob MGDTN_TMA_NST: 2..4 stages
    case 2: launch_tma<P, MODE, DOT, 2>(L, colour, x, y, r, d, step, partials, grid, pdl, st); break;
    case 3: launch_tma<P, MODE, DOT, 3>(L, colour, x, y, r, d, step, partials, grid, pdl, st); break;
    default: launch_tma<P, MODE, DOT, 4>(L, colour, x, y, r, d, step, partials, grid, pdl, st); break;
  }
}

// ---------------------------------------------------------------- fused launch
static int fused_mode() {   // MGDTN_FUSED: 0 two launches (default), 1 grid barrier, 2 chunk flags
  static int v = -1;
  if (v < 0) v = env_int("MGDTN_FUSED", 0);
  return v;
}
static bool use_fused() { return fused_mode() != 0 && apply_impl() != 1; }
// mode 3: the grid-barrier variant on the P1 levels only (short, launch-bound passes)
static bool fused_for(const LevelDev& L) {
  const int m = fused_mode();
  if (m == 3) return L.p == 1 && apply_impl() != 1;
  return (m == 1 || m == 2) && apply_impl() == 2;
}



template <int P>
static int fused_nst() {   // the fused kernel is built for the default stage count only
  return TmaCfg<P>::NST;
}

// resident CTAs per SM of a fused instantiation (occupancy calculator, cached)
template <int P, int MODE, bool DOT, int NST, bool FLAGS>
static int fused_resident() {
  static int v = 0;
  if (v == 0) {
    const size_t smem = (size_t)NST * TmaCfg<P>::CHUNK_BYTES;
    cudaFuncSetAttribute(k_apply_fused<P, MODE, DOT, NST, FLAGS>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int nb = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_apply_fused<P, MODE, DOT, NST, FLAGS>, 32,
                                                  smem);
    v = nb > 0 ? nb : 1;
  }
  return v;
}

template <int P, int NST>
static int fused_grid_p(const LevelDev& L) {
  // every instantiation of one (P, NST) has the same smem; AM_SMOOTH stands for all
  const int res = fused_resident<P, AM_SMOOTH, false, NST, false>();
  int cps = tma_cps(L.p);
  if (cps > res) cps = res;
  return balanced_grid(L.nchunk, (int64_t)num_sms() * cps);
}

template <int P>
static int fused_grid(const LevelDev& L) {
  return fused_grid_p<P, TmaCfg<P>::NST>(L);
}

int apply2_grid(const LevelDev& L, int mode) {
  if (strip_ok(L, mode)) return strip_grid(L) + strip_fixup_grid(L);
  if (!fused_for(L) || L.sync == nullptr || L.imask != 0 || mode == AM_GSC || L.ns)
    return apply_grid_mode(L, mode);
  switch (L.p) {
    case 1: return fused_grid<1>(L);
    case 2: return fused_grid<2>(L);
    case 3: return fused_grid<3>(L);
    default: return fused_grid<4>(L);
  }
}

template <int P, int MODE, bool DOT, int NST>
static void launch_fused_t(const LevelDev& L, const double* x, double* y, const double* r,
                           double* d, int step, double* partials, int grid, bool pdl,
                           cudaStream_t st) {
  const size_t smem = (size_t)NST * TmaCfg<P>::CHUNK_BYTES;
  if (fused_mode() == 2) {
    const int res = fused_resident<P, MODE, DOT, NST, true>();   // also sets the smem attribute
    if (grid > res * num_sms()) grid = res * num_sms();           // one resident wave at most
    launch_ex(k_apply_fused<P, MODE, DOT, NST, true>, grid, 32, smem, pdl, st, L, x, y, r, d, step,
              partials, pdl ? 1 : 0);
  } else {
    const int res = fused_resident<P, MODE, DOT, NST, false>();
    if (grid > res * num_sms()) grid = res * num_sms();
    launch_ex(k_apply_fused<P, MODE, DOT, NST, false>, grid, 32, smem, pdl, st, L, x, y, r, d, step,
              partials, pdl ? 1 : 0);
  }
}

template <int P, int MODE, bool DOT>
static void launch_fused_one(const LevelDev& L, const double* x, double* y, const double* r,
                             double* d, int step, double* partials, int grid, bool pdl,
                             cudaStream_t st) {
  launch_fused_t<P, MODE, DOT, TmaCfg<P>::NST>(L, x, y, r, d, step, partials, grid, pdl, st);
}

template <int P>
static void dispatch_fused(const LevelDev& L, int mode, const double* x, double* y,
                           const double* r, double* d, int step, double* partials, int grid,
                           bool pdl, cudaStream_t st) {
  switch (mode) {
    case AM_APPLY:
      if (partials)
        launch_fused_one<P, AM_APPLY, true>(L, x, y, r, d, step, partials, grid, pdl, st);
      else
        launch_fused_one<P, AM_APPLY, false>(L, x, y, r, d, step, partials, grid, pdl, st);
      break;
    case AM_RESID:
      launch_fused_one<P, AM_RESID, false>(L, x, y, r, d, step, partials, grid, pdl, st);
      break;
    case AM_DINV:
      if (partials)
        launch_fused_one<P, AM_DINV, true>(L, x, y, r, d, step, partials, grid, pdl, st);
      else
        launch_fused_one<P, AM_DINV, false>(L, x, y, r, d, step, partials, grid, pdl, st);
      break;
    default:
      launch_fused_one<P, AM_SMOOTH, false>(L, x, y, r, d, step, partials, grid, pdl, st);
      break;
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

int launch_apply2(const LevelDev& L, int mode, const double* x, double* y, const double* r,
                  double* d, int step, double* partials, bool pdl, cudaStream_t st) {
  if (strip_ok(L, mode)) {
    switch (L.p) {
      case 1: launch_strip_p<1>(L, mode, x, y, r, partials, pdl, st); break;
      case 2: launch_strip_p<2>(L, mode, x, y, r, partials, pdl, st); break;
      case 3: launch_strip_p<3>(L, mode, x, y, r, partials, pdl, st); break;
      default: launch_strip_p<4>(L, mode, x, y, r, partials, pdl, st); break;
    }
    return 2;
  }
  if (!fused_for(L) || L.sync == nullptr || L.imask != 0 || mode == AM_GSC || L.ns) {   // fused: 1 GPU
    int n = launch_apply(L, 0, AM_W0, x, y, nullptr, nullptr, 0, nullptr, pdl, st);
    return n + launch_apply(L, 1, mode, x, y, r, d, step, partials, pdl, st);
  }
  const int grid = apply2_grid(L, mode);
  switch (L.p) {
    case 1: dispatch_fused<1>(L, mode, x, y, r, d, step, partials, grid, pdl, st); break;
    case 2: dispatch_fused<2>(L, mode, x, y, r, d, step, partials, grid, pdl, st); break;
    case 3: dispatch_fused<3>(L, mode, x, y, r, d, step, partials, grid, pdl, st); break;
    default: dispatch_fused<4>(L, mode, x, y, r, d, step, partials, grid, pdl, st); break;
  }
  return 1;
}

}  // namespace mgdtn
