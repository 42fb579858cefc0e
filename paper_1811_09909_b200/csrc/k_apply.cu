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

#include "bodies.cuh"

namespace mgdtn {

__device__ __forceinline__ uint64_t evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
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
  // chunks of this CTA: c_k = blockIdx.x + k * gridDim.x
  const int nmine = (int)blockIdx.x < nchunk ? (nchunk - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
  if (lane == 0) {
#pragma unroll
    for (int s = 0; s < NST; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  __syncwarp();
  auto issue = [&](int k) {   // lane 0: chunk k of this CTA into stage k % NST
    const int c = (int)blockIdx.x + k * (int)gridDim.x;
    const int s = k % NST;
    mbar_expect_tx(&bars[s], C::CHUNK_BYTES);
    tma_bulk_g2s(stage_buf + (size_t)s * NPK * 32, Sbase + (int64_t)c * NPK * 32, C::CHUNK_BYTES,
                 &bars[s], pol);
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
  for (int k = 0; k < nmine; ++k) {
    const int c = (int)blockIdx.x + k * (int)gridDim.x;
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
    if (act) {   // every global read of the element, independent of the stage: overlaps the wait
      int i, j;
      slot_elem(L.nx, colour, s, i, j);
      elem_edges(L.nx, L.ny, i, j, ed, bd);
      gather_x<K1>(x, ed, bd, xv);
      epi_load<K1, MODE>(L, ed, bd, y, r, d, t, dd);
    }
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
    if (act) epi_store<K1, MODE, DOT>(L, ed, bd, xv, yv, t, dd, x, y, d, step, c1, c2, dot);
  }
  if (DOT) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
    if (lane == 0) partials[blockIdx.x] = dot;
  }
}

// ---------------------------------------------------------------- direct-load apply (A/B)
template <int P, int MODE, bool DOT>
__global__ void __launch_bounds__(128) k_apply_ldg(const LevelDev L, int colour,
                                                   const double* x, double* y,
                                                   const double* __restrict__ r, double* d,
                                                   int step, double* __restrict__ partials,
                                                   int early) {
  (void)early;
  constexpr int K1 = P + 1;
  constexpr int M = 4 * K1;
  constexpr int NPK = M * (M + 1) / 2;
  const int64_t nec = L.ne >> 1;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const uint64_t pol = evict_first_policy();
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
    elem_edges(L.nx, L.ny, i, j, ed, bd);
    double xv[M], yv[M], t[M], dd[M];
    gather_x<K1>(x, ed, bd, xv);
    epi_load<K1, MODE>(L, ed, bd, y, r, d, t, dd);
#pragma unroll
    for (int a = 0; a < M; ++a) yv[a] = 0.0;
    const double* Sp = L.S + ((((int64_t)colour * L.nchunk + (s >> 5)) * NPK) << 5) + (s & 31);
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
    epi_store<K1, MODE, DOT>(L, ed, bd, xv, yv, t, dd, x, y, d, step, c1, c2, dot);
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

// ---------------------------------------------------------------- host side
static bool use_ldg() {
  static int v = -1;
  if (v < 0) {
    const char* e = std::getenv("MGDTN_APPLY");
    v = (e && std::strcmp(e, "ldg") == 0) ? 1 : 0;
  }
  return v == 1;
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

int apply_grid(const LevelDev& L) {
  const int64_t nec = L.ne / 2;
  if (use_ldg()) {
    int64_t g = (nec + 127) / 128;
    const int64_t gmax = 148 * 8;
    return (int)(g < gmax ? (g > 0 ? g : 1) : gmax);
  }
  const int64_t nchunk = (nec + 31) / 32;
  const int64_t gmax = 148 * tma_cps(L.p);
  return (int)(nchunk < gmax ? (nchunk > 0 ? nchunk : 1) : gmax);
}

template <int P, int MODE, bool DOT, int NST>
static void launch_tma(const LevelDev& L, int colour, const double* x, double* y, const double* r,
                       double* d, int step, double* partials, int grid, bool pdl,
                       cudaStream_t st) {
  const size_t smem = (size_t)NST * TmaCfg<P>::CHUNK_BYTES;
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(k_apply_tma<P, MODE, DOT, NST>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr_set = true;
  }
  launch_ex(k_apply_tma<P, MODE, DOT, NST>, grid, 32, smem, pdl, st, L, colour, x, y, r, d, step,
           partials, pdl ? 1 : 0);
}

template <int P, int MODE, bool DOT>
static void launch_one(const LevelDev& L, int colour, const double* x, double* y, const double* r,
                       double* d, int step, double* partials, int grid, bool pdl,
                       cudaStream_t st) {
  if (use_ldg()) {
    launch_ex(k_apply_ldg<P, MODE, DOT>, grid, 128, 0, pdl, st, L, colour, x, y, r, d, step,
             partials, 0);
    return;
  }
  using C = TmaCfg<P>;
  int nst = tma_nst();
  if (nst <= 0 || nst * C::CHUNK_BYTES > 220 * 1024) nst = C::NST;
  switch (nst) {
    case 2: launch_tma<P, MODE, DOT, 2>(L, colour, x, y, r, d, step, partials, grid, pdl, st); break;
    case 3: launch_tma<P, MODE, DOT, 3>(L, colour, x, y, r, d, step, partials, grid, pdl, st); break;
    case 4: launch_tma<P, MODE, DOT, 4>(L, colour, x, y, r, d, step, partials, grid, pdl, st); break;
    case 5: launch_tma<P, MODE, DOT, 5>(L, colour, x, y, r, d, step, partials, grid, pdl, st); break;
    default: launch_tma<P, MODE, DOT, 6>(L, colour, x, y, r, d, step, partials, grid, pdl, st); break;
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
    default:
      launch_one<P, AM_SMOOTH, false>(L, colour, x, y, r, d, step, partials, grid, pdl, st);
      break;
  }
}

int launch_apply(const LevelDev& L, int colour, int mode, const double* x, double* y,
                 const double* r, double* d, int step, double* partials, bool pdl,
                 cudaStream_t st) {
  const int grid = apply_grid(L);
  switch (L.p) {
    case 1: dispatch_apply<1>(L, colour, mode, x, y, r, d, step, partials, grid, pdl, st); break;
    case 2: dispatch_apply<2>(L, colour, mode, x, y, r, d, step, partials, grid, pdl, st); break;
    case 3: dispatch_apply<3>(L, colour, mode, x, y, r, d, step, partials, grid, pdl, st); break;
    default: dispatch_apply<4>(L, colour, mode, x, y, r, d, step, partials, grid, pdl, st); break;
  }
  return 1;
}

}  // namespace mgdtn
