// Trace-operator apply y = A_k x = sum_T G_T^T S_T G_T x (PAPER.md:305-325,
// 330-344: A is the sum of the element DtN maps) with a conflict-free
// 2-colour scatter: colour-0 elements write their edge outputs, colour-1
// elements (which share no edge with each other) read-modify-write them and
// run the fused epilogue (residual, smoothing update, dot product).
//
// Thread per element; the packed symmetric S_T (npk = m(m+1)/2 doubles) is
// streamed once with L1-bypassing, L2-evict-first loads (warp-contiguous 256 B
// segments, see kernels.cuh); x_T (m values) is gathered from the 4 edges.
// HBM-bound: 8*npk bytes per element against 2*m*m flops.
#include "kernels.cuh"

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

template <int P, int MODE, bool DOT>
__global__ void __launch_bounds__(128) k_apply(const LevelDev L, int colour,
                                               const double* x, double* y,
                                               const double* __restrict__ r, double* d,
                                               int step, double* __restrict__ partials) {
  constexpr int K1 = P + 1;
  constexpr int M = 4 * K1;
  constexpr int NPK = M * (M + 1) / 2;
  const int64_t nec = L.ne >> 1;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const uint64_t pol = evict_first_policy();
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
    double xv[M], yv[M];
#pragma unroll
    for (int f = 0; f < 4; ++f) {
#pragma unroll
      for (int a = 0; a < K1; ++a) xv[f * K1 + a] = bd[f] ? 0.0 : x[ed[f] * K1 + a];
    }
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
#pragma unroll
    for (int f = 0; f < 4; ++f) {
      const int64_t base = ed[f] * K1;
      if (MODE == AM_W0) {
#pragma unroll
        for (int a = 0; a < K1; ++a) y[base + a] = bd[f] ? 0.0 : yv[f * K1 + a];
      } else if (MODE == AM_APPLY) {
#pragma unroll
        for (int a = 0; a < K1; ++a) {
          double v = bd[f] ? 0.0 : y[base + a] + yv[f * K1 + a];
          y[base + a] = v;
          if (DOT) dot = fma(xv[f * K1 + a], v, dot);
        }
      } else if (MODE == AM_RESID) {
#pragma unroll
        for (int a = 0; a < K1; ++a)
          y[base + a] = bd[f] ? 0.0 : r[base + a] - (y[base + a] + yv[f * K1 + a]);
      } else {  // AM_SMOOTH: x is updated in place (x aliases the smoothed iterate)
        if (!bd[f]) {
          double res[K1];
#pragma unroll
          for (int a = 0; a < K1; ++a) res[a] = r[base + a] - (y[base + a] + yv[f * K1 + a]);
          const double* Di = L.Dinv + ed[f] * (K1 * K1);
          double* xo = const_cast<double*>(x);
#pragma unroll
          for (int a = 0; a < K1; ++a) {
            double c = 0.0;
#pragma unroll
            for (int b = 0; b < K1; ++b) c = fma(Di[a * K1 + b], res[b], c);
            double dn = c2 * c;
            if (L.smoother == 1) {
              if (step > 0) dn = fma(c1, d[base + a], dn);
              d[base + a] = dn;
            }
            xo[base + a] = xv[f * K1 + a] + dn;
          }
        }
      }
    }
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

int apply_grid(const LevelDev& L) {
  int64_t nec = L.ne / 2;
  int64_t g = (nec + 127) / 128;
  const int64_t gmax = 148 * 8;
  return (int)(g < gmax ? (g > 0 ? g : 1) : gmax);
}

template <int P>
static void dispatch_apply(const LevelDev& L, int colour, int mode, const double* x, double* y,
                           const double* r, double* d, int step, double* partials, int grid,
                           cudaStream_t st) {
  switch (mode) {
    case AM_W0:
      k_apply<P, AM_W0, false><<<grid, 128, 0, st>>>(L, colour, x, y, r, d, step, partials);
      break;
    case AM_APPLY:
      if (partials)
        k_apply<P, AM_APPLY, true><<<grid, 128, 0, st>>>(L, colour, x, y, r, d, step, partials);
      else
        k_apply<P, AM_APPLY, false><<<grid, 128, 0, st>>>(L, colour, x, y, r, d, step, partials);
      break;
    case AM_RESID:
      k_apply<P, AM_RESID, false><<<grid, 128, 0, st>>>(L, colour, x, y, r, d, step, partials);
      break;
    default:
      k_apply<P, AM_SMOOTH, false><<<grid, 128, 0, st>>>(L, colour, x, y, r, d, step, partials);
      break;
  }
}

int launch_apply(const LevelDev& L, int colour, int mode, const double* x, double* y,
                 const double* r, double* d, int step, double* partials, int dot_grid,
                 cudaStream_t st) {
  int grid = dot_grid > 0 ? dot_grid : apply_grid(L);
  switch (L.p) {
    case 1: dispatch_apply<1>(L, colour, mode, x, y, r, d, step, partials, grid, st); break;
    case 2: dispatch_apply<2>(L, colour, mode, x, y, r, d, step, partials, grid, st); break;
    case 3: dispatch_apply<3>(L, colour, mode, x, y, r, d, step, partials, grid, st); break;
    default: dispatch_apply<4>(L, colour, mode, x, y, r, d, step, partials, grid, st); break;
  }
  return 1;
}

}  // namespace mgdtn
