// Single-pass streamed trace apply on the D4-orbit levels (one GPU): y = A x,
// w = r - A x, and the smoothing step e' = e + d (block-Jacobi / Chebyshev on
// edge blocks) in ONE pass over the elements, with every
// vector read and written once (the two-colour passes of k_apply_orb read x
// twice and write, re-read and re-write y).
//
// Geometry.  The mesh is cut into strips of SC = 64 element columns and each
// strip into segments of rows.  A CTA sweeps one segment upwards, SR = 2 element
// rows per step (thread per element).  It owns the bottom and left edges of its
// elements (and the mesh's top / right boundary edges next to them).  An owned
// edge sums the contributions of its two elements (A = sum_T G_T^T S_T G_T,
// PAPER.md:305-325): the element below a row's bottom edge is the previous step's
// top row (its top-edge contribution is carried in shared memory), the element
// left of the strip's first column belongs to the neighbouring strip and is
// recomputed here for that one row block ("halo"), and a segment starts with a
// prologue step that only produces the carry of the row below it.  So no two
// CTAs ever exchange partial sums and the result needs no second pass.
//
// Streaming.  Everything a step reads -- x on its edges, the elements' D4 orbit
// values (d4.cuh; a strip row of one colour is one 32-element chunk record), and
// for the residual / smoothing epilogue r, d and the centrosymmetric D_e^-1 orbits
// of its owned edges -- is a contiguous row range, copied by one thread with
// cp.async.bulk (TMA) into an NS-stage shared-memory ring (one mbarrier per stage),
// NS-1 steps ahead of the step being computed.  dOmega entries of x are masked
// when read (inputs are not required to hold 0 there).  The smoothing step writes its result out of place
// (xo): a neighbouring strip may still be reading x on the shared edges.
// Partition-interface levels, the power iteration and LU-SGS keep the two-colour
// kernels (k_apply.cu).
#include "bodies.cuh"
#include "d4.cuh"

namespace mgdtn {

// one element row of a 64-column strip per step; 4 threads per element (one per edge's
// row block of the element map); 2 CTAs per SM
constexpr int SW_C = 64, SW_R = 1, SW_T = 4 * SW_C * SW_R, SW_W = SW_C + 4;   // staged row width
constexpr int SW_CPS = 2;   // CTAs per SM (SW_R = 2 with 1 CTA per SM: 1052 ms vs 1022 ms per 30 c5 iterations)

__device__ __forceinline__ uint32_t sw_smem(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void sw_bulk(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          sw_smem(dst)),
      "l"(src), "r"(bytes), "r"(sw_smem(bar))
      : "memory");
}
__device__ __forceinline__ void sw_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra W_%=;\n}\n" ::"r"(sw_smem(bar)),
      "r"(parity)
      : "memory");
}
// Edges [e0, e0 + n) of a vector with K doubles per edge are copied from the even edge
// e0 & ~1 on (a bulk copy needs 16-byte aligned source, destination and size; vectors
// are 256-byte aligned and every level has an even edge count, so the rounded range
// stays inside the vector).  Edge e then sits at (e - (e0 & ~1)) * K.
__device__ __forceinline__ uint32_t sw_bytes(int64_t e0, int n, int K) {
  return (uint32_t)((((e0 + n + 1) & ~(int64_t)1) - (e0 & ~(int64_t)1)) * K * 8);
}
// shared-memory layout (doubles) of one pipeline stage and of the step-local buffers.
// A staged row holds up to SW_W edges.
template <int P, int MODE>
struct SweepCfg {
  static constexpr int K1 = P + 1, NORB = D4<P>::NORB, NCS = D4<P>::NCS;
  static constexpr bool R = MODE == AM_RESID || MODE == AM_SMOOTH, SMO = MODE == AM_SMOOTH;
  static constexpr int ROW = SW_W * K1;
  static constexpr int XH = (SW_R + 1) * ROW;               // H rows j0 .. j0+SW_R
  static constexpr int XV = SW_R * ROW;                     // V rows j0 .. j0+SW_R-1
  static constexpr int SS = SW_R * 2 * NORB * 32;           // [rr][colour][o][lane] chunk records
  static constexpr int SH = ((SW_R * NORB + 1) / 2) * 2;    // [rr][o] left halo element
  static constexpr int OWN = 2 * SW_R * SW_C;               // owned edges: H rows, then V rows
  static constexpr int RR = R ? 2 * SW_R * ROW : 0;         // r on the owned rows (H, then V)
  static constexpr int DD = SMO ? 2 * SW_R * ROW : 0;       // d (Chebyshev)
  static constexpr int DS = SMO ? NCS * 2 * SW_R * SW_W : 0;   // [o][row][edge] D_e^-1 orbits
  static constexpr int STAGE = XH + XV + SS + SH + RR + DD + DS;
  static constexpr int Y = 2 * OWN * K1;                    // lo / hi contributions (x2: by step)
  static constexpr int CARRY = 3 * SW_C * K1;               // top-edge contributions, 3 steps
  static constexpr int budget = (216 * 1024 / SW_CPS) / 8 - 2 * Y - CARRY;
  static constexpr int NS = budget / STAGE >= 4 ? 4 : budget / STAGE >= 3 ? 3 : 2;
  static constexpr int DOUBLES = NS * STAGE + 2 * Y + CARRY;
  static constexpr int BYTES = DOUBLES * 8;
};

struct SweepGeom {
  int nstrip, nseg, seg;   // strips of SW_C columns, segments of `seg` rows (multiple of SW_R)
};

// Warp-specialised: warp NCW (the producer) walks the CTA's steps ahead of the
// consumers and fills the NS-stage ring -- bulk copies of the contiguous rows (one
// lane per copy) plus 8-byte cp.async of the left halo element's orbit values, all
// completing on the stage's "full" mbarrier -- after the consumers have released the
// stage on its "empty" mbarrier.  The NCW consumer warps only wait for data: per step
// they form the element contributions, meet at one named barrier, and finish the owned
// edges.  The contribution slots are double-buffered and the row carry triple-buffered
// by step, so one barrier per step orders everything (a warp passes the barrier of
// step k only when every warp has finished the epilogue of step k-1).
constexpr int SW_NCW = SW_T / 32;   // consumer warps

template <int P, int MODE, bool DOT>
__global__ void __launch_bounds__(SW_T + 32, SW_CPS)
    k_apply_sweep(const LevelDev L, SweepGeom G, const double* __restrict__ x, double* y,
                  const double* __restrict__ r, double* d, double* xo, int step,
                  double* __restrict__ partials) {
  using D = D4<P>;
  using C = SweepCfg<P, MODE>;
  constexpr int K1 = P + 1, M = 4 * K1, NORB = D::NORB, NCS = D::NCS, NS = C::NS;
  constexpr int OWN = C::OWN, ROW = C::ROW;
  extern __shared__ __align__(128) double sm[];
  double* Ybuf = sm + NS * C::STAGE;    // [2][lo | hi][OWN][K1]
  double* carry = Ybuf + 2 * C::Y;      // [3][SW_C][K1]
  __shared__ __align__(8) uint64_t full[NS], empty[NS];
  __shared__ double red[SW_NCW];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nx = L.nx, ny = L.ny;
  const int64_t nh = (int64_t)nx * (ny + 1);
  const int nwork = G.nstrip * G.nseg;
  if (tid == 0) {
    for (int q = 0; q < NS; ++q) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 33;" ::"r"(sw_smem(&full[q])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sw_smem(&empty[q])), "r"(SW_NCW));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  pdl_enter();
  double c1 = 0.0, c2 = 0.0;
  if (MODE == AM_SMOOTH) {
    c1 = L.coef[2 * step];
    c2 = L.coef[2 * step + 1];
  }
  const bool cheb_d = MODE == AM_SMOOTH && L.smoother == 1 && step > 0;
  double dot = 0.0;
  int g = 0;   // global step counter of this CTA: stage g % NS, phase (g / NS) & 1
  for (int w = blockIdx.x; w < nwork; w += gridDim.x) {
    const int i0 = (w % G.nstrip) * SW_C, jb = (w / G.nstrip) * G.seg;
    const int je = min(ny, jb + G.seg);
    const int j00 = jb > 0 ? jb - SW_R : 0;   // first step: the prologue (carry only)
    const int nsteps = (je - j00 + SW_R - 1) / SW_R;
    const int lo_i = i0 > 0 ? i0 - 1 : 0;     // first staged column
    const int hi_i = min(i0 + SW_C + 1, nx + 1);
    if (warp == SW_NCW) {
      // ================================================================ producer
      for (int k = 0; k < nsteps; ++k, ++g) {
        const int sidx = g % NS;
        if (g >= NS) sw_wait(&empty[sidx], ((g / NS) - 1) & 1);
        double* st = sm + sidx * C::STAGE;
        const int j0 = j00 + k * SW_R;
        const bool pro = jb > 0 && k == 0;
        // copy idx -> (dst, src, bytes); order: x H rows, x V rows, chunk records, r, d, D
        auto copy_desc = [&](int idx, double*& dst, const double*& src) -> uint32_t {
          if (idx <= SW_R) {
            const int rr = idx;
            if (j0 + rr > ny) return 0;
            const int64_t e0 = (int64_t)(j0 + rr) * nx + lo_i;
            dst = st + rr * ROW;
            src = x + (e0 & ~(int64_t)1) * K1;
            return sw_bytes(e0, i0 + SW_C - lo_i, K1);
          }
          idx -= SW_R + 1;
          if (idx < SW_R) {
            const int rr = idx;
            if (j0 + rr >= ny) return 0;
            const int64_t e0 = nh + (int64_t)(j0 + rr) * (nx + 1) + lo_i;
            dst = st + C::XH + rr * ROW;
            src = x + (e0 & ~(int64_t)1) * K1;
            return sw_bytes(e0, hi_i - lo_i, K1);
          }
          idx -= SW_R;
          if (idx < 2 * SW_R) {
            const int rr = idx >> 1, cl = idx & 1;
            if (j0 + rr >= ny) return 0;
            const int64_t q = ((int64_t)(j0 + rr) * (nx >> 1) + (i0 >> 1)) >> 5;
            dst = st + C::XH + C::XV + (rr * 2 + cl) * NORB * 32;
            src = L.So + ((int64_t)cl * L.nchunk + q) * NORB * 32;
            return NORB * 256;
          }
          idx -= 2 * SW_R;
          if (!C::R || pro) return 0;
          const int nvec = C::SMO ? (cheb_d ? 2 + NCS : 1 + NCS) : 1;
          if (idx >= nvec * 2 * SW_R) return 0;
          const int vq = idx / (2 * SW_R), row = idx % (2 * SW_R), hv = row / SW_R, rr = row % SW_R;
          if (j0 + rr >= je) return 0;
          const int64_t e0 = hv == 0 ? (int64_t)(j0 + rr) * nx + i0 : nh + (int64_t)(j0 + rr) * (nx + 1) + i0;
          double* RR = st + C::XH + C::XV + C::SS + C::SH;
          if (vq == 0) {
            dst = RR + row * ROW;
            src = r + (e0 & ~(int64_t)1) * K1;
            return sw_bytes(e0, SW_C, K1);
          }
          if (C::SMO && cheb_d && vq == 1) {
            dst = RR + C::RR + row * ROW;
            src = d + (e0 & ~(int64_t)1) * K1;
            return sw_bytes(e0, SW_C, K1);
          }
          const int o = vq - (cheb_d ? 2 : 1);
          const int64_t f0 = (int64_t)o * L.nedge + e0;
          dst = RR + C::RR + C::DD + (o * 2 * SW_R + row) * SW_W;
          src = L.Dso + (f0 & ~(int64_t)1);
          return sw_bytes(f0, SW_C, 1);
        };
        constexpr int NCOPY = (SW_R + 1) + SW_R + 2 * SW_R + (C::SMO ? (2 + NCS) : C::R ? 1 : 0) * 2 * SW_R;
        constexpr int NU = (NCOPY + 31) / 32;
        double* dsts[NU];
        const double* srcs[NU];
        uint32_t nb[NU];
        uint32_t mine = 0;
#pragma unroll
        for (int u = 0; u < NU; ++u) {
          nb[u] = 0;
          if (lane + 32 * u < NCOPY) nb[u] = copy_desc(lane + 32 * u, dsts[u], srcs[u]);
          mine += nb[u];
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, o);
        if (lane == 0)
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sw_smem(&full[sidx])),
                       "r"(mine)
                       : "memory");
        __syncwarp();
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
#pragma unroll
        for (int u = 0; u < NU; ++u)
          if (nb[u]) sw_bulk(dsts[u], srcs[u], nb[u], &full[sidx]);
        // the left halo element's orbit values (scattered: 8-byte cp.async)
        if (!pro && i0 > 0) {
          for (int q = lane; q < SW_R * NORB; q += 32) {
            const int rr = q / NORB, o = q - rr * NORB, j = j0 + rr;
            const bool v = j < je;
            const double* src = L.So;
            if (v) {
              int colour;
              int64_t s;
              elem_slot(nx, i0 - 1, j, colour, s);
              src = L.So + ((((int64_t)colour * L.nchunk + (s >> 5)) * NORB + o) << 5) + (s & 31);
            }
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(
                             sw_smem(st + C::XH + C::XV + C::SS + q)),
                         "l"(src), "r"(v ? 8 : 0)
                         : "memory");
          }
        }
        asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(sw_smem(&full[sidx]))
                     : "memory");
      }
      continue;
    }
    // ================================================================ consumers
    for (int k = 0; k < nsteps; ++k, ++g) {
      const int sidx = g % NS;
      sw_wait(&full[sidx], (g / NS) & 1);
      const double* st = sm + sidx * C::STAGE;
      const double* XH = st;
      const double* XV = XH + C::XH;
      const double* SS = XV + C::XV;
      const double* SH = SS + C::SS;
      const double* RR = SH + C::SH;
      const double* DD = RR + C::RR;
      const double* DS = DD + C::DD;
      const int j0 = j00 + k * SW_R;
      const bool pro = jb > 0 && k == 0;
      double* Ylo = Ybuf + (g & 1) * C::Y;
      double* Yhi = Ylo + OWN * K1;
      const double* cold = carry + (g % 3) * SW_C * K1;
      double* cnew = carry + ((g + 1) % 3) * SW_C * K1;
      // staged edge position of H(i, j0+rr) / V(i, j0+rr): i - i0 + hoff / voff[rr]
      const int hoff = (int)((lo_i + (int64_t)j0 * nx) & 1) + (i0 - lo_i);   // nx even: every row
      int voff[SW_R];
#pragma unroll
      for (int rr = 0; rr < SW_R; ++rr)
        voff[rr] = (int)((nh + (int64_t)(j0 + rr) * (nx + 1) + lo_i) & 1) + (i0 - lo_i);
      // ---- elements: four threads per element, thread f forming the row block of edge f,
      // y_f = S_T[f, :] x_T.  A warp holds one edge role of the 32 elements of one colour
      // of the row, so its orbit reads are one conflict-free 256-byte row of the record.
      {
        const int rr = warp / 8, wr = warp % 8, f = wr >> 1, col = wr & 1;
        const int j = j0 + rr;
        const int cc = 2 * lane + ((col + j) & 1), i = i0 + cc;
        if (j < je) {
          double xv[M];
          const double* xb = XH + rr * ROW + (cc + hoff) * K1;         // H(i, j)
          const double* xt = XH + (rr + 1) * ROW + (cc + hoff) * K1;   // H(i, j+1)
          const double* xl = XV + rr * ROW + (cc + voff[rr]) * K1;     // V(i, j)
          const double* xr = xl + K1;                                  // V(i+1, j)
          const bool mb = j == 0, mt = j + 1 == ny, ml = i == 0, mr = i + 1 == nx;   // dOmega
#pragma unroll
          for (int a = 0; a < K1; ++a) {
            xv[0 * K1 + a] = mb ? 0.0 : xb[a];
            xv[1 * K1 + a] = mr ? 0.0 : xr[a];
            xv[2 * K1 + a] = mt ? 0.0 : xt[a];
            xv[3 * K1 + a] = ml ? 0.0 : xl[a];
          }
          const double* Sp = SS + (rr * 2 + col) * NORB * 32 + lane;
          double yv[K1];
#define SW_ROWS(FF)                                                                   \
  _Pragma("unroll") for (int a = 0; a < K1; ++a) {                                    \
    double acc = 0.0;                                                                 \
    _Pragma("unroll") for (int b = 0; b < M; ++b)                                     \
        acc = fma(Sp[D::orb(D::pk((FF) * K1 + a, b)) * 32], xv[b], acc);              \
    yv[a] = acc;                                                                      \
  }
          if (f == 0) { SW_ROWS(0) } else if (f == 1) { SW_ROWS(1) }
          else if (f == 2) { SW_ROWS(2) } else { SW_ROWS(3) }
#undef SW_ROWS
          if (f == 2) {   // top edge: the next row's bottom edge (carry after the last row)
            double* dst = rr + 1 < SW_R ? Ylo + ((rr + 1) * SW_C + cc) * K1 : cnew + cc * K1;
#pragma unroll
            for (int a = 0; a < K1; ++a) dst[a] = yv[a];
          } else if (!pro) {
            const int hq = rr * SW_C + cc, vq = SW_R * SW_C + rr * SW_C + cc;
            double* dst = f == 0 ? Yhi + hq * K1                                        // bottom
                        : f == 3 ? Yhi + vq * K1                                        // left
                        : (cc + 1 < SW_C ? Ylo + (vq + 1) * K1 : nullptr);              // right
            if (dst) {
#pragma unroll
              for (int a = 0; a < K1; ++a) dst[a] = yv[a];
            }
          }
        }
        // the left neighbour strip's element (i0-1, j0): row block of its right edge,
        // one thread per row (orbit values staged in SH)
        if (!pro && i0 > 0 && tid < SW_R * K1 && j0 + tid / K1 < je) {
          const int hr = tid / K1, a = tid % K1, ih = i0 - 1, jh = j0 + hr;
          double xv[M];
          const double* xb = XH + hr * ROW + (hoff - 1) * K1;
          const double* xt = XH + (hr + 1) * ROW + (hoff - 1) * K1;
          const double* xl = XV + hr * ROW + (voff[hr] - 1) * K1;
          const double* xr = xl + K1;
          const bool mb = jh == 0, mt = jh + 1 == ny, ml = ih == 0;
#pragma unroll
          for (int q = 0; q < K1; ++q) {
            xv[0 * K1 + q] = mb ? 0.0 : xb[q];
            xv[1 * K1 + q] = xr[q];
            xv[2 * K1 + q] = mt ? 0.0 : xt[q];
            xv[3 * K1 + q] = ml ? 0.0 : xl[q];
          }
          double acc = 0.0;
#pragma unroll
          for (int b = 0; b < M; ++b) {
            int o = 0;
#pragma unroll
            for (int q = 0; q < K1; ++q)
              if (q == a) o = D::orb(D::pk(K1 + q, b));
            acc = fma(SH[hr * NORB + o], xv[b], acc);
          }
          Ylo[(SW_R * SW_C + hr * SW_C) * K1 + a] = acc;
        }
      }
      asm volatile("bar.sync 1, %0;" ::"n"(SW_T) : "memory");   // consumers only
      // ---- owned edges (thread per edge): y_e = lo + hi, then the epilogue
      if (!pro) {
        for (int q = tid; q < OWN + SW_R + SW_C; q += SW_T) {
          int64_t e;
          bool bnd;
          const double* xs = nullptr;
          int ro = 0;   // staged position in the r / d rows and the D rows
          double yy[K1];
          if (q >= OWN) {   // the mesh's right / top boundary edges next to this step
            const int u = q - OWN;
            if (u < SW_R) {
              if (i0 + SW_C != nx || j0 + u >= je) continue;
              e = nh + (int64_t)(j0 + u) * (nx + 1) + nx;
            } else {
              if (je != ny || j0 + SW_R < ny) continue;
              e = (int64_t)ny * nx + i0 + (u - SW_R);
            }
            bnd = true;
          } else {
            const int hv = q / (SW_R * SW_C), rr = (q / SW_C) % SW_R, cc = q % SW_C;
            const int i = i0 + cc, j = j0 + rr;
            if (j >= je) continue;
            int64_t e0;
            if (hv == 0) {
              e0 = (int64_t)j * nx + i0;
              bnd = j == 0;
              xs = XH + rr * ROW + (cc + hoff) * K1;
            } else {
              e0 = nh + (int64_t)j * (nx + 1) + i0;
              bnd = i == 0;
              xs = XV + rr * ROW + (cc + voff[rr]) * K1;
            }
            e = e0 + cc;
            ro = (hv * SW_R + rr) * SW_W + cc + (int)(e0 & 1);   // rows start at e0 & ~1
            if (!bnd) {
              const double* lo = (hv == 0 && rr == 0) ? cold + cc * K1 : Ylo + q * K1;
#pragma unroll
              for (int a = 0; a < K1; ++a) yy[a] = lo[a] + Yhi[q * K1 + a];
            }
          }
          const int64_t base = e * K1;
          double out[K1];
          if (bnd) {   // dOmega: y = 0; the smoothed iterate keeps 0 there
#pragma unroll
            for (int a = 0; a < K1; ++a) out[a] = 0.0;
            st_edge<K1>((MODE == AM_SMOOTH ? xo : y) + base, out);
            continue;
          }
          if (MODE == AM_APPLY) {
#pragma unroll
            for (int a = 0; a < K1; ++a) {
              out[a] = yy[a];
              if (DOT) dot = fma(xs[a], yy[a], dot);
            }
            st_edge<K1>(y + base, out);
          } else if (MODE == AM_RESID) {
#pragma unroll
            for (int a = 0; a < K1; ++a) out[a] = RR[ro * K1 + a] - yy[a];
            st_edge<K1>(y + base, out);
          } else {   // AM_SMOOTH: res = r - A x, dn = c2 D^-1 res (+ c1 d), d = dn, xo = x + dn
            double res[K1], dn[K1];
#pragma unroll
            for (int a = 0; a < K1; ++a) res[a] = RR[ro * K1 + a] - yy[a];
#pragma unroll
            for (int a = 0; a < K1; ++a) {
              double cc2 = 0.0;
#pragma unroll
              for (int b = 0; b < K1; ++b)
                cc2 = fma(DS[D::cs(D::pe(a, b)) * 2 * SW_R * SW_W + ro], res[b], cc2);
              dn[a] = c2 * cc2;
              if (L.smoother == 1 && step > 0) dn[a] = fma(c1, DD[ro * K1 + a], dn[a]);
              out[a] = xs[a] + dn[a];
            }
            if (L.smoother == 1) st_edge<K1>(d + base, dn);
            st_edge<K1>(xo + base, out);
          }
        }
      }
      __syncwarp();
      if (lane == 0)
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sw_smem(&empty[sidx])) : "memory");
    }
  }
  if (DOT && warp < SW_NCW) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
    if (lane == 0) red[warp] = dot;
    asm volatile("bar.sync 1, %0;" ::"n"(SW_T) : "memory");
    if (tid == 0) {
      double s = 0.0;
      for (int q = 0; q < SW_NCW; ++q) s += red[q];
      partials[blockIdx.x] = s;
    }
  }
}

static int sweep_sms() {
  static int v = 0;
  if (v == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    if (v <= 0) v = 148;
  }
  return v;
}

// Strips x segments: segments of at least 8 steps while there are enough of them to
// give every SM a few work items; a persistent grid of one CTA per SM walks them.
static SweepGeom sweep_geom(const LevelDev& L) {
  SweepGeom g;
  g.nstrip = (L.nx + SW_C - 1) / SW_C;
  const int want = 4 * SW_CPS * sweep_sms();
  int seg = (int)(((int64_t)L.ny * g.nstrip + want - 1) / want);
  seg = ((seg + SW_R - 1) / SW_R) * SW_R;
  if (seg < 8 * SW_R) seg = 8 * SW_R;
  if (seg > L.ny) seg = ((L.ny + SW_R - 1) / SW_R) * SW_R;
  g.seg = seg;
  g.nseg = (L.ny + seg - 1) / seg;
  return g;
}

// strips must be whole chunks of the orbit records (64 columns, nx % 64 == 0); other
// meshes keep the two-colour passes, and so do meshes too small to give every SM a
// few segments of >= 16 rows (config 2's 256 x 256: 64 work items for 148 SMs)
// Off by default (MG_OPT_SWEEP = 1 turns it on): with the dependents of every pass released
// at its exit, the two-colour orbit passes are as fast at config 5 (38.7 ms per iteration
// either way) and faster at config 3 (2428 vs 3127 ms; the p <= 2 sweep loses to the
// 2-4 KB-per-chunk orbit ring), profiles/r02_sweep_probe.txt.
bool tile_level(const LevelDev& L) {
  return L.sweep > 0 && L.orb && L.imask == 0 && !L.ns && L.nx % SW_C == 0;
}

int apply_tile_grid(const LevelDev& L) {
  const SweepGeom g = sweep_geom(L);
  int n = g.nstrip * g.nseg;
  if (L.grid_cap > 0 && n > L.grid_cap) n = L.grid_cap;
  return n < SW_CPS * sweep_sms() ? n : SW_CPS * sweep_sms();
}

template <int P, int MODE, bool DOT>
static void launch_sweep_t(const LevelDev& L, const double* x, double* y, const double* r,
                           double* d, double* xo, int step, double* partials, cudaStream_t st) {
  using C = SweepCfg<P, MODE>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_apply_sweep<P, MODE, DOT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         C::BYTES);
    attr = true;
  }
  launch_ex(k_apply_sweep<P, MODE, DOT>, apply_tile_grid(L), SW_T + 32, (size_t)C::BYTES, true, st, L,
            sweep_geom(L), x, y, r, d, xo, step, partials);
}

template <int P>
static void launch_sweep_p(const LevelDev& L, int mode, const double* x, double* y, const double* r,
                           double* d, double* xo, int step, double* partials, cudaStream_t st) {
  switch (mode) {
    case AM_APPLY:
      if (partials) launch_sweep_t<P, AM_APPLY, true>(L, x, y, r, d, xo, step, partials, st);
      else launch_sweep_t<P, AM_APPLY, false>(L, x, y, r, d, xo, step, partials, st);
      break;
    case AM_RESID: launch_sweep_t<P, AM_RESID, false>(L, x, y, r, d, xo, step, partials, st); break;
    default: launch_sweep_t<P, AM_SMOOTH, false>(L, x, y, r, d, xo, step, partials, st); break;
  }
}

int launch_apply_tile(const LevelDev& L, int mode, const double* x, double* y, const double* r,
                      double* d, double* xo, int step, double* partials, cudaStream_t st) {
  switch (L.p) {
    case 1: launch_sweep_p<1>(L, mode, x, y, r, d, xo, step, partials, st); break;
    case 2: launch_sweep_p<2>(L, mode, x, y, r, d, xo, step, partials, st); break;
    case 3: launch_sweep_p<3>(L, mode, x, y, r, d, xo, step, partials, st); break;
    default: launch_sweep_p<4>(L, mode, x, y, r, d, xo, step, partials, st); break;
  }
  return 1;
}

}  // namespace mgdtn
