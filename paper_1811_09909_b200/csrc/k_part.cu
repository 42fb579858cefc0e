// Partitioned levels (multi-GPU): kernels around the halo
// exchange of partition-interface edges.
//
// Elements are sharded in px x py blocks; each rank stores every edge of its
// elements, so an edge on a partition interface is held by the two ranks that
// share it.  The trace apply y = sum_T G_T^T S_T G_T x is a
// sum over elements, so on an interface edge each rank holds only its own
// elements' partial sum after the local colour passes; the ranks exchange those
// partial sums (one message per neighbour) and finish the edge in
// k_itf_epilogue.  Every two-term sum is commutative in IEEE arithmetic, and the
// three-term restriction sum is evaluated as J^T res + (own + remote), so both
// copies of a duplicated dof receive bitwise the same value on both ranks and
// the iterates stay consistent without any broadcast.
//
// Buffer layout (per level and direction): [4 sides][max(nx, ny) * k1] doubles,
// side f holds its edges in side_edge() order (the neighbour's matching side
// lists the same global edges in the same order).
#include "bodies.cuh"

namespace mgdtn {

#define GTID ((int64_t)blockIdx.x * blockDim.x + threadIdx.x)
#define GNT ((int64_t)gridDim.x * blockDim.x)

static inline int grid_for(int64_t work, int threads, int cap) {
  int64_t g = (work + threads - 1) / threads;
  if (g < 1) g = 1;
  return (int)(g < cap ? g : cap);
}

int itf_stride(const LevelDev& L) { return (L.nx > L.ny ? L.nx : L.ny) * L.k1; }

// total interface edges of a level (the 4 sides are enumerated one after the other)
__device__ __forceinline__ bool itf_item(const LevelDev& L, int64_t w, int& f, int& q) {
  for (f = 0; f < 4; ++f) {
    const int n = ((L.imask >> f) & 1) ? side_len(L.nx, L.ny, f) : 0;
    if (w < n) {
      q = (int)w;
      return true;
    }
    w -= n;
  }
  return false;
}

__host__ __device__ int64_t itf_edges(const LevelDev& L) {
  int64_t n = 0;
  for (int f = 0; f < 4; ++f)
    if ((L.imask >> f) & 1) n += side_len(L.nx, L.ny, f);
  return n;
}

// ---------------------------------------------------------------- apply halo
__global__ void k_itf_pack(LevelDev L, const double* __restrict__ y, double* send, int stride) {
  pdl_enter();
  const int K1 = L.k1;
  const int64_t n = itf_edges(L);
  for (int64_t w = GTID; w < n; w += GNT) {
    int f, q;
    itf_item(L, w, f, q);
    const int64_t e = side_edge(L.nx, L.ny, f, q);
    for (int a = 0; a < K1; ++a) send[(int64_t)f * stride + q * K1 + a] = y[e * K1 + a];
  }
}

int launch_itf_pack(const LevelDev& L, const double* y, double* send, cudaStream_t st) {
  launch_ex(k_itf_pack, grid_for(itf_edges(L), 128, 148), 128, 0, true, st, L, y, send,
            itf_stride(L));
  return 1;
}

constexpr int ITF_BLOCKS = 16;   // fixed grid of the interface epilogue (partials slots)

// Finish an apply on the interface edges: y_full = y_own + y_remote, then the
// colour-1 epilogue of `mode` (bodies.cuh epi_store) on those edges.  DOT:
// dot-product partials of the edges this rank owns, into partials[0..ITF_BLOCKS).
template <int MODE, bool DOT>
__global__ void __launch_bounds__(128) k_itf_epilogue(LevelDev L, double* x, double* y,
                                                      const double* __restrict__ r, double* d,
                                                      int step, const double* __restrict__ recv,
                                                      int stride, double* partials) {
  pdl_enter();
  const int K1 = L.k1;
  const int64_t n = itf_edges(L);
  const int nomask = nonowned_mask(L.imask);
  double c1 = 0.0, c2 = 0.0;
  if (MODE == AM_SMOOTH) {
    c1 = L.coef[2 * step];
    c2 = L.coef[2 * step + 1];
  }
  double dot = 0.0;
  for (int64_t w = GTID; w < n; w += GNT) {
    int f, q;
    itf_item(L, w, f, q);
    const int64_t e = side_edge(L.nx, L.ny, f, q);
    const int64_t base = e * K1;
    const bool own = !((nomask >> f) & 1);
    double yf[MAX_K1];
    for (int a = 0; a < K1; ++a) yf[a] = y[base + a] + recv[(int64_t)f * stride + q * K1 + a];
    if (MODE == AM_APPLY) {
      for (int a = 0; a < K1; ++a) {
        y[base + a] = yf[a];
        if (DOT && own) dot = fma(x[base + a], yf[a], dot);
      }
    } else if (MODE == AM_RESID) {
      for (int a = 0; a < K1; ++a) y[base + a] = r[base + a] - yf[a];
    } else {
      double res[MAX_K1];
      for (int a = 0; a < K1; ++a) {
        if (MODE == AM_DINV) {
          res[a] = yf[a];
          y[base + a] = yf[a];
        } else {
          res[a] = r[base + a] - yf[a];
        }
      }
      const double* Di = L.Dinv + e;
      for (int a = 0; a < K1; ++a) {
        double c = 0.0;
        for (int b = 0; b < K1; ++b) c = fma(Di[(int64_t)(a * K1 + b) * L.nedge], res[b], c);
        if (MODE == AM_DINV) {
          x[base + a] = c;
          if (DOT && own) dot = fma(c, res[a], dot);
        } else {
          double dn = c2 * c;
          if (L.smoother == 1) {
            if (step > 0) dn = fma(c1, d[base + a], dn);
            d[base + a] = dn;
          }
          x[base + a] += dn;
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

int itf_blocks() { return ITF_BLOCKS; }

int launch_itf_epilogue(const LevelDev& L, int mode, double* x, double* y, const double* r,
                        double* d, int step, const double* recv, double* partials,
                        cudaStream_t st) {
  const int s = itf_stride(L);
  const int g = ITF_BLOCKS;
  switch (mode) {
    case AM_APPLY:
      if (partials)
        launch_ex(k_itf_epilogue<AM_APPLY, true>, g, 128, 0, true, st, L, x, y, r, d, step, recv,
                  s, partials);
      else
        launch_ex(k_itf_epilogue<AM_APPLY, false>, g, 128, 0, true, st, L, x, y, r, d, step, recv,
                  s, partials);
      break;
    case AM_RESID:
      launch_ex(k_itf_epilogue<AM_RESID, false>, g, 128, 0, true, st, L, x, y, r, d, step, recv, s,
                partials);
      break;
    case AM_DINV:
      if (partials)
        launch_ex(k_itf_epilogue<AM_DINV, true>, g, 128, 0, true, st, L, x, y, r, d, step, recv,
                  s, partials);
      else
        launch_ex(k_itf_epilogue<AM_DINV, false>, g, 128, 0, true, st, L, x, y, r, d, step, recv,
                  s, partials);
      break;
    default:
      launch_ex(k_itf_epilogue<AM_SMOOTH, false>, g, 128, 0, true, st, L, x, y, r, d, step, recv,
                s, partials);
      break;
  }
  return 1;
}

// ---------------------------------------------------------------- restriction halo
// own macro's P_M^T res_I term on every interface coarse edge of C (slots of the
// macro's local coarse edges: bottom 0,1  right 2,3  top 4,5  left 6,7)
__global__ void k_restrict_pack(LevelDev C, const double* __restrict__ cbuf, double* send,
                                int stride) {
  pdl_enter();
  const int64_t n = itf_edges(C);
  const int nxc = C.nx, nyc = C.ny;
  for (int64_t w = GTID; w < n; w += GNT) {
    int f, q;
    itf_item(C, w, f, q);
    int64_t M;
    int slot;
    if (f == 0) { M = q; slot = 0; }
    else if (f == 2) { M = (int64_t)(nyc - 1) * nxc + q; slot = 4; }
    else if (f == 3) { M = (int64_t)q * nxc; slot = 6; }
    else { M = (int64_t)q * nxc + nxc - 1; slot = 2; }
    send[(int64_t)f * stride + q * 2] = cbuf[M * 8 + slot];
    send[(int64_t)f * stride + q * 2 + 1] = cbuf[M * 8 + slot + 1];
  }
}

// rc = J^T res + (own + remote) on the interface coarse edges (+ the fused first
// smoothing step of the coarse level, as restrict_edges_body does elsewhere)
__global__ void k_restrict_itf(LevelDev C, double* rc, const double* __restrict__ send,
                               const double* __restrict__ recv, int stride, int fuse, double* ec,
                               double* dc) {
  pdl_enter();
  const int64_t n = itf_edges(C);
  const double c2 = fuse ? C.coef[1] : 0.0;
  for (int64_t w = GTID; w < n; w += GNT) {
    int f, q;
    itf_item(C, w, f, q);
    const int64_t E = side_edge(C.nx, C.ny, f, q);
    const int64_t o = (int64_t)f * stride + q * 2;
    const double v0 = rc[E * 2] + (send[o] + recv[o]);
    const double v1 = rc[E * 2 + 1] + (send[o + 1] + recv[o + 1]);
    rc[E * 2] = v0;
    rc[E * 2 + 1] = v1;
    if (fuse) {
      const double* Di = C.Dinv + E;
      const int64_t sd = C.nedge;
      const double e0 = c2 * (Di[0] * v0 + Di[sd] * v1);
      const double e1 = c2 * (Di[2 * sd] * v0 + Di[3 * sd] * v1);
      ec[E * 2] = e0;
      ec[E * 2 + 1] = e1;
      if (C.smoother == 1) {
        dc[E * 2] = e0;
        dc[E * 2 + 1] = e1;
      }
    }
  }
}

int launch_restrict_halo_pack(const LevelDev& C, const double* cbuf, double* send,
                              cudaStream_t st) {
  launch_ex(k_restrict_pack, grid_for(itf_edges(C), 128, 148), 128, 0, true, st, C, cbuf, send,
            itf_stride(C));
  return 1;
}

int launch_restrict_halo_finish(const LevelDev& C, double* rc, const double* send,
                                const double* recv, bool fuse, double* ec, double* dc,
                                cudaStream_t st) {
  launch_ex(k_restrict_itf, grid_for(itf_edges(C), 128, 148), 128, 0, true, st, C, rc, send, recv,
            itf_stride(C), fuse ? 1 : 0, ec, dc);
  return 1;
}

// ---------------------------------------------------------------- edge blocks on interfaces
// k_edge_blocks leaves this rank's partial D_e (not inverted) in Dinv on the
// interface edges; pack it, and after the exchange invert D_own + D_remote.
__global__ void k_eblk_pack(LevelDev L, double* send, int stride) {
  const int K1 = L.k1;
  const int64_t n = itf_edges(L);
  for (int64_t w = GTID; w < n; w += GNT) {
    int f, q;
    itf_item(L, w, f, q);
    const int64_t e = side_edge(L.nx, L.ny, f, q);
    for (int t = 0; t < K1 * K1; ++t)
      send[(int64_t)f * stride + (int64_t)q * K1 * K1 + t] = L.Dinv[(int64_t)t * L.nedge + e];
  }
}

__global__ void k_eblk_finish(LevelDev L, const double* __restrict__ recv, int stride,
                              DevError* err) {
  const int K1 = L.k1;
  const int64_t n = itf_edges(L);
  for (int64_t w = GTID; w < n; w += GNT) {
    int f, q;
    itf_item(L, w, f, q);
    const int64_t e = side_edge(L.nx, L.ny, f, q);
    double D[MAX_K1 * MAX_K1];
    for (int t = 0; t < K1 * K1; ++t)
      D[t] = L.Dinv[(int64_t)t * L.nedge + e] + recv[(int64_t)f * stride + (int64_t)q * K1 * K1 + t];
    double inv[MAX_K1 * MAX_K1];
    if (!chol_inverse(D, K1, inv)) report_error(err, -4, e);
    for (int t = 0; t < K1 * K1; ++t) L.Dinv[(int64_t)t * L.nedge + e] = inv[t];
  }
}

int eblk_stride(const LevelDev& L) { return (L.nx > L.ny ? L.nx : L.ny) * L.k1 * L.k1; }

int launch_eblk_pack(const LevelDev& L, double* send, cudaStream_t st) {
  k_eblk_pack<<<grid_for(itf_edges(L), 128, 148), 128, 0, st>>>(L, send, eblk_stride(L));
  return 1;
}
int launch_eblk_finish(const LevelDev& L, const double* recv, DevError* err, cudaStream_t st) {
  k_eblk_finish<<<grid_for(itf_edges(L), 128, 148), 128, 0, st>>>(L, recv, eblk_stride(L), err);
  return 1;
}

// ---------------------------------------------------------------- gather level (local <-> replicated global)
// rank blocks: rank = ry * px + rx owns global elements [rx*bx, (rx+1)*bx) x [ry*by, (ry+1)*by)
// of the level; `all` = the allgathered local vectors [nranks][ndof_loc].
__device__ __forceinline__ void global_to_local_edge(int64_t Eg, int nxg, int nyg, int bx, int by,
                                                     int px, int py, int& rank, int64_t& el) {
  const int64_t nhg = (int64_t)nxg * (nyg + 1);
  if (Eg < nhg) {
    const int gj = (int)(Eg / nxg), gi = (int)(Eg - (int64_t)gj * nxg);
    const int rx = gi / bx;
    int ry = gj / by;
    if (ry > py - 1) ry = py - 1;
    rank = ry * px + rx;
    el = hedge(bx, gi - rx * bx, gj - ry * by);
  } else {
    const int64_t r = Eg - nhg;
    const int gj = (int)(r / (nxg + 1)), gi = (int)(r - (int64_t)gj * (nxg + 1));
    int rx = gi / bx;
    if (rx > px - 1) rx = px - 1;
    const int ry = gj / by;
    rank = ry * px + rx;
    el = vedge(bx, by, gi - rx * bx, gj - ry * by);
  }
}

__global__ void k_gather_vec(LevelDev G, int bx, int by, int px, int py, int64_t ndof_loc,
                             const double* __restrict__ all, double* out) {
  pdl_enter();
  const int K1 = G.k1;
  for (int64_t Eg = GTID; Eg < G.nedge; Eg += GNT) {
    int rank;
    int64_t el;
    global_to_local_edge(Eg, G.nx, G.ny, bx, by, px, py, rank, el);
    for (int a = 0; a < K1; ++a) out[Eg * K1 + a] = all[(int64_t)rank * ndof_loc + el * K1 + a];
  }
}

__global__ void k_scatter_vec(LevelDev Lc, int ox, int oy, int nxg, int nyg,
                              const double* __restrict__ glob, double* loc) {
  pdl_enter();
  const int K1 = Lc.k1;
  const int64_t nh = (int64_t)Lc.nx * (Lc.ny + 1);
  const int64_t nhg = (int64_t)nxg * (nyg + 1);
  for (int64_t e = GTID; e < Lc.nedge; e += GNT) {
    int64_t Eg;
    if (e < nh) {
      const int j = (int)(e / Lc.nx), i = (int)(e - (int64_t)j * Lc.nx);
      Eg = (int64_t)(oy + j) * nxg + (ox + i);
    } else {
      const int64_t r = e - nh;
      const int j = (int)(r / (Lc.nx + 1)), i = (int)(r - (int64_t)j * (Lc.nx + 1));
      Eg = nhg + (int64_t)(oy + j) * (nxg + 1) + (ox + i);
    }
    for (int a = 0; a < K1; ++a) loc[e * K1 + a] = glob[Eg * K1 + a];
  }
}

// allgathered dense local element maps [nranks][ne_loc][m][m] -> the global level's packed S
__global__ void k_gather_S(LevelDev G, int bx, int by, int px, const double* __restrict__ dense) {
  const int m = G.m;
  for (int64_t eg = GTID; eg < G.ne; eg += GNT) {
    const int gj = (int)(eg / G.nx), gi = (int)(eg - (int64_t)gj * G.nx);
    const int rank = (gj / by) * px + gi / bx;
    const int64_t el = (int64_t)(gj % by) * bx + (gi % bx);
    const double* src = dense + ((int64_t)rank * bx * by + el) * m * m;
    int colour;
    int64_t s;
    elem_slot(G.nx, gi, gj, colour, s);
    double* dst = G.S + s_offset(G.nchunk, G.npk, colour, s, 0);
    for (int a = 0; a < m; ++a)
      for (int b = a; b < m; ++b) dst[(int64_t)pk_index(a, b, m) * 32] = src[a * m + b];
  }
}

int launch_gather_vec(const LevelDev& G, int bx, int by, int px, int py, int64_t ndof_loc,
                      const double* all, double* out, cudaStream_t st) {
  launch_ex(k_gather_vec, grid_for(G.nedge, 128, 148 * 8), 128, 0, true, st, G, bx, by, px, py,
            ndof_loc, all, out);
  return 1;
}
int launch_scatter_vec(const LevelDev& Lc, int ox, int oy, int nxg, int nyg, const double* glob,
                       double* loc, cudaStream_t st) {
  launch_ex(k_scatter_vec, grid_for(Lc.nedge, 128, 148 * 8), 128, 0, true, st, Lc, ox, oy, nxg,
            nyg, glob, loc);
  return 1;
}
int launch_gather_S(const LevelDev& G, int bx, int by, int px, const double* dense,
                    cudaStream_t st) {
  k_gather_S<<<grid_for(G.ne, 128, 148 * 8), 128, 0, st>>>(G, bx, by, px, dense);
  return 1;
}

}  // namespace mgdtn
