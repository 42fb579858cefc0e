// Setup kernels: batched element-local static condensation (H1), the
// right-hand side, p-coarsening (H2), per-agglomerate Galerkin coarse DtN
// (H3), edge-block diagonals (H4) and the coarsest dense factor (H5).
#include <cstdlib>

#include "bodies.cuh"
#include "d4.cuh"

namespace mgdtn {

// ============================================================================
// H1: element DtN maps.  PAPER.md:305-316 ("express the local volume unknowns
// ... element-by-element, as a function of the skeletal unknowns"); HDG
// Eqs. HDG/HDG_flux, SIPG-H Eq. SIPG_H.
// After eliminating u (HDG) the local problem of a side-h square is
//   Q q = R lambda + f_w,  flux = R^T q - S0 lambda,   Q = K A + t F, t = tau h,
// so S_T = S0 - R^T Q^-1 R and b_T = R^T Q^-1 f_w.  The pencil (A, F) is
// diagonalised once per p on the host (refelem.h RefTables::Pencil:
// T Q T^T = diag(d_i), d_i = K lam_i + t mu_i), which turns the batched
// per-element factorisation into a sum of rank-1 terms with per-element weights:
//   S_T[a][b] = S0[a][b] - sum_i w_ia w_ib / d_i,   w_i = t At_i + K Bk_i.
// CTA = M/2 warps on one chunk of 32 same-colour elements (the S_T layout of
// kernels.cuh); lane = element, warp w owns rows w and M-1-w (balanced), so each
// packed entry is written by one lane as a coalesced 256-byte warp store.  No
// factorisation, no serial dependency: ~NV*NPK*2 FMA per element.
// ============================================================================
__device__ __forceinline__ void pk_row_col(int kk, int m, int& i, int& j) {
  i = 0;
  int rowlen = m;
  while (kk >= rowlen) {
    kk -= rowlen;
    ++i;
    --rowlen;
  }
  j = i + kk;
}

template <int P>
struct LocalShape {
  static constexpr int K1 = P + 1, NV = K1 * K1, M = 4 * K1, NPK = M * (M + 1) / 2;
};

template <int P>
__global__ void __launch_bounds__(32 * (2 * (P + 1))) k_local_dtn(LevelDev L, RefDev R, double h,
                                                              const double* __restrict__ K,
                                                              const int8_t* __restrict__ method,
                                                              const double* __restrict__ tau,
                                                              DevError* err, int project) {
  using Sh = LocalShape<P>;
  constexpr int NV = Sh::NV, M = Sh::M, NPK = Sh::NPK, NW = M / 2;
  __shared__ double sAt[2][NV * M], sBk[2][NV * M];
  __shared__ double sW[M * M], sH[M * M];
  __shared__ double sc[NV][32];   // 1 / d_i per lane-element
  __shared__ double srow[M][32];  // row sums S_T 1 per lane-element (projection)
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int q = threadIdx.x; q < NV * M; q += blockDim.x) {
    sAt[0][q] = R.pAt[0][q];
    sAt[1][q] = R.pAt[1][q];
    sBk[0][q] = R.pBk[0][q];
    sBk[1][q] = R.pBk[1][q];
  }
  for (int q = threadIdx.x; q < M * M; q += blockDim.x) {
    sW[q] = R.W[q];
    sH[q] = R.H[q];
  }
  const int64_t nec = L.ne >> 1;
  const int64_t nchunk_tot = 2 * (int64_t)L.nchunk;
  for (int64_t cc = blockIdx.x; cc < nchunk_tot; cc += gridDim.x) {
    const int colour = (int)(cc / L.nchunk);
    const int64_t chunk = cc - (int64_t)colour * L.nchunk;
    const int64_t s = chunk * 32 + lane;
    const bool act = s < nec;
    double Kc = 1.0, t = 1.0;
    int meth = 0;
    int64_t e = -1;
    if (act) {
      int i, j;
      slot_elem(L.nx, colour, s, i, j);
      e = (int64_t)j * L.nx + i;
      Kc = K[e];
      t = tau[e] * h;
      meth = method[e];
      if (!(Kc > 0.0) || !(t > 0.0) || (meth != 0 && meth != 1)) {
        if (w == 0) report_error(err, -1, e);
        Kc = 1.0;
        t = 1.0;
        meth = 0;
      }
    }
    __syncthreads();   // sc of the previous chunk consumed; tables loaded
    for (int i = w; i < NV; i += NW) {
      const double d = fma(Kc, R.plam[meth][i], t * R.pmu[meth][i]);
      if (act && !(d > 0.0)) report_error(err, -4, e);   // Q not SPD (under-penalised)
      sc[i][lane] = 1.0 / d;
    }
    __syncthreads();
    const double* At = sAt[meth];
    const double* Bk = sBk[meth];
    double* dst = L.S + (((int64_t)colour * L.nchunk + chunk) * NPK) * 32 + lane;
    {
      // the warp's two rows a1 < a2 in one sweep over (i, b): each w_ib (two shared
      // loads) feeds both rows' FMAs (same arithmetic per entry as one row at a time)
      const int a1 = w, a2 = M - 1 - w;
      double acc1[M], acc2[M];
#pragma unroll
      for (int b = 0; b < M; ++b) {
        acc1[b] = (meth == 0 ? Kc * sW[a1 * M + b] : 0.0) + t * sH[a1 * M + b];
        acc2[b] = (meth == 0 ? Kc * sW[a2 * M + b] : 0.0) + t * sH[a2 * M + b];
      }
      for (int i = 0; i < NV; ++i) {
        const double si = sc[i][lane];
        const double wa1 = fma(t, At[i * M + a1], Kc * Bk[i * M + a1]) * si;
        const double wa2 = fma(t, At[i * M + a2], Kc * Bk[i * M + a2]) * si;
#pragma unroll
        for (int b = 0; b < M; ++b) {
          if (b >= a1) {
            const double wib = fma(t, At[i * M + b], Kc * Bk[i * M + b]);
            acc1[b] = fma(-wa1, wib, acc1[b]);
            if (b >= a2) acc2[b] = fma(-wa2, wib, acc2[b]);
          }
        }
      }
      if (act) {
        const int base1 = a1 * (2 * M - a1 + 1) / 2 - a1;   // kk(a, b) = base + b
        const int base2 = a2 * (2 * M - a2 + 1) / 2 - a2;
#pragma unroll
        for (int b = 0; b < M; ++b) {
          if (b >= a1) dst[(int64_t)(base1 + b) * 32] = acc1[b];
          if (b >= a2) dst[(int64_t)(base2 + b) * 32] = acc2[b];
        }
      }
    }
    if (project) {
      // S_T 1 = 0 exactly for the DtN map (constant traces: u = 0, q = lambda = c solve
      // the local problem with zero flux).  The elimination
      // leaves a rounding-level constant-mode error (amplified by the coarse Schur
      // complements, R5); replace S by its nearest symmetric matrix with
      // S 1 = 0, P S P with P = I - 1 1^T / m.
      __syncthreads();   // every row of the chunk stored
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        const int a = half == 0 ? w : M - 1 - w;
        double rs = 0.0;
#pragma unroll
        for (int b = 0; b < M; ++b) {
          const int lo = a < b ? a : b, hi = a < b ? b : a;
          rs += act ? dst[(int64_t)(lo * (2 * M - lo + 1) / 2 + (hi - lo)) * 32] : 0.0;
        }
        srow[a][lane] = rs;
      }
      __syncthreads();
      double sig = 0.0;
#pragma unroll
      for (int b = 0; b < M; ++b) sig += srow[b][lane];
      const double inv_m = 1.0 / M, c0 = sig * inv_m * inv_m;
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        const int a = half == 0 ? w : M - 1 - w;
        if (!act) continue;
        const int base = a * (2 * M - a + 1) / 2 - a;
#pragma unroll
        for (int b = 0; b < M; ++b)
          if (b >= a) {
            double* q = dst + (int64_t)(base + b) * 32;
            *q = (*q - (srow[a][lane] + srow[b][lane]) * inv_m) + c0;
          }
      }
    }
  }
}

int launch_local_dtn(const LevelDev& L, const RefDev& R, double h, const double* K,
                     const int8_t* method, const double* tau, DevError* err, cudaStream_t st) {
  const int64_t nct = 2 * (int64_t)L.nchunk;
  const int grid = (int)(nct < 148 * 8 ? nct : 148 * 8);
  static int project = -1;   // MGDTN_DTN_PROJECT=0: no constant-mode projection (A/B)
  if (project < 0) {
    const char* e = std::getenv("MGDTN_DTN_PROJECT");
    project = (e && std::atoi(e) == 0) ? 0 : 1;
  }
  if (L.ns) return launch_local_dtn_ns(L, R, h, K, method, tau, err, project, st);
  switch (L.p) {
    case 1: k_local_dtn<1><<<grid, 32 * 4, 0, st>>>(L, R, h, K, method, tau, err, project); break;
    case 2: k_local_dtn<2><<<grid, 32 * 6, 0, st>>>(L, R, h, K, method, tau, err, project); break;
    case 3: k_local_dtn<3><<<grid, 32 * 8, 0, st>>>(L, R, h, K, method, tau, err, project); break;
    default: k_local_dtn<4><<<grid, 32 * 10, 0, st>>>(L, R, h, K, method, tau, err, project); break;
  }
  return 1;
}

// ============================================================================
// Right-hand side: b_T = R^T Q^-1 f_w = sum_i w_i f'_i / d_i (pencil form, see
// H1; f'_i = h^2 sum_q fqT[q][i] f_q from the (p+4)^2 Gauss samples), minus
// the Dirichlet lift S_T lambda_D (stored S_T) on elements touching dOmega;
// scattered with the 2-colour rule of the apply (colour 0 writes, colour 1
// adds, reading Q4).  Thread per element.
// ============================================================================
template <int P>
__global__ void __launch_bounds__(128) k_local_rhs(
    LevelDev L, RefDev R, double h, const double* __restrict__ K,
    const int8_t* __restrict__ method, const double* __restrict__ tau,
    const double* __restrict__ f_qp, double f_const, const double* __restrict__ lamD, double* g,
    int colour) {
  using Sh = LocalShape<P>;
  constexpr int NV = Sh::NV, M = Sh::M, K1 = Sh::K1, NPK = Sh::NPK;
  const int64_t nec = L.ne >> 1;
  const int nq2 = R.nqf * R.nqf;
  for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < nec;
       s += (int64_t)gridDim.x * blockDim.x) {
    int i, j;
    slot_elem(L.nx, colour, s, i, j);
    const int64_t e = (int64_t)j * L.nx + i;
    const double Kc = K[e], t = tau[e] * h;
    const int meth = method[e] == 1 ? 1 : 0;
    const double* fqT = R.pfq[meth];
    double fp[NV];
#pragma unroll
    for (int a = 0; a < NV; ++a) fp[a] = 0.0;
    // the element's (p+4)^2 samples, 8 loads in flight per thread (a chain of one
    // dependent load per sample was the kernel's latency); same FMA order per fp[a]
    constexpr int QB = 8;
    int q = 0;
    for (; q + QB <= nq2; q += QB) {
      double fv[QB];
#pragma unroll
      for (int u = 0; u < QB; ++u) fv[u] = f_qp ? f_qp[e * nq2 + q + u] : f_const;
#pragma unroll
      for (int u = 0; u < QB; ++u)
#pragma unroll
        for (int a = 0; a < NV; ++a) fp[a] = fma(fqT[(q + u) * NV + a], fv[u], fp[a]);
    }
    for (; q < nq2; ++q) {
      const double fv = f_qp ? f_qp[e * nq2 + q] : f_const;
#pragma unroll
      for (int a = 0; a < NV; ++a) fp[a] = fma(fqT[q * NV + a], fv, fp[a]);
    }
#pragma unroll
    for (int a = 0; a < NV; ++a)
      fp[a] *= h * h / fma(Kc, R.plam[meth][a], t * R.pmu[meth][a]);
    double b[M];
#pragma unroll
    for (int a = 0; a < M; ++a) {
      double acc = 0.0;
#pragma unroll
      for (int q = 0; q < NV; ++q)
        acc = fma(fma(t, R.pAt[meth][q * M + a], Kc * R.pBk[meth][q * M + a]), fp[q], acc);
      b[a] = acc;
    }
    int64_t ed[4];
    bool bd[4];
    elem_edges(L.nx, L.ny, i, j, ed, bd, L.dmask);
    if (lamD && (bd[0] || bd[1] || bd[2] || bd[3])) {   // b -= S_T lambda_D
      double lt[M];
#pragma unroll
      for (int f = 0; f < 4; ++f)
#pragma unroll
        for (int a = 0; a < K1; ++a) lt[f * K1 + a] = bd[f] ? lamD[ed[f] * K1 + a] : 0.0;
      const double* Sp = L.S + ((((int64_t)colour * L.nchunk + (s >> 5)) * NPK) << 5) + (s & 31);
#pragma unroll
      for (int a = 0; a < M; ++a) {
#pragma unroll
        for (int c = a; c < M; ++c) {
          const double sv = Sp[(int64_t)(a * (2 * M - a + 1) / 2 + (c - a)) * 32];
          b[a] = fma(-sv, lt[c], b[a]);
          if (c != a) b[c] = fma(-sv, lt[a], b[c]);
        }
      }
    }
#pragma unroll
    for (int f = 0; f < 4; ++f) {
      if (bd[f]) continue;
#pragma unroll
      for (int a = 0; a < K1; ++a) {
        const int64_t idx = ed[f] * K1 + a;
        g[idx] = colour == 0 ? b[f * K1 + a] : g[idx] + b[f * K1 + a];
      }
    }
  }
}

int launch_local_rhs(const LevelDev& L, const RefDev& R, double h, const double* K,
                     const int8_t* method, const double* tau, const double* f_qp,
                     double f_const, const double* lamD, double* g, DevError* err,
                     cudaStream_t st) {
  (void)err;
  if (L.ns) return launch_local_rhs_ns(L, R, h, K, method, tau, f_qp, f_const, lamD, g, st);
  int64_t gsz = (L.ne / 2 + 127) / 128;
  int grid = (int)(gsz < 148 * 16 ? gsz : 148 * 16);
  if (grid < 1) grid = 1;
  for (int c = 0; c < 2; ++c) {
    switch (L.p) {
      case 1: k_local_rhs<1><<<grid, 128, 0, st>>>(L, R, h, K, method, tau, f_qp, f_const, lamD, g, c); break;
      case 2: k_local_rhs<2><<<grid, 128, 0, st>>>(L, R, h, K, method, tau, f_qp, f_const, lamD, g, c); break;
      case 3: k_local_rhs<3><<<grid, 128, 0, st>>>(L, R, h, K, method, tau, f_qp, f_const, lamD, g, c); break;
      default: k_local_rhs<4><<<grid, 128, 0, st>>>(L, R, h, K, method, tau, f_qp, f_const, lamD, g, c); break;
    }
  }
  return 2;
}

// ============================================================================
// volume recovery ("the local volume unknowns
// can be recovered in an element-by-element fashion completely independent of
// each other").  With the local pencil (refelem.h), Q = T^-1 diag(d) T^-T and
//   q_T = Q^-1 (R lambda_T + f_w) = T^T diag(1/d) (W lambda_T + f'),
// W = t At + K Bk (rows w_i), f'_i = h^2 sum_q fqT[q,i] f_q, d_i = K lam_i + t mu_i
// (the same factors the element DtN and the right-hand side use).  q_T: GLL nodal
// coefficients [(p+1)^2] in element-id order.  With q_exact samples at the
// (p+4)^2 Gauss points: per-block partial sums of h^2 sum_q w_q (q_T(x_q) - q_ex)^2.
// ============================================================================
template <int P>
__global__ void __launch_bounds__(128) k_recover(LevelDev L, RefDev R, double h,
                                                 const double* __restrict__ K,
                                                 const int8_t* __restrict__ method,
                                                 const double* __restrict__ tau,
                                                 const double* __restrict__ lam,
                                                 const double* __restrict__ f_qp, double f_const,
                                                 double* q_out, const double* __restrict__ qex,
                                                 double* partials) {
  using Sh = LocalShape<P>;
  constexpr int NV = Sh::NV, M = Sh::M, K1 = Sh::K1;
  const int nq2 = R.nqf * R.nqf;
  double err = 0.0;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < L.ne;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int j = (int)(e / L.nx), i = (int)(e - (int64_t)j * L.nx);
    const double Kc = K[e], t = tau[e] * h;
    const int meth = method[e] == 1 ? 1 : 0;
    int64_t ed[4];
    bool bd[4];
    elem_edges(L.nx, L.ny, i, j, ed, bd, L.dmask);
    double lt[M];
#pragma unroll
    for (int f = 0; f < 4; ++f)
#pragma unroll
      for (int a = 0; a < K1; ++a) lt[f * K1 + a] = lam[ed[f] * K1 + a];
    double c[NV];
    for (int v = 0; v < NV; ++v) {
      double acc = 0.0;
      for (int q = 0; q < nq2; ++q)
        acc = fma(R.pfq[meth][q * NV + v], f_qp ? f_qp[e * nq2 + q] : f_const, acc);
      acc *= h * h;
#pragma unroll
      for (int a = 0; a < M; ++a)
        acc = fma(fma(t, R.pAt[meth][v * M + a], Kc * R.pBk[meth][v * M + a]), lt[a], acc);
      c[v] = acc / fma(Kc, R.plam[meth][v], t * R.pmu[meth][v]);
    }
    double qv[NV];
    for (int k = 0; k < NV; ++k) {
      double acc = 0.0;
      for (int v = 0; v < NV; ++v) acc = fma(R.pTt[meth][k * NV + v], c[v], acc);
      qv[k] = acc;
      q_out[e * NV + k] = acc;
    }
    if (qex) {
      double s = 0.0;
      for (int q = 0; q < nq2; ++q) {
        double val = 0.0;
        for (int k = 0; k < NV; ++k) val = fma(R.vq[q * NV + k], qv[k], val);
        const double d = val - qex[e * nq2 + q];
        s = fma(R.wq[q] * d, d, s);
      }
      err = fma(h * h, s, err);
    }
  }
  if (qex) {
    __shared__ double red[4];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) err += __shfl_xor_sync(0xffffffffu, err, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = err;
    __syncthreads();
    if (threadIdx.x == 0) partials[blockIdx.x] = (red[0] + red[1]) + (red[2] + red[3]);
  }
}

int launch_recover(const LevelDev& L, const RefDev& R, double h, const double* K,
                   const int8_t* method, const double* tau, const double* lam,
                   const double* f_qp, double f_const, double* q_out, const double* qex_qp,
                   double* partials, int* grid_out, cudaStream_t st) {
  if (L.ns)
    return launch_recover_ns(L, R, h, K, method, tau, lam, f_qp, f_const, q_out, qex_qp,
                             partials, grid_out, st);
  int64_t g = (L.ne + 127) / 128;
  const int grid = (int)(g < 148 * 8 ? (g > 0 ? g : 1) : 148 * 8);
  if (grid_out) *grid_out = grid;
  switch (L.p) {
    case 1: k_recover<1><<<grid, 128, 0, st>>>(L, R, h, K, method, tau, lam, f_qp, f_const, q_out, qex_qp, partials); break;
    case 2: k_recover<2><<<grid, 128, 0, st>>>(L, R, h, K, method, tau, lam, f_qp, f_const, q_out, qex_qp, partials); break;
    case 3: k_recover<3><<<grid, 128, 0, st>>>(L, R, h, K, method, tau, lam, f_qp, f_const, q_out, qex_qp, partials); break;
    default: k_recover<4><<<grid, 128, 0, st>>>(L, R, h, K, method, tau, lam, f_qp, f_const, q_out, qex_qp, partials); break;
  }
  return 1;
}

// Dirichlet values: per-edge L2 projection of g_D onto P^p (reading Q4).
__global__ void k_dirichlet(LevelDev L, RefDev R, const double* __restrict__ gD, double* lamD) {
  const int nb = 2 * L.nx + 2 * L.ny;
  const int K1 = L.k1, nq = R.nqf;
  for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < nb; b += gridDim.x * blockDim.x) {
    int64_t e;
    int side;
    if (b < L.nx) { e = hedge(L.nx, b, 0); side = 0; }
    else if (b < 2 * L.nx) { e = hedge(L.nx, b - L.nx, L.ny); side = 2; }
    else if (b < 2 * L.nx + L.ny) { e = vedge(L.nx, L.ny, 0, b - 2 * L.nx); side = 3; }
    else { e = vedge(L.nx, L.ny, L.nx, b - 2 * L.nx - L.ny); side = 1; }
    if (!((L.dmask >> side) & 1)) {   // partition interface: not on dOmega
      for (int a = 0; a < K1; ++a) lamD[e * K1 + a] = 0.0;
      continue;
    }
    double mom[MAX_K1];
    for (int a = 0; a < K1; ++a) {
      double acc = 0.0;
      for (int q = 0; q < nq; ++q) acc += R.ew[q * K1 + a] * gD[(int64_t)b * nq + q];
      mom[a] = acc;
    }
    for (int a = 0; a < K1; ++a) {
      double v = 0.0;
      for (int c = 0; c < K1; ++c) v += R.H1inv[a * K1 + c] * mom[c];
      lamD[e * K1 + a] = v;
    }
  }
}

int launch_dirichlet(const LevelDev& L, const RefDev& R, const double* gD_qp, double* lamD,
                     cudaStream_t st) {
  int nb = 2 * L.nx + 2 * L.ny;
  k_dirichlet<<<(nb + 127) / 128, 128, 0, st>>>(L, R, gD_qp, lamD);
  return 1;
}

// ============================================================================
// H2: p-coarsening S^(1)_T = J_p^T S_T J_p (Eq. ANm1), per
// element, J_p = blockdiag over the 4 edges of [(1-s_a), s_a].
// ============================================================================
__device__ __forceinline__ double s_get(const double* base, int m, int ns, int a, int b) {
  return base[(int64_t)s_index(a, b, m, ns) * 32];
}

// One thread per element; J_p is block diagonal (one [(p+1) x 2] block per edge),
// so per row block f: T_f = S_{f,:} J_p (K1 x 8, from the packed rows of edge f),
// then rows 2f, 2f+1 of J_p^T S J_p = J_f^T T_f.  Compile-time indices throughout.
// NS: full row-major storage on both levels (nonsymmetric context): every entry of
// J_p^T S_T J_p is formed (the symmetric path forms the upper triangle).
template <int P, bool NS>
__global__ void __launch_bounds__(128) k_p_coarsen_acc(LevelDev F, LevelDev C,
                                                       const double* __restrict__ Jp) {
  constexpr int K1 = P + 1, M = 4 * K1, NC = NS ? 64 : 36;
  double J[K1][2];
#pragma unroll
  for (int a = 0; a < K1; ++a) {
    J[a][0] = Jp[a * 2];
    J[a][1] = Jp[a * 2 + 1];
  }
  const int64_t nec = F.ne >> 1;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < 2 * nec;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int colour = (int)(t / nec);
    const int64_t s = t - colour * nec;
    const double* src = F.S + s_offset(F.nchunk, F.npk, colour, s, 0);
    double* dst = C.S + s_offset(C.nchunk, C.npk, colour, s, 0);
    double acc[NC];
#pragma unroll
    for (int q = 0; q < NC; ++q) acc[q] = 0.0;
#pragma unroll
    for (int a = 0; a < M; ++a) {
#pragma unroll
      for (int b = NS ? 0 : a; b < M; ++b) {
        const int f = a / K1, al = a % K1, g = b / K1, bl = b % K1;
        const double v = __ldg(src + (int64_t)(NS ? a * M + b : pk_index(a, b, M)) * 32);
#pragma unroll
        for (int ca = 0; ca < 2; ++ca)
#pragma unroll
          for (int cb = 0; cb < 2; ++cb) {
            const int A = 2 * f + ca, B = 2 * g + cb;
            if (NS) {
              acc[A * 8 + B] = fma(J[al][ca] * J[bl][cb], v, acc[A * 8 + B]);
            } else if (f < g) {   // off-diagonal edge blocks: a < b always
              acc[pk_index(A, B, 8)] = fma(J[al][ca] * J[bl][cb], v, acc[pk_index(A, B, 8)]);
            } else if (A <= B) {  // same edge: the pair (a, b) and, if a != b, (b, a)
              acc[pk_index(A, B, 8)] = fma(J[al][ca] * J[bl][cb], v, acc[pk_index(A, B, 8)]);
              if (a != b)
                acc[pk_index(A, B, 8)] = fma(J[bl][ca] * J[al][cb], v, acc[pk_index(A, B, 8)]);
            }
          }
      }
    }
#pragma unroll
    for (int q = 0; q < NC; ++q) dst[(int64_t)q * 32] = acc[q];
  }
}

int launch_p_coarsen(const LevelDev& F, const LevelDev& C, const double* Jp, cudaStream_t st) {
  int64_t n = F.ne;
  int grid = (int)((n + 127) / 128 < 148 * 16 ? (n + 127) / 128 : 148 * 16);
  if (F.ns) {
    switch (F.p) {
      case 2: k_p_coarsen_acc<2, true><<<grid, 128, 0, st>>>(F, C, Jp); break;
      case 3: k_p_coarsen_acc<3, true><<<grid, 128, 0, st>>>(F, C, Jp); break;
      default: k_p_coarsen_acc<4, true><<<grid, 128, 0, st>>>(F, C, Jp); break;
    }
  } else {
    switch (F.p) {
      case 2: k_p_coarsen_acc<2, false><<<grid, 128, 0, st>>>(F, C, Jp); break;
      case 3: k_p_coarsen_acc<3, false><<<grid, 128, 0, st>>>(F, C, Jp); break;
      default: k_p_coarsen_acc<4, false><<<grid, 128, 0, st>>>(F, C, Jp); break;
    }
  }
  return 1;
}

// ============================================================================
// H3: 2x2 agglomeration (Eqs. 3.3, 3.5, Akm1; Prop. DtN
// A_{k-1} is the Schur complement obtained by eliminating
// the trace unknowns inside each macro-element).  Per macro (I,J), with the
// 4 children's 8x8 DtN maps, assemble the reduced 16x16 matrix over
// [interior dofs (8) | coarse macro-edge dofs (8)]:
//     Kr = sum_c G_c^T S_c G_c,   G_c: child dof -> interior dof (identity)
//                                          or J-interpolated coarse dof,
// so Kr_II = A_II(M), Kr_IC = A_IB J, Kr_CC = J^T A_BB J (per macro), and
//     A_II^-1 (stored), P_M = -A_II^-1 A_IB J (stored),
//     S_c = J^T (A_BB - A_BI A_II^-1 A_IB) J = Kr_CC + Kr_IC^T P_M.
// Interior edge order: H(2I,2J+1), H(2I+1,2J+1), V(2I+1,2J), V(2I+1,2J+1);
// coarse dof order = coarse element local order {bottom, right, top, left} x 2.
// ============================================================================
// child c (0:(0,0) 1:(1,0) 2:(0,1) 3:(1,1)), local edge f -> code:
// code < 4: interior edge index; code >= 4: macro edge (code-4)>>1, half (code-4)&1
__constant__ int c_child_map[4][4] = {
    {4 + 0 * 2 + 0, 2, 0, 4 + 3 * 2 + 0},
    {4 + 0 * 2 + 1, 4 + 1 * 2 + 0, 1, 2},
    {0, 3, 4 + 2 * 2 + 0, 4 + 3 * 2 + 1},
    {1, 4 + 1 * 2 + 1, 4 + 2 * 2 + 1, 3}};

constexpr int AGG_WARPS = 4;

// dense_out != nullptr: the coarse maps go to dense_out[M][8][8] (element-id order of
// the coarse block; both triangles) instead of the packed chunk layout -- the gather
// level's per-rank block, whose element count may be odd
// Nonsymmetric context (F.ns): A_II is inverted by Gauss-Jordan with partial
// pivoting, S_c = Kr_CC + Kr_CI P_M is formed in full, and the restriction's macro
// term of Eq. 3.5, Q_M = -J^T A_BI A_II^-1 = -Kr_CI A_II^-1 (not P_M^T when A is
// nonsymmetric), is stored transposed in Rm (Rm[a*8 + c] = Q_M[c][a], the layout in
// which the restriction reads P_M on a symmetric level).
__global__ void __launch_bounds__(32 * AGG_WARPS) k_agglomerate(LevelDev F, LevelDev C,
                                                                double* KIIinv, double* Pm,
                                                                DevError* err,
                                                                double* dense_out, double* Rm) {
  __shared__ double smK[AGG_WARPS][16 * 16];
  __shared__ double smG[AGG_WARPS][8 * 16];
  __shared__ double smU[AGG_WARPS][8 * 16];
  __shared__ double smS[AGG_WARPS][64];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* Kr = smK[w];
  double* G = smG[w];
  double* U = smU[w];
  double* Sc = smS[w];
  const int nxc = F.nx >> 1, nyc = F.ny >> 1;
  const int64_t nmac = (int64_t)nxc * nyc;
  for (int64_t M = (int64_t)blockIdx.x * AGG_WARPS + w; M < nmac;
       M += (int64_t)gridDim.x * AGG_WARPS) {
    const int I = (int)(M % nxc), J = (int)(M / nxc);
    for (int q = lane; q < 256; q += 32) Kr[q] = 0.0;
    __syncwarp();
    for (int c = 0; c < 4; ++c) {
      const int ci = 2 * I + (c & 1), cj = 2 * J + (c >> 1);
      int colour;
      int64_t s;
      elem_slot(F.nx, ci, cj, colour, s);
      const double* src = F.S + s_offset(F.nchunk, F.npk, colour, s, 0);
      // child S (dense 8x8) into Sc, G_c (8 x 16) into G
      for (int q = lane; q < 64; q += 32) {
        int a = q >> 3, b = q & 7;
        Sc[q] = s_get(src, 8, F.ns, a, b);
      }
      for (int q = lane; q < 128; q += 32) G[q] = 0.0;
      __syncwarp();
      if (lane < 8) {
        int f = lane >> 1, a = lane & 1;
        int code = c_child_map[c][f];
        if (code < 4) {
          G[lane * 16 + code * 2 + a] = 1.0;
        } else {
          int E = (code - 4) >> 1, half = (code - 4) & 1;
          // fine node a of half `half`: value at parameter (half + a)/2 of the macro edge
          double sp = 0.5 * (half + a);
          G[lane * 16 + 8 + E * 2 + 0] = 1.0 - sp;
          G[lane * 16 + 8 + E * 2 + 1] = sp;
        }
      }
      __syncwarp();
      // U = S_c G_c (8 x 16)
      for (int q = lane; q < 128; q += 32) {
        int a = q >> 4, col = q & 15;
        double acc = 0.0;
        for (int b = 0; b < 8; ++b) acc += Sc[a * 8 + b] * G[b * 16 + col];
        U[q] = acc;
      }
      __syncwarp();
      // Kr += G_c^T U
      for (int q = lane; q < 256; q += 32) {
        int r = q >> 4, col = q & 15;
        double acc = 0.0;
        for (int a = 0; a < 8; ++a) acc += G[a * 16 + r] * U[a * 16 + col];
        Kr[q] += acc;
      }
      __syncwarp();
    }
    if (F.ns) {
      // A_II^-1 (Gauss-Jordan, partial pivoting) into G[0..63]; scratch Sc
      if (lane == 0) {
        double Kii[64];
        for (int q = 0; q < 64; ++q) Kii[q] = Kr[(q >> 3) * 16 + (q & 7)];
        if (!gj_inverse(Kii, 8, G, Sc)) report_error(err, -3, M);
      }
      __syncwarp();
      for (int q = lane; q < 64; q += 32) {
        const int a = q >> 3, b = q & 7;
        KIIinv[M * 64 + q] = G[q];
        double pm = 0.0, qm = 0.0;
        for (int r = 0; r < 8; ++r) {
          pm = fma(-G[a * 8 + r], Kr[r * 16 + 8 + b], pm);          // P_M[a][b]
          qm = fma(-Kr[(8 + b) * 16 + r], G[r * 8 + a], qm);        // Q_M[b][a]
        }
        Pm[M * 64 + q] = pm;
        U[a * 16 + b] = pm;
        Rm[M * 64 + q] = qm;
      }
      __syncwarp();
      int colour;
      int64_t s;
      elem_slot(C.nx, I, J, colour, s);
      double* dst = C.S + s_offset(C.nchunk, C.npk, colour, s, 0);
      for (int q = lane; q < 64; q += 32) {
        const int a = q >> 3, b = q & 7;
        double acc = Kr[(8 + a) * 16 + 8 + b];
        for (int r = 0; r < 8; ++r) acc = fma(Kr[(8 + a) * 16 + r], U[r * 16 + b], acc);
        dst[(int64_t)q * 32] = acc;
      }
      __syncwarp();
      continue;
    }
    // A_II^-1 and A_II^-1 Kr_IC by Gauss-Jordan on [Kr_II | I | Kr_IC] (8 x 24, no
    // pivoting: A_II is SPD), all lanes per elimination step: left 16 columns in G
    // (row stride 16), right 8 in U (row stride 16).  Every lane reads its entries,
    // the pivot row and the pivot column before any lane writes (one __syncwarp).
    for (int q = lane; q < 128; q += 32) {
      const int r = q >> 4, j = q & 15;
      G[q] = j < 8 ? Kr[r * 16 + j] : (j - 8 == r ? 1.0 : 0.0);
      U[q] = j < 8 ? Kr[r * 16 + 8 + j] : 0.0;
    }
    __syncwarp();
    bool ok = true;
    for (int k = 0; k < 8; ++k) {
      const double piv = G[k * 16 + k];
      if (!(piv > 0.0)) ok = false;
      const double ipiv = piv > 0.0 ? 1.0 / piv : 0.0;
      double nv[6];
#pragma unroll
      for (int u = 0; u < 6; ++u) {   // 192 entries, 6 per lane
        const int q = lane + 32 * u, r = q / 24, j = q - (q / 24) * 24;
        double* X = j < 16 ? G + r * 16 + j : U + r * 16 + (j - 16);
        const double pk = (j < 16 ? G[k * 16 + j] : U[k * 16 + (j - 16)]) * ipiv;
        nv[u] = r == k ? pk : fma(-G[r * 16 + k], pk, *X);
      }
      __syncwarp();
#pragma unroll
      for (int u = 0; u < 6; ++u) {
        const int q = lane + 32 * u, r = q / 24, j = q - (q / 24) * 24;
        double* X = j < 16 ? G + r * 16 + j : U + r * 16 + (j - 16);
        *X = nv[u];
      }
      __syncwarp();
    }
    if (!ok && lane == 0) report_error(err, -4, M);
    for (int q = lane; q < 64; q += 32) {
      const int a = q >> 3, b = q & 7;
      // symmetric A_II: its inverse as the packed upper triangle (36 of 64 doubles; the
      // local correction's dominant stream at the 4096^2 P1 level, lc_restrict_body)
      if (a <= b) KIIinv[M * 36 + pk_index(a, b, 8)] = G[a * 16 + 8 + b];
      const double pm = -U[a * 16 + b];
      Pm[M * 64 + q] = pm;
      U[a * 16 + b] = pm;   // keep P_M for S_c
    }
    __syncwarp();
    // S_c = Kr_CC + Kr_IC^T P_M, packed upper (36), into the coarse storage
    if (dense_out) {
      for (int kk = lane; kk < 36; kk += 32) {
        int a, b;
        pk_row_col(kk, 8, a, b);
        double acc = Kr[(8 + a) * 16 + 8 + b];
        for (int r = 0; r < 8; ++r) acc += Kr[r * 16 + 8 + a] * U[r * 16 + b];
        dense_out[M * 64 + a * 8 + b] = acc;
        dense_out[M * 64 + b * 8 + a] = acc;
      }
    } else {
      int colour;
      int64_t s;
      elem_slot(C.nx, I, J, colour, s);
      double* dst = C.S + s_offset(C.nchunk, 36, colour, s, 0);
      for (int kk = lane; kk < 36; kk += 32) {
        int a, b;
        pk_row_col(kk, 8, a, b);
        double acc = Kr[(8 + a) * 16 + 8 + b];
        for (int r = 0; r < 8; ++r) acc += Kr[r * 16 + 8 + a] * U[r * 16 + b];
        dst[(int64_t)kk * 32] = acc;
      }
    }
    __syncwarp();
  }
}

int launch_agglomerate(const LevelDev& F, const LevelDev& C, double* KIIinv, double* Pm,
                       DevError* err, cudaStream_t st, double* dense_out, double* Rm) {
  int64_t nmac = (int64_t)(F.nx / 2) * (F.ny / 2);
  int64_t g = (nmac + AGG_WARPS - 1) / AGG_WARPS;
  int grid = (int)(g < 148 * 16 ? g : 148 * 16);
  k_agglomerate<<<grid, 32 * AGG_WARPS, 0, st>>>(F, C, KIIinv, Pm, err, dense_out, Rm);
  return 1;
}

// Reading R10: the exact coarse maps annihilate constant traces too (a macro's harmonic
// extension of a constant is that constant, and J_p / J_M map constants to constants),
// so every p = 1 level's maps -- p-coarsened or agglomerated -- are replaced by P S P,
// P = I - 11^T/8, as the fine maps are (R5).  Without it the rounding-level constant-mode
// error of each level accumulates coherently through the Galerkin chain.
__global__ void k_project_const8(LevelDev L) {
  constexpr int M = 8, NPK = 36;
  const int64_t nslot = (int64_t)L.nchunk * 32;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < 2 * nslot;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int colour = q >= nslot ? 1 : 0;
    const int64_t s = q - colour * nslot;
    double* Sp = L.S + (((int64_t)colour * L.nchunk + (s >> 5)) * NPK) * 32 + (s & 31);
    double v[NPK], rs[M];
#pragma unroll
    for (int kk = 0; kk < NPK; ++kk) v[kk] = Sp[kk * 32];
    double sig = 0.0;
#pragma unroll
    for (int a = 0; a < M; ++a) {
      double t = 0.0;
#pragma unroll
      for (int b = 0; b < M; ++b) {
        const int lo = a < b ? a : b, hi = a < b ? b : a;
        t += v[lo * (2 * M - lo + 1) / 2 + (hi - lo)];
      }
      rs[a] = t;
      sig += t;
    }
    const double c0 = sig / (M * M);
#pragma unroll
    for (int a = 0; a < M; ++a)
#pragma unroll
      for (int b = a; b < M; ++b) {
        const int kk = a * (2 * M - a + 1) / 2 + (b - a);
        Sp[kk * 32] = (v[kk] - (rs[a] + rs[b]) / M) + c0;
      }
  }
}
int launch_project_const(const LevelDev& L, cudaStream_t st) {
  if (L.ns || L.p != 1) return 0;
  const int64_t n = (int64_t)L.nchunk * 64;
  const int grid = (int)((n + 127) / 128 < 2368 ? (n + 127) / 128 : 2368);
  k_project_const8<<<grid, 128, 0, st>>>(L);
  return 1;
}

// ============================================================================
// H4: edge-block diagonal D_e = sum_{T owns e} S_T[e,e] and its inverse
// (block-Jacobi with edge blocks).
// ============================================================================
__global__ void k_edge_blocks(LevelDev L, DevError* err) {
  const int K1 = L.k1, m = L.m;
  const int64_t nh = (int64_t)L.nx * (L.ny + 1);
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < L.nedge;
       e += (int64_t)gridDim.x * blockDim.x) {
    double D[MAX_K1 * MAX_K1];
    double* out = L.Dinv + e;   // SoA, stride nedge
    const int64_t sd = L.nedge;
    const int side = edge_side(L.nx, L.ny, e);
    if (side >= 0 && ((L.dmask >> side) & 1)) {
      for (int q = 0; q < K1 * K1; ++q) out[q * sd] = 0.0;
      continue;
    }
    int ei[2], ej[2], ef[2];
    if (e < nh) {
      int j = (int)(e / L.nx), i = (int)(e % L.nx);
      ei[0] = i; ej[0] = j - 1; ef[0] = 2;   // element below, its top edge
      ei[1] = i; ej[1] = j;     ef[1] = 0;   // element above, its bottom edge
    } else {
      int64_t r = e - nh;
      int j = (int)(r / (L.nx + 1)), i = (int)(r % (L.nx + 1));
      ei[0] = i - 1; ej[0] = j; ef[0] = 1;   // left element, its right edge
      ei[1] = i;     ej[1] = j; ef[1] = 3;   // right element, its left edge
    }
    for (int q = 0; q < K1 * K1; ++q) D[q] = 0.0;
    for (int t = 0; t < 2; ++t) {
      // on a partition interface one of the two elements lives on the neighbour rank
      if (ei[t] < 0 || ei[t] >= L.nx || ej[t] < 0 || ej[t] >= L.ny) continue;
      int colour;
      int64_t s;
      elem_slot(L.nx, ei[t], ej[t], colour, s);
      const double* src = L.S + s_offset(L.nchunk, L.npk, colour, s, 0);
      for (int a = 0; a < K1; ++a)
        for (int b = 0; b < K1; ++b)
          D[a * K1 + b] += s_get(src, m, L.ns, ef[t] * K1 + a, ef[t] * K1 + b);
    }
    if (side >= 0) {   // interface: this rank's partial block; inverted after the halo (k_part.cu)
      for (int q = 0; q < K1 * K1; ++q) out[q * sd] = D[q];
      continue;
    }
    double inv[MAX_K1 * MAX_K1];
    if (L.ns) {   // nonsymmetric block: Gauss-Jordan with partial pivoting
      double scr[MAX_K1 * MAX_K1];
      if (!gj_inverse(D, K1, inv, scr)) report_error(err, -3, e);
    } else if (!chol_inverse(D, K1, inv)) {
      report_error(err, -4, e);
    }
    for (int q = 0; q < K1 * K1; ++q) out[q * sd] = inv[q];
  }
}

int launch_edge_blocks(const LevelDev& L, DevError* err, cudaStream_t st) {
  int64_t g = (L.nedge + 127) / 128;
  int grid = (int)(g < 148 * 16 ? g : 148 * 16);
  k_edge_blocks<<<grid, 128, 0, st>>>(L, err);
  return 1;
}

// D_e^-1 of every free edge into the colour-1 element-chunk layout LevelDev::Dc
__global__ void k_dinv_pack(LevelDev L) {
  const int K1 = L.k1, NDE = K1 * (K1 + 1) / 2;
  const int64_t nec = L.ne >> 1;
  const int64_t nslot = (int64_t)L.nchunk * 32;
  for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < nslot;
       s += (int64_t)gridDim.x * blockDim.x) {
    int64_t ed[4] = {0, 0, 0, 0};
    bool bd[4] = {true, true, true, true};
    if (s < nec) {
      int i, j;
      slot_elem(L.nx, 1, s, i, j);
      elem_edges(L.nx, L.ny, i, j, ed, bd, L.dmask);
    }
    double* dst = L.Dc + ((s >> 5) * L.ndi) * 32 + (s & 31);
    for (int f = 0; f < 4; ++f)
      for (int a = 0; a < K1; ++a)
        for (int b = a; b < K1; ++b) {
          const int row = f * NDE + pk_index(a, b, K1);
          dst[(int64_t)row * 32] = bd[f] ? 0.0 : L.Dinv[(int64_t)(a * K1 + b) * L.nedge + ed[f]];
        }
  }
}
// orbit level (R9): D_e^-1 is centrosymmetric (d4.cuh); each orbit of the upper
// triangle is replaced by its mean (in place, both triangles), and the orbit values go
// to the SoA Dso (edge-parallel kernels)
template <int P>
__global__ void k_dinv_orb(LevelDev L) {
  using D = D4<P>;
  constexpr int K1 = P + 1;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < L.nedge;
       e += (int64_t)gridDim.x * blockDim.x) {
    double* Di = L.Dinv + e;
    double sum[D::NCS];
#pragma unroll
    for (int o = 0; o < D::NCS; ++o) sum[o] = 0.0;
#pragma unroll
    for (int a = 0; a < K1; ++a)
#pragma unroll
      for (int b = a; b < K1; ++b) sum[D::cs(D::pe(a, b))] += Di[(int64_t)(a * K1 + b) * L.nedge];
    double v[D::NCS];
#pragma unroll
    for (int o = 0; o < D::NCS; ++o) {
      v[o] = sum[o] / (double)D::ccnt(o);
      L.Dso[(int64_t)o * L.nedge + e] = v[o];
    }
#pragma unroll
    for (int a = 0; a < K1; ++a)
#pragma unroll
      for (int b = 0; b < K1; ++b) Di[(int64_t)(a * K1 + b) * L.nedge] = v[D::cs(D::pe(a, b))];
  }
}
// Dso -> the colour-1 element-chunk records Dco streamed by k_apply_orb
template <int P>
__global__ void k_dinv_pack_orb(LevelDev L) {
  using D = D4<P>;
  const int64_t nec = L.ne >> 1;
  const int64_t nslot = (int64_t)L.nchunk * 32;
  for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < nslot;
       s += (int64_t)gridDim.x * blockDim.x) {
    int64_t ed[4] = {0, 0, 0, 0};
    bool bd[4] = {true, true, true, true};
    if (s < nec) {
      int i, j;
      slot_elem(L.nx, 1, s, i, j);
      elem_edges(L.nx, L.ny, i, j, ed, bd, L.dmask);
    }
    double* dst = L.Dco + (s >> 5) * 4 * D::NCS * 32 + (s & 31);
#pragma unroll
    for (int f = 0; f < 4; ++f)
#pragma unroll
      for (int o = 0; o < D::NCS; ++o)
        dst[(f * D::NCS + o) * 32] = bd[f] ? 0.0 : L.Dso[(int64_t)o * L.nedge + ed[f]];
  }
}

int launch_dinv_pack(const LevelDev& L, cudaStream_t st) {
  const int64_t n = (int64_t)L.nchunk * 32;
  const int grid = (int)((n + 127) / 128 < 1184 ? (n + 127) / 128 : 1184);
  if (L.orb) {
    const int ge = (int)((L.nedge + 127) / 128 < 1184 ? (L.nedge + 127) / 128 : 1184);
    switch (L.p) {
      case 1: k_dinv_orb<1><<<ge, 128, 0, st>>>(L); k_dinv_pack_orb<1><<<grid, 128, 0, st>>>(L); break;
      case 2: k_dinv_orb<2><<<ge, 128, 0, st>>>(L); k_dinv_pack_orb<2><<<grid, 128, 0, st>>>(L); break;
      case 3: k_dinv_orb<3><<<ge, 128, 0, st>>>(L); k_dinv_pack_orb<3><<<grid, 128, 0, st>>>(L); break;
      default: k_dinv_orb<4><<<ge, 128, 0, st>>>(L); k_dinv_pack_orb<4><<<grid, 128, 0, st>>>(L); break;
    }
    return 2;
  }
  k_dinv_pack<<<grid, 128, 0, st>>>(L);
  return 1;
}

// orbit storage (R9): every element map of the level is replaced by its D4 orbit
// averages (mean over the packed entries of each orbit, in packed order), in place,
// and the orbit values are written to the chunk records So
template <int P>
__global__ void k_orbit_pack(LevelDev L) {
  using D = D4<P>;
  constexpr int NPK = D::NPK, NORB = D::NORB;
  const int64_t nslot = (int64_t)L.nchunk * 32;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < 2 * nslot;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int colour = q >= nslot ? 1 : 0;
    const int64_t s = q - colour * nslot;
    const int64_t rec = (int64_t)colour * L.nchunk + (s >> 5);
    double* Sp = L.S + rec * NPK * 32 + (s & 31);
    double sum[NORB];
#pragma unroll
    for (int o = 0; o < NORB; ++o) sum[o] = 0.0;
#pragma unroll
    for (int kk = 0; kk < NPK; ++kk) sum[D::orb(kk)] += Sp[kk * 32];
    double* Op = L.So + rec * NORB * 32 + (s & 31);
#pragma unroll
    for (int o = 0; o < NORB; ++o) {
      sum[o] = sum[o] / (double)D::cnt(o);
      Op[o * 32] = sum[o];
    }
#pragma unroll
    for (int kk = 0; kk < NPK; ++kk) Sp[kk * 32] = sum[D::orb(kk)];
  }
}
int launch_orbit_pack(const LevelDev& L, cudaStream_t st) {
  if (!L.orb) return 0;
  const int64_t n = (int64_t)L.nchunk * 64;
  const int grid = (int)((n + 127) / 128 < 2368 ? (n + 127) / 128 : 2368);
  switch (L.p) {
    case 1: k_orbit_pack<1><<<grid, 128, 0, st>>>(L); break;
    case 2: k_orbit_pack<2><<<grid, 128, 0, st>>>(L); break;
    case 3: k_orbit_pack<3><<<grid, 128, 0, st>>>(L); break;
    default: k_orbit_pack<4><<<grid, 128, 0, st>>>(L); break;
  }
  return 1;
}

// dense [ne][m][m] (element-id order) <-> packed interleaved storage
__global__ void k_dense_to_packed(LevelDev L, const double* __restrict__ src) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < L.ne;
       e += (int64_t)gridDim.x * blockDim.x) {
    int i = (int)(e % L.nx), j = (int)(e / L.nx), colour;
    int64_t s;
    elem_slot(L.nx, i, j, colour, s);
    double* dst = L.S + s_offset(L.nchunk, L.npk, colour, s, 0);
    const double* a0 = src + e * L.m * L.m;
    for (int a = 0; a < L.m; ++a)
      for (int b = L.ns ? 0 : a; b < L.m; ++b)
        dst[(int64_t)s_index(a, b, L.m, L.ns) * 32] = a0[a * L.m + b];
  }
}
__global__ void k_packed_to_dense(LevelDev L, double* __restrict__ dst) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < L.ne;
       e += (int64_t)gridDim.x * blockDim.x) {
    int i = (int)(e % L.nx), j = (int)(e / L.nx), colour;
    int64_t s;
    elem_slot(L.nx, i, j, colour, s);
    const double* src = L.S + s_offset(L.nchunk, L.npk, colour, s, 0);
    double* a0 = dst + e * L.m * L.m;
    for (int a = 0; a < L.m; ++a)
      for (int b = 0; b < L.m; ++b) a0[a * L.m + b] = s_get(src, L.m, L.ns, a, b);
  }
}
int launch_dense_to_packed(const LevelDev& L, const double* src, cudaStream_t st) {
  int grid = (int)((L.ne + 127) / 128 < 1184 ? (L.ne + 127) / 128 : 1184);
  k_dense_to_packed<<<grid, 128, 0, st>>>(L, src);
  return 1;
}
int launch_packed_to_dense(const LevelDev& L, double* dst, cudaStream_t st) {
  int grid = (int)((L.ne + 127) / 128 < 1184 ? (L.ne + 127) / 128 : 1184);
  k_packed_to_dense<<<grid, 128, 0, st>>>(L, dst);
  return 1;
}

// selected elements, dense [n][m][m]
__global__ void k_gather_dense(LevelDev L, const int64_t* __restrict__ elems, int64_t n,
                               double* __restrict__ dst) {
  const int m = L.m;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n * m * m;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = q / (m * m);
    const int ab = (int)(q % (m * m)), a = ab / m, b = ab % m;
    const int64_t e = elems[t];
    if (e < 0 || e >= L.ne) {
      dst[q] = 0.0;
      continue;
    }
    int colour;
    int64_t s;
    elem_slot(L.nx, (int)(e % L.nx), (int)(e / L.nx), colour, s);
    dst[q] = s_get(L.S + s_offset(L.nchunk, L.npk, colour, s, 0), m, L.ns, a, b);
  }
}

int launch_gather_dense(const LevelDev& L, const int64_t* elems, int64_t n, double* dst,
                        cudaStream_t st) {
  const int64_t tot = n * L.m * L.m;
  int grid = (int)((tot + 127) / 128 < 1184 ? (tot + 127) / 128 : 1184);
  k_gather_dense<<<grid > 0 ? grid : 1, 128, 0, st>>>(L, elems, n, dst);
  return 1;
}

// ============================================================================
// H5: coarsest level, B_1 = A_1^-1 by a direct solver.
// One CTA assembles the dense free-dof matrix, factors it (Cholesky) and
// forms the explicit inverse used by every V-cycle.
// ============================================================================
__global__ void k_coarse_factor(LevelDev L, const int* __restrict__ fpos, int nf, double* A,
                                double* Ainv, DevError* err) {
  const int tid = threadIdx.x, nt = blockDim.x;
  // small coarsest level (the 2x2 macro mesh: nf = 8, 4 elements): every thread owns
  // entries of A and sums their contributions in the serial loop's order (elements,
  // then a, then b), from a shared copy of the element-to-free-dof maps -- the same
  // sums as the one-thread assembly below, without its chain of dependent global
  // read-modify-writes
  constexpr int SGI = 1024, SNF = 32;
  __shared__ int sgi[SGI];
  __shared__ double sA[SNF * SNF], sI[SNF * SNF];   // A and A^-1 of a small coarsest level
  const bool par = nf <= SNF && L.ne * L.m <= SGI;
  double* Aw = par ? sA : A;
  double* Iw = par ? sI : Ainv;
  if (par) {
    for (int q = tid; q < L.ne * L.m; q += nt) {
      const int64_t e = q / L.m;
      const int a = q - (int)e * L.m;
      const int i = (int)(e % L.nx), j = (int)(e / L.nx);
      int64_t ed[4];
      bool bd[4];
      elem_edges(L.nx, L.ny, i, j, ed, bd, L.dmask);
      sgi[q] = fpos[ed[a / L.k1] * L.k1 + a % L.k1];
    }
    __syncthreads();
    for (int q = tid; q < nf * nf; q += nt) {
      const int gr = q / nf, gc = q - gr * nf;
      double acc = 0.0;
      for (int64_t e = 0; e < L.ne; ++e) {
        const int* gi = sgi + e * L.m;
        const double* src = nullptr;
        for (int a = 0; a < L.m; ++a) {
          if (gi[a] != gr) continue;
          for (int b = 0; b < L.m; ++b) {
            if (gi[b] != gc) continue;
            if (!src) {
              int colour;
              int64_t s;
              elem_slot(L.nx, (int)(e % L.nx), (int)(e / L.nx), colour, s);
              src = L.S + s_offset(L.nchunk, L.npk, colour, s, 0);
            }
            acc += s_get(src, L.m, L.ns, a, b);
          }
        }
      }
      Aw[q] = acc;
    }
  } else {
    for (int q = tid; q < nf * nf; q += nt) A[q] = 0.0;
  }
  __syncthreads();
  if (!par && tid == 0) {
    for (int64_t e = 0; e < L.ne; ++e) {
      int i = (int)(e % L.nx), j = (int)(e / L.nx), colour;
      int64_t s;
      elem_slot(L.nx, i, j, colour, s);
      const double* src = L.S + s_offset(L.nchunk, L.npk, colour, s, 0);
      int64_t ed[4];
      bool bd[4];
      elem_edges(L.nx, L.ny, i, j, ed, bd, L.dmask);
      int gi[4 * MAX_K1];
      for (int f = 0; f < 4; ++f)
        for (int a = 0; a < L.k1; ++a) gi[f * L.k1 + a] = fpos[ed[f] * L.k1 + a];
      for (int a = 0; a < L.m; ++a)
        for (int b = 0; b < L.m; ++b)
          if (gi[a] >= 0 && gi[b] >= 0) A[gi[a] * nf + gi[b]] += s_get(src, L.m, L.ns, a, b);
    }
  }
  __syncthreads();
  if (L.ns) {   // nonsymmetric A_1: Gauss-Jordan with partial pivoting (A is the scratch)
    if (tid == 0 && !gj_inverse(Aw, nf, Iw, Aw)) report_error(err, -3, -2);
    __syncthreads();
    if (par)
      for (int q = tid; q < nf * nf; q += nt) {
        A[q] = sA[q];
        Ainv[q] = sI[q];
      }
    return;
  }
  __shared__ int bad;
  if (tid == 0) bad = 0;
  __syncthreads();
  for (int jc = 0; jc < nf; ++jc) {
    if (tid == 0) {
      double d = Aw[jc * nf + jc];
      if (!(d > 0.0)) { bad = 1; d = 1e-300; }
      Aw[jc * nf + jc] = sqrt(d);
    }
    __syncthreads();
    const double dj = Aw[jc * nf + jc];
    for (int i = jc + 1 + tid; i < nf; i += nt) Aw[i * nf + jc] /= dj;
    __syncthreads();
    const int r = nf - jc - 1;
    for (int q = tid; q < r * r; q += nt) {
      int ii = jc + 1 + q / r, cc = jc + 1 + q % r;
      if (cc <= ii) Aw[ii * nf + cc] -= Aw[ii * nf + jc] * Aw[cc * nf + jc];
    }
    __syncthreads();
  }
  if (tid == 0 && bad) report_error(err, -4, -2);
  // inverse, one column per thread
  for (int c = tid; c < nf; c += nt) {
    for (int a = 0; a < nf; ++a) {
      double s = (a == c) ? 1.0 : 0.0;
      for (int k = 0; k < a; ++k) s -= Aw[a * nf + k] * Iw[k * nf + c];
      Iw[a * nf + c] = s / Aw[a * nf + a];
    }
    for (int a = nf - 1; a >= 0; --a) {
      double s = Iw[a * nf + c];
      for (int k = a + 1; k < nf; ++k) s -= Aw[k * nf + a] * Iw[k * nf + c];
      Iw[a * nf + c] = s / Aw[a * nf + a];
    }
  }
  if (par) {
    __syncthreads();
    for (int q = tid; q < nf * nf; q += nt) {
      A[q] = sA[q];
      Ainv[q] = sI[q];
    }
  }
}

int launch_coarse_assemble_factor(const LevelDev& L, const int* fpos, int nf, double* A1,
                                  double* A1inv, DevError* err, cudaStream_t st) {
  k_coarse_factor<<<1, 256, 0, st>>>(L, fpos, nf, A1, A1inv, err);
  return 1;
}

__global__ void k_coarse_solve(const int* __restrict__ fidx, int nf,
                               const double* __restrict__ Ainv, const double* __restrict__ r,
                               double* e) {
  pdl_enter();
  coarse_solve_body(fidx, nf, Ainv, r, e, threadIdx.x, blockDim.x);
}

int launch_coarse_solve(const LevelDev& L, const int* fidx, int nf, const double* A1inv,
                        const double* r, double* e, cudaStream_t st) {
  (void)L;
  launch_ex(k_coarse_solve, 1, 256, 0, true, st, fidx, nf, A1inv, r, e);
  return 1;
}

}  // namespace mgdtn
