// Setup kernels: batched element-local static condensation (H1), the
// right-hand side, p-coarsening (H2), per-agglomerate Galerkin coarse DtN
// (H3), edge-block diagonals (H4) and the coarsest dense factor (H5).
#include "bodies.cuh"

namespace mgdtn {

// ============================================================================
// H1: element DtN maps.  PAPER.md:305-316 ("express the local volume unknowns
// ... element-by-element, as a function of the skeletal unknowns"); HDG
// Eqs. HDG/HDG_flux, SIPG-H Eq. SIPG_H.
// One warp per element, local matrices in shared memory:
//   Q = K G + t F (HDG) | K LN + t F (SIPG),  R = K P + t E | t E - K Nl,
//   Q = L L^T,  Y = L^-1 R,  S_T = S0 - Y^T Y,  S0 = K W + t H | t H,  t = tau h.
// ============================================================================
template <int P>
struct LocalShape {
  static constexpr int K1 = P + 1, NV = K1 * K1, M = 4 * K1, NPK = M * (M + 1) / 2;
};

constexpr int LOC_WARPS = 4;

template <int P>
__device__ __forceinline__ bool local_factor(const RefDev& R, double Kc, double t, int meth,
                                             double* Q, double* Rm, int lane) {
  using Sh = LocalShape<P>;
  constexpr int NV = Sh::NV, M = Sh::M;
  for (int idx = lane; idx < NV * NV; idx += 32)
    Q[idx] = (meth == 0 ? Kc * R.G[idx] : Kc * R.LN[idx]) + t * R.F[idx];
  for (int idx = lane; idx < NV * M; idx += 32)
    Rm[idx] = meth == 0 ? fma(Kc, R.P[idx], t * R.E[idx]) : t * R.E[idx] - Kc * R.Nl[idx];
  __syncwarp();
  bool ok = true;
  // right-looking Cholesky, lower triangle in place
  for (int jc = 0; jc < NV; ++jc) {
    double dj = Q[jc * NV + jc];
    if (!(dj > 0.0)) ok = false;
    dj = sqrt(fmax(dj, 1e-300));
    __syncwarp();
    if (lane == 0) Q[jc * NV + jc] = dj;
    for (int i = jc + 1 + lane; i < NV; i += 32) Q[i * NV + jc] /= dj;
    __syncwarp();
    const int nt = NV - jc - 1;
    for (int q = lane; q < nt * nt; q += 32) {
      int ii = jc + 1 + q / nt, cc = jc + 1 + q % nt;
      if (cc <= ii) Q[ii * NV + cc] -= Q[ii * NV + jc] * Q[cc * NV + jc];
    }
    __syncwarp();
  }
  // Y = L^-1 R, lanes over the m columns
  if (lane < M) {
    for (int i = 0; i < NV; ++i) {
      double s = Rm[i * M + lane];
      for (int k = 0; k < i; ++k) s -= Q[i * NV + k] * Rm[k * M + lane];
      Rm[i * M + lane] = s / Q[i * NV + i];
    }
  }
  __syncwarp();
  return ok;
}

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
__global__ void __launch_bounds__(32 * LOC_WARPS) k_local_dtn(LevelDev L, RefDev R, double h,
                                                              const double* __restrict__ K,
                                                              const int8_t* __restrict__ method,
                                                              const double* __restrict__ tau,
                                                              DevError* err) {
  using Sh = LocalShape<P>;
  constexpr int NV = Sh::NV, M = Sh::M, NPK = Sh::NPK;
  __shared__ double smQ[LOC_WARPS][NV * NV];
  __shared__ double smR[LOC_WARPS][NV * M];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* Q = smQ[w];
  double* Rm = smR[w];
  for (int64_t e = (int64_t)blockIdx.x * LOC_WARPS + w; e < L.ne;
       e += (int64_t)gridDim.x * LOC_WARPS) {
    const double Kc = K[e];
    const double t = tau[e] * h;
    const int meth = method[e];
    if (!(Kc > 0.0) || !(t > 0.0) || (meth != 0 && meth != 1)) {
      if (lane == 0) report_error(err, -1, e);
      continue;
    }
    bool ok = local_factor<P>(R, Kc, t, meth, Q, Rm, lane);
    if (!ok && lane == 0) report_error(err, -4, e);
    const int i = (int)(e % L.nx), j = (int)(e / L.nx);
    int colour;
    int64_t s;
    elem_slot(L.nx, i, j, colour, s);
    double* dst = L.S + s_offset(L.nchunk, NPK, colour, s, 0);
    for (int kk = lane; kk < NPK; kk += 32) {
      int a, b;
      pk_row_col(kk, M, a, b);
      double v = (meth == 0 ? Kc * R.W[a * M + b] : 0.0) + t * R.H[a * M + b];
      for (int r = 0; r < NV; ++r) v -= Rm[r * M + a] * Rm[r * M + b];
      dst[(int64_t)kk * 32] = v;
    }
    __syncwarp();
  }
}

int launch_local_dtn(const LevelDev& L, const RefDev& R, double h, const double* K,
                     const int8_t* method, const double* tau, DevError* err, cudaStream_t st) {
  int64_t g = (L.ne + LOC_WARPS - 1) / LOC_WARPS;
  int grid = (int)(g < 148 * 32 ? g : 148 * 32);
  switch (L.p) {
    case 1: k_local_dtn<1><<<grid, 32 * LOC_WARPS, 0, st>>>(L, R, h, K, method, tau, err); break;
    case 2: k_local_dtn<2><<<grid, 32 * LOC_WARPS, 0, st>>>(L, R, h, K, method, tau, err); break;
    case 3: k_local_dtn<3><<<grid, 32 * LOC_WARPS, 0, st>>>(L, R, h, K, method, tau, err); break;
    default: k_local_dtn<4><<<grid, 32 * LOC_WARPS, 0, st>>>(L, R, h, K, method, tau, err); break;
  }
  return 1;
}

// ============================================================================
// Right-hand side: b_T = R^T Q^-1 f_w (flux rows at lambda = 0), minus the
// Dirichlet lift S_T lambda_D, scattered with the same 2-colour rule as the
// apply (colour 0 writes, colour 1 adds, reading Q4).
// ============================================================================
template <int P>
__global__ void __launch_bounds__(32 * LOC_WARPS) k_local_rhs(
    LevelDev L, RefDev R, double h, const double* __restrict__ K,
    const int8_t* __restrict__ method, const double* __restrict__ tau,
    const double* __restrict__ f_qp, double f_const, const double* __restrict__ lamD, double* g,
    int colour) {
  using Sh = LocalShape<P>;
  constexpr int NV = Sh::NV, M = Sh::M, K1 = Sh::K1;
  __shared__ double smQ[LOC_WARPS][NV * NV];
  __shared__ double smR[LOC_WARPS][NV * M];
  __shared__ double smv[LOC_WARPS][NV + 2 * M];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* Q = smQ[w];
  double* Rm = smR[w];
  double* z = smv[w];
  double* lamT = smv[w] + NV;
  double* bT = smv[w] + NV + M;
  const int64_t nec = L.ne >> 1;
  const int nq = R.nqf;
  for (int64_t s = (int64_t)blockIdx.x * LOC_WARPS + w; s < nec;
       s += (int64_t)gridDim.x * LOC_WARPS) {
    int i, j;
    slot_elem(L.nx, colour, s, i, j);
    const int64_t e = (int64_t)j * L.nx + i;
    const double Kc = K[e], t = tau[e] * h;
    const int meth = method[e];
    local_factor<P>(R, Kc, t, meth, Q, Rm, lane);
    int64_t ed[4];
    bool bd[4];
    elem_edges(L.nx, L.ny, i, j, ed, bd);
    // f_w = h^2 sum_q fq[q][i] f_q
    for (int a = lane; a < NV; a += 32) {
      double acc = 0.0;
      for (int q = 0; q < nq * nq; ++q)
        acc += R.fq[q * NV + a] * (f_qp ? f_qp[e * nq * nq + q] : f_const);
      z[a] = h * h * acc;
    }
    for (int c = lane; c < M; c += 32) {
      int f = c / K1;
      lamT[c] = (bd[f] && lamD) ? lamD[ed[f] * K1 + (c % K1)] : 0.0;
    }
    __syncwarp();
    if (lane == 0) {  // z = L^-1 f_w
      for (int a = 0; a < NV; ++a) {
        double sacc = z[a];
        for (int k = 0; k < a; ++k) sacc -= Q[a * NV + k] * z[k];
        z[a] = sacc / Q[a * NV + a];
      }
    }
    __syncwarp();
    if (lane < M) {
      // b = Y^T z - S lamD,  S = S0 - Y^T Y
      double b = 0.0;
      for (int r = 0; r < NV; ++r) b += Rm[r * M + lane] * z[r];
      double sl = 0.0;
      for (int c = 0; c < M; ++c) {
        if (lamT[c] == 0.0) continue;
        double sv = (meth == 0 ? Kc * R.W[lane * M + c] : 0.0) + t * R.H[lane * M + c];
        for (int r = 0; r < NV; ++r) sv -= Rm[r * M + lane] * Rm[r * M + c];
        sl += sv * lamT[c];
      }
      bT[lane] = b - sl;
    }
    __syncwarp();
    if (lane < M) {
      int f = lane / K1;
      if (!bd[f]) {
        int64_t idx = ed[f] * K1 + (lane % K1);
        g[idx] = colour == 0 ? bT[lane] : g[idx] + bT[lane];
      }
    }
    __syncwarp();
  }
}

int launch_local_rhs(const LevelDev& L, const RefDev& R, double h, const double* K,
                     const int8_t* method, const double* tau, const double* f_qp,
                     double f_const, const double* lamD, double* g, DevError* err,
                     cudaStream_t st) {
  (void)err;
  int64_t gsz = (L.ne / 2 + LOC_WARPS - 1) / LOC_WARPS;
  int grid = (int)(gsz < 148 * 32 ? gsz : 148 * 32);
  for (int c = 0; c < 2; ++c) {
    switch (L.p) {
      case 1: k_local_rhs<1><<<grid, 32 * LOC_WARPS, 0, st>>>(L, R, h, K, method, tau, f_qp, f_const, lamD, g, c); break;
      case 2: k_local_rhs<2><<<grid, 32 * LOC_WARPS, 0, st>>>(L, R, h, K, method, tau, f_qp, f_const, lamD, g, c); break;
      case 3: k_local_rhs<3><<<grid, 32 * LOC_WARPS, 0, st>>>(L, R, h, K, method, tau, f_qp, f_const, lamD, g, c); break;
      default: k_local_rhs<4><<<grid, 32 * LOC_WARPS, 0, st>>>(L, R, h, K, method, tau, f_qp, f_const, lamD, g, c); break;
    }
  }
  return 2;
}

// Dirichlet values: per-edge L2 projection of g_D onto P^p (reading Q4).
__global__ void k_dirichlet(LevelDev L, RefDev R, const double* __restrict__ gD, double* lamD) {
  const int nb = 2 * L.nx + 2 * L.ny;
  const int K1 = L.k1, nq = R.nqf;
  for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < nb; b += gridDim.x * blockDim.x) {
    int64_t e;
    if (b < L.nx) e = hedge(L.nx, b, 0);
    else if (b < 2 * L.nx) e = hedge(L.nx, b - L.nx, L.ny);
    else if (b < 2 * L.nx + L.ny) e = vedge(L.nx, L.ny, 0, b - 2 * L.nx);
    else e = vedge(L.nx, L.ny, L.nx, b - 2 * L.nx - L.ny);
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
__device__ __forceinline__ double pk_get(const double* base, int m, int a, int b) {
  if (a > b) { int t = a; a = b; b = t; }
  return base[(int64_t)pk_index(a, b, m) * 32];
}

__global__ void k_p_coarsen(LevelDev F, LevelDev C, const double* __restrict__ Jp) {
  const int K1 = F.k1, m = F.m;
  const int64_t nec = F.ne >> 1;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < 2 * nec;
       t += (int64_t)gridDim.x * blockDim.x) {
    int colour = (int)(t / nec);
    int64_t s = t - colour * nec;
    const double* src = F.S + s_offset(F.nchunk, F.npk, colour, s, 0);
    double* dst = C.S + s_offset(C.nchunk, C.npk, colour, s, 0);
    for (int A = 0; A < 8; ++A)
      for (int B = A; B < 8; ++B) {
        int f = A >> 1, al = A & 1, g = B >> 1, be = B & 1;
        double acc = 0.0;
        for (int a = 0; a < K1; ++a) {
          double inner = 0.0;
          for (int b = 0; b < K1; ++b) inner += pk_get(src, m, f * K1 + a, g * K1 + b) * Jp[b * 2 + be];
          acc += Jp[a * 2 + al] * inner;
        }
        dst[(int64_t)pk_index(A, B, 8) * 32] = acc;
      }
  }
}

int launch_p_coarsen(const LevelDev& F, const LevelDev& C, const double* Jp, cudaStream_t st) {
  int64_t n = F.ne;
  int grid = (int)((n + 127) / 128 < 148 * 16 ? (n + 127) / 128 : 148 * 16);
  k_p_coarsen<<<grid, 128, 0, st>>>(F, C, Jp);
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

__global__ void __launch_bounds__(32 * AGG_WARPS) k_agglomerate(LevelDev F, LevelDev C,
                                                                double* KIIinv, double* Pm,
                                                                DevError* err) {
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
      const double* src = F.S + s_offset(F.nchunk, 36, colour, s, 0);
      // child S (dense 8x8) into Sc, G_c (8 x 16) into G
      for (int q = lane; q < 64; q += 32) {
        int a = q >> 3, b = q & 7;
        Sc[q] = pk_get(src, 8, a, b);
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
    // Cholesky of Kr_II (8x8, lower, in Sc)
    for (int q = lane; q < 64; q += 32) Sc[q] = Kr[(q >> 3) * 16 + (q & 7)];
    __syncwarp();
    bool ok = true;
    if (lane == 0) {
      for (int jc = 0; jc < 8; ++jc) {
        double d = Sc[jc * 8 + jc];
        for (int k = 0; k < jc; ++k) d -= Sc[jc * 8 + k] * Sc[jc * 8 + k];
        if (!(d > 0.0)) { ok = false; d = 1e-300; }
        d = sqrt(d);
        Sc[jc * 8 + jc] = d;
        for (int i2 = jc + 1; i2 < 8; ++i2) {
          double sacc = Sc[i2 * 8 + jc];
          for (int k = 0; k < jc; ++k) sacc -= Sc[i2 * 8 + k] * Sc[jc * 8 + k];
          Sc[i2 * 8 + jc] = sacc / d;
        }
      }
      if (!ok) report_error(err, -4, M);
    }
    __syncwarp();
    // columns: lanes 0..7 -> A_II^-1 e_col ; lanes 8..15 -> A_II^-1 Kr_IC[:, col]
    if (lane < 16) {
      double v[8];
      for (int a = 0; a < 8; ++a)
        v[a] = lane < 8 ? (a == lane ? 1.0 : 0.0) : Kr[a * 16 + 8 + (lane - 8)];
      for (int a = 0; a < 8; ++a) {
        double sacc = v[a];
        for (int k = 0; k < a; ++k) sacc -= Sc[a * 8 + k] * v[k];
        v[a] = sacc / Sc[a * 8 + a];
      }
      for (int a = 7; a >= 0; --a) {
        double sacc = v[a];
        for (int k = a + 1; k < 8; ++k) sacc -= Sc[k * 8 + a] * v[k];
        v[a] = sacc / Sc[a * 8 + a];
      }
      if (lane < 8) {
        for (int a = 0; a < 8; ++a) KIIinv[M * 64 + a * 8 + lane] = v[a];
      } else {
        for (int a = 0; a < 8; ++a) {
          Pm[M * 64 + a * 8 + (lane - 8)] = -v[a];
          U[a * 16 + (lane - 8)] = -v[a];   // keep P_M for S_c
        }
      }
    }
    __syncwarp();
    // S_c = Kr_CC + Kr_IC^T P_M, packed upper (36), into the coarse storage
    {
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
                       DevError* err, cudaStream_t st) {
  int64_t nmac = (int64_t)(F.nx / 2) * (F.ny / 2);
  int64_t g = (nmac + AGG_WARPS - 1) / AGG_WARPS;
  int grid = (int)(g < 148 * 16 ? g : 148 * 16);
  k_agglomerate<<<grid, 32 * AGG_WARPS, 0, st>>>(F, C, KIIinv, Pm, err);
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
    if (edge_on_boundary(L.nx, L.ny, e)) {
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
      int colour;
      int64_t s;
      elem_slot(L.nx, ei[t], ej[t], colour, s);
      const double* src = L.S + s_offset(L.nchunk, L.npk, colour, s, 0);
      for (int a = 0; a < K1; ++a)
        for (int b = 0; b < K1; ++b) D[a * K1 + b] += pk_get(src, m, ef[t] * K1 + a, ef[t] * K1 + b);
    }
    // Cholesky + explicit inverse
    double Lc[MAX_K1 * MAX_K1];
    bool ok = true;
    for (int j = 0; j < K1; ++j) {
      double d = D[j * K1 + j];
      for (int k = 0; k < j; ++k) d -= Lc[j * K1 + k] * Lc[j * K1 + k];
      if (!(d > 0.0)) { ok = false; d = 1e-300; }
      d = sqrt(d);
      Lc[j * K1 + j] = d;
      for (int i = j + 1; i < K1; ++i) {
        double s = D[i * K1 + j];
        for (int k = 0; k < j; ++k) s -= Lc[i * K1 + k] * Lc[j * K1 + k];
        Lc[i * K1 + j] = s / d;
      }
    }
    if (!ok) report_error(err, -4, e);
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
      for (int a = 0; a < K1; ++a) out[(a * K1 + c) * sd] = v[a];
    }
  }
}

int launch_edge_blocks(const LevelDev& L, DevError* err, cudaStream_t st) {
  int64_t g = (L.nedge + 127) / 128;
  int grid = (int)(g < 148 * 16 ? g : 148 * 16);
  k_edge_blocks<<<grid, 128, 0, st>>>(L, err);
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
      for (int b = a; b < L.m; ++b) dst[(int64_t)pk_index(a, b, L.m) * 32] = a0[a * L.m + b];
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
      for (int b = 0; b < L.m; ++b) a0[a * L.m + b] = pk_get(src, L.m, a, b);
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

// ============================================================================
// H5: coarsest level, B_1 = A_1^-1 by a direct solver.
// One CTA assembles the dense free-dof matrix, factors it (Cholesky) and
// forms the explicit inverse used by every V-cycle.
// ============================================================================
__global__ void k_coarse_factor(LevelDev L, const int* __restrict__ fpos, int nf, double* A,
                                double* Ainv, DevError* err) {
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int q = tid; q < nf * nf; q += nt) A[q] = 0.0;
  __syncthreads();
  if (tid == 0) {
    for (int64_t e = 0; e < L.ne; ++e) {
      int i = (int)(e % L.nx), j = (int)(e / L.nx), colour;
      int64_t s;
      elem_slot(L.nx, i, j, colour, s);
      const double* src = L.S + s_offset(L.nchunk, L.npk, colour, s, 0);
      int64_t ed[4];
      bool bd[4];
      elem_edges(L.nx, L.ny, i, j, ed, bd);
      int gi[4 * MAX_K1];
      for (int f = 0; f < 4; ++f)
        for (int a = 0; a < L.k1; ++a) gi[f * L.k1 + a] = fpos[ed[f] * L.k1 + a];
      for (int a = 0; a < L.m; ++a)
        for (int b = 0; b < L.m; ++b)
          if (gi[a] >= 0 && gi[b] >= 0) A[gi[a] * nf + gi[b]] += pk_get(src, L.m, a, b);
    }
  }
  __syncthreads();
  __shared__ int bad;
  if (tid == 0) bad = 0;
  __syncthreads();
  for (int jc = 0; jc < nf; ++jc) {
    if (tid == 0) {
      double d = A[jc * nf + jc];
      if (!(d > 0.0)) { bad = 1; d = 1e-300; }
      A[jc * nf + jc] = sqrt(d);
    }
    __syncthreads();
    const double dj = A[jc * nf + jc];
    for (int i = jc + 1 + tid; i < nf; i += nt) A[i * nf + jc] /= dj;
    __syncthreads();
    const int r = nf - jc - 1;
    for (int q = tid; q < r * r; q += nt) {
      int ii = jc + 1 + q / r, cc = jc + 1 + q % r;
      if (cc <= ii) A[ii * nf + cc] -= A[ii * nf + jc] * A[cc * nf + jc];
    }
    __syncthreads();
  }
  if (tid == 0 && bad) report_error(err, -4, -2);
  // inverse, one column per thread
  for (int c = tid; c < nf; c += nt) {
    for (int a = 0; a < nf; ++a) {
      double s = (a == c) ? 1.0 : 0.0;
      for (int k = 0; k < a; ++k) s -= A[a * nf + k] * Ainv[k * nf + c];
      Ainv[a * nf + c] = s / A[a * nf + a];
    }
    for (int a = nf - 1; a >= 0; --a) {
      double s = Ainv[a * nf + c];
      for (int k = a + 1; k < nf; ++k) s -= A[k * nf + a] * Ainv[k * nf + c];
      Ainv[a * nf + c] = s / A[a * nf + a];
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
  coarse_solve_body(fidx, nf, Ainv, r, e, threadIdx.x, blockDim.x);
}

int launch_coarse_solve(const LevelDev& L, const int* fidx, int nf, const double* A1inv,
                        const double* r, double* e, cudaStream_t st) {
  (void)L;
  k_coarse_solve<<<1, 256, 0, st>>>(fidx, nf, A1inv, r, e);
  return 1;
}

}  // namespace mgdtn
