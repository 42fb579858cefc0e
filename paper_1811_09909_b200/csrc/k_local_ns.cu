// Element-local solves of a NONSYMMETRIC context (IIPG-H and
// NIPG-H, Eq. IPG_H, s_f = 0 / -1; HDG and SIPG-H run through
// the same generic form there).  Per element, with t = tau h (refelem.h tables):
//   HDG (u eliminated first):   Q = K G + t F,                 Y = K P + t E,
//                               Bf^T = Y,                      S0 = K W + t H
//   IPDG-H (s_f = 1, 0, -1):    Q = K (L - N - s_f N^T) + t F,  Y = t E - s_f K Nl,
//                               Bf^T = t E - K Nl,             S0 = t H
//   S_T = S0 - Bf Q^-1 Y  (= -d flux / d lambda),  b_T = Bf Q^-1 f_w,
//   q_T = Q^-1 (Y lambda_T + f_w)  (volume recovery).
// For s_f != 1 Q is nonsymmetric, so the symmetric path's host-diagonalised
// pencil does not apply: one warp per element factors Q (NV = (p+1)^2 <= 25) by
// Gaussian elimination with partial pivoting in shared memory and solves for all
// right-hand sides at once.  S_T is stored full (row-major, LevelDev::ns).
#include "bodies.cuh"

namespace mgdtn {

namespace {

constexpr int NS_WARPS = 4;

__device__ __forceinline__ double s_f_of(int meth) {
  return meth == 1 ? 1.0 : meth == 2 ? 0.0 : -1.0;   // SIPG-H, IIPG-H, NIPG-H
}

// Q (NV x NV, row-major) into shared memory, lanes over entries
template <int NV>
__device__ __forceinline__ void ns_assemble_Q(const RefDev& R, int meth, double Kc, double t,
                                              double* Q, int lane) {
  const double sf = s_f_of(meth);
  for (int q = lane; q < NV * NV; q += 32) {
    const int i = q / NV, j = q - (q / NV) * NV;
    double v;
    if (meth == 0) v = fma(Kc, __ldg(R.G + q), t * __ldg(R.F + q));
    else
      v = fma(Kc, __ldg(R.Lv + q) - __ldg(R.Nv + q) - sf * __ldg(R.Nv + j * NV + i),
              t * __ldg(R.F + q));
    Q[q] = v;
  }
}

// Y[i][b] (coupling of volume row i to trace dof b) and Bf^T[i][a] (flux row a)
template <int M>
__device__ __forceinline__ double ns_Y(const RefDev& R, int meth, double Kc, double t, int i,
                                       int b) {
  const int q = i * M + b;
  if (meth == 0) return fma(Kc, __ldg(R.P + q), t * __ldg(R.E + q));
  return fma(-s_f_of(meth) * Kc, __ldg(R.Nl + q), t * __ldg(R.E + q));
}
template <int M>
__device__ __forceinline__ double ns_BfT(const RefDev& R, int meth, double Kc, double t, int i,
                                         int a) {
  const int q = i * M + a;
  if (meth == 0) return fma(Kc, __ldg(R.P + q), t * __ldg(R.E + q));
  return fma(-Kc, __ldg(R.Nl + q), t * __ldg(R.E + q));
}

// X <- Q^-1 X (X: NV x nc row-major) by Gaussian elimination with partial pivoting,
// one warp; Q is overwritten by its factors.  Returns false on a zero pivot.
template <int NV>
__device__ bool warp_lu_solve(double* Q, double* X, int nc, int lane) {
  static_assert(NV <= 32, "one pivot candidate per lane");
  bool ok = true;
  for (int k = 0; k < NV; ++k) {
    const int r = k + lane;
    double v = r < NV ? fabs(Q[r * NV + k]) : -1.0;
    int idx = r;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double v2 = __shfl_xor_sync(0xffffffffu, v, o);
      const int i2 = __shfl_xor_sync(0xffffffffu, idx, o);
      if (v2 > v || (v2 == v && i2 < idx)) {
        v = v2;
        idx = i2;
      }
    }
    if (!(v > 0.0)) {   // singular: keep going on a unit pivot, report once
      ok = false;
      if (lane == 0) Q[k * NV + k] = 1.0;
      idx = k;
    }
    if (idx != k) {
      for (int c = lane; c < NV + nc; c += 32) {
        double* a = c < NV ? Q + k * NV + c : X + k * nc + (c - NV);
        double* b = c < NV ? Q + idx * NV + c : X + idx * nc + (c - NV);
        const double tmp = *a;
        *a = *b;
        *b = tmp;
      }
    }
    __syncwarp();
    const double piv = Q[k * NV + k];
    if (lane < NV - k - 1) Q[(k + 1 + lane) * NV + k] /= piv;
    __syncwarp();
    const int w = NV - k - 1 + nc;   // trailing columns of [Q | X]
    const int tot = (NV - k - 1) * w;
    for (int q = lane; q < tot; q += 32) {
      const int rr = k + 1 + q / w, cc = q - (q / w) * w;
      const double l = Q[rr * NV + k];
      if (cc < NV - k - 1) Q[rr * NV + k + 1 + cc] -= l * Q[k * NV + k + 1 + cc];
      else X[rr * nc + (cc - (NV - k - 1))] -= l * X[k * nc + (cc - (NV - k - 1))];
    }
    __syncwarp();
  }
  for (int k = NV - 1; k >= 0; --k) {
    const double dk = Q[k * NV + k];
    for (int c = lane; c < nc; c += 32) X[k * nc + c] /= dk;
    __syncwarp();
    for (int q = lane; q < k * nc; q += 32) {
      const int rr = q / nc, c = q - (q / nc) * nc;
      X[rr * nc + c] -= Q[rr * NV + k] * X[k * nc + c];
    }
    __syncwarp();
  }
  return ok;
}

// per-element checks shared by the three kernels; false -> element skipped (error reported)
__device__ __forceinline__ bool ns_element_ok(double Kc, double t, int meth, DevError* err,
                                              int64_t e, int lane) {
  if (Kc > 0.0 && t > 0.0 && meth >= 0 && meth <= 3) return true;
  if (lane == 0 && err) report_error(err, -1, e);
  return false;
}

// f_w,i = h^2 sum_q fq[q,i] f_q (weights folded into fq) into X[i * nc + col]
template <int NV>
__device__ __forceinline__ void ns_load(const RefDev& R, double h, const double* f_qp,
                                        double f_const, int64_t e, double* X, int nc, int col,
                                        int lane) {
  const int nq2 = R.nqf * R.nqf;
  for (int i = lane; i < NV; i += 32) {
    double acc = 0.0;
    for (int q = 0; q < nq2; ++q)
      acc = fma(__ldg(R.fq + q * NV + i), f_qp ? f_qp[e * nq2 + q] : f_const, acc);
    X[i * nc + col] = h * h * acc;
  }
}

}  // namespace

// ---------------------------------------------------------------- H1 (nonsymmetric): S_T
template <int P>
__global__ void __launch_bounds__(32 * NS_WARPS) k_local_dtn_ns(LevelDev L, RefDev R, double h,
                                                               const double* __restrict__ K,
                                                               const int8_t* __restrict__ method,
                                                               const double* __restrict__ tau,
                                                               DevError* err, int project) {
  constexpr int K1 = P + 1, NV = K1 * K1, M = 4 * K1;
  constexpr int QS = NV * NV > M * M ? NV * NV : M * M;   // M^2 > NV^2 for p <= 2
  __shared__ double sQ[NS_WARPS][QS];        // Q, then (aliased) S_T
  __shared__ double sX[NS_WARPS][NV * M];
  __shared__ double sRC[NS_WARPS][2 * M];    // row / column sums (projection)
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* Q = sQ[w];
  double* X = sX[w];
  double* rs = sRC[w];
  const int64_t nec = L.ne >> 1;
  for (int64_t tt = (int64_t)blockIdx.x * NS_WARPS + w; tt < 2 * nec;
       tt += (int64_t)gridDim.x * NS_WARPS) {
    const int colour = (int)(tt / nec);
    const int64_t s = tt - colour * nec;
    int i, j;
    slot_elem(L.nx, colour, s, i, j);
    const int64_t e = (int64_t)j * L.nx + i;
    const double Kc = K[e], t = tau[e] * h;
    const int meth = method[e];
    if (!ns_element_ok(Kc, t, meth, err, e, lane)) continue;
    ns_assemble_Q<NV>(R, meth, Kc, t, Q, lane);
    for (int q = lane; q < NV * M; q += 32) X[q] = ns_Y<M>(R, meth, Kc, t, q / M, q % M);
    __syncwarp();
    if (!warp_lu_solve<NV>(Q, X, M, lane) && lane == 0) report_error(err, -3, e);
    // S = S0 - Bf X into Q's storage (Q no longer needed)
    double* S = Q;
    for (int q = lane; q < M * M; q += 32) {
      const int a = q / M, b = q - (q / M) * M;
      double acc = (meth == 0 ? Kc * __ldg(R.W + q) : 0.0) + t * __ldg(R.H + q);
      for (int v = 0; v < NV; ++v) acc = fma(-ns_BfT<M>(R, meth, Kc, t, v, a), X[v * M + b], acc);
      S[q] = acc;
    }
    __syncwarp();
    double* dst = L.S + s_offset(L.nchunk, L.npk, colour, s, 0);
    if (project) {
      // constants are a right AND a left null vector of S_T (q = lambda = c solves the
      // local problem; test w = 1 gives a lambda-independent total flux), F2:
      // S <- P S P, P = I - 1 1^T / m (reading R5)
      if (lane < M) {
        double r = 0.0, c = 0.0;
        for (int b = 0; b < M; ++b) {
          r += S[lane * M + b];
          c += S[b * M + lane];
        }
        rs[lane] = r;
        rs[M + lane] = c;
      }
      __syncwarp();
      double sig = 0.0;
      for (int b = 0; b < M; ++b) sig += rs[b];
      const double inv_m = 1.0 / M, c0 = sig * inv_m * inv_m;
      for (int q = lane; q < M * M; q += 32) {
        const int a = q / M, b = q - (q / M) * M;
        dst[(int64_t)q * 32] = (S[q] - (rs[a] + rs[M + b]) * inv_m) + c0;
      }
    } else {
      for (int q = lane; q < M * M; q += 32) dst[(int64_t)q * 32] = S[q];
    }
    __syncwarp();
  }
}

// ---------------------------------------------------------------- right-hand side (nonsymmetric)
// b_T = Bf Q^-1 f_w, minus S_T lambda_D on elements touching dOmega; 2-colour scatter
template <int P>
__global__ void __launch_bounds__(32 * NS_WARPS) k_local_rhs_ns(
    LevelDev L, RefDev R, double h, const double* __restrict__ K,
    const int8_t* __restrict__ method, const double* __restrict__ tau,
    const double* __restrict__ f_qp, double f_const, const double* __restrict__ lamD, double* g,
    int colour) {
  constexpr int K1 = P + 1, NV = K1 * K1, M = 4 * K1;
  __shared__ double sQ[NS_WARPS][NV * NV];
  __shared__ double sX[NS_WARPS][NV];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* Q = sQ[w];
  double* X = sX[w];
  const int64_t nec = L.ne >> 1;
  for (int64_t s = (int64_t)blockIdx.x * NS_WARPS + w; s < nec;
       s += (int64_t)gridDim.x * NS_WARPS) {
    int i, j;
    slot_elem(L.nx, colour, s, i, j);
    const int64_t e = (int64_t)j * L.nx + i;
    const double Kc = K[e], t = tau[e] * h;
    const int meth = method[e];
    if (!ns_element_ok(Kc, t, meth, nullptr, e, lane)) continue;
    ns_assemble_Q<NV>(R, meth, Kc, t, Q, lane);
    ns_load<NV>(R, h, f_qp, f_const, e, X, 1, 0, lane);
    __syncwarp();
    warp_lu_solve<NV>(Q, X, 1, lane);
    int64_t ed[4];
    bool bd[4];
    elem_edges(L.nx, L.ny, i, j, ed, bd, L.dmask);
    if (lane < M) {
      const int a = lane, f = a / K1, al = a - f * K1;
      double b = 0.0;
      for (int v = 0; v < NV; ++v) b = fma(ns_BfT<M>(R, meth, Kc, t, v, a), X[v], b);
      if (lamD && (bd[0] || bd[1] || bd[2] || bd[3])) {   // b -= S_T lambda_D
        const double* Sp = L.S + s_offset(L.nchunk, L.npk, colour, s, 0);
        for (int g2 = 0; g2 < 4; ++g2) {
          if (!bd[g2]) continue;
          for (int c = 0; c < K1; ++c)
            b = fma(-Sp[(int64_t)(a * M + g2 * K1 + c) * 32], lamD[ed[g2] * K1 + c], b);
        }
      }
      if (!bd[f]) {
        const int64_t idx = ed[f] * K1 + al;
        g[idx] = colour == 0 ? b : g[idx] + b;
      }
    }
    __syncwarp();
  }
}

// ---------------------------------------------------------------- volume recovery (nonsymmetric)
template <int P>
__global__ void __launch_bounds__(32 * NS_WARPS) k_recover_ns(
    LevelDev L, RefDev R, double h, const double* __restrict__ K,
    const int8_t* __restrict__ method, const double* __restrict__ tau,
    const double* __restrict__ lam, const double* __restrict__ f_qp, double f_const,
    double* q_out, const double* __restrict__ qex, double* partials) {
  constexpr int K1 = P + 1, NV = K1 * K1, M = 4 * K1;
  __shared__ double sQ[NS_WARPS][NV * NV];
  __shared__ double sX[NS_WARPS][NV];
  __shared__ double sL[NS_WARPS][M];
  __shared__ double red[NS_WARPS];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* Q = sQ[w];
  double* X = sX[w];
  double* lt = sL[w];
  const int nq2 = R.nqf * R.nqf;
  double err = 0.0;
  for (int64_t e = (int64_t)blockIdx.x * NS_WARPS + w; e < L.ne;
       e += (int64_t)gridDim.x * NS_WARPS) {
    const int j = (int)(e / L.nx), i = (int)(e - (int64_t)j * L.nx);
    const double Kc = K[e], t = tau[e] * h;
    const int meth = method[e];
    if (!ns_element_ok(Kc, t, meth, nullptr, e, lane)) continue;
    int64_t ed[4];
    bool bd[4];
    elem_edges(L.nx, L.ny, i, j, ed, bd, L.dmask);
    if (lane < M) lt[lane] = lam[ed[lane / K1] * K1 + lane % K1];
    ns_assemble_Q<NV>(R, meth, Kc, t, Q, lane);
    ns_load<NV>(R, h, f_qp, f_const, e, X, 1, 0, lane);
    __syncwarp();
    for (int v = lane; v < NV; v += 32) {   // + Y lambda_T
      double acc = X[v];
      for (int b = 0; b < M; ++b) acc = fma(ns_Y<M>(R, meth, Kc, t, v, b), lt[b], acc);
      X[v] = acc;
    }
    __syncwarp();
    warp_lu_solve<NV>(Q, X, 1, lane);
    for (int v = lane; v < NV; v += 32) q_out[e * NV + v] = X[v];
    if (qex) {
      double sacc = 0.0;
      for (int q = lane; q < nq2; q += 32) {
        double val = 0.0;
        for (int k = 0; k < NV; ++k) val = fma(R.vq[q * NV + k], X[k], val);
        const double dq = val - qex[e * nq2 + q];
        sacc = fma(R.wq[q] * dq, dq, sacc);
      }
      err = fma(h * h, sacc, err);
    }
    __syncwarp();
  }
  if (qex) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) err += __shfl_xor_sync(0xffffffffu, err, o);
    if (lane == 0) red[w] = err;
    __syncthreads();
    if (threadIdx.x == 0) partials[blockIdx.x] = (red[0] + red[1]) + (red[2] + red[3]);
  }
}

// ---------------------------------------------------------------- launchers
static int ns_grid(int64_t items) {
  const int64_t g = (items + NS_WARPS - 1) / NS_WARPS;
  return (int)(g < 148 * 16 ? (g > 0 ? g : 1) : 148 * 16);
}

int launch_local_dtn_ns(const LevelDev& L, const RefDev& R, double h, const double* K,
                        const int8_t* method, const double* tau, DevError* err, int project,
                        cudaStream_t st) {
  const int grid = ns_grid(L.ne);
  switch (L.p) {
    case 1: k_local_dtn_ns<1><<<grid, 32 * NS_WARPS, 0, st>>>(L, R, h, K, method, tau, err, project); break;
    case 2: k_local_dtn_ns<2><<<grid, 32 * NS_WARPS, 0, st>>>(L, R, h, K, method, tau, err, project); break;
    case 3: k_local_dtn_ns<3><<<grid, 32 * NS_WARPS, 0, st>>>(L, R, h, K, method, tau, err, project); break;
    default: k_local_dtn_ns<4><<<grid, 32 * NS_WARPS, 0, st>>>(L, R, h, K, method, tau, err, project); break;
  }
  return 1;
}

int launch_local_rhs_ns(const LevelDev& L, const RefDev& R, double h, const double* K,
                        const int8_t* method, const double* tau, const double* f_qp,
                        double f_const, const double* lamD, double* g, cudaStream_t st) {
  const int grid = ns_grid(L.ne / 2);
  for (int c = 0; c < 2; ++c) {
    switch (L.p) {
      case 1: k_local_rhs_ns<1><<<grid, 32 * NS_WARPS, 0, st>>>(L, R, h, K, method, tau, f_qp, f_const, lamD, g, c); break;
      case 2: k_local_rhs_ns<2><<<grid, 32 * NS_WARPS, 0, st>>>(L, R, h, K, method, tau, f_qp, f_const, lamD, g, c); break;
      case 3: k_local_rhs_ns<3><<<grid, 32 * NS_WARPS, 0, st>>>(L, R, h, K, method, tau, f_qp, f_const, lamD, g, c); break;
      default: k_local_rhs_ns<4><<<grid, 32 * NS_WARPS, 0, st>>>(L, R, h, K, method, tau, f_qp, f_const, lamD, g, c); break;
    }
  }
  return 2;
}

int launch_recover_ns(const LevelDev& L, const RefDev& R, double h, const double* K,
                      const int8_t* method, const double* tau, const double* lam,
                      const double* f_qp, double f_const, double* q_out, const double* qex_qp,
                      double* partials, int* grid_out, cudaStream_t st) {
  const int grid = ns_grid(L.ne);
  if (grid_out) *grid_out = grid;
  switch (L.p) {
    case 1: k_recover_ns<1><<<grid, 32 * NS_WARPS, 0, st>>>(L, R, h, K, method, tau, lam, f_qp, f_const, q_out, qex_qp, partials); break;
    case 2: k_recover_ns<2><<<grid, 32 * NS_WARPS, 0, st>>>(L, R, h, K, method, tau, lam, f_qp, f_const, q_out, qex_qp, partials); break;
    case 3: k_recover_ns<3><<<grid, 32 * NS_WARPS, 0, st>>>(L, R, h, K, method, tau, lam, f_qp, f_const, q_out, qex_qp, partials); break;
    default: k_recover_ns<4><<<grid, 32 * NS_WARPS, 0, st>>>(L, R, h, K, method, tau, lam, f_qp, f_const, q_out, qex_qp, partials); break;
  }
  return 1;
}

}  // namespace mgdtn
