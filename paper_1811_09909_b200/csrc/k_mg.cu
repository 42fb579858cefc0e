// V-cycle transfer / smoothing kernels and PCG vector kernels.
//
// Transfers: p-level I_N = J_N, Q_{N-1} = J_N^T (per
// edge); h-levels I_k = [P_M ; J], Q_{k-1} = [P_M^T , J^T] with
// P_M = -A_II^-1 A_IB J per macro.  Local correction T_k = [A_II^-1 0; 0 0]
// (Eq. 3.11) per macro.  Reductions are deterministic two-stage trees.
#include "kernels.cuh"

namespace mgdtn {

static inline int cap_grid(int64_t work, int threads, int cap) {
  int64_t g = (work + threads - 1) / threads;
  if (g < 1) g = 1;
  return (int)(g < cap ? g : cap);
}

// ---------------------------------------------------------------- smoothing, first step
// e = 0 -> first smoothing step needs no apply: e = c2_0 Dinv r (d = e for Chebyshev).
__global__ void k_smooth_first(LevelDev L, const double* __restrict__ r, double* e, double* d) {
  const int K1 = L.k1;
  const double c2 = L.coef[1];
  for (int64_t ed = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; ed < L.nedge;
       ed += (int64_t)gridDim.x * blockDim.x) {
    if (edge_on_boundary(L.nx, L.ny, ed)) continue;
    const double* Di = L.Dinv + ed * K1 * K1;
    for (int a = 0; a < K1; ++a) {
      double c = 0.0;
      for (int b = 0; b < K1; ++b) c = fma(Di[a * K1 + b], r[ed * K1 + b], c);
      double v = c2 * c;
      e[ed * K1 + a] = v;
      if (L.smoother == 1) d[ed * K1 + a] = v;
    }
  }
}

int launch_smooth_first(const LevelDev& L, const double* r, double* e, double* d,
                        cudaStream_t st) {
  k_smooth_first<<<cap_grid(L.nedge, 128, 148 * 8), 128, 0, st>>>(L, r, e, d);
  return 1;
}

// ---------------------------------------------------------------- local correction + restriction (macro part)
__device__ __forceinline__ void macro_interior_edges(const LevelDev& F, int I, int J,
                                                     int64_t ie[4]) {
  ie[0] = hedge(F.nx, 2 * I, 2 * J + 1);
  ie[1] = hedge(F.nx, 2 * I + 1, 2 * J + 1);
  ie[2] = vedge(F.nx, F.ny, 2 * I + 1, 2 * J);
  ie[3] = vedge(F.nx, F.ny, 2 * I + 1, 2 * J + 1);
}

__global__ void k_lc_restrict(LevelDev F, const double* __restrict__ res, double* e,
                              const double* __restrict__ KIIinv, const double* __restrict__ Pm,
                              double* cbuf, int do_lc, int do_restrict) {
  const int nxc = F.nx >> 1;
  const int64_t nmac = (int64_t)nxc * (F.ny >> 1);
  for (int64_t M = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; M < nmac;
       M += (int64_t)gridDim.x * blockDim.x) {
    const int I = (int)(M % nxc), J = (int)(M / nxc);
    int64_t ie[4];
    macro_interior_edges(F, I, J, ie);
    double rI[8];
#pragma unroll
    for (int l = 0; l < 4; ++l) {
      rI[2 * l] = res[ie[l] * 2];
      rI[2 * l + 1] = res[ie[l] * 2 + 1];
    }
    if (do_lc) {
      const double* Ki = KIIinv + M * 64;
#pragma unroll
      for (int a = 0; a < 8; ++a) {
        double c = 0.0;
#pragma unroll
        for (int b = 0; b < 8; ++b) c = fma(Ki[a * 8 + b], rI[b], c);
        e[ie[a >> 1] * 2 + (a & 1)] += c;
      }
    }
    if (do_restrict) {
      const double* P = Pm + M * 64;
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        double acc = 0.0;
#pragma unroll
        for (int a = 0; a < 8; ++a) acc = fma(P[a * 8 + c], rI[a], acc);
        cbuf[M * 8 + c] = acc;
      }
    }
  }
}

int launch_lc_restrict(const LevelDev& F, const double* res, double* e, const double* KIIinv,
                       const double* Pm, double* cbuf, bool do_lc, bool do_restrict,
                       cudaStream_t st) {
  int64_t nmac = (int64_t)(F.nx / 2) * (F.ny / 2);
  k_lc_restrict<<<cap_grid(nmac, 128, 148 * 8), 128, 0, st>>>(F, res, e, KIIinv, Pm, cbuf,
                                                              do_lc, do_restrict);
  return 1;
}

// ---------------------------------------------------------------- restriction (coarse-edge part)
// rc = J^T res_B + sum_{M adjacent} (P_M^T res_I)[slot]; optionally fused with the
// coarse level's first smoothing step.
__global__ void k_restrict_edges(LevelDev F, LevelDev C, const double* __restrict__ res,
                                 const double* __restrict__ cbuf, double* rc, int fuse,
                                 double* ec, double* dc) {
  const int nxc = C.nx, nyc = C.ny;
  const int64_t nh = (int64_t)nxc * (nyc + 1);
  const double c2 = fuse ? C.coef[1] : 0.0;
  for (int64_t E = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; E < C.nedge;
       E += (int64_t)gridDim.x * blockDim.x) {
    double v0 = 0.0, v1 = 0.0;
    bool bnd;
    if (E < nh) {
      const int J = (int)(E / nxc), I = (int)(E % nxc);
      bnd = (J == 0 || J == nyc);
      if (!bnd) {
        const int64_t f0 = hedge(F.nx, 2 * I, 2 * J), f1 = hedge(F.nx, 2 * I + 1, 2 * J);
        const double a0 = res[f0 * 2], a1 = res[f0 * 2 + 1], b0 = res[f1 * 2], b1 = res[f1 * 2 + 1];
        v0 = a0 + 0.5 * a1 + 0.5 * b0;
        v1 = 0.5 * a1 + 0.5 * b0 + b1;
        const int64_t Mb = (int64_t)(J - 1) * nxc + I, Ma = (int64_t)J * nxc + I;
        v0 += cbuf[Mb * 8 + 4] + cbuf[Ma * 8 + 0];
        v1 += cbuf[Mb * 8 + 5] + cbuf[Ma * 8 + 1];
      }
    } else {
      const int64_t rr = E - nh;
      const int J = (int)(rr / (nxc + 1)), I = (int)(rr % (nxc + 1));
      bnd = (I == 0 || I == nxc);
      if (!bnd) {
        const int64_t f0 = vedge(F.nx, F.ny, 2 * I, 2 * J), f1 = vedge(F.nx, F.ny, 2 * I, 2 * J + 1);
        const double a0 = res[f0 * 2], a1 = res[f0 * 2 + 1], b0 = res[f1 * 2], b1 = res[f1 * 2 + 1];
        v0 = a0 + 0.5 * a1 + 0.5 * b0;
        v1 = 0.5 * a1 + 0.5 * b0 + b1;
        const int64_t Ml = (int64_t)J * nxc + (I - 1), Mr = (int64_t)J * nxc + I;
        v0 += cbuf[Ml * 8 + 2] + cbuf[Mr * 8 + 6];
        v1 += cbuf[Ml * 8 + 3] + cbuf[Mr * 8 + 7];
      }
    }
    rc[E * 2] = v0;
    rc[E * 2 + 1] = v1;
    if (fuse && !bnd) {
      const double* Di = C.Dinv + E * 4;
      double e0 = c2 * (Di[0] * v0 + Di[1] * v1);
      double e1 = c2 * (Di[2] * v0 + Di[3] * v1);
      ec[E * 2] = e0;
      ec[E * 2 + 1] = e1;
      if (C.smoother == 1) {
        dc[E * 2] = e0;
        dc[E * 2 + 1] = e1;
      }
    }
  }
}

int launch_restrict_edges(const LevelDev& F, const LevelDev& C, const double* res,
                          const double* cbuf, double* rc, bool fuse_first, double* ec,
                          double* dc, cudaStream_t st) {
  k_restrict_edges<<<cap_grid(C.nedge, 128, 148 * 8), 128, 0, st>>>(F, C, res, cbuf, rc,
                                                                    fuse_first, ec, dc);
  return 1;
}

// ---------------------------------------------------------------- prolongation (macro)
// e_I += P_M e_c(M); e_B += J e_c on the macro's bottom and left macro-edges
// (every interior macro-edge is the bottom or left edge of exactly one macro).
__global__ void k_prolong_macro(LevelDev F, LevelDev C, const double* __restrict__ ec,
                                const double* __restrict__ Pm, double* e) {
  const int nxc = C.nx, nyc = C.ny;
  const int64_t nmac = (int64_t)nxc * nyc;
  for (int64_t M = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; M < nmac;
       M += (int64_t)gridDim.x * blockDim.x) {
    const int I = (int)(M % nxc), J = (int)(M / nxc);
    int64_t ce[4];
    bool cb[4];
    elem_edges(nxc, nyc, I, J, ce, cb);
    double c[8];
#pragma unroll
    for (int f = 0; f < 4; ++f) {
      c[2 * f] = cb[f] ? 0.0 : ec[ce[f] * 2];
      c[2 * f + 1] = cb[f] ? 0.0 : ec[ce[f] * 2 + 1];
    }
    int64_t ie[4];
    macro_interior_edges(F, I, J, ie);
    const double* P = Pm + M * 64;
#pragma unroll
    for (int a = 0; a < 8; ++a) {
      double acc = 0.0;
#pragma unroll
      for (int b = 0; b < 8; ++b) acc = fma(P[a * 8 + b], c[b], acc);
      e[ie[a >> 1] * 2 + (a & 1)] += acc;
    }
    if (!cb[0]) {  // bottom macro-edge
      const double c0 = c[0], c1 = c[1], cm = 0.5 * (c0 + c1);
      const int64_t f0 = hedge(F.nx, 2 * I, 2 * J), f1 = hedge(F.nx, 2 * I + 1, 2 * J);
      e[f0 * 2] += c0;
      e[f0 * 2 + 1] += cm;
      e[f1 * 2] += cm;
      e[f1 * 2 + 1] += c1;
    }
    if (!cb[3]) {  // left macro-edge
      const double c0 = c[6], c1 = c[7], cm = 0.5 * (c0 + c1);
      const int64_t f0 = vedge(F.nx, F.ny, 2 * I, 2 * J), f1 = vedge(F.nx, F.ny, 2 * I, 2 * J + 1);
      e[f0 * 2] += c0;
      e[f0 * 2 + 1] += cm;
      e[f1 * 2] += cm;
      e[f1 * 2 + 1] += c1;
    }
  }
}

int launch_prolong_macro(const LevelDev& F, const LevelDev& C, const double* ec,
                         const double* Pm, double* e, cudaStream_t st) {
  int64_t nmac = (int64_t)C.nx * C.ny;
  k_prolong_macro<<<cap_grid(nmac, 128, 148 * 8), 128, 0, st>>>(F, C, ec, Pm, e);
  return 1;
}

// ---------------------------------------------------------------- p-level transfers (per edge)
__global__ void k_p_restrict(LevelDev F, LevelDev C, const double* __restrict__ Jp,
                             const double* __restrict__ res, double* rc, int fuse, double* ec,
                             double* dc) {
  const int K1 = F.k1;
  const double c2 = fuse ? C.coef[1] : 0.0;
  for (int64_t E = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; E < F.nedge;
       E += (int64_t)gridDim.x * blockDim.x) {
    if (edge_on_boundary(F.nx, F.ny, E)) {
      rc[E * 2] = 0.0;
      rc[E * 2 + 1] = 0.0;
      continue;
    }
    double v0 = 0.0, v1 = 0.0;
    for (int a = 0; a < K1; ++a) {
      const double x = res[E * K1 + a];
      v0 = fma(Jp[a * 2], x, v0);
      v1 = fma(Jp[a * 2 + 1], x, v1);
    }
    rc[E * 2] = v0;
    rc[E * 2 + 1] = v1;
    if (fuse) {
      const double* Di = C.Dinv + E * 4;
      double e0 = c2 * (Di[0] * v0 + Di[1] * v1);
      double e1 = c2 * (Di[2] * v0 + Di[3] * v1);
      ec[E * 2] = e0;
      ec[E * 2 + 1] = e1;
      if (C.smoother == 1) {
        dc[E * 2] = e0;
        dc[E * 2 + 1] = e1;
      }
    }
  }
}

int launch_p_restrict(const LevelDev& F, const LevelDev& C, const double* Jp,
                      const double* res, double* rc, bool fuse_first, double* ec, double* dc,
                      cudaStream_t st) {
  k_p_restrict<<<cap_grid(F.nedge, 128, 148 * 8), 128, 0, st>>>(F, C, Jp, res, rc, fuse_first,
                                                                ec, dc);
  return 1;
}

__global__ void k_p_prolong(LevelDev F, const double* __restrict__ Jp,
                            const double* __restrict__ ec, double* e) {
  const int K1 = F.k1;
  for (int64_t E = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; E < F.nedge;
       E += (int64_t)gridDim.x * blockDim.x) {
    if (edge_on_boundary(F.nx, F.ny, E)) continue;
    const double c0 = ec[E * 2], c1 = ec[E * 2 + 1];
    for (int a = 0; a < K1; ++a) e[E * K1 + a] += fma(Jp[a * 2], c0, Jp[a * 2 + 1] * c1);
  }
}

int launch_p_prolong(const LevelDev& F, const double* Jp, const double* ec, double* e,
                     cudaStream_t st) {
  k_p_prolong<<<cap_grid(F.nedge, 128, 148 * 8), 128, 0, st>>>(F, Jp, ec, e);
  return 1;
}

// ---------------------------------------------------------------- reductions
__device__ __forceinline__ double block_sum(double v) {
  __shared__ double red[32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  const int nw = blockDim.x >> 5;
  double t = 0.0;
  if (w == 0) {
    t = lane < nw ? red[lane] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  }
  return t;  // valid in thread 0
}

int vec_grid(int64_t n) { return cap_grid(n, 256, 148 * 4); }

__global__ void k_dot(const double* __restrict__ a, const double* __restrict__ b, int64_t n,
                      double* partials) {
  double s = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    s = fma(a[i], b[i], s);
  s = block_sum(s);
  if (threadIdx.x == 0) partials[blockIdx.x] = s;
}

int launch_dot(const double* a, const double* b, int64_t n, double* partials, int grid,
               cudaStream_t st) {
  k_dot<<<grid, 256, 0, st>>>(a, b, n, partials);
  return 1;
}

// scal layout (PCG): [0] rz, [1] pAp, [2] rr, [3] alpha, [4] beta, [5] gg, [6..] misc
__global__ void k_reduce(const double* __restrict__ partials, int n, double* scal, int slot,
                         int op) {
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) s += partials[i];
  s = block_sum(s);
  if (threadIdx.x == 0) {
    if (op == 1) {          // alpha = rz / pAp (pAp <= 0 is checked by the host: breakdown)
      scal[3] = scal[0] / s;
    } else if (op == 2) {   // beta = rz_new / rz_old, then rz = rz_new
      scal[4] = s / scal[0];
    }
    scal[slot] = s;
  }
}

int launch_reduce(const double* partials, int n, double* scal, int slot, int op, DevError* err,
                  cudaStream_t st) {
  (void)err;
  k_reduce<<<1, 1024, 0, st>>>(partials, n, scal, slot, op);
  return 1;
}

__global__ void k_pcg_update(double* x, double* r, const double* __restrict__ p,
                             const double* __restrict__ ap, const double* __restrict__ scal,
                             int64_t n, double* partials) {
  const double alpha = scal[3];
  double s = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    x[i] = fma(alpha, p[i], x[i]);
    const double ri = fma(-alpha, ap[i], r[i]);
    r[i] = ri;
    s = fma(ri, ri, s);
  }
  s = block_sum(s);
  if (threadIdx.x == 0) partials[blockIdx.x] = s;
}

int launch_pcg_update(double* x, double* r, const double* p, const double* ap,
                      const double* scal, int64_t n, double* partials, int grid,
                      cudaStream_t st) {
  k_pcg_update<<<grid, 256, 0, st>>>(x, r, p, ap, scal, n, partials);
  return 1;
}

__global__ void k_pcg_pupdate(double* p, const double* __restrict__ z,
                              const double* __restrict__ scal, int64_t n) {
  const double beta = scal[4];
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    p[i] = fma(beta, p[i], z[i]);
}

int launch_pcg_pupdate(double* p, const double* z, const double* scal, int64_t n,
                       cudaStream_t st) {
  k_pcg_pupdate<<<vec_grid(n), 256, 0, st>>>(p, z, scal, n);
  return 1;
}

// ---------------------------------------------------------------- lambda_max (Q11)
__global__ void k_pow_init(LevelDev L, double* v) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < L.ndof;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = i / L.k1;
    v[i] = edge_on_boundary(L.nx, L.ny, e) ? 0.0 : 1.0 + (double)(i % 7) / 7.0;
  }
}

int launch_pow_init(const LevelDev& L, double* v, cudaStream_t st) {
  k_pow_init<<<vec_grid(L.ndof), 256, 0, st>>>(L, v);
  return 1;
}

// u = Dinv y per edge; partials[2*b] = sum u.u, partials[2*b+1] = sum u.y
__global__ void k_edge_dinv(LevelDev L, const double* __restrict__ y, double* u,
                            double* partials) {
  const int K1 = L.k1;
  double s_uu = 0.0, s_uy = 0.0;
  for (int64_t ed = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; ed < L.nedge;
       ed += (int64_t)gridDim.x * blockDim.x) {
    if (edge_on_boundary(L.nx, L.ny, ed)) {
      for (int a = 0; a < K1; ++a) u[ed * K1 + a] = 0.0;
      continue;
    }
    const double* Di = L.Dinv + ed * K1 * K1;
    for (int a = 0; a < K1; ++a) {
      double c = 0.0;
      for (int b = 0; b < K1; ++b) c = fma(Di[a * K1 + b], y[ed * K1 + b], c);
      u[ed * K1 + a] = c;
      s_uu = fma(c, c, s_uu);
      s_uy = fma(c, y[ed * K1 + a], s_uy);
    }
  }
  double a = block_sum(s_uu);
  if (threadIdx.x == 0) partials[blockIdx.x] = a;
  double b = block_sum(s_uy);
  if (threadIdx.x == 0) partials[gridDim.x + blockIdx.x] = b;
}

int launch_edge_dinv(const LevelDev& L, const double* y, double* u, double* partials,
                     int grid, cudaStream_t st) {
  k_edge_dinv<<<grid, 256, 0, st>>>(L, y, u, partials);
  return 1;
}

__global__ void k_scale_by_norm(double* v, const double* __restrict__ u, int64_t n,
                                const double* __restrict__ scal, int slot) {
  const double inv = 1.0 / sqrt(scal[slot]);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    v[i] = u[i] * inv;
}

int launch_scale_by_norm(double* v, const double* u, int64_t n, const double* scal, int slot,
                         cudaStream_t st) {
  k_scale_by_norm<<<vec_grid(n), 256, 0, st>>>(v, u, n, scal, slot);
  return 1;
}

// scal[6] = u.u (last), scal[7] = u.y_prev (last), scal[8] = v.Av:
// lambda_hat = v.Av / v.Dv with v = u/|u| -> v.Dv = u.y_prev / u.u.
// Chebyshev coefficients (O8): theta = (b+a)/2, delta = (b-a)/2, sigma = theta/delta,
// step 0: c1 = 0, c2 = 1/theta; step k: rho_k = 1/(2 sigma - rho_{k-1}),
// c1 = rho_k rho_{k-1}, c2 = 2 rho_k / delta.
__global__ void k_lmax_finish(const double* __restrict__ scal, double safety, double ratio,
                              int nu_max, double* lam_out, double* coef) {
  const double vDv = scal[7] / scal[6];
  const double lam = safety * scal[8] / vDv;
  *lam_out = lam;
  const double b = lam, a = lam / ratio;
  const double theta = 0.5 * (b + a), delta = 0.5 * (b - a), sigma = theta / delta;
  double rho = 1.0 / sigma;
  coef[0] = 0.0;
  coef[1] = 1.0 / theta;
  for (int k = 1; k < nu_max; ++k) {
    const double rn = 1.0 / (2.0 * sigma - rho);
    coef[2 * k] = rn * rho;
    coef[2 * k + 1] = 2.0 * rn / delta;
    rho = rn;
  }
}

int launch_lmax_finish(const double* scal, double safety, double ratio, int nu_max,
                       double* lam_out, double* coef, cudaStream_t st) {
  k_lmax_finish<<<1, 1, 0, st>>>(scal, safety, ratio, nu_max, lam_out, coef);
  return 1;
}

__global__ void k_set_bj_coef(double omega, double* coef) {
  int k = threadIdx.x;
  if (k < MAX_NU) {
    coef[2 * k] = 0.0;
    coef[2 * k + 1] = omega;
  }
}

int launch_set_bj_coef(double omega, double* coef, cudaStream_t st) {
  k_set_bj_coef<<<1, 32, 0, st>>>(omega, coef);
  return 1;
}

__global__ void k_copy(double* dst, const double* __restrict__ src, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

int launch_copy(double* dst, const double* src, int64_t n, cudaStream_t st) {
  k_copy<<<vec_grid(n), 256, 0, st>>>(dst, src, n);
  return 1;
}

__global__ void k_zero(double* dst, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = 0.0;
}

int launch_zero(double* dst, int64_t n, cudaStream_t st) {
  k_zero<<<vec_grid(n), 256, 0, st>>>(dst, n);
  return 1;
}

// dst = src with the dOmega (Dirichlet) entries set to 0 (inputs are ignored there)
__global__ void k_copy_masked(LevelDev L, double* dst, const double* __restrict__ src) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < L.ndof;
       i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = edge_on_boundary(L.nx, L.ny, i / L.k1) ? 0.0 : src[i];
}

int launch_copy_masked(const LevelDev& L, double* dst, const double* src, cudaStream_t st) {
  k_copy_masked<<<vec_grid(L.ndof), 256, 0, st>>>(L, dst, src);
  return 1;
}

__global__ void k_add(double* dst, const double* __restrict__ src, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    dst[i] += src[i];
}

int launch_add(double* dst, const double* src, int64_t n, cudaStream_t st) {
  k_add<<<vec_grid(n), 256, 0, st>>>(dst, src, n);
  return 1;
}

}  // namespace mgdtn
