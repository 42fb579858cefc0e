// Host-side reference-element tables for the element-local solves.
//
// Unit square, volume space Q^p with GLL nodal basis (index i = b*(p+1)+a,
// a along x), trace space P^p per edge with GLL nodes in the edge's global
// orientation, local edges {0 bottom, 1 right, 2 top, 3 left}.  Exact Gauss
// quadrature.  The element matrices of a side-h square depend only on
// (K, tau*h) (SURVEY.md 8(c) "Scaling"), so these h-free tables plus two
// scalars per element fully determine each local solve (PAPER.md:184-199,
// 230-233, 305-316).
#pragma once
#include <vector>

namespace mgdtn {

struct RefTables {
  int p = 0, k1 = 0, nv = 0, m = 0;
  std::vector<double> gll;            // [k1]
  // HDG staged elimination (u eliminated first):
  //   Q = K*G + t*F, R = K*P + t*E, S0 = K*W + t*H, t = tau*h
  std::vector<double> G, F;           // [nv*nv]
  std::vector<double> P, E;           // [nv*m]
  std::vector<double> W, H;           // [m*m]
  // SIPG-H: Q = K*LN + t*F, R = t*E - K*Nl, S0 = t*H, LN = L - N - N^T
  std::vector<double> LN;             // [nv*nv]
  std::vector<double> Nl;             // [nv*m]
  // IPDG-H with general s_f (Eq. IPG_H): Q = K*(L - N - s_f N^T) + t*F, R = t*E - s_f K*Nl,
  // flux rows (t*E - K*Nl)^T; L_ij = (grad phi_j, grad phi_i), N_ij = <grad phi_j.n, phi_i>_dT
  std::vector<double> L, N;           // [nv*nv]
  // source quadrature on the input sampling grid (p+4 Gauss per direction):
  //   fw_i = h^2 * sum_{qy,qx} fq[qy,qx,i] * f(qy,qx)
  int nqf = 0;
  std::vector<double> fq;             // [nqf*nqf*nv] (weights folded in)
  std::vector<double> vq;             // [nqf*nqf*nv] basis values at those points (no weights)
  std::vector<double> wq;             // [nqf*nqf] tensor Gauss weights on the unit square
  // boundary-data projection: lambda = H1inv * (sum_q ew[q,a] g_q)
  std::vector<double> ew;             // [nqf*k1] (weights folded in)
  std::vector<double> H1inv;          // [k1*k1]
  // p-injection J_p: fine node a from P1 endpoint values (c0, c1)
  std::vector<double> Jp;             // [k1*2]
  // Simultaneous diagonalisation of the local pencil (A, F), A = G (HDG) or LN
  // (SIPG-H): with B = A + c F SPD (B = L L^T), C = L^-1 A L^-T = V diag V^T and
  // T = V^T L^-1, every local matrix Q = K A + t F becomes T Q T^T =
  // diag(K lam_i + t mu_i) (lam_i = (T A T^T)_ii, mu_i = (T F T^T)_ii, taken as
  // Rayleigh quotients, not 1 - ..., so F-null modes keep mu_i ~ 1e-30).  Hence
  //   S_T = S0 - sum_i w_i w_i^T / (K lam_i + t mu_i),  w_i = t At_i + K Bk_i,
  //   b_T = sum_i w_i f'_i / (K lam_i + t mu_i),      f'_i = h^2 sum_q fqT[q,i] f_q,
  // with At = T E, Bk = T P (HDG) or -T Nl (SIPG-H); S0 = K W + t H (HDG), t H (SIPG-H).
  struct Pencil {
    double c = 1.0;
    std::vector<double> lam, mu;      // [nv]
    std::vector<double> At, Bk;       // [nv*m]
    std::vector<double> fqT;          // [nqf*nqf*nv]
    std::vector<double> Tt;           // [nv*nv] T^T (volume recovery: q = T^T diag(1/d) (w lam + f'))
  };
  Pencil pen[2];                      // [0] HDG, [1] SIPG-H
};

// Builds the tables for order p (1..4).  Pure host C++ (Legendre recurrences,
// Newton iterations, dense Cholesky), no library calls.
RefTables build_ref_tables(int p);

// 1D helpers (exposed for tests of the host code)
std::vector<double> gll_nodes01(int p);
void gauss01(int nq, std::vector<double>& x, std::vector<double>& w);

}  // namespace mgdtn
