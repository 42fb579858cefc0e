// Reference-element tables (host C++).  See refelem.h.
//
// Derivation of the staged HDG elimination (tested with
// v = (phi_i, 0), (0, phi_i) and w = phi_i, HDG_local2 integrated by parts):
//   (1/K) M u_x - Dx^T q + Cx lam = 0           => u_x = K M^-1 (Dx^T q - Cx lam)
//   Dx u_x + Dy u_y + tau F q - tau E lam = f_w
//   => (K G + tau F) q = f_w + (K P + tau E) lam
//   flux rows <u_hat.n, mu> = (K P + tau E)^T q - (K W + tau H) lam
//   => S_T = S0 - R^T Q^-1 R,  b_T = R^T Q^-1 f_w.
// With a side-h square: M = h^2 Mhat, D = h Dhat, C,E,F,H = h * hat, so
// G, P, W are h-free and only t = tau*h enters (SURVEY.md 8(c) Scaling).
#include "refelem.h"

#include <cmath>
#include <stdexcept>

namespace mgdtn {

static void legendre(int n, double x, double& P, double& dP) {
  double p0 = 1.0, p1 = x;
  if (n == 0) { P = 1.0; dP = 0.0; return; }
  for (int k = 1; k < n; ++k) {
    double p2 = ((2.0 * k + 1.0) * x * p1 - k * p0) / (k + 1.0);
    p0 = p1;
    p1 = p2;
  }
  P = p1;
  dP = n * (x * p1 - p0) / (x * x - 1.0);
}

std::vector<double> gll_nodes01(int p) {
  std::vector<double> x(p + 1);
  x[0] = -1.0;
  x[p] = 1.0;
  for (int i = 1; i < p; ++i) {
    double t = -std::cos(M_PI * i / p);
    for (int it = 0; it < 100; ++it) {
      double P, dP;
      legendre(p, t, P, dP);
      double d2P = (2.0 * t * dP - p * (p + 1.0) * P) / (1.0 - t * t);
      double dt = dP / d2P;
      t -= dt;
      if (std::fabs(dt) < 1e-16) break;
    }
    x[i] = t;
  }
  for (auto& v : x) v = 0.5 * (v + 1.0);
  return x;
}

void gauss01(int nq, std::vector<double>& x, std::vector<double>& w) {
  x.assign(nq, 0.0);
  w.assign(nq, 0.0);
  for (int i = 0; i < nq; ++i) {
    double t = std::cos(M_PI * (i + 0.75) / (nq + 0.5));
    double P = 0, dP = 1;
    for (int it = 0; it < 100; ++it) {
      legendre(nq, t, P, dP);
      double dt = P / dP;
      t -= dt;
      if (std::fabs(dt) < 1e-16) break;
    }
    legendre(nq, t, P, dP);
    // ascending order on [0,1]
    x[nq - 1 - i] = 0.5 * (t + 1.0);
    w[nq - 1 - i] = 0.5 * 2.0 / ((1.0 - t * t) * dP * dP);
  }
}

static double lag(const std::vector<double>& nd, int a, double x) {
  double v = 1.0;
  for (size_t b = 0; b < nd.size(); ++b)
    if ((int)b != a) v *= (x - nd[b]) / (nd[a] - nd[b]);
  return v;
}

static double dlag(const std::vector<double>& nd, int a, double x) {
  double s = 0.0;
  for (size_t c = 0; c < nd.size(); ++c) {
    if ((int)c == a) continue;
    double t = 1.0 / (nd[a] - nd[c]);
    for (size_t b = 0; b < nd.size(); ++b)
      if ((int)b != a && b != c) t *= (x - nd[b]) / (nd[a] - nd[b]);
    s += t;
  }
  return s;
}

// dense SPD solve X = A^-1 B (A n x n row-major, B n x r), Cholesky
static std::vector<double> spd_solve(std::vector<double> A, int n, std::vector<double> B, int r) {
  for (int j = 0; j < n; ++j) {
    double d = A[j * n + j];
    for (int k = 0; k < j; ++k) d -= A[j * n + k] * A[j * n + k];
    if (!(d > 0)) throw std::runtime_error("reference mass matrix not SPD");
    d = std::sqrt(d);
    A[j * n + j] = d;
    for (int i = j + 1; i < n; ++i) {
      double s = A[i * n + j];
      for (int k = 0; k < j; ++k) s -= A[i * n + k] * A[j * n + k];
      A[i * n + j] = s / d;
    }
  }
  for (int c = 0; c < r; ++c) {
    for (int i = 0; i < n; ++i) {
      double s = B[i * r + c];
      for (int k = 0; k < i; ++k) s -= A[i * n + k] * B[k * r + c];
      B[i * r + c] = s / A[i * n + i];
    }
    for (int i = n - 1; i >= 0; --i) {
      double s = B[i * r + c];
      for (int k = i + 1; k < n; ++k) s -= A[k * n + i] * B[k * r + c];
      B[i * r + c] = s / A[i * n + i];
    }
  }
  return B;
}

// cyclic Jacobi eigen-decomposition of a symmetric n x n matrix (accurate to a
// few ulps of ||A||): A = V diag(lam) V^T, V column-major in v[row*n + col]
static void jacobi_eig(std::vector<double> A, int n, std::vector<double>& lam,
                       std::vector<double>& V) {
  V.assign(n * n, 0.0);
  for (int i = 0; i < n; ++i) V[i * n + i] = 1.0;
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0, tot = 0.0;
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) {
        tot += A[i * n + j] * A[i * n + j];
        if (i != j) off += A[i * n + j] * A[i * n + j];
      }
    if (off <= 1e-34 * tot) break;
    for (int pp = 0; pp < n; ++pp)
      for (int q = pp + 1; q < n; ++q) {
        const double apq = A[pp * n + q];
        if (apq == 0.0) continue;
        const double th = (A[q * n + q] - A[pp * n + pp]) / (2.0 * apq);
        const double t = (th >= 0 ? 1.0 : -1.0) / (std::fabs(th) + std::sqrt(th * th + 1.0));
        const double cs = 1.0 / std::sqrt(t * t + 1.0), sn = t * cs;
        for (int k = 0; k < n; ++k) {   // columns pp, q
          const double akp = A[k * n + pp], akq = A[k * n + q];
          A[k * n + pp] = cs * akp - sn * akq;
          A[k * n + q] = sn * akp + cs * akq;
        }
        for (int k = 0; k < n; ++k) {   // rows pp, q
          const double apk = A[pp * n + k], aqk = A[q * n + k];
          A[pp * n + k] = cs * apk - sn * aqk;
          A[q * n + k] = sn * apk + cs * aqk;
        }
        for (int k = 0; k < n; ++k) {
          const double vkp = V[k * n + pp], vkq = V[k * n + q];
          V[k * n + pp] = cs * vkp - sn * vkq;
          V[k * n + q] = sn * vkp + cs * vkq;
        }
      }
  }
  lam.assign(n, 0.0);
  for (int i = 0; i < n; ++i) lam[i] = A[i * n + i];
}

// lower Cholesky factor (false if not SPD with margin)
static bool cholesky(const std::vector<double>& B, int n, std::vector<double>& Lc, double margin) {
  Lc.assign(n * n, 0.0);
  for (int j = 0; j < n; ++j) {
    double d = B[j * n + j];
    for (int k = 0; k < j; ++k) d -= Lc[j * n + k] * Lc[j * n + k];
    if (!(d > margin * B[j * n + j])) return false;
    d = std::sqrt(d);
    Lc[j * n + j] = d;
    for (int i = j + 1; i < n; ++i) {
      double s = B[i * n + j];
      for (int k = 0; k < j; ++k) s -= Lc[i * n + k] * Lc[j * n + k];
      Lc[i * n + j] = s / d;
    }
  }
  return true;
}

// pencil tables (refelem.h RefTables::Pencil) for Q = K A + t F with
// w = t E + K Bm (rows of the local right-hand sides)
static RefTables::Pencil make_pencil(const std::vector<double>& A, const std::vector<double>& F,
                                     const std::vector<double>& E, const std::vector<double>& Bm,
                                     const std::vector<double>& fq, int nv, int m, int nqf2) {
  RefTables::Pencil P;
  std::vector<double> B(nv * nv), Lc;
  for (P.c = 1.0;; P.c *= 2.0) {
    for (int i = 0; i < nv * nv; ++i) B[i] = A[i] + P.c * F[i];
    if (cholesky(B, nv, Lc, 1e-3)) break;
    if (P.c > 1e6) throw std::runtime_error("no SPD pencil");
  }
  // Linv (lower triangular)
  std::vector<double> Li(nv * nv, 0.0);
  for (int c = 0; c < nv; ++c)
    for (int i = 0; i < nv; ++i) {
      double s = (i == c) ? 1.0 : 0.0;
      for (int k = 0; k < i; ++k) s -= Lc[i * nv + k] * Li[k * nv + c];
      Li[i * nv + c] = s / Lc[i * nv + i];
    }
  // C = Li A Li^T
  std::vector<double> LA(nv * nv, 0.0), C(nv * nv, 0.0);
  for (int i = 0; i < nv; ++i)
    for (int j = 0; j < nv; ++j) {
      double s = 0;
      for (int k = 0; k <= i; ++k) s += Li[i * nv + k] * A[k * nv + j];
      LA[i * nv + j] = s;
    }
  for (int i = 0; i < nv; ++i)
    for (int j = 0; j < nv; ++j) {
      double s = 0;
      for (int k = 0; k <= j; ++k) s += LA[i * nv + k] * Li[j * nv + k];
      C[i * nv + j] = s;
    }
  for (int i = 0; i < nv; ++i)
    for (int j = 0; j < i; ++j) C[i * nv + j] = C[j * nv + i] = 0.5 * (C[i * nv + j] + C[j * nv + i]);
  std::vector<double> ev, V;
  jacobi_eig(C, nv, ev, V);
  // T = V^T Li
  std::vector<double> T(nv * nv, 0.0);
  for (int i = 0; i < nv; ++i)
    for (int j = 0; j < nv; ++j) {
      double s = 0;
      for (int k = j; k < nv; ++k) s += V[k * nv + i] * Li[k * nv + j];
      T[i * nv + j] = s;
    }
  auto quad = [&](const std::vector<double>& X, int i) {
    double s = 0;
    for (int a = 0; a < nv; ++a) {
      double r = 0;
      for (int b = 0; b < nv; ++b) r += X[a * nv + b] * T[i * nv + b];
      s += T[i * nv + a] * r;
    }
    return s;
  };
  P.lam.assign(nv, 0.0);
  P.mu.assign(nv, 0.0);
  for (int i = 0; i < nv; ++i) {
    P.lam[i] = quad(A, i);
    P.mu[i] = quad(F, i);
  }
  P.At.assign(nv * m, 0.0);
  P.Bk.assign(nv * m, 0.0);
  for (int i = 0; i < nv; ++i)
    for (int a = 0; a < m; ++a) {
      double s1 = 0, s2 = 0;
      for (int k = 0; k < nv; ++k) {
        s1 += T[i * nv + k] * E[k * m + a];
        s2 += T[i * nv + k] * Bm[k * m + a];
      }
      P.At[i * m + a] = s1;
      P.Bk[i * m + a] = s2;
    }
  P.Tt.assign(nv * nv, 0.0);
  for (int i = 0; i < nv; ++i)
    for (int k = 0; k < nv; ++k) P.Tt[k * nv + i] = T[i * nv + k];
  P.fqT.assign(nqf2 * nv, 0.0);
  for (int q = 0; q < nqf2; ++q)
    for (int i = 0; i < nv; ++i) {
      double s = 0;
      for (int k = 0; k < nv; ++k) s += T[i * nv + k] * fq[q * nv + k];
      P.fqT[q * nv + i] = s;
    }
  return P;
}

RefTables build_ref_tables(int p) {
  if (p < 1 || p > 4) throw std::runtime_error("p must be in 1..4");
  RefTables T;
  const int k1 = p + 1, nv = k1 * k1, m = 4 * k1;
  T.p = p; T.k1 = k1; T.nv = nv; T.m = m;
  T.gll = gll_nodes01(p);
  const auto& nd = T.gll;
  std::vector<double> xq, wq;
  gauss01(p + 2, xq, wq);
  const int nq = p + 2;

  std::vector<double> M(nv * nv, 0.0), Dx(nv * nv, 0.0), Dy(nv * nv, 0.0), L(nv * nv, 0.0);
  for (int qy = 0; qy < nq; ++qy)
    for (int qx = 0; qx < nq; ++qx) {
      double w = wq[qx] * wq[qy], X = xq[qx], Y = xq[qy];
      std::vector<double> ph(nv), gx(nv), gy(nv);
      for (int b = 0; b < k1; ++b)
        for (int a = 0; a < k1; ++a) {
          int i = b * k1 + a;
          ph[i] = lag(nd, a, X) * lag(nd, b, Y);
          gx[i] = dlag(nd, a, X) * lag(nd, b, Y);
          gy[i] = lag(nd, a, X) * dlag(nd, b, Y);
        }
      for (int i = 0; i < nv; ++i)
        for (int j = 0; j < nv; ++j) {
          M[i * nv + j] += w * ph[i] * ph[j];
          Dx[i * nv + j] += w * gx[j] * ph[i];     // (d_x phi_j, phi_i)
          Dy[i * nv + j] += w * gy[j] * ph[i];
          L[i * nv + j] += w * (gx[i] * gx[j] + gy[i] * gy[j]);
        }
    }
  // edges
  const double nrm[4][2] = {{0, -1}, {1, 0}, {0, 1}, {-1, 0}};
  std::vector<double> E(nv * m, 0.0), F(nv * nv, 0.0), H(m * m, 0.0), N(nv * nv, 0.0),
      Nl(nv * m, 0.0);
  for (int f = 0; f < 4; ++f)
    for (int q = 0; q < nq; ++q) {
      double s = xq[q], w = wq[q];
      double X = (f == 0 || f == 2) ? s : (f == 1 ? 1.0 : 0.0);
      double Y = (f == 1 || f == 3) ? s : (f == 2 ? 1.0 : 0.0);
      std::vector<double> ph(nv), gn(nv), mu(k1);
      for (int b = 0; b < k1; ++b)
        for (int a = 0; a < k1; ++a) {
          int i = b * k1 + a;
          ph[i] = lag(nd, a, X) * lag(nd, b, Y);
          double gx = dlag(nd, a, X) * lag(nd, b, Y);
          double gy = lag(nd, a, X) * dlag(nd, b, Y);
          gn[i] = nrm[f][0] * gx + nrm[f][1] * gy;
        }
      for (int a = 0; a < k1; ++a) mu[a] = lag(nd, a, s);
      for (int i = 0; i < nv; ++i) {
        for (int a = 0; a < k1; ++a) {
          E[i * m + f * k1 + a] += w * mu[a] * ph[i];
          Nl[i * m + f * k1 + a] += w * mu[a] * gn[i];
        }
        for (int j = 0; j < nv; ++j) {
          F[i * nv + j] += w * ph[i] * ph[j];
          N[i * nv + j] += w * gn[j] * ph[i];
        }
      }
      for (int a = 0; a < k1; ++a)
        for (int b = 0; b < k1; ++b) H[(f * k1 + a) * m + f * k1 + b] += w * mu[a] * mu[b];
    }
  std::vector<double> Cx(nv * m), Cy(nv * m);
  for (int i = 0; i < nv; ++i)
    for (int c = 0; c < m; ++c) {
      int f = c / k1;
      Cx[i * m + c] = nrm[f][0] * E[i * m + c];
      Cy[i * m + c] = nrm[f][1] * E[i * m + c];
    }
  // M^-1 Dx^T, M^-1 Dy^T (nv x nv), M^-1 Cx, M^-1 Cy (nv x m)
  std::vector<double> DxT(nv * nv), DyT(nv * nv);
  for (int i = 0; i < nv; ++i)
    for (int j = 0; j < nv; ++j) {
      DxT[i * nv + j] = Dx[j * nv + i];
      DyT[i * nv + j] = Dy[j * nv + i];
    }
  auto MiDxT = spd_solve(M, nv, DxT, nv);
  auto MiDyT = spd_solve(M, nv, DyT, nv);
  auto MiCx = spd_solve(M, nv, Cx, m);
  auto MiCy = spd_solve(M, nv, Cy, m);
  T.G.assign(nv * nv, 0.0);
  T.P.assign(nv * m, 0.0);
  T.W.assign(m * m, 0.0);
  for (int i = 0; i < nv; ++i)
    for (int j = 0; j < nv; ++j) {
      double s = 0;
      for (int k = 0; k < nv; ++k) s += Dx[i * nv + k] * MiDxT[k * nv + j] + Dy[i * nv + k] * MiDyT[k * nv + j];
      T.G[i * nv + j] = s;
    }
  for (int i = 0; i < nv; ++i)
    for (int c = 0; c < m; ++c) {
      double s = 0;
      for (int k = 0; k < nv; ++k) s += Dx[i * nv + k] * MiCx[k * m + c] + Dy[i * nv + k] * MiCy[k * m + c];
      T.P[i * m + c] = s;
    }
  for (int a = 0; a < m; ++a)
    for (int b = 0; b < m; ++b) {
      double s = 0;
      for (int k = 0; k < nv; ++k) s += Cx[k * m + a] * MiCx[k * m + b] + Cy[k * m + a] * MiCy[k * m + b];
      T.W[a * m + b] = s;
    }
  T.F = F;
  T.E = E;
  T.H = H;
  T.LN.assign(nv * nv, 0.0);
  for (int i = 0; i < nv; ++i)
    for (int j = 0; j < nv; ++j) T.LN[i * nv + j] = L[i * nv + j] - N[i * nv + j] - N[j * nv + i];
  T.Nl = Nl;
  T.L = L;
  T.N = N;
  // source / boundary-data quadrature on the p+4 Gauss sampling grid
  std::vector<double> xf, wf;
  T.nqf = p + 4;
  gauss01(T.nqf, xf, wf);
  T.fq.assign(T.nqf * T.nqf * nv, 0.0);
  for (int qy = 0; qy < T.nqf; ++qy)
    for (int qx = 0; qx < T.nqf; ++qx)
      for (int b = 0; b < k1; ++b)
        for (int a = 0; a < k1; ++a)
          T.fq[(qy * T.nqf + qx) * nv + b * k1 + a] =
              wf[qy] * wf[qx] * lag(nd, a, xf[qx]) * lag(nd, b, xf[qy]);
  T.vq.assign(T.nqf * T.nqf * nv, 0.0);
  T.wq.assign(T.nqf * T.nqf, 0.0);
  for (int qy = 0; qy < T.nqf; ++qy)
    for (int qx = 0; qx < T.nqf; ++qx) {
      T.wq[qy * T.nqf + qx] = wf[qy] * wf[qx];
      for (int b = 0; b < k1; ++b)
        for (int a = 0; a < k1; ++a)
          T.vq[(qy * T.nqf + qx) * nv + b * k1 + a] = lag(nd, a, xf[qx]) * lag(nd, b, xf[qy]);
    }
  T.ew.assign(T.nqf * k1, 0.0);
  for (int q = 0; q < T.nqf; ++q)
    for (int a = 0; a < k1; ++a) T.ew[q * k1 + a] = wf[q] * lag(nd, a, xf[q]);
  std::vector<double> H1(k1 * k1, 0.0), I1(k1 * k1, 0.0);
  for (int a = 0; a < k1; ++a) {
    I1[a * k1 + a] = 1.0;
    for (int b = 0; b < k1; ++b) H1[a * k1 + b] = H[a * m + b];   // edge 0 block
  }
  T.H1inv = spd_solve(H1, k1, I1, k1);
  T.Jp.assign(k1 * 2, 0.0);
  for (int a = 0; a < k1; ++a) {
    T.Jp[a * 2 + 0] = 1.0 - nd[a];
    T.Jp[a * 2 + 1] = nd[a];
  }
  std::vector<double> mNl(nv * m);
  for (int i = 0; i < nv * m; ++i) mNl[i] = -T.Nl[i];
  T.pen[0] = make_pencil(T.G, T.F, T.E, T.P, T.fq, nv, m, T.nqf * T.nqf);
  T.pen[1] = make_pencil(T.LN, T.F, T.E, mNl, T.fq, nv, m, T.nqf * T.nqf);
  return T;
}

}  // namespace mgdtn
