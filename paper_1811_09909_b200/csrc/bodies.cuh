// Device bodies of the V-cycle operations, written as grid-stride loops over
// (t0, nt) so that the same code runs as a standalone kernel (t0 = global
// thread id, nt = grid threads) and inside the cluster-resident coarse-tail
// kernel k_coarse_tail (t0 = rank in the cluster, nt = cluster threads).
//
// Transfers: p-level I_N = J_N, Q_{N-1} = J_N^T (per
// edge); h-levels I_k = [P_M ; J], Q_{k-1} = [P_M^T , J^T] with
// P_M = -A_II^-1 A_IB J per macro.  Local correction T_k = [A_II^-1 0; 0 0]
// (Eq. 3.11) per macro.  Smoothers on edge blocks.
#pragma once
#include "kernels.cuh"

namespace mgdtn {

// ---------------------------------------------------------------- apply pieces
// The K1 doubles of one edge with 16-byte accesses where the address allows (an edge
// starts 16-byte aligned iff e*K1 is even).  In a colour pass the 32 lanes of a warp
// hold every other element of a row, so their edges of one role all have one parity:
// the branch does not diverge, and a warp's access to an edge block takes ceil(K1/2)
// instead of K1 L1 wavefront groups (the gathers of a thread-per-element pass are
// L1-wavefront-bound: 32 lanes x 8 bytes at an 80-byte stride touch 20 lines each).
template <int K1>
__device__ __forceinline__ void ld_edge(const double* p, double* v) {
  if (K1 % 2 == 0) {
#pragma unroll
    for (int q = 0; q < K1 / 2; ++q) {
      const double2 t = reinterpret_cast<const double2*>(p)[q];
      v[2 * q] = t.x;
      v[2 * q + 1] = t.y;
    }
  } else if ((reinterpret_cast<uintptr_t>(p) & 15) == 0) {
#pragma unroll
    for (int q = 0; q < K1 / 2; ++q) {
      const double2 t = reinterpret_cast<const double2*>(p)[q];
      v[2 * q] = t.x;
      v[2 * q + 1] = t.y;
    }
    v[K1 - 1] = p[K1 - 1];
  } else {
    v[0] = p[0];
#pragma unroll
    for (int q = 0; q < K1 / 2; ++q) {
      const double2 t = reinterpret_cast<const double2*>(p + 1)[q];
      v[1 + 2 * q] = t.x;
      v[2 + 2 * q] = t.y;
    }
  }
}
template <int K1>
__device__ __forceinline__ void st_edge(double* p, const double* v) {
  if (K1 % 2 == 0) {
#pragma unroll
    for (int q = 0; q < K1 / 2; ++q) reinterpret_cast<double2*>(p)[q] = make_double2(v[2 * q], v[2 * q + 1]);
  } else if ((reinterpret_cast<uintptr_t>(p) & 15) == 0) {
#pragma unroll
    for (int q = 0; q < K1 / 2; ++q) reinterpret_cast<double2*>(p)[q] = make_double2(v[2 * q], v[2 * q + 1]);
    p[K1 - 1] = v[K1 - 1];
  } else {
    p[0] = v[0];
#pragma unroll
    for (int q = 0; q < K1 / 2; ++q)
      reinterpret_cast<double2*>(p + 1)[q] = make_double2(v[1 + 2 * q], v[2 + 2 * q]);
  }
}

template <int K1>
__device__ __forceinline__ void gather_x(const double* x, const int64_t ed[4], const bool bd[4],
                                         double* xv) {
#pragma unroll
  for (int f = 0; f < 4; ++f) {
    if (bd[f]) {
#pragma unroll
      for (int a = 0; a < K1; ++a) xv[f * K1 + a] = 0.0;
    } else {
      ld_edge<K1>(x + ed[f] * K1, xv + f * K1);
    }
  }
}

// Epilogue of one element, in two phases so that no load waits behind a store
// (y / x / d are plain pointers the compiler must assume may alias):
//   epi_load  -- every value the epilogue reads (y, r, d) is loaded up front
//                (before the matvec; in the TMA kernel before the stage wait):
//                AM_APPLY: t = y;  AM_RESID / AM_SMOOTH: t = r - y;  AM_SMOOTH: dd = d
//   epi_store -- AM_W0: y = y_T;  AM_APPLY: y = t + y_T (dot += x.y);
//                AM_RESID: y = t - y_T = r - A x;
//                AM_SMOOTH: res = t - y_T, dn = c2 D_e^-1 res (+ c1 dd), d = dn, x += dn
//                AM_DINV: y = t + y_T = A x, x = D_e^-1 (A x) (dot += x_new . y)
// Edges on dOmega: y written as 0 (W0/APPLY/RESID), untouched by AM_SMOOTH.
// NC: r may be read through the non-coherent path (true unless r is written
// earlier in the same kernel, as in k_coarse_tail).
// itf: bit f set if edge f is a partition interface edge (multi-GPU): the
// colour-1 pass stores only this rank's partial sum there (y = y_T) and the
// interface epilogue (k_itf_epilogue) finishes it after the halo exchange.
// FMASK: the edges (bits) this call handles (the two-warp apply splits them)
template <int K1, int MODE, bool NC = true, int FMASK = 15>
__device__ __forceinline__ void epi_load(const LevelDev& L, const int64_t ed[4], const bool bd[4],
                                         const double* y, const double* __restrict__ r,
                                         const double* d, double* t, double* dd, int itf = 0) {
  if (MODE == AM_W0) return;
#pragma unroll
  for (int f = 0; f < 4; ++f) {
    if (!((FMASK >> f) & 1)) continue;
    if ((itf >> f) & 1) {
#pragma unroll
      for (int a = 0; a < K1; ++a) {
        t[f * K1 + a] = 0.0;
        dd[f * K1 + a] = 0.0;
      }
      continue;
    }
    const int64_t base = ed[f] * K1;
    double yo[K1], rv[K1], dv[K1];
#pragma unroll
    for (int a = 0; a < K1; ++a) yo[a] = rv[a] = dv[a] = 0.0;
    if (!bd[f]) {
      ld_edge<K1>(y + base, yo);
      if (MODE != AM_APPLY && MODE != AM_DINV) {
        if (NC) {
#pragma unroll
          for (int a = 0; a < K1; ++a) rv[a] = __ldg(r + base + a);
        } else {
          ld_edge<K1>(r + base, rv);
        }
      }
      if (MODE == AM_SMOOTH && L.smoother == 1) ld_edge<K1>(d + base, dv);
    }
#pragma unroll
    for (int a = 0; a < K1; ++a) {
      if (MODE == AM_APPLY || MODE == AM_DINV) t[f * K1 + a] = yo[a];
      else t[f * K1 + a] = bd[f] ? 0.0 : rv[a] - yo[a];
      if (MODE == AM_SMOOTH) dd[f * K1 + a] = dv[a];
    }
  }
}

template <int K1, int MODE, bool DOT, int FMASK = 15>
__device__ __forceinline__ void epi_store(const LevelDev& L, const int64_t ed[4], const bool bd[4],
                                          const double* xv, const double* yv, const double* t,
                                          const double* dd, const double* x, double* y, double* d,
                                          int step, double c1, double c2, double& dot,
                                          int itf = 0) {
#pragma unroll
  for (int f = 0; f < 4; ++f) {
    if (!((FMASK >> f) & 1)) continue;
    const int64_t base = ed[f] * K1;
    if (MODE != AM_W0 && ((itf >> f) & 1)) {   // partial sum only; finished after the halo
      st_edge<K1>(y + base, yv + f * K1);
      continue;
    }
    if (MODE == AM_W0 || MODE == AM_APPLY || MODE == AM_RESID) {
      double v[K1];
#pragma unroll
      for (int a = 0; a < K1; ++a) {
        v[a] = bd[f] ? 0.0
             : MODE == AM_W0 ? yv[f * K1 + a]
             : MODE == AM_APPLY ? t[f * K1 + a] + yv[f * K1 + a]
                               : t[f * K1 + a] - yv[f * K1 + a];
        if (MODE == AM_APPLY && DOT) dot = fma(xv[f * K1 + a], v[a], dot);
      }
      st_edge<K1>(y + base, v);
    } else if (MODE == AM_DINV) {  // power iteration on D^-1 A: x <- D^-1 A x in place
      if (!bd[f]) {
        double yf[K1];
#pragma unroll
        for (int a = 0; a < K1; ++a) {
          yf[a] = t[f * K1 + a] + yv[f * K1 + a];
          y[base + a] = yf[a];
        }
        const double* Di = L.Dinv + ed[f];
        double* xo = const_cast<double*>(x);
#pragma unroll
        for (int a = 0; a < K1; ++a) {
          double c = 0.0;
#pragma unroll
          for (int b = 0; b < K1; ++b) c = fma(__ldg(Di + (a * K1 + b) * L.nedge), yf[b], c);
          xo[base + a] = c;
          if (DOT) dot = fma(c, yf[a], dot);   // v_{k+1} . D v_{k+1}  (D v_{k+1} = A v_k)
        }
      } else {
#pragma unroll
        for (int a = 0; a < K1; ++a) y[base + a] = 0.0;
      }
    } else {  // AM_SMOOTH: x is updated in place (x aliases the smoothed iterate)
      if (!bd[f]) {
        double res[K1];
#pragma unroll
        for (int a = 0; a < K1; ++a) res[a] = t[f * K1 + a] - yv[f * K1 + a];
        const double* Di = L.Dinv + ed[f];   // SoA: coalesced across neighbouring elements
        double* xo = const_cast<double*>(x);
#pragma unroll
        for (int a = 0; a < K1; ++a) {
          double c = 0.0;
#pragma unroll
          for (int b = 0; b < K1; ++b) c = fma(__ldg(Di + (a * K1 + b) * L.nedge), res[b], c);
          double dn = c2 * c;
          if (L.smoother == 1) {
            if (step > 0) dn = fma(c1, dd[f * K1 + a], dn);
            d[base + a] = dn;
          }
          xo[base + a] = xv[f * K1 + a] + dn;
        }
      }
    }
  }
}

// y_T = S_T x_T from a packed symmetric S_T whose entry kk sits at Sp[kk * 32]
template <int M, typename LD>
__device__ __forceinline__ void packed_matvec(const double* xv, double* yv, LD load) {
#pragma unroll
  for (int a = 0; a < M; ++a) yv[a] = 0.0;
#pragma unroll
  for (int a = 0; a < M; ++a) {
#pragma unroll
    for (int b = a; b < M; ++b) {
      const int kk = a * (2 * M - a + 1) / 2 + (b - a);
      const double sv = load(kk);
      yv[a] = fma(sv, xv[b], yv[a]);
      if (b != a) yv[b] = fma(sv, xv[a], yv[b]);
    }
  }
}

// one colour pass over the elements (thread per element, plain loads; used for
// the L2-resident coarse levels inside k_coarse_tail)
template <int P, int MODE, bool NC = true, bool DOT = false>
__device__ __forceinline__ double apply_pass_body(const LevelDev& L, int colour, const double* x,
                                                  double* y, const double* r, double* d, int step,
                                                  int64_t t0, int64_t nt) {
  constexpr int K1 = P + 1, M = 4 * K1, NPK = M * (M + 1) / 2;
  const int64_t nec = L.ne >> 1;
  double c1 = 0.0, c2 = 0.0;
  if (MODE == AM_SMOOTH) {
    c1 = L.coef[2 * step];
    c2 = L.coef[2 * step + 1];
  }
  double dot = 0.0;
  for (int64_t s = t0; s < nec; s += nt) {
    int i, j;
    slot_elem(L.nx, colour, s, i, j);
    int64_t ed[4];
    bool bd[4];
    elem_edges(L.nx, L.ny, i, j, ed, bd, L.dmask);
    double xv[M], yv[M], t[M], dd[M];
    gather_x<K1>(x, ed, bd, xv);
    epi_load<K1, MODE, NC>(L, ed, bd, y, r, d, t, dd);
    const double* Sp = L.S + ((((int64_t)colour * L.nchunk + (s >> 5)) * NPK) << 5) + (s & 31);
    packed_matvec<M>(xv, yv, [&](int kk) { return Sp[kk << 5]; });
    epi_store<K1, MODE, DOT>(L, ed, bd, xv, yv, t, dd, x, y, d, step, c1, c2, dot);
  }
  return dot;
}

// power-iteration start vector (Q11): v_i = 1 + (i mod 7)/7 on free dofs, i = GLOBAL
// dof id (the same vector on 1 GPU and on any partition; duplicated interface dofs agree)
__device__ __forceinline__ void pow_init_body(const LevelDev& L, double* v, int64_t t0, int64_t nt) {
  for (int64_t i = t0; i < L.ndof; i += nt) {
    const int64_t e = (unsigned)i / (unsigned)L.k1;
    const int64_t gi = global_edge(L, e) * L.k1 + (i - e * L.k1);
    v[i] = edge_on_boundary(L.nx, L.ny, e, L.dmask) ? 0.0 : 1.0 + (double)(gi % 7) / 7.0;
  }
}

// ---------------------------------------------------------------- smoothing, first step
// e = 0 -> first smoothing step needs no apply: e = c2_0 Dinv r (d = e for Chebyshev).
__device__ __forceinline__ void smooth_first_body(const LevelDev& L, const double* __restrict__ r,
                                                  double* e, double* d, int64_t t0, int64_t nt) {
  const int K1 = L.k1;
  const double c2 = L.coef[1];
  for (int64_t ed = t0; ed < L.nedge; ed += nt) {
    if (edge_on_boundary(L.nx, L.ny, ed, L.dmask)) continue;
    const double* Di = L.Dinv + ed;
    for (int a = 0; a < K1; ++a) {
      double c = 0.0;
      for (int b = 0; b < K1; ++b) c = fma(Di[(a * K1 + b) * L.nedge], r[ed * K1 + b], c);
      double v = c2 * c;
      e[ed * K1 + a] = v;
      if (L.smoother == 1) d[ed * K1 + a] = v;
    }
  }
}

// ---------------------------------------------------------------- local correction + restriction (macro part)
__device__ __forceinline__ void macro_interior_edges(const LevelDev& F, int I, int J,
                                                     int64_t ie[4]) {
  ie[0] = hedge(F.nx, 2 * I, 2 * J + 1);
  ie[1] = hedge(F.nx, 2 * I + 1, 2 * J + 1);
  ie[2] = vedge(F.nx, F.ny, 2 * I + 1, 2 * J);
  ie[3] = vedge(F.nx, F.ny, 2 * I + 1, 2 * J + 1);
}

// h-prolongation term (I_k ec)_E of fine P1 edge E (Eqs. 3.3 / 3.4): an edge inside a 2x2
// macro gets its two rows of P_M ec_M (P_M = -A_II^-1 A_IB J), an edge on a macro side the
// linear interpolation J of its coarse edge's two values (skip: that coarse edge is on
// dOmega, no dofs).  k_prolong_edges and the folded colour-0 pass (AM_W0H) share it.
__device__ __forceinline__ double2 prolong_edge_term(int nx, int ny, int nxc, int nyc, int cdmask,
                                                     const double* __restrict__ ec,
                                                     const double* __restrict__ Pm, int64_t E,
                                                     bool& skip) {
  const int64_t nhF = (int64_t)nx * (ny + 1);
  int I, J, k = -1, half = 0;
  int64_t cE = 0;
  skip = false;
  if (E < nhF) {
    const int j = (int)((unsigned)E / (unsigned)nx), i = (int)E - j * nx;
    I = i >> 1;
    J = j >> 1;
    if (j & 1) k = i & 1;                       // ie[0] / ie[1]
    else { cE = hedge(nxc, I, J); half = i & 1; }
  } else {
    const int64_t r = E - nhF;
    const int j = (int)((unsigned)r / (unsigned)(nx + 1)), i = (int)r - j * (nx + 1);
    I = i >> 1;
    J = j >> 1;
    if (i & 1) k = 2 + (j & 1);                 // ie[2] / ie[3]
    else { cE = vedge(nxc, nyc, I, J); half = j & 1; }
  }
  if (k >= 0) {
    int64_t ce[4];
    bool cb[4];
    elem_edges(nxc, nyc, I, J, ce, cb, cdmask);
    double c[8];
#pragma unroll
    for (int f = 0; f < 4; ++f) {
      const double2 t = cb[f] ? make_double2(0.0, 0.0) : reinterpret_cast<const double2*>(ec)[ce[f]];
      c[2 * f] = t.x;
      c[2 * f + 1] = t.y;
    }
    const double2* P = reinterpret_cast<const double2*>(Pm + ((int64_t)J * nxc + I) * 64 + k * 16);
    double a0 = 0.0, a1 = 0.0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const double2 p0 = __ldg(P + q), p1 = __ldg(P + 4 + q);
      a0 = fma(p0.x, c[2 * q], a0);
      a0 = fma(p0.y, c[2 * q + 1], a0);
      a1 = fma(p1.x, c[2 * q], a1);
      a1 = fma(p1.y, c[2 * q + 1], a1);
    }
    return make_double2(a0, a1);
  }
  if (edge_on_boundary(nxc, nyc, cE, cdmask)) {
    skip = true;
    return make_double2(0.0, 0.0);
  }
  const double2 t = reinterpret_cast<const double2*>(ec)[cE];
  const double cm = 0.5 * (t.x + t.y);
  return half ? make_double2(cm, t.y) : make_double2(t.x, cm);
}

// step 3 (e_I += A_II^-1 res_I per macro) and the macro part of Q_{k-1}
// (cbuf = P_M^T res_I per macro).  Work item = (macro M, row c): 8 threads per
// macro, each one output row, so the 2 x 64 matrix loads of a macro are spread
// over 8 threads (coalesced 512-byte rows / columns) instead of one dependent
// chain per thread.
__device__ __forceinline__ void lc_restrict_body(const LevelDev& F, const double* __restrict__ res,
                                                 double* e, const double* __restrict__ KIIinv,
                                                 const double* __restrict__ Pm, double* cbuf,
                                                 int do_lc, int do_restrict, int64_t t0,
                                                 int64_t nt) {
  const int nxc = F.nx >> 1;
  const int64_t nmac = (int64_t)nxc * (F.ny >> 1);
  for (int64_t w = t0; w < nmac * 8; w += nt) {
    const int64_t M = w >> 3;
    const int c = (int)(w & 7);
    const int J = (int)((unsigned)M / (unsigned)nxc), I = (int)M - J * nxc;
    int64_t ie[4];
    macro_interior_edges(F, I, J, ie);
    double rI[8];
#pragma unroll
    for (int l = 0; l < 4; ++l) {
      rI[2 * l] = res[ie[l] * 2];
      rI[2 * l + 1] = res[ie[l] * 2 + 1];
    }
    if (do_lc) {
      double acc = 0.0;
      if (F.ns) {   // full 8 x 8 (nonsymmetric A_II)
        const double* Ki = KIIinv + M * 64 + c * 8;
#pragma unroll
        for (int b = 0; b < 8; ++b) acc = fma(Ki[b], rI[b], acc);
      } else {      // packed upper triangle of the symmetric inverse
        const double* Ki = KIIinv + M * 36;
#pragma unroll
        for (int b = 0; b < 8; ++b)
          acc = fma(Ki[c <= b ? pk_index(c, b, 8) : pk_index(b, c, 8)], rI[b], acc);
      }
      e[ie[c >> 1] * 2 + (c & 1)] += acc;
    }
    if (do_restrict) {
      const double* P = Pm + M * 64 + c;
      double acc = 0.0;
#pragma unroll
      for (int a = 0; a < 8; ++a) acc = fma(P[a * 8], rI[a], acc);
      cbuf[M * 8 + c] = acc;
    }
  }
}

// restriction, coarse-edge part: rc = J^T res_B + sum_{M adjacent} (P_M^T res_I)[slot];
// optionally fused with the coarse level's first smoothing step.
__device__ __forceinline__ void restrict_edges_body(const LevelDev& F, const LevelDev& C,
                                                    const double* __restrict__ res,
                                                    const double* __restrict__ cbuf, double* rc,
                                                    int fuse, double* ec, double* dc, int64_t t0,
                                                    int64_t nt) {
  const int nxc = C.nx, nyc = C.ny;
  const int64_t nh = (int64_t)nxc * (nyc + 1);
  const double c2 = fuse ? C.coef[1] : 0.0;
  for (int64_t E = t0; E < C.nedge; E += nt) {
    double v0 = 0.0, v1 = 0.0;
    // coarse edge on a local mesh side: on dOmega (no dofs) or a partition interface
    // (J^T res only here; the two adjacent macros' P_M^T terms live on two ranks and
    // are added by k_restrict_itf after the halo exchange)
    const int sd = edge_side(nxc, nyc, E);
    const bool bnd = sd >= 0 && ((C.dmask >> sd) & 1);
    const bool itf = sd >= 0 && !bnd;
    if (E < nh) {
      const int J = (int)((unsigned)E / (unsigned)nxc), I = (int)E - J * nxc;
      if (!bnd) {
        const int64_t f0 = hedge(F.nx, 2 * I, 2 * J), f1 = hedge(F.nx, 2 * I + 1, 2 * J);
        const double a0 = res[f0 * 2], a1 = res[f0 * 2 + 1], b0 = res[f1 * 2], b1 = res[f1 * 2 + 1];
        v0 = a0 + 0.5 * a1 + 0.5 * b0;
        v1 = 0.5 * a1 + 0.5 * b0 + b1;
        if (!itf) {
          const int64_t Mb = (int64_t)(J - 1) * nxc + I, Ma = (int64_t)J * nxc + I;
          v0 += cbuf[Mb * 8 + 4] + cbuf[Ma * 8 + 0];
          v1 += cbuf[Mb * 8 + 5] + cbuf[Ma * 8 + 1];
        }
      }
    } else {
      const int64_t rr = E - nh;
      const int J = (int)((unsigned)rr / (unsigned)(nxc + 1)), I = (int)rr - J * (nxc + 1);
      if (!bnd) {
        const int64_t f0 = vedge(F.nx, F.ny, 2 * I, 2 * J), f1 = vedge(F.nx, F.ny, 2 * I, 2 * J + 1);
        const double a0 = res[f0 * 2], a1 = res[f0 * 2 + 1], b0 = res[f1 * 2], b1 = res[f1 * 2 + 1];
        v0 = a0 + 0.5 * a1 + 0.5 * b0;
        v1 = 0.5 * a1 + 0.5 * b0 + b1;
        if (!itf) {
          const int64_t Ml = (int64_t)J * nxc + (I - 1), Mr = (int64_t)J * nxc + I;
          v0 += cbuf[Ml * 8 + 2] + cbuf[Mr * 8 + 6];
          v1 += cbuf[Ml * 8 + 3] + cbuf[Mr * 8 + 7];
        }
      }
    }
    rc[E * 2] = v0;
    rc[E * 2 + 1] = v1;
    if (fuse && !bnd && !itf) {
      const double* Di = C.Dinv + E;
      const int64_t sd = C.nedge;
      double e0 = c2 * (Di[0] * v0 + Di[sd] * v1);
      double e1 = c2 * (Di[2 * sd] * v0 + Di[3 * sd] * v1);
      ec[E * 2] = e0;
      ec[E * 2 + 1] = e1;
      if (C.smoother == 1) {
        dc[E * 2] = e0;
        dc[E * 2 + 1] = e1;
      }
    }
  }
}

// prolongation (macro): e_I += P_M e_c(M); e_B += J e_c on the macro's bottom and
// left macro-edges (every interior macro-edge is the bottom or left edge of
// exactly one macro).  Work item = (macro M, t in 0..7): row t of P_M e_c, and
// value t of the bottom (t < 4) / left (t >= 4) macro-edge's J e_c.
__device__ __forceinline__ void prolong_macro_body(const LevelDev& F, const LevelDev& C,
                                                   const double* __restrict__ ec,
                                                   const double* __restrict__ Pm, double* e,
                                                   int64_t t0, int64_t nt) {
  const int nxc = C.nx, nyc = C.ny;
  const int64_t nmac = (int64_t)nxc * nyc;
  for (int64_t w = t0; w < nmac * 8; w += nt) {
    const int64_t M = w >> 3;
    const int t = (int)(w & 7);
    const int J = (int)((unsigned)M / (unsigned)nxc), I = (int)M - J * nxc;
    int64_t ce[4];
    bool cb[4];
    elem_edges(nxc, nyc, I, J, ce, cb, C.dmask);
    double c[8];
#pragma unroll
    for (int f = 0; f < 4; ++f) {
      c[2 * f] = cb[f] ? 0.0 : ec[ce[f] * 2];
      c[2 * f + 1] = cb[f] ? 0.0 : ec[ce[f] * 2 + 1];
    }
    int64_t ie[4];
    macro_interior_edges(F, I, J, ie);
    const double* P = Pm + M * 64 + t * 8;
    double acc = 0.0;
#pragma unroll
    for (int b = 0; b < 8; ++b) acc = fma(P[b], c[b], acc);
    e[ie[t >> 1] * 2 + (t & 1)] += acc;
    // J on the macro-edge: fine edge f0 (lower coordinate) gets (c0, (c0+c1)/2),
    // f1 gets ((c0+c1)/2, c1)
    const int side = t < 4 ? 0 : 3;       // bottom / left
    if (!cb[side]) {
      const int u = t & 3;
      const double c0 = c[2 * side], c1 = c[2 * side + 1], cm = 0.5 * (c0 + c1);
      const int64_t f = side == 0 ? hedge(F.nx, 2 * I + (u >> 1), 2 * J)
                                  : vedge(F.nx, F.ny, 2 * I, 2 * J + (u >> 1));
      const double v = u == 0 ? c0 : u == 3 ? c1 : cm;
      e[f * 2 + (u & 1)] += v;
    }
  }
}

// ---------------------------------------------------------------- p-level transfers (per edge)
__device__ __forceinline__ void p_restrict_body(const LevelDev& F, const LevelDev& C,
                                                const double* __restrict__ Jp,
                                                const double* __restrict__ res, double* rc,
                                                int fuse, double* ec, double* dc, int64_t t0,
                                                int64_t nt) {
  const int K1 = F.k1;
  const double c2 = fuse ? C.coef[1] : 0.0;
  for (int64_t E = t0; E < F.nedge; E += nt) {
    if (edge_on_boundary(F.nx, F.ny, E, F.dmask)) {
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
      const double* Di = C.Dinv + E;
      const int64_t sd = C.nedge;
      double e0 = c2 * (Di[0] * v0 + Di[sd] * v1);
      double e1 = c2 * (Di[2 * sd] * v0 + Di[3 * sd] * v1);
      ec[E * 2] = e0;
      ec[E * 2 + 1] = e1;
      if (C.smoother == 1) {
        dc[E * 2] = e0;
        dc[E * 2 + 1] = e1;
      }
    }
  }
}

__device__ __forceinline__ void p_prolong_body(const LevelDev& F, const double* __restrict__ Jp,
                                               const double* __restrict__ ec, double* e,
                                               int64_t t0, int64_t nt) {
  const int K1 = F.k1;
  for (int64_t E = t0; E < F.nedge; E += nt) {
    if (edge_on_boundary(F.nx, F.ny, E, F.dmask)) continue;
    const double c0 = ec[E * 2], c1 = ec[E * 2 + 1];
    for (int a = 0; a < K1; ++a) e[E * K1 + a] += fma(Jp[a * 2], c0, Jp[a * 2 + 1] * c1);
  }
}

// ---------------------------------------------------------------- coarsest solve, vectors
__device__ __forceinline__ void coarse_solve_body(const int* __restrict__ fidx, int nf,
                                                  const double* __restrict__ Ainv,
                                                  const double* __restrict__ r, double* e,
                                                  int64_t t0, int64_t nt) {
  for (int64_t t = t0; t < nf; t += nt) {
    double acc = 0.0;
    for (int c = 0; c < nf; ++c) acc += Ainv[t * nf + c] * r[fidx[c]];
    e[fidx[t]] = acc;
  }
}

__device__ __forceinline__ void zero_body(double* dst, int64_t n, int64_t t0, int64_t nt) {
  for (int64_t i = t0; i < n; i += nt) dst[i] = 0.0;
}

// Power iteration (Q11) without per-step normalisation: v_{k+1} = D^-1 A v_k
// (the Rayleigh quotient is scale invariant).  scal[7] = v.Dv (v = v_last,
// D v_last = A v_{last-1}), scal[8] = v.Av.  lambda_hat = safety * v.Av / v.Dv.
// Chebyshev coefficients (O8): theta = (b+a)/2, delta = (b-a)/2, sigma = theta/delta,
// step 0: c1 = 0, c2 = 1/theta; step k: rho_k = 1/(2 sigma - rho_{k-1}),
// c1 = rho_k rho_{k-1}, c2 = 2 rho_k / delta.
__device__ __forceinline__ void lmax_finish_body(double vAv, double vDv, double safety,
                                                 double ratio, int nu_max, double* lam_out,
                                                 double* coef) {
  const double lam = safety * vAv / vDv;
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

}  // namespace mgdtn
