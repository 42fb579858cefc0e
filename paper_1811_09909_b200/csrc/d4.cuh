// Symmetry-reduced storage of the element DtN maps of a uniform square mesh.
//
// On an n x n mesh of squares with a scalar K per element (the only meshes the
// ABI accepts, mg_quad_mesh), every element's local problem (PAPER.md:186-199
// for HDG, 230-233 for SIPG-H) is invariant under the 8 symmetries of the
// square (the dihedral group D4): a rotation or reflection g maps the element
// onto itself, permutes its four edges and, since the GLL trace nodes are
// symmetric (s_{p-a} = 1 - s_a), permutes its 4(p+1) trace dofs.  The DtN map
// therefore commutes with these permutations, S_T = P_g S_T P_g^T, and an entry
// S_T[i][j] depends only on the D4 orbit of the pair {i, j}.  The number of
// orbits is 7 / 14 / 22 / 33 for p = 1..4 (against 36 / 78 / 136 / 210 packed
// entries), so a level whose element maps are all D4-invariant (the finest
// level, and its p-coarsened P1 level: J_p is D4-equivariant) is stored as one
// value per orbit and element (reading R9).  The p = 1 levels
// obtained by 2x2 agglomeration are not (the four children carry different K).
//
// The edge blocks D_e are sums of two elements' diagonal
// blocks for edge e; the reflection through the perpendicular bisector of e maps
// both elements onto themselves and reverses e, so D_e (and D_e^-1) is
// centrosymmetric: D[a][b] = D[p-a][p-b].  Stored per orbit of {a, b} under that
// reversal: 2 / 4 / 6 / 9 values per edge for p = 1..4 (against 3 / 6 / 10 / 15).
//
// Local trace dofs: (f, a) -> f*(p+1) + a, edges {0 bottom, 1 right, 2 top,
// 3 left}, each in its global orientation (+x for 0 and 2, +y for 1 and 3);
// the same numbering as the packed maps (kernels.cuh).  Tables are constexpr:
// inside unrolled loops every orbit index folds to an immediate.
#pragma once

namespace mgdtn {

template <int P>
struct D4 {
  static constexpr int K1 = P + 1, M = 4 * K1, NPK = M * (M + 1) / 2, NDE = K1 * (K1 + 1) / 2;

  // image of local dof i under group element g (g = 0..7: bit 2 swaps x and y, then
  // bit 0 flips x -> 1 - x, bit 1 flips y -> 1 - y)
  __host__ __device__ static constexpr int perm(int g, int i) {
    const int f = i / K1, a = i % K1;
    // endpoints (t = 0, t = 1) of edge f on the unit square
    const int e0x = f == 1 ? 1 : 0, e0y = f == 2 ? 1 : 0;
    const int e1x = f == 3 ? 0 : 1, e1y = (f == 0) ? 0 : 1;
    const int s0x = (g & 4) ? e0y : e0x, s0y = (g & 4) ? e0x : e0y;
    const int s1x = (g & 4) ? e1y : e1x, s1y = (g & 4) ? e1x : e1y;
    const int q0x = (g & 1) ? 1 - s0x : s0x, q0y = (g & 2) ? 1 - s0y : s0y;
    const int q1x = (g & 1) ? 1 - s1x : s1x, q1y = (g & 2) ? 1 - s1y : s1y;
    int fe = 0;
    bool rev = false;
    if (q0y == q1y) {   // horizontal image: bottom or top, parameter along +x
      fe = q0y == 0 ? 0 : 2;
      rev = q0x > q1x;
    } else {            // vertical image: left or right, parameter along +y
      fe = q0x == 0 ? 3 : 1;
      rev = q0y > q1y;
    }
    return fe * K1 + (rev ? P - a : a);
  }
  // packed upper-triangle index of (i, j) (kernels.cuh pk_index)
  __host__ __device__ static constexpr int pk(int i, int j) {
    return i <= j ? i * (2 * M - i + 1) / 2 + (j - i) : j * (2 * M - j + 1) / 2 + (i - j);
  }
  // packed index of (a, b) inside one k1 x k1 symmetric block
  __host__ __device__ static constexpr int pe(int a, int b) {
    return a <= b ? a * (2 * K1 - a + 1) / 2 + (b - a) : b * (2 * K1 - b + 1) / 2 + (a - b);
  }

  struct Tab {
    int orb[NPK];   // orbit of packed entry kk (numbered in order of first appearance)
    int cnt[NPK];   // members per orbit
    int norb;
    int cs[NDE];    // orbit of block entry pe(a,b) under (a,b) -> (p-a, p-b)
    int ccnt[NDE];
    int ncs;
  };
  __host__ __device__ static constexpr Tab make() {
    Tab t{};
    for (int q = 0; q < NPK; ++q) {
      t.orb[q] = -1;
      t.cnt[q] = 0;
    }
    int n = 0;
    for (int i = 0; i < M; ++i)
      for (int j = i; j < M; ++j) {
        if (t.orb[pk(i, j)] >= 0) continue;
        for (int g = 0; g < 8; ++g) {
          const int r = pk(perm(g, i), perm(g, j));
          if (t.orb[r] < 0) t.orb[r] = n;
        }
        ++n;
      }
    for (int q = 0; q < NPK; ++q) t.cnt[t.orb[q]]++;
    t.norb = n;
    for (int q = 0; q < NDE; ++q) {
      t.cs[q] = -1;
      t.ccnt[q] = 0;
    }
    n = 0;
    for (int a = 0; a < K1; ++a)
      for (int b = a; b < K1; ++b) {
        if (t.cs[pe(a, b)] >= 0) continue;
        t.cs[pe(a, b)] = n;
        t.cs[pe(P - a, P - b)] = n;
        ++n;
      }
    for (int q = 0; q < NDE; ++q) t.ccnt[t.cs[q]]++;
    t.ncs = n;
    return t;
  }
  __host__ __device__ static constexpr int orb(int kk) {
    constexpr Tab t = make();
    return t.orb[kk];
  }
  __host__ __device__ static constexpr int cnt(int o) {
    constexpr Tab t = make();
    return t.cnt[o];
  }
  __host__ __device__ static constexpr int cs(int q) {
    constexpr Tab t = make();
    return t.cs[q];
  }
  __host__ __device__ static constexpr int ccnt(int o) {
    constexpr Tab t = make();
    return t.ccnt[o];
  }
  static constexpr int NORB = make().norb;   // values per element
  static constexpr int NCS = make().ncs;     // values per edge block
};

static_assert(D4<1>::NORB == 7 && D4<2>::NORB == 14 && D4<3>::NORB == 22 && D4<4>::NORB == 33,
              "D4 orbit counts of the packed element maps");
static_assert(D4<1>::NCS == 2 && D4<2>::NCS == 4 && D4<3>::NCS == 6 && D4<4>::NCS == 9,
              "centrosymmetric orbit counts of the edge blocks");

__host__ __device__ inline int d4_norb(int p) {
  return p == 1 ? D4<1>::NORB : p == 2 ? D4<2>::NORB : p == 3 ? D4<3>::NORB : D4<4>::NORB;
}
__host__ __device__ inline int d4_ncs(int p) {
  return p == 1 ? D4<1>::NCS : p == 2 ? D4<2>::NCS : p == 3 ? D4<3>::NCS : D4<4>::NCS;
}

}  // namespace mgdtn
