// Invariant checks of a set-up hierarchy (mg_check_invariants, SURVEY 5 "debug mode"):
//   - every element map of every level annihilates constants (readings
//     R5 / R10 make this exact up to rounding): max_T ||S_T 1||_inf / max|S_T|;
//   - no NaN / Inf in the element maps, the edge-block inverses and the orbit records;
//   - the conflict-free two-colour apply equals an independent scatter with atomicAdd
//     (thread per element, no colouring) on the finest level.
#include "bodies.cuh"

namespace mgdtn {

__device__ __forceinline__ void atomic_max_pos(double* addr, double v) {
  // v >= 0: the IEEE bit patterns of non-negative doubles order like the values
  atomicMax(reinterpret_cast<unsigned long long*>(addr), (unsigned long long)__double_as_longlong(v));
}

// out[0] = max over elements of ||S_T 1||_inf / max_ab |S_T[a][b]| (packed storage, any m);
// out[1] += number of non-finite entries
__global__ void k_check_maps(LevelDev L, double* out) {
  const int m = L.m;
  const int64_t nec = L.ne >> 1;
  double worst = 0.0, bad = 0.0;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < 2 * nec;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int colour = q >= nec ? 1 : 0;
    const int64_t s = q - colour * nec;
    const double* Sp = L.S + s_offset(L.nchunk, L.npk, colour, s, 0);
    double mx = 0.0, rmax = 0.0;
    for (int a = 0; a < m; ++a) {
      double rs = 0.0;
      for (int b = 0; b < m; ++b) {
        const double v = Sp[(int64_t)s_index(a, b, m, L.ns) * 32];
        if (!isfinite(v)) bad += 1.0;
        rs += v;
        mx = fmax(mx, fabs(v));
      }
      rmax = fmax(rmax, fabs(rs));
    }
    if (mx > 0) worst = fmax(worst, rmax / mx);
  }
  if (worst > 0) atomic_max_pos(out, worst);
  if (bad > 0) atomicAdd(out + 1, bad);
}

// out[1] += non-finite entries of a device array
__global__ void k_check_finite(const double* v, int64_t n, double* out) {
  double bad = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    if (!isfinite(v[i])) bad += 1.0;
  if (bad > 0) atomicAdd(out + 1, bad);
}

// y = A x by atomic scatter-add: every element adds S_T x_T to its four edges (dOmega rows
// skipped); y must be zero on entry
template <int P>
__global__ void k_apply_atomic(LevelDev L, const double* __restrict__ x, double* y) {
  constexpr int K1 = P + 1, M = 4 * K1;
  for (int64_t el = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; el < L.ne;
       el += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(el % L.nx), j = (int)(el / L.nx);
    int colour;
    int64_t s;
    elem_slot(L.nx, i, j, colour, s);
    int64_t ed[4];
    bool bd[4];
    elem_edges(L.nx, L.ny, i, j, ed, bd, L.dmask);
    double xv[M], yv[M];
    gather_x<K1>(x, ed, bd, xv);
    const double* Sp = L.S + s_offset(L.nchunk, L.npk, colour, s, 0);
    packed_matvec<M>(xv, yv, [&](int kk) { return Sp[(int64_t)kk * 32]; });
    for (int f = 0; f < 4; ++f) {
      if (bd[f]) continue;
      for (int a = 0; a < K1; ++a) atomicAdd(y + ed[f] * K1 + a, yv[f * K1 + a]);
    }
  }
}

int launch_check_maps(const LevelDev& L, double* out, cudaStream_t st) {
  const int64_t n = L.ne;
  const int grid = (int)((n + 255) / 256 < 2368 ? (n + 255) / 256 : 2368);
  k_check_maps<<<grid > 0 ? grid : 1, 256, 0, st>>>(L, out);
  return 1;
}
int launch_check_finite(const double* v, int64_t n, double* out, cudaStream_t st) {
  if (!v || n <= 0) return 0;
  const int grid = (int)((n + 255) / 256 < 2368 ? (n + 255) / 256 : 2368);
  k_check_finite<<<grid, 256, 0, st>>>(v, n, out);
  return 1;
}
int launch_apply_atomic(const LevelDev& L, const double* x, double* y, cudaStream_t st) {
  if (L.ns) return -1;
  const int grid = (int)((L.ne + 127) / 128 < 2368 ? (L.ne + 127) / 128 : 2368);
  switch (L.p) {
    case 1: k_apply_atomic<1><<<grid, 128, 0, st>>>(L, x, y); break;
    case 2: k_apply_atomic<2><<<grid, 128, 0, st>>>(L, x, y); break;
    case 3: k_apply_atomic<3><<<grid, 128, 0, st>>>(L, x, y); break;
    default: k_apply_atomic<4><<<grid, 128, 0, st>>>(L, x, y); break;
  }
  return 1;
}

}  // namespace mgdtn
