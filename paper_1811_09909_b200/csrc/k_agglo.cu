// Seed-point agglomeration of an unstructured quad mesh (SURVEY.md 8(f) f4,
// PAPER.md:491-498, section 3.1.2; readings A1-A3 in DESIGN.md section 3):
//   level 1      graph Voronoi cells of the seeds on the element dual graph,
//                ties to the lower seed index (A1): a level-synchronous
//                multi-source BFS whose per-element key (hop << 32 | seed) is
//                lowered with atomicMin, one launch per BFS layer;
//   level k + 1  every level-k agglomerate split in four (A2): west / east
//                halves by rank under (cx, cy, id), then south / north by rank
//                under (cy, cx, id) inside each half.  The ranks come from
//                stable LSD radix sorts of the element ids (CUB, least
//                significant key first, the agglomerate label last): an
//                element's rank is its sorted position minus its agglomerate's
//                offset (count + one-CTA exclusive scan);
//   skeleton     an edge is on the level-k skeleton iff it is on the domain
//                boundary or its two elements carry different labels (A3).
// Integer output only: the comparisons are exact, so the labels are bit-equal
// to any implementation of the same readings (tests/test_gpu_agglomerate.py).
// Also here: the arc-length parameterisation of the macro-edges (A5,
// mg_macro_edge_params) and their P^p transfer blocks (A6, mg_macro_edge_transfer).
// This is setup-time work (once per mesh), not part of the solve.
#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include <cub/device/device_radix_sort.cuh>

#include "mgdtn.h"
#include "refelem.h"

namespace {

constexpr unsigned long long KEY_NONE = ~0ull;

// keys reset; an edge naming an element outside [0, ne) (or no first element) is an error
__global__ void k_seed_init(unsigned long long* key, int64_t ne, const int32_t* edge_elem,
                            int64_t nedge, int* err) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < ne) key[t] = KEY_NONE;
  if (t < nedge) {
    const int32_t a = edge_elem[2 * t], b = edge_elem[2 * t + 1];
    if (a < 0 || a >= ne || b < -1 || b >= ne) atomicExch(err, 1);
  }
}

__global__ void k_seed_set(unsigned long long* key, int64_t ne, const int32_t* seeds, int nseed,
                           int* err) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nseed) return;
  const int32_t s = seeds[k];
  if (s < 0 || s >= ne) {
    atomicExch(err, 1);
    return;
  }
  atomicMin(key + s, (unsigned long long)(uint32_t)k);   // hop 0; duplicate seeds: lower index
}

// one BFS layer: every element at hop d offers (d + 1, its seed) to its neighbours
__global__ void k_bfs_layer(unsigned long long* key, const int32_t* __restrict__ edge_elem,
                            int64_t nedge, uint32_t d, int* changed) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= nedge) return;
  const int32_t a = edge_elem[2 * e], b = edge_elem[2 * e + 1];
  if (b < 0) return;
  const unsigned long long ka = key[a], kb = key[b];
  const unsigned long long nxt = (unsigned long long)(d + 1) << 32;
  if (ka != KEY_NONE && (uint32_t)(ka >> 32) == d) {
    const unsigned long long c = nxt | (ka & 0xffffffffull);
    if (c < kb) {
      atomicMin(key + b, c);
      *changed = 1;
    }
  }
  if (kb != KEY_NONE && (uint32_t)(kb >> 32) == d) {
    const unsigned long long c = nxt | (kb & 0xffffffffull);
    if (c < ka) {
      atomicMin(key + a, c);
      *changed = 1;
    }
  }
}

__global__ void k_label1(const unsigned long long* key, int64_t ne, int32_t* lab,
                         unsigned long long* bad) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= ne) return;
  const unsigned long long k = key[t];
  if (k == KEY_NONE) {
    atomicMin(bad, (unsigned long long)t);
    lab[t] = -1;
  } else {
    lab[t] = (int32_t)(k & 0xffffffffull);
  }
}

__global__ void k_count(const int32_t* lab, int64_t ne, int32_t* cnt) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < ne) atomicAdd(cnt + lab[t], 1);
}

// exclusive scan of cnt[0..G) into off[0..G) by one CTA (setup-time, G <= ne)
__global__ void k_scan(const int32_t* cnt, int64_t G, int64_t* off) {
  __shared__ int64_t part[1024];
  const int tid = threadIdx.x, nt = blockDim.x;
  const int64_t per = (G + nt - 1) / nt, lo = tid * per, hi = lo + per < G ? lo + per : G;
  int64_t s = 0;
  for (int64_t g = lo; g < hi; ++g) s += cnt[g];
  part[tid] = s;
  __syncthreads();
  if (tid == 0) {
    int64_t run = 0;
    for (int i = 0; i < nt; ++i) {
      const int64_t v = part[i];
      part[i] = run;
      run += v;
    }
  }
  __syncthreads();
  s = part[tid];
  for (int64_t g = lo; g < hi; ++g) {
    off[g] = s;
    s += cnt[g];
  }
}

// ---- four-way split (A2) by stable LSD sorts: the element ids start in id order, then
// are stably sorted by the least significant key first, so after the sort by the
// agglomerate label they are in (label, key1, key2, id) order and an element's rank in
// its agglomerate is its position minus the agglomerate's offset.
__global__ void k_iota(int32_t* perm, int64_t ne) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < ne) perm[i] = (int32_t)i;
}

// sort key of position i: v[perm[i]], -0.0 folded into +0.0 (the radix order of the bit
// patterns then equals the order of operator<; NaN is rejected up front)
__global__ void k_gather_d(const int32_t* __restrict__ perm, const double* __restrict__ v,
                           int64_t ne, double* key) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= ne) return;
  const double x = v[perm[i]];
  key[i] = x == 0.0 ? 0.0 : x;
}

__global__ void k_gather_i(const int32_t* __restrict__ perm, const int32_t* __restrict__ v,
                           int64_t ne, int32_t* key) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < ne) key[i] = v[perm[i]];
}

// west / east half: the first ceil(m/2) of an agglomerate in (cx, cy, id) order are west;
// sub = 2 * label + east keys the second split
__global__ void k_half(const int32_t* __restrict__ perm, int64_t ne, const int32_t* __restrict__ lab,
                       const int64_t* __restrict__ off, const int32_t* __restrict__ cnt,
                       int32_t* sub) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= ne) return;
  const int32_t t = perm[i], g = lab[t];
  sub[t] = 2 * g + (i - off[g] >= (cnt[g] + 1) / 2);
}

// south / north quarter: the first ceil(h/2) of a half in (cy, cx, id) order are south
__global__ void k_quarter(const int32_t* __restrict__ perm, int64_t ne,
                          const int32_t* __restrict__ sub, const int64_t* __restrict__ off,
                          const int32_t* __restrict__ cnt, int32_t* nlab) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= ne) return;
  const int32_t t = perm[i], h = sub[t];
  nlab[t] = 2 * h + (i - off[h] >= (cnt[h] + 1) / 2);
}

__global__ void k_check_keys(const double* cx, const double* cy, int64_t ne, int* err) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < ne && (cx[t] != cx[t] || cy[t] != cy[t])) atomicExch(err, 1);
}

__global__ void k_skeleton(const int32_t* __restrict__ edge_elem, int64_t nedge,
                           const int32_t* __restrict__ lab, uint8_t* skel) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= nedge) return;
  const int32_t a = edge_elem[2 * e], b = edge_elem[2 * e + 1];
  skel[e] = b < 0 || lab[a] != lab[b];
}

// ---- level macro-edges (reading A4): the fine skeleton edges grouped by their pair
// (lo, hi) of agglomerates (lo = -1 on the domain boundary), numbered in lexicographic
// pair order.  Counting-sorted into 2G buckets: bucket a < G holds agglomerate a's share
// of the domain boundary (the single pair (-1, a)), bucket G + lo the interior edges of
// pairs (lo, *); inside a bucket (at most about one agglomerate's perimeter) the distinct
// hi values are found and ranked by comparison.  Bucket order = lexicographic pair order.
__device__ __forceinline__ bool edge_pair(const int32_t* __restrict__ edge_elem,
                                          const int32_t* __restrict__ lab, int64_t e, int32_t& lo,
                                          int32_t& hi) {
  const int32_t a = edge_elem[2 * e], b = edge_elem[2 * e + 1];
  if (b < 0) {
    lo = -1;
    hi = lab[a];
    return true;
  }
  const int32_t la = lab[a], lb = lab[b];
  lo = la < lb ? la : lb;
  hi = la < lb ? lb : la;
  return la != lb;
}

__device__ __forceinline__ int64_t bucket_of(int32_t lo, int32_t hi, int64_t G) {
  return lo < 0 ? hi : G + lo;
}

__global__ void k_me_count(const int32_t* edge_elem, int64_t nedge, const int32_t* lab, int64_t G,
                           int32_t* cnt) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= nedge) return;
  int32_t lo, hi;
  if (edge_pair(edge_elem, lab, e, lo, hi)) atomicAdd(cnt + bucket_of(lo, hi, G), 1);
}

__global__ void k_me_scatter(const int32_t* edge_elem, int64_t nedge, const int32_t* lab, int64_t G,
                             const int64_t* off, int32_t* cur, int32_t* elist) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= nedge) return;
  int32_t lo, hi;
  if (edge_pair(edge_elem, lab, e, lo, hi)) {
    const int64_t q = bucket_of(lo, hi, G);
    elist[off[q] + atomicAdd(cur + q, 1)] = (int32_t)e;
  }
}

// first[e] = e is the lowest-numbered edge of its pair; dcnt[bucket] counts the pairs
__global__ void k_me_first(const int32_t* __restrict__ edge_elem, int64_t nsk,
                           const int32_t* __restrict__ lab, int64_t G,
                           const int32_t* __restrict__ elist, const int64_t* __restrict__ off,
                           const int32_t* __restrict__ cnt, uint8_t* first, int32_t* dcnt) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nsk) return;
  const int32_t e = elist[i];
  int32_t lo, hi;
  edge_pair(edge_elem, lab, e, lo, hi);
  const int64_t q = bucket_of(lo, hi, G), o = off[q];
  const int32_t m = cnt[q];
  bool f = true;
  for (int32_t j = 0; j < m && f; ++j) {
    const int32_t u = elist[o + j];
    int32_t ul, uh;
    edge_pair(edge_elem, lab, u, ul, uh);
    if (uh == hi && u < e) f = false;
  }
  first[e] = f;
  if (f) atomicAdd(dcnt + q, 1);
}

__global__ void k_me_rank(const int32_t* __restrict__ edge_elem, int64_t nedge,
                          const int32_t* __restrict__ lab, int64_t G,
                          const int32_t* __restrict__ elist, const int64_t* __restrict__ off,
                          const int32_t* __restrict__ cnt, const uint8_t* __restrict__ first,
                          const int64_t* __restrict__ doff, int32_t* medge) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= nedge) return;
  int32_t lo, hi;
  if (!edge_pair(edge_elem, lab, e, lo, hi)) {
    medge[e] = -1;
    return;
  }
  const int64_t q = bucket_of(lo, hi, G), o = off[q];
  const int32_t m = cnt[q];
  int32_t rank = 0;
  for (int32_t j = 0; j < m; ++j) {
    const int32_t u = elist[o + j];
    if (!first[u]) continue;
    int32_t ul, uh;
    edge_pair(edge_elem, lab, u, ul, uh);
    rank += uh < hi;
  }
  medge[e] = (int32_t)(doff[q] + rank);
}

inline unsigned nblk(int64_t n, int t = 256) { return (unsigned)((n + t - 1) / t > 0 ? (n + t - 1) / t : 1); }

struct Scratch {
  cudaStream_t st;
  std::vector<void*> p;
  template <class T>
  T* get(size_t n) {
    void* q = nullptr;
    if (cudaMallocAsync(&q, n * sizeof(T) + 16, st) != cudaSuccess) return nullptr;
    p.push_back(q);
    return (T*)q;
  }
  ~Scratch() {
    for (void* q : p) cudaFreeAsync(q, st);
  }
};

}  // namespace

extern "C" int mg_agglomerate_seeds(int64_t ne, int64_t nedge, const int32_t* edge_elem,
                                    const double* cx, const double* cy, int32_t nseed,
                                    const int32_t* seeds, int32_t nlev, int32_t* labels,
                                    uint8_t* skel, int32_t* medge, int64_t* nmedge,
                                    void* stream, int64_t* bad_index) {
  if (bad_index) *bad_index = -1;
  if (ne <= 0 || ne > INT32_MAX || nedge <= 0 || nseed <= 0 || nlev < 2 || !edge_elem || !cx ||
      !cy || !seeds || !labels || !skel || (medge && !nmedge))
    return MG_ERR_ARG;
  // level k has nseed * 4^(k-1) ids; keep the last one within int32
  long double G = nseed;
  for (int k = 2; k < nlev; ++k) G *= 4;
  if (G > (long double)INT32_MAX) return MG_ERR_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  int rc = MG_OK;
  {
    Scratch S{st, {}};
    unsigned long long* key = S.get<unsigned long long>(ne);
    unsigned long long* bad = S.get<unsigned long long>(1);
    int* flags = S.get<int>(2);   // [0] seed error, [1] BFS changed
    // counting-sort buffers: G agglomerates (splits) or 2G pair buckets (macro-edges)
    int32_t* cnt = S.get<int32_t>(2 * (size_t)G);
    int32_t* cur = S.get<int32_t>(2 * (size_t)G);
    int64_t* off = S.get<int64_t>(2 * (size_t)G);
    int32_t* dcnt = S.get<int32_t>(2 * (size_t)G);
    int64_t* doff = S.get<int64_t>(2 * (size_t)G);
    int32_t* list = S.get<int32_t>(ne > nedge ? ne : nedge);
    uint8_t* east = S.get<uint8_t>(ne > nedge ? ne : nedge);
    // split sorts: permutation / key double buffers and CUB's temporary storage
    int32_t* permA = S.get<int32_t>(ne);
    int32_t* permB = S.get<int32_t>(ne);
    double* dkA = S.get<double>(ne);
    double* dkB = S.get<double>(ne);
    int32_t* ikA = S.get<int32_t>(ne);
    int32_t* ikB = S.get<int32_t>(ne);
    int32_t* sub = S.get<int32_t>(ne);
    size_t tb_d = 0, tb_i = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tb_d, dkA, dkB, permA, permB, (int)ne, 0, 64, st);
    cub::DeviceRadixSort::SortPairs(nullptr, tb_i, ikA, ikB, permA, permB, (int)ne, 0, 32, st);
    const size_t tbytes = tb_d > tb_i ? tb_d : tb_i;
    void* temp = S.get<unsigned char>(tbytes);
    if (!key || !bad || !flags || !cnt || !cur || !off || !dcnt || !doff || !list || !east ||
        !permA || !permB || !dkA || !dkB || !ikA || !ikB || !sub || !temp)
      return MG_ERR_CUDA;
    int32_t* perm = permA;   // current permutation (the other buffer receives each sort)
    auto other = [&](int32_t* q) { return q == permA ? permB : permA; };
    auto sort_by_d = [&](const double* v) {   // stable sort of perm by v[perm[i]]
      k_gather_d<<<nblk(ne), 256, 0, st>>>(perm, v, ne, dkA);
      size_t tb = tbytes;
      cub::DeviceRadixSort::SortPairs(temp, tb, dkA, dkB, perm, other(perm), (int)ne, 0, 64, st);
      perm = other(perm);
    };
    auto sort_by_i = [&](const int32_t* v, int64_t bound) {   // keys in [0, bound)
      int bits = 1;
      while (bits < 31 && ((int64_t)1 << bits) < bound) ++bits;
      k_gather_i<<<nblk(ne), 256, 0, st>>>(perm, v, ne, ikA);
      size_t tb = tbytes;
      cub::DeviceRadixSort::SortPairs(temp, tb, ikA, ikB, perm, other(perm), (int)ne, 0, bits, st);
      perm = other(perm);
    };
    int hflags[2] = {0, 0};
    cudaMemsetAsync(flags, 0, 2 * sizeof(int), st);
    cudaMemsetAsync(bad, 0xff, sizeof(unsigned long long), st);
    k_seed_init<<<nblk(ne > nedge ? ne : nedge), 256, 0, st>>>(key, ne, edge_elem, nedge, flags);
    k_seed_set<<<nblk(nseed), 256, 0, st>>>(key, ne, seeds, nseed, flags);
    k_check_keys<<<nblk(ne), 256, 0, st>>>(cx, cy, ne, flags);
    cudaMemcpyAsync(hflags, flags, sizeof(int), cudaMemcpyDeviceToHost, st);
    if (cudaStreamSynchronize(st) != cudaSuccess) return MG_ERR_CUDA;
    if (hflags[0]) return MG_ERR_ARG;   // seed or edge element id out of range
    // BFS layers in batches of 16 between host checks (extra layers are no-ops)
    for (uint32_t d = 0;; d += 16) {
      cudaMemsetAsync(flags + 1, 0, sizeof(int), st);
      for (uint32_t q = 0; q < 16; ++q)
        k_bfs_layer<<<nblk(nedge), 256, 0, st>>>(key, edge_elem, nedge, d + q, flags + 1);
      cudaMemcpyAsync(hflags, flags, 2 * sizeof(int), cudaMemcpyDeviceToHost, st);
      if (cudaStreamSynchronize(st) != cudaSuccess) return MG_ERR_CUDA;
      if (!hflags[1]) break;
    }
    k_label1<<<nblk(ne), 256, 0, st>>>(key, ne, labels, bad);
    k_skeleton<<<nblk(nedge), 256, 0, st>>>(edge_elem, nedge, labels, skel);
    unsigned long long hbad = 0;
    cudaMemcpyAsync(&hbad, bad, sizeof(hbad), cudaMemcpyDeviceToHost, st);
    if (cudaStreamSynchronize(st) != cudaSuccess) return MG_ERR_CUDA;
    if (hbad != KEY_NONE) {   // an element no seed reaches
      if (bad_index) *bad_index = (int64_t)hbad;
      return MG_ERR_SHAPE;
    }
    int64_t Gk = nseed;
    for (int k = 1; k < nlev; ++k, Gk *= 4) {
      const int32_t* lab = labels + (size_t)(k - 1) * ne;
      if (medge) {   // level-k macro-edges (A4); `east` doubles as the first-of-pair flags
        int32_t* me = medge + (size_t)(k - 1) * nedge;
        const int64_t B = 2 * Gk;
        cudaMemsetAsync(cnt, 0, (size_t)B * sizeof(int32_t), st);
        cudaMemsetAsync(cur, 0, (size_t)B * sizeof(int32_t), st);
        cudaMemsetAsync(dcnt, 0, (size_t)B * sizeof(int32_t), st);
        k_me_count<<<nblk(nedge), 256, 0, st>>>(edge_elem, nedge, lab, Gk, cnt);
        k_scan<<<1, 1024, 0, st>>>(cnt, B, off);
        k_me_scatter<<<nblk(nedge), 256, 0, st>>>(edge_elem, nedge, lab, Gk, off, cur, list);
        int64_t hoff = 0;
        int32_t hcnt = 0;
        cudaMemcpyAsync(&hoff, off + B - 1, sizeof(hoff), cudaMemcpyDeviceToHost, st);
        cudaMemcpyAsync(&hcnt, cnt + B - 1, sizeof(hcnt), cudaMemcpyDeviceToHost, st);
        if (cudaStreamSynchronize(st) != cudaSuccess) return MG_ERR_CUDA;
        const int64_t nsk = hoff + hcnt;   // skeleton edges of level k
        k_me_first<<<nblk(nsk), 256, 0, st>>>(edge_elem, nsk, lab, Gk, list, off, cnt, east, dcnt);
        k_scan<<<1, 1024, 0, st>>>(dcnt, B, doff);
        k_me_rank<<<nblk(nedge), 256, 0, st>>>(edge_elem, nedge, lab, Gk, list, off, cnt, east, doff,
                                                me);
        int32_t hd = 0;
        cudaMemcpyAsync(&hoff, doff + B - 1, sizeof(hoff), cudaMemcpyDeviceToHost, st);
        cudaMemcpyAsync(&hd, dcnt + B - 1, sizeof(hd), cudaMemcpyDeviceToHost, st);
        if (cudaStreamSynchronize(st) != cudaSuccess) return MG_ERR_CUDA;
        nmedge[k - 1] = hoff + hd;
      }
      if (k + 1 == nlev) break;
      int32_t* nlab = labels + (size_t)k * ne;
      // west / east: order (label, cx, cy, id)
      cudaMemsetAsync(cnt, 0, (size_t)Gk * sizeof(int32_t), st);
      k_count<<<nblk(ne), 256, 0, st>>>(lab, ne, cnt);
      k_scan<<<1, 1024, 0, st>>>(cnt, Gk, off);
      k_iota<<<nblk(ne), 256, 0, st>>>(perm, ne);
      sort_by_d(cy);
      sort_by_d(cx);
      sort_by_i(lab, Gk);
      k_half<<<nblk(ne), 256, 0, st>>>(perm, ne, lab, off, cnt, sub);
      // south / north: order (2 label + east, cy, cx, id)
      cudaMemsetAsync(cnt, 0, (size_t)(2 * Gk) * sizeof(int32_t), st);
      k_count<<<nblk(ne), 256, 0, st>>>(sub, ne, cnt);
      k_scan<<<1, 1024, 0, st>>>(cnt, 2 * Gk, off);
      k_iota<<<nblk(ne), 256, 0, st>>>(perm, ne);
      sort_by_d(cx);
      sort_by_d(cy);
      sort_by_i(sub, 2 * Gk);
      k_quarter<<<nblk(ne), 256, 0, st>>>(perm, ne, sub, off, cnt, nlab);
      k_skeleton<<<nblk(nedge), 256, 0, st>>>(edge_elem, nedge, nlab, skel + (size_t)k * nedge);
    }
    if (cudaGetLastError() != cudaSuccess) rc = MG_ERR_CUDA;
  }
  if (cudaStreamSynchronize(st) != cudaSuccess) rc = MG_ERR_CUDA;
  return rc;
}

// ---- macro-edge arc-length parameterisation (reading A5) ----
// Every fine-edge end of a macro-edge becomes a record keyed (macro-edge, vertex); after
// a radix sort the records of one vertex are adjacent, so each end learns its partner:
// the other edge of the same macro-edge at that vertex (-1: a path end, -2: a vertex
// shared by more than two of its edges).  One thread per fine edge then walks its path:
// to both ends (path check: no branch, no loop, one piece = the macro-edge's size), then
// from the start end (least in (vx, vy, id)) forward, summing the edge lengths in path
// order twice (total, then up to itself), the same additions in the same order as a
// sequential sweep.  O(L) per edge for a path of L edges (setup-time).
namespace {

constexpr unsigned long long REC_NONE = ~0ull;

__global__ void k_ep_records(const int32_t* __restrict__ medge, const int32_t* __restrict__ ev,
                             int64_t nedge, int64_t nmedge, int64_t nvert, unsigned long long* key,
                             int32_t* val, int32_t* size, int* err) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= 2 * nedge) return;
  const int64_t e = r >> 1;
  int32_t q = medge[e];
  const int32_t v = ev[r];
  if (v < 0 || v >= nvert || q >= nmedge) {
    atomicExch(err, 1);
    q = -1;
  }
  key[r] = q >= 0 && v >= 0 && v < nvert
               ? ((unsigned long long)(uint32_t)q << 32) | (uint32_t)v : REC_NONE;
  val[r] = (int32_t)r;
  if (q >= 0 && (r & 1) == 0) atomicAdd(size + q, 1);
}

__global__ void k_ep_partner(const unsigned long long* __restrict__ key,
                             const int32_t* __restrict__ val, int64_t nrec, int32_t* partner) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nrec) return;
  const unsigned long long k = key[i];
  if (k == REC_NONE) return;
  int64_t lo = i, hi = i + 1;
  while (lo > 0 && key[lo - 1] == k) --lo;
  while (hi < nrec && key[hi] == k) ++hi;
  const int64_t deg = hi - lo;
  partner[val[i]] = deg == 1 ? -1 : deg == 2 ? val[i == lo ? lo + 1 : lo] : -2;
}

__device__ __forceinline__ double edge_len(const double* vx, const double* vy, int32_t a,
                                           int32_t b) {
  const double dx = vx[b] - vx[a], dy = vy[b] - vy[a];
  return sqrt(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)));   // no FMA contraction
}

__global__ void k_ep_param(const int32_t* __restrict__ medge, const int32_t* __restrict__ ev,
                           int64_t nedge, const int32_t* __restrict__ partner,
                           const int32_t* __restrict__ size, const double* __restrict__ vx,
                           const double* __restrict__ vy, double* s) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= nedge) return;
  s[2 * e] = s[2 * e + 1] = -1.0;
  const int32_t q = medge[e];
  if (q < 0) return;
  const int32_t m = size[q];
  // walk to the end beyond side c0 of e; returns the end record (edge << 1 | side) or -1
  auto walk_end = [&](int c0, int32_t& steps) -> int64_t {
    int64_t f = e;
    int c = c0;
    steps = 0;
    for (;;) {
      const int32_t p = partner[2 * f + c];
      if (p == -1) return (f << 1) | c;
      if (p == -2) return -1;
      f = p >> 1;
      c = 1 - (p & 1);
      if (f == e || ++steps >= m) return -1;   // a loop, or longer than the macro-edge
    }
  };
  int32_t s0 = 0, s1 = 0;
  const int64_t A = walk_end(0, s0), B = walk_end(1, s1);
  if (A < 0 || B < 0 || s0 + s1 + 1 != m) return;   // not one open path
  const int32_t va = ev[A], vb = ev[B];
  const bool a_first = vx[va] < vx[vb] || (vx[va] == vx[vb] && (vy[va] < vy[vb] ||
                                                                 (vy[va] == vy[vb] && va < vb)));
  const int64_t S = a_first ? A : B;   // start record: the path enters there
  double total = 0.0;
  {
    int64_t f = S >> 1;
    int c = (int)(S & 1);
    for (;;) {
      total += edge_len(vx, vy, ev[2 * f + c], ev[2 * f + 1 - c]);
      const int32_t p = partner[2 * f + 1 - c];
      if (p == -1) break;
      f = p >> 1;
      c = p & 1;
    }
  }
  double cum = 0.0;
  int64_t f = S >> 1;
  int c = (int)(S & 1);
  for (;;) {
    const double ln = edge_len(vx, vy, ev[2 * f + c], ev[2 * f + 1 - c]);
    if (f == e) {
      s[2 * e + c] = cum / total;
      s[2 * e + 1 - c] = (cum + ln) / total;
      return;
    }
    cum += ln;
    const int32_t p = partner[2 * f + 1 - c];
    f = p >> 1;
    c = p & 1;
  }
}

}  // namespace

extern "C" int mg_macro_edge_params(int64_t nedge, const int32_t* medge, int64_t nmedge,
                                    const int32_t* edge_vert, int64_t nvert, const double* vx,
                                    const double* vy, double* s, void* stream) {
  if (nedge <= 0 || nedge > INT32_MAX / 2 || nmedge < 0 || nmedge > INT32_MAX || nvert <= 0 ||
      nvert > INT32_MAX || !medge || !edge_vert || !vx || !vy || !s)
    return MG_ERR_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t nrec = 2 * nedge;
  int rc = MG_OK;
  {
    Scratch S{st, {}};
    unsigned long long* kA = S.get<unsigned long long>(nrec);
    unsigned long long* kB = S.get<unsigned long long>(nrec);
    int32_t* vA = S.get<int32_t>(nrec);
    int32_t* vB = S.get<int32_t>(nrec);
    int32_t* partner = S.get<int32_t>(nrec);
    int32_t* size = S.get<int32_t>(nmedge + 1);
    int* err = S.get<int>(1);
    size_t tb = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tb, kA, kB, vA, vB, (int)nrec, 0, 64, st);
    void* temp = S.get<unsigned char>(tb);
    if (!kA || !kB || !vA || !vB || !partner || !size || !err || !temp) return MG_ERR_CUDA;
    cudaMemsetAsync(size, 0, (size_t)(nmedge + 1) * sizeof(int32_t), st);
    cudaMemsetAsync(err, 0, sizeof(int), st);
    k_ep_records<<<nblk(nrec), 256, 0, st>>>(medge, edge_vert, nedge, nmedge, nvert, kA, vA, size,
                                             err);
    int herr = 0;
    cudaMemcpyAsync(&herr, err, sizeof(int), cudaMemcpyDeviceToHost, st);
    if (cudaStreamSynchronize(st) != cudaSuccess) return MG_ERR_CUDA;
    if (herr) return MG_ERR_ARG;   // a vertex or macro-edge id out of range
    size_t tb2 = tb;
    cub::DeviceRadixSort::SortPairs(temp, tb2, kA, kB, vA, vB, (int)nrec, 0, 64, st);
    k_ep_partner<<<nblk(nrec), 256, 0, st>>>(kB, vB, nrec, partner);
    k_ep_param<<<nblk(nedge), 256, 0, st>>>(medge, edge_vert, nedge, partner, size, vx, vy, s);
    if (cudaGetLastError() != cudaSuccess) rc = MG_ERR_CUDA;
  }
  if (cudaStreamSynchronize(st) != cudaSuccess) rc = MG_ERR_CUDA;
  return rc;
}

// ---- P^p transfer blocks of the parameterised macro-edges (reading A6) ----
// Fine node a of edge e sits at s = s0 + (s1 - s0) t_a on its macro-edge; the block row
// is the macro-edge's GLL Lagrange basis there, l_j(s) = prod_{m != j} (s - t_m) /
// (t_j - t_m) in increasing m (the injection M_{k-1} -> M_k).
namespace {

struct Gll {
  double t[8];
};

__global__ void k_me_transfer(const double* __restrict__ s, int64_t nedge, int p, Gll g,
                              double* J) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= nedge) return;
  const int k1 = p + 1;
  const double s0 = s[2 * e], s1 = s[2 * e + 1];
  double* Je = J + e * k1 * k1;
  for (int a = 0; a < k1; ++a) {
    const double x = __dadd_rn(s0, __dmul_rn(s1 - s0, g.t[a]));   // as written, no FMA
    for (int j = 0; j < k1; ++j) {
      double v = 1.0;
      for (int m = 0; m < k1; ++m)
        if (m != j) v *= (x - g.t[m]) / (g.t[j] - g.t[m]);
      Je[a * k1 + j] = s0 < 0.0 ? 0.0 : v;
    }
  }
}

}  // namespace

extern "C" int mg_macro_edge_transfer(int64_t nedge, const double* s, int32_t p, double* J,
                                      void* stream) {
  if (nedge <= 0 || p < 1 || p > 7 || !s || !J) return MG_ERR_ARG;
  const std::vector<double> t = mgdtn::gll_nodes01(p);
  Gll g{};
  for (int a = 0; a <= p; ++a) g.t[a] = t[a];
  cudaStream_t st = (cudaStream_t)stream;
  k_me_transfer<<<nblk(nedge, 128), 128, 0, st>>>(s, nedge, p, g, J);
  if (cudaGetLastError() != cudaSuccess) return MG_ERR_CUDA;
  return cudaStreamSynchronize(st) == cudaSuccess ? MG_OK : MG_ERR_CUDA;
}
