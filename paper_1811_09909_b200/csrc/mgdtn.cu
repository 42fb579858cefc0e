// C-ABI implementation (include/mgdtn.h): level structure, workspace carve-up,
// setup sequence, V-cycle (Algorithm 1), PCG driver and the
// CUDA-graph capture of the per-iteration kernel sequences.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "../../include/mgdtn.h"
#include "comm.h"
#include "d4.cuh"
#include "kernels.cuh"
#include "refelem.h"
#include "tail.h"

namespace mgdtn {

enum LevelKind { KIND_COARSEST = 0, KIND_P = 1, KIND_H = 2 };

struct HostLevel {
  LevelDev d{};
  int kind = KIND_COARSEST;
  double h = 0.0;
  size_t o_S = 0, o_Dinv = 0, o_Dc = 0, o_coef = 0, o_lam = 0, o_r = 0, o_e = 0, o_w = 0, o_d = 0;
  size_t o_So = 0, o_Dco = 0, o_Dso = 0;   // orbit storage (R9, d4.cuh)
  size_t o_clist = 0;   // partitioned orbit level: colour-1 chunks, interface ones first
  int* clist = nullptr;
  int nclB = 0, nclI = 0;
  size_t o_KIIinv = 0, o_Pm = 0, o_Rm = 0, o_cbuf = 0, o_lpart = 0;
  double* lpart = nullptr;   // per-level partial sums + 16 scalars (concurrent power iterations)
  double *KIIinv = nullptr, *Pm = nullptr, *cbuf = nullptr;
  double* Rm = nullptr;      // restriction's macro matrix: Pm (symmetric) or -J^T A_BI A_II^-1
                             // transposed (nonsymmetric context, Eq. 3.5)
  double *r = nullptr, *e = nullptr, *w = nullptr, *dv = nullptr, *lam = nullptr;
};

struct Ctx {
  mg_quad_mesh mesh{};
  int p = 1;
  bool ns = false;              // MG_BUILD_NONSYMMETRIC: full S_T storage, LU blocks, Eq. 3.5 restriction
  std::vector<HostLevel> lev;   // lev[0] = finest (paper's level N)
  cudaStream_t st = nullptr;
  RefTables ref;
  size_t ref_doubles = 0;
  // workspace
  char* ws = nullptr;
  size_t ws_bytes = 0, ws_need = 0;
  size_t o_err = 0, o_ref = 0, o_part = 0, o_scal = 0, o_sscal = 0, o_x = 0, o_p = 0, o_ap = 0,
         o_lamD = 0, o_g = 0, o_fpos = 0, o_fidx = 0, o_A1 = 0, o_A1inv = 0, o_K = 0, o_tau = 0,
         o_meth = 0;
  int nf = 0;
  int npart = 0;
  RefDev refdev{};
  DevError* err = nullptr;
  double *part = nullptr, *scal = nullptr, *sscal = nullptr, *x = nullptr, *pv = nullptr,
         *ap = nullptr, *lamD = nullptr, *gbuf = nullptr, *A1 = nullptr, *A1inv = nullptr;
  int *fpos = nullptr, *fidx = nullptr;
  double *Kc = nullptr, *tauc = nullptr;   // internal copies of the element data (rhs)
  int8_t* methc = nullptr;
  // staging for mg_solve_host
  char* stg = nullptr;
  size_t stg_bytes = 0;
  // state
  bool setup_done = false;
  mg_smoother_cfg sm{};
  std::string last_err;
  long long last_idx = -1;
  long long launches = 0, last_solve_launches = 0;
  double* pinned = nullptr;
  cudaGraphExec_t gS = nullptr;   // whole PCG solve: prologue + conditional WHILE loop
  cudaGraphExec_t gV = nullptr;   // one V-cycle, fine L.r -> L.e (GMRES / MG-solver / mg_vcycle)
  cudaGraphExec_t gPA = nullptr, gPBA = nullptr;   // partitioned PCG over NCCL: the first
  long long nPA = 0, nPBA = 0;                      // iteration's A-part, then B + A parts
  long long nV = 0;               // kernels in gV
  const double* vres = nullptr;   // the fine work vector that holds gV's result
  cudaGraphExec_t gU = nullptr;   // the whole setup after the input copies (forked streams as
  long long nU = 0;               // graph branches); captured for the smoother config gU_sm
  mg_smoother_cfg gU_sm{};
  cudaGraphConditionalHandle cond = 0;
  long long nPro = 0, nBody = 0;  // kernels in the prologue / in one loop iteration
  bool use_graphs = true;
  long long gather_ne = 1LL << 16;   // MG_OPT_GATHER_NE
  int tail_start = -1;            // first level run by k_coarse_tail (-1: none)
  bool tail_vcycle = true;        // V-cycle levels >= tail_start through k_coarse_tail
  bool tail_lmax = true;          // their Chebyshev power iterations through k_tail_lmax
  bool tail_dense = false;        // B_tail as an explicit matrix (k_tail_basis / k_tail_dense)
  bool keep_fine_maps = false;    // MG_OPT_KEEP_FINE_MAPS: setup keeps the finest level's maps
  int nft = 0;                    // free dofs of the top tail level
  size_t o_Bt = 0, o_tfidx = 0;
  double* Bt = nullptr;
  int* tfidx = nullptr;
  TailParams tail{};
  size_t o_ist = 0, o_hist = 0;
  int* ist = nullptr;             // device PCG state (k_pcg_check)
  double* dhist = nullptr;        // device residual history [HIST_CAP]
  // ---- element-block partition over ranks; nranks == 1: single GPU
  Comm* comm = nullptr;
  int rank = 0, nranks = 1, px = 1, py = 1, rx = 0, ry = 0;
  int nbr[4] = {-1, -1, -1, -1};   // neighbour rank across local side f (bottom, right, top, left)
  int Lg = -1;                     // first replicated level (every rank holds it whole); the
                                   // levels above it hold this rank's element block only
  HostLevel lgl;                   // this rank's block of level Lg (restriction / prolongation)
  size_t o_hs = 0, o_hr = 0, o_gall = 0, o_sden = 0, o_sall = 0, halo_doubles = 0;
  int comm_rc = 0;                 // first communicator failure (reported by the next sync point)
  double comm_timeout_s = 300.0;   // host waits on a partitioned context give up after this
                                   // (mg_set_option MG_OPT_COMM_TIMEOUT_MS); NCCL is aborted
  // setup: the levels' Chebyshev power iterations are independent and run on their
  // own streams (fork / join with events on the ctx stream)
  cudaStream_t cst = nullptr;      // partitioned: halo exchange overlapped with interior work
  cudaEvent_t evB = nullptr, evC = nullptr;
  std::vector<cudaStream_t> side;
  std::vector<cudaEvent_t> side_ev, fork_evs;
  // mg_solve_host: the source-term / boundary-data uploads run on their own stream,
  // overlapped with mg_setup_dtn (which does not read them)
  cudaStream_t copy_st = nullptr;
  bool pu_pending = false;          // pcg_iter_B left p = z + beta p to the next apply (AM_W0U)
  const double* zp = nullptr;       // its z
  cudaEvent_t copy_ev0 = nullptr, copy_ev1 = nullptr;
  double *hsend = nullptr, *hrecv = nullptr, *gall = nullptr, *sden = nullptr, *sall = nullptr;
};

static bool partitioned(const Ctx* c) { return c->nranks > 1; }

// NVTX ranges (nsys / ncu --nvtx): the setup, every level of a V-cycle (its smoothing,
// residual and transfers) and every PCG iteration of the host-driven loops.  Host-side
// markers: inside a captured graph they mark the capture, and the replays run unmarked.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};
struct LevelNames {
  char buf[64][24];
  LevelNames() {
    for (int k = 0; k < 64; ++k) std::snprintf(buf[k], sizeof(buf[k]), "mg/vcycle/li%d", k);
  }
};
static const char* level_range_name(int li) {
  static const LevelNames names;   // thread-safe initialisation (virtual ranks are threads)
  return names.buf[li < 0 ? 0 : li > 63 ? 63 : li];
}

static int fail(Ctx* c, int code, const std::string& msg, long long idx = -1) {
  if (c) {
    c->last_err = msg;
    c->last_idx = idx;
  }
  return code;
}

static int cuda_check(Ctx* c, cudaError_t e, const char* where) {
  if (e == cudaSuccess) return MG_OK;
  return fail(c, MG_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

#define CK(expr)                                   \
  do {                                             \
    int _rc = cuda_check(c, (expr), #expr);        \
    if (_rc != MG_OK) return _rc;                  \
  } while (0)

#define RC(expr)                                   \
  do {                                             \
    int _rc = (expr);                              \
    if (_rc != MG_OK) return _rc;                  \
  } while (0)

static size_t align_up(size_t x) { return (x + 255) & ~(size_t)255; }

// host wait for a stream: on a partitioned context through the communicator, which polls
// NCCL's asynchronous errors and gives up after comm_timeout_s (a lost peer never hangs
// the caller); plain cudaStreamSynchronize otherwise
static int sync_st(Ctx* c, cudaStream_t st) {
  if (c->comm && c->nranks > 1) {
    if (c->comm->wait(st, c->comm_timeout_s) != 0) {
      if (c->comm_rc == 0) c->comm_rc = MG_ERR_NCCL;
      return fail(c, MG_ERR_NCCL, "communicator: " + c->comm->err);
    }
    return MG_OK;
  }
  return cuda_check(c, cudaStreamSynchronize(st), "cudaStreamSynchronize");
}

constexpr int HIST_CAP = 16384;   // device residual history; larger maxit -> host loop

// ---------------------------------------------------------------- hierarchy
static int env_or(const char* name, int dflt) {
  const char* e = std::getenv(name);
  return e ? std::atoi(e) : dflt;
}

static void init_level(HostLevel& L, int nx, int ny, int p, double h, int kind) {
  LevelDev& d = L.d;
  d.nx = nx;
  d.ny = ny;
  d.p = p;
  d.k1 = p + 1;
  d.m = 4 * (p + 1);
  d.npk = d.m * (d.m + 1) / 2;
  d.ne = (int64_t)nx * ny;
  d.nedge = (int64_t)nx * (ny + 1) + (int64_t)(nx + 1) * ny;
  d.ndof = d.nedge * d.k1;
  d.nchunk = (int)((d.ne / 2 + 31) / 32);
  d.dmask = 15;
  d.imask = 0;
  d.ox = 0;
  d.oy = 0;
  d.gnx = nx;
  d.gny = ny;
  d.orb = 0;
  d.So = d.Dco = d.Dso = nullptr;
  d.sweep = 0;
  d.gather = 0;
  d.grid_cap = 0;
  d.ndi = 4 * d.k1 * (d.k1 + 1) / 2;
  L.h = h;
  L.kind = kind;
}

static void layout(Ctx* c) {
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off = align_up(off + (bytes ? bytes : 8));
    return o;
  };
  c->o_err = take(sizeof(DevError));
  c->o_ref = take(c->ref_doubles * sizeof(double));
  c->npart = 4 * 148 * 16 + 64;   // >= any apply / vector grid (at most 16 CTAs per SM)
  c->o_part = take((size_t)c->npart * sizeof(double));
  c->o_scal = take(16 * sizeof(double));
  c->o_sscal = take(16 * sizeof(double));
  c->o_ist = take(4 * sizeof(int));
  c->o_hist = take(HIST_CAP * sizeof(double));
  const int64_t ndofN = c->lev[0].d.ndof;
  c->o_x = take(ndofN * sizeof(double));
  c->o_p = take(ndofN * sizeof(double));
  c->o_ap = take(ndofN * sizeof(double));
  c->o_lamD = take(ndofN * sizeof(double));
  c->o_g = take(ndofN * sizeof(double));
  c->o_K = take(c->lev[0].d.ne * sizeof(double));
  c->o_tau = take(c->lev[0].d.ne * sizeof(double));
  c->o_meth = take(c->lev[0].d.ne * sizeof(int8_t));
  for (auto& L : c->lev) {
    const LevelDev& d = L.d;
    L.o_S = take((size_t)2 * d.nchunk * d.npk * 32 * sizeof(double));
    L.o_Dinv = take((size_t)d.nedge * d.k1 * d.k1 * sizeof(double));
    if (d.orb && d.imask) L.o_clist = take((size_t)d.nchunk * sizeof(int));
    if (d.orb) {   // orbit records replace the packed colour-1 D_e^-1 stream
      L.o_So = take((size_t)2 * d.nchunk * d4_norb(d.p) * 32 * sizeof(double));
      L.o_Dco = take((size_t)d.nchunk * 4 * d4_ncs(d.p) * 32 * sizeof(double));
      L.o_Dso = take((size_t)d.nedge * d4_ncs(d.p) * sizeof(double));
    } else {
      L.o_Dc = take((size_t)d.nchunk * d.ndi * 32 * sizeof(double));
    }
    L.o_coef = take(2 * MAX_NU * sizeof(double));
    L.o_lpart = take((size_t)(c->npart + 16) * sizeof(double));
    L.o_lam = take(sizeof(double));
    L.o_r = take(d.ndof * sizeof(double));
    L.o_e = take(d.ndof * sizeof(double));
    L.o_w = take(d.ndof * sizeof(double));
    L.o_d = take(d.ndof * sizeof(double));
    if (L.kind == KIND_H) {
      int64_t nmac = (int64_t)(d.nx / 2) * (d.ny / 2);
      // A_II^-1: packed upper triangle (36) in symmetric contexts, full 8 x 8 otherwise
      L.o_KIIinv = take(nmac * (c->ns ? 64 : 36) * sizeof(double));
      L.o_Pm = take(nmac * 64 * sizeof(double));
      if (c->ns) L.o_Rm = take(nmac * 64 * sizeof(double));
      L.o_cbuf = take(nmac * 8 * sizeof(double));
    }
  }
  const HostLevel& C1 = c->lev.back();
  c->o_fpos = take(C1.d.ndof * sizeof(int));
  c->o_fidx = take((size_t)c->nf * sizeof(int));
  c->o_A1 = take((size_t)c->nf * c->nf * sizeof(double));
  c->o_A1inv = take((size_t)c->nf * c->nf * sizeof(double));
  if (c->tail_dense) {
    c->o_Bt = take((size_t)c->nft * c->nft * sizeof(double));
    c->o_tfidx = take((size_t)c->nft * sizeof(int));
  }
  if (partitioned(c)) {
    HostLevel& G = c->lgl;
    const LevelDev& d = G.d;
    G.o_r = take(d.ndof * sizeof(double));
    G.o_e = take(d.ndof * sizeof(double));
    size_t hd = 0;
    for (int li = 0; li < c->Lg; ++li) {
      const LevelDev& l = c->lev[li].d;
      hd = std::max(hd, (size_t)4 * std::max(l.nx, l.ny) * l.k1 * l.k1);
    }
    hd = std::max(hd, (size_t)4 * std::max(d.nx, d.ny) * d.k1 * d.k1);
    c->halo_doubles = hd;
    c->o_hs = take(hd * sizeof(double));
    c->o_hr = take(hd * sizeof(double));
    c->o_gall = take((size_t)c->nranks * d.ndof * sizeof(double));
    c->o_sden = take((size_t)d.ne * 64 * sizeof(double));
    c->o_sall = take((size_t)c->nranks * d.ne * 64 * sizeof(double));
  }
  c->ws_need = off;
}

static void bind_pointers(Ctx* c) {
  char* b = c->ws;
  auto D = [&](size_t o) { return reinterpret_cast<double*>(b + o); };
  c->err = reinterpret_cast<DevError*>(b + c->o_err);
  c->part = D(c->o_part);
  c->scal = D(c->o_scal);
  c->sscal = D(c->o_sscal);
  c->ist = reinterpret_cast<int*>(b + c->o_ist);
  c->dhist = D(c->o_hist);
  c->x = D(c->o_x);
  c->pv = D(c->o_p);
  c->ap = D(c->o_ap);
  c->lamD = D(c->o_lamD);
  c->gbuf = D(c->o_g);
  c->fpos = reinterpret_cast<int*>(b + c->o_fpos);
  c->fidx = reinterpret_cast<int*>(b + c->o_fidx);
  c->A1 = D(c->o_A1);
  c->A1inv = D(c->o_A1inv);
  if (c->tail_dense) {
    c->Bt = D(c->o_Bt);
    c->tfidx = reinterpret_cast<int*>(b + c->o_tfidx);
  }
  if (partitioned(c)) {
    HostLevel& G = c->lgl;   // vectors only (its coarse maps go straight to sden)
    G.r = D(G.o_r);
    G.e = D(G.o_e);
    c->hsend = D(c->o_hs);
    c->hrecv = D(c->o_hr);
    c->gall = D(c->o_gall);
    c->sden = D(c->o_sden);
    c->sall = D(c->o_sall);
  }
  c->Kc = D(c->o_K);
  c->tauc = D(c->o_tau);
  c->methc = reinterpret_cast<int8_t*>(b + c->o_meth);
  for (auto& L : c->lev) {
    L.d.S = D(L.o_S);
    L.d.Dinv = D(L.o_Dinv);
    // packed-symmetric D_e^-1 (symmetric packed levels) or the orbit records
    L.d.Dc = (c->ns || L.d.orb) ? nullptr : D(L.o_Dc);
    if (L.d.orb && L.d.imask) L.clist = reinterpret_cast<int*>(b + L.o_clist);
    if (L.d.orb) {
      L.d.So = D(L.o_So);
      L.d.Dco = D(L.o_Dco);
      L.d.Dso = D(L.o_Dso);
    }
    L.d.coef = D(L.o_coef);
    L.lpart = D(L.o_lpart);
    L.lam = D(L.o_lam);
    L.r = D(L.o_r);
    L.e = D(L.o_e);
    L.w = D(L.o_w);
    L.dv = D(L.o_d);
    if (L.kind == KIND_H) {
      L.KIIinv = D(L.o_KIIinv);
      L.Pm = D(L.o_Pm);
      L.Rm = c->ns ? D(L.o_Rm) : L.Pm;
      L.cbuf = D(L.o_cbuf);
    }
  }
  // reference tables
  double* R = D(c->o_ref);
  const RefTables& T = c->ref;
  size_t o = 0;
  auto put = [&](const std::vector<double>& v) {
    const double* p = R + o;
    o += v.size();
    return p;
  };
  RefDev& rd = c->refdev;
  rd.p = T.p;
  rd.k1 = T.k1;
  rd.nv = T.nv;
  rd.m = T.m;
  rd.nqf = T.nqf;
  rd.G = put(T.G);
  rd.F = put(T.F);
  rd.P = put(T.P);
  rd.E = put(T.E);
  rd.W = put(T.W);
  rd.H = put(T.H);
  rd.LN = put(T.LN);
  rd.Nl = put(T.Nl);
  rd.fq = put(T.fq);
  rd.ew = put(T.ew);
  rd.H1inv = put(T.H1inv);
  rd.Jp = put(T.Jp);
  for (int k = 0; k < 2; ++k) {
    rd.plam[k] = put(T.pen[k].lam);
    rd.pmu[k] = put(T.pen[k].mu);
    rd.pAt[k] = put(T.pen[k].At);
    rd.pBk[k] = put(T.pen[k].Bk);
    rd.pfq[k] = put(T.pen[k].fqT);
    rd.pTt[k] = put(T.pen[k].Tt);
  }
  rd.vq = put(T.vq);
  rd.wq = put(T.wq);
  rd.Lv = put(T.L);
  rd.Nv = put(T.N);
}

// Levels from tail_start down run as ONE launch of k_coarse_tail (k_coarse.cu):
// p = 1 levels with at most MGDTN_TAIL_NE elements (default 256 = 16 x 16; 0 =
// off), one CTA whose level data stay in L1 (profiles/r01_ab_tail.txt: a
// single CTA over <= 16x16 levels beats the per-step launches; multi-CTA
// clusters and larger tails lose to them).  MGDTN_TAIL_VCYCLE=0 /
// MGDTN_TAIL_LMAX=0 keep the V-cycle / the Chebyshev power iteration on launches.

// gather-form apply (k_apply_gather) on the packed P1 levels with at most gather_ne
// elements (MG_OPT_GATHER_NE), one-GPU or replicated
static void plan_gather(Ctx* c) {
  for (auto& L : c->lev) {
    LevelDev& d = L.d;
    d.gather = (!c->ns && !d.orb && d.p == 1 && d.imask == 0 && d.dmask == 15 &&
                d.ne <= c->gather_ne) ? 1 : 0;
  }
}

static void plan_tail(Ctx* c) {
  const char* env = std::getenv("MGDTN_TAIL_NE");
  const long long tail_ne = env ? std::atoll(env) : 256;
  c->tail_vcycle = env_or("MGDTN_TAIL_VCYCLE", 1) == 1;
  c->tail_lmax = env_or("MGDTN_TAIL_LMAX", 1) == 1;
  const int nlev = (int)c->lev.size();
  c->tail_start = -1;
  if (tail_ne <= 0 || c->ns) return;   // the tail kernels read packed-symmetric maps
  for (int li = c->Lg > 0 ? c->Lg : 0; li < nlev; ++li) {   // replicated levels only
    const LevelDev& d = c->lev[li].d;
    if (d.p == 1 && d.ne <= tail_ne && nlev - li >= 2 && nlev - li <= MAX_TAIL &&
        (li == 0 || c->lev[li - 1].kind == KIND_H || c->lev[li - 1].kind == KIND_P)) {
      bool all_h = true;
      for (int k = li; k < nlev - 1; ++k) all_h = all_h && c->lev[k].kind == KIND_H;
      if (all_h) {
        c->tail_start = li;
        break;
      }
    }
  }
}

// B_tail explicit (MGDTN_TAIL_DENSE, default on): the whole tail V-cycle is a
// fixed linear operator on the top tail level's free dofs; it is tabulated once
// per setup (one tail V-cycle per unit vector, all columns in one launch) and
// applied as one dense matvec per V-cycle.
static void plan_tail_dense(Ctx* c) {
  c->tail_dense = false;
  c->nft = 0;
  if (c->tail_start < 0 || !c->tail_vcycle || env_or("MGDTN_TAIL_DENSE", 1) == 0) return;
  const LevelDev& d = c->lev[c->tail_start].d;
  const int64_t nf = ((int64_t)d.nx * (d.ny - 1) + (int64_t)(d.nx - 1) * d.ny) * d.k1;
  if (nf <= 0 || nf > 2048) return;
  c->nft = (int)nf;
  c->tail_dense = true;
}

static void fill_tail(Ctx* c) {
  if (c->tail_start < 0) return;
  TailParams& T = c->tail;
  const int nlev = (int)c->lev.size();
  T.nlev = nlev - c->tail_start;
  // shared-memory copies of the tail vectors (k_coarse.cu), if they fit (MGDTN_TAIL_SMEM=0: off)
  int64_t nd = 0;
  for (int k = c->tail_start; k < nlev; ++k) {
    const LevelDev& d = c->lev[k].d;
    nd += 4 * d.ndof + (k < nlev - 1 ? (int64_t)(d.nx / 2) * (d.ny / 2) * 8 : 0);
  }
  T.smem_doubles = (env_or("MGDTN_TAIL_SMEM", 1) != 0 && nd * 8 <= 200 * 1024) ? (int)nd : 0;
  if (T.smem_doubles == 0) c->tail_dense = false;   // the basis kernel needs shared-memory vectors
  T.fidx = c->fidx;
  T.nf = c->nf;
  T.A1inv = c->A1inv;
  for (int k = 0; k < T.nlev; ++k) {
    const HostLevel& L = c->lev[c->tail_start + k];
    TailLevel& t = T.lev[k];
    t.d = L.d;
    t.r = L.r;
    t.e = L.e;
    t.w = L.w;
    t.dv = L.dv;
    t.KIIinv = L.KIIinv;
    t.Pm = L.Pm;
    t.cbuf = L.cbuf;
    t.lam = L.lam;
  }
}

static int upload_static(Ctx* c) {
  // reference tables
  std::vector<double> all;
  const RefTables& T = c->ref;
  for (const auto* v : {&T.G, &T.F, &T.P, &T.E, &T.W, &T.H, &T.LN, &T.Nl, &T.fq, &T.ew, &T.H1inv,
                        &T.Jp})
    all.insert(all.end(), v->begin(), v->end());
  for (int k = 0; k < 2; ++k)
    for (const auto* v : {&T.pen[k].lam, &T.pen[k].mu, &T.pen[k].At, &T.pen[k].Bk, &T.pen[k].fqT,
                          &T.pen[k].Tt})
      all.insert(all.end(), v->begin(), v->end());
  all.insert(all.end(), T.vq.begin(), T.vq.end());
  all.insert(all.end(), T.wq.begin(), T.wq.end());
  all.insert(all.end(), T.L.begin(), T.L.end());
  all.insert(all.end(), T.N.begin(), T.N.end());
  CK(cudaMemcpyAsync(c->ws + c->o_ref, all.data(), all.size() * sizeof(double),
                     cudaMemcpyHostToDevice, c->st));
  // coarsest free-dof maps
  const LevelDev& d = c->lev.back().d;
  std::vector<int> fpos(d.ndof, -1), fidx;
  for (int64_t e = 0; e < d.nedge; ++e) {
    if (edge_on_boundary(d.nx, d.ny, e)) continue;
    for (int a = 0; a < d.k1; ++a) {
      fpos[e * d.k1 + a] = (int)fidx.size();
      fidx.push_back((int)(e * d.k1 + a));
    }
  }
  CK(cudaMemcpyAsync(c->fpos, fpos.data(), fpos.size() * sizeof(int), cudaMemcpyHostToDevice,
                     c->st));
  if (!fidx.empty())
    CK(cudaMemcpyAsync(c->fidx, fidx.data(), fidx.size() * sizeof(int), cudaMemcpyHostToDevice,
                       c->st));
  for (auto& L : c->lev) {   // split colour-1 pass of the partitioned orbit levels
    if (!L.clist) continue;
    const LevelDev& d = L.d;
    const int64_t nec = d.ne / 2;
    std::vector<int> bl, il;
    for (int q = 0; q < d.nchunk; ++q) {
      bool itf = false;
      for (int64_t sl = (int64_t)q * 32; sl < (int64_t)q * 32 + 32 && sl < nec && !itf; ++sl) {
        int i, j;
        slot_elem(d.nx, 1, sl, i, j);
        itf = elem_itf(d.nx, d.ny, i, j, d.imask) != 0;
      }
      (itf ? bl : il).push_back(q);
    }
    L.nclB = (int)bl.size();
    L.nclI = (int)il.size();
    bl.insert(bl.end(), il.begin(), il.end());
    CK(cudaMemcpyAsync(L.clist, bl.data(), bl.size() * sizeof(int), cudaMemcpyHostToDevice, c->st));
  }
  if (c->tail_dense) {
    const LevelDev& t = c->lev[c->tail_start].d;
    std::vector<int> tf;
    for (int64_t e = 0; e < t.nedge; ++e) {
      if (edge_on_boundary(t.nx, t.ny, e)) continue;
      for (int a = 0; a < t.k1; ++a) tf.push_back((int)(e * t.k1 + a));
    }
    CK(cudaMemcpyAsync(c->tfidx, tf.data(), tf.size() * sizeof(int), cudaMemcpyHostToDevice,
                       c->st));
  }
  RC(sync_st(c, c->st));
  return MG_OK;
}

static void drop_graphs(Ctx* c) {
  if (c->gS) cudaGraphExecDestroy(c->gS);
  c->gS = nullptr;
  if (c->gPA) cudaGraphExecDestroy(c->gPA);
  c->gPA = nullptr;
  if (c->gPBA) cudaGraphExecDestroy(c->gPBA);
  c->gPBA = nullptr;
  if (c->gV) cudaGraphExecDestroy(c->gV);
  c->gV = nullptr;
  if (c->gU) cudaGraphExecDestroy(c->gU);
  c->gU = nullptr;
}

static int check_device_error(Ctx* c) {
  DevError h{};
  CK(cudaMemcpyAsync(&h, c->err, sizeof(DevError), cudaMemcpyDeviceToHost, c->st));
  RC(sync_st(c, c->st));
  if (c->comm_rc) return c->comm_rc;
  if (h.code == 0) return MG_OK;
  CK(cudaMemsetAsync(c->err, 0, sizeof(DevError), c->st));
  switch (h.code) {
    case -4:
      return fail(c, MG_ERR_NOT_SPD,
                  "Cholesky failed (local block, edge block, macro A_II or A_1); index "
                  "(element / edge / macro; -2 = coarsest) reported",
                  h.index);
    case -1:
      return fail(c, MG_ERR_ARG,
                  c->ns ? "invalid K / tau / method at element"
                        : "invalid K / tau / method at element (IIPG-H / NIPG-H need a "
                          "MG_BUILD_NONSYMMETRIC context)",
                  h.index);
    case -3:
      return fail(c, MG_ERR_SINGULAR_LOCAL,
                  "LU pivot vanished (local block, edge block, macro A_II or A_1); index "
                  "(element / edge / macro; -2 = coarsest) reported",
                  h.index);
    default:
      return fail(c, MG_ERR_SINGULAR_LOCAL, "device error", h.index);
  }
}

// ---------------------------------------------------------------- communication (partitioned levels)
static void comm_fail(Ctx* c, int rc) {
  if (rc != 0 && c->comm_rc == 0) {
    c->comm_rc = MG_ERR_NCCL;
    c->last_err = "communicator: " + (c->comm ? c->comm->err : std::string("none"));
  }
}

// exchange c->hsend -> c->hrecv with the neighbours across the interface sides of
// level d: `per` doubles per interface edge, side stride `stride` doubles
static void halo_exchange(Ctx* c, const LevelDev& d, int stride, int per,
                          cudaStream_t st = nullptr) {
  int cnt[4];
  for (int f = 0; f < 4; ++f) cnt[f] = ((d.imask >> f) & 1) ? side_len(d.nx, d.ny, f) * per : 0;
  comm_fail(c, c->comm->halo(c->nbr, c->hsend, c->hrecv, stride, cnt, st ? st : c->st));
}

// scal[slot] = sum of partials over every rank (then the k_reduce op)
static void reduce_scal(Ctx* c, const double* partials, int n, double* scal, int slot, int op) {
  if (!partitioned(c)) {
    c->launches += launch_reduce(partials, n, scal, slot, op, nullptr, c->st);
    return;
  }
  constexpr int TMP = 14;
  c->launches += launch_reduce(partials, n, scal, TMP, 0, nullptr, c->st);
  comm_fail(c, c->comm->allreduce_sum(scal + TMP, 1, c->st));
  c->launches += launch_scalar_op(scal, TMP, slot, op, c->st);
}

// ---------------------------------------------------------------- apply / smoothing building blocks
// one apply in `mode` (bodies.cuh epilogues); on a partitioned level the colour
// passes leave partial sums on the interface edges, which are exchanged and
// finished by k_itf_epilogue (k_part.cu)
// MG_OPT_SWEEP = 1 runs the smoothing step of a one-GPU orbit level as one streamed
// pass (k_tile.cu): it reads x, r, d once instead of the two-colour pair's x twice and
// y three times, but measured slower than the pair (profiles/r02_sweep_probe.txt), so
// it is off by default.
static bool tiled(const LevelDev& d, int mode) { return tile_level(d) && mode == AM_SMOOTH; }
// small P1 levels: one gather-form pass per apply / residual / smoothing step
// (k_apply_gather) instead of the pair of colour passes
static bool gathered(const LevelDev& d, int mode) {
  return gather_level(d) && (mode == AM_APPLY || mode == AM_RESID || mode == AM_SMOOTH);
}
static void apply_mode(Ctx* c, const HostLevel& L, int mode, const double* x, double* y,
                       const double* r, double* d, int step, double* partials) {
  if (tiled(L.d, mode) && mode != AM_SMOOTH) {
    c->launches += launch_apply_tile(L.d, mode, x, y, r, d, nullptr, step, partials, c->st);
    return;
  }
  if (gathered(L.d, mode) && !partials && mode != AM_SMOOTH) {
    c->launches += launch_apply_gather(L.d, mode, x, y, r, d, nullptr, step, c->st);
    return;
  }
  if (L.clist && c->cst) {
    // partitioned orbit level ("boundary elements first, start NCCL, then
    // interior"): colour 0 everywhere, then the colour-1 chunks that touch a partition
    // interface; their partial sums go out (pack, halo, interface epilogue) on the
    // communication stream while the other colour-1 chunks -- which touch no interface
    // edge -- run on the main stream
    LevelDev dB = L.d, dI = L.d;
    dB.clist = L.clist;
    dB.ncl = L.nclB;
    dI.clist = L.clist + L.nclB;
    dI.ncl = L.nclI;
    const int gB = L.nclB ? apply_grid_mode(dB, mode) : 0;
    const int gI = L.nclI ? apply_grid_mode(dI, mode) : 0;
    c->launches += launch_apply(L.d, 0, AM_W0, x, y, nullptr, nullptr, 0, nullptr, true, c->st);
    if (L.nclB) c->launches += launch_apply(dB, 1, mode, x, y, r, d, step, partials, true, c->st);
    cudaEventRecord(c->evB, c->st);
    cudaStreamWaitEvent(c->cst, c->evB, 0);
    c->launches += launch_itf_pack(L.d, y, c->hsend, c->cst);
    halo_exchange(c, L.d, itf_stride(L.d), L.d.k1, c->cst);
    c->launches += launch_itf_epilogue(L.d, mode, const_cast<double*>(x), y, r, d, step, c->hrecv,
                                       partials ? partials + gB + gI : nullptr, c->cst);
    cudaEventRecord(c->evC, c->cst);
    if (L.nclI)
      c->launches += launch_apply(dI, 1, mode, x, y, r, d, step, partials ? partials + gB : nullptr,
                                  true, c->st);
    cudaStreamWaitEvent(c->st, c->evC, 0);
    return;
  }
  c->launches += launch_apply2(L.d, mode, x, y, r, d, step, partials, true, c->st);
  if (L.d.imask) {
    c->launches += launch_itf_pack(L.d, y, c->hsend, c->st);
    halo_exchange(c, L.d, itf_stride(L.d), L.d.k1);
    c->launches += launch_itf_epilogue(L.d, mode, const_cast<double*>(x), y, r, d, step, c->hrecv,
                                       partials ? partials + apply2_grid(L.d, mode) : nullptr,
                                       c->st);
  }
}
// number of dot-product partials apply_mode writes
static int apply_parts(const HostLevel& L, int mode) {
  const LevelDev& d = L.d;
  if (tiled(d, mode)) return apply_tile_grid(d);
  if (L.clist) {   // split colour-1 pass (apply_mode)
    LevelDev dB = d, dI = d;
    dB.clist = L.clist;
    dB.ncl = L.nclB;
    dI.clist = L.clist + L.nclB;
    dI.ncl = L.nclI;
    return (L.nclB ? apply_grid_mode(dB, mode) : 0) + (L.nclI ? apply_grid_mode(dI, mode) : 0) +
           itf_blocks();
  }
  return apply2_grid(d, mode) + (d.imask ? itf_blocks() : 0);
}

static inline void apply_full(Ctx* c, const HostLevel& L, const double* x, double* y,
                              double* partials) {
  apply_mode(c, L, AM_APPLY, x, y, nullptr, nullptr, 0, partials);
}

// The level's iterate lives in one of its two work vectors L.e / L.w: the tiled
// smoothing pass writes its result out of place (a neighbouring tile may still read
// the old iterate on the shared edges), so the iterate alternates between them; the
// two-colour passes update it in place (and use the other vector as scratch).
static inline double* other(const HostLevel& L, const double* cur) { return cur == L.e ? L.w : L.e; }

// Chebyshev step 1 after a first step from e = 0 reads its direction d_0 from the iterate
// x_1 (equal bit for bit; STEP_D_FROM_X), so the first step need not store d: one-GPU
// orbit levels run by the launch-per-step V-cycle through the pair of colour passes.
// Config 5: one fewer vector write (first step) and read (step 1) on the two 4096^2 levels.
static bool dfx_ok(const Ctx* c, int li) {
  const HostLevel& L = c->lev[li];
  return c->sm.kind == MG_SMOOTH_CHEBYSHEV && L.d.orb && !L.d.imask && !L.clist && !partitioned(c) &&
         !tiled(L.d, AM_SMOOTH) && !gathered(L.d, AM_SMOOTH) &&
         (c->tail_start < 0 || li < c->tail_start) && env_or("MGDTN_DFX", 1) != 0;
}

// one smoothing step on the iterate `cur`; returns where the new iterate is
static inline double* smooth_step(Ctx* c, HostLevel& L, int step, double* cur, bool dfx = false,
                                  bool nod = false, double* zpart = nullptr) {
  if (c->sm.kind == MG_SMOOTH_LUSGS) {
    // one LU-SGS step: forward block Gauss-Seidel sweep over the
    // four edge colours, then backward (oracle/multigrid.py)
    static const int order[8] = {0, 1, 2, 3, 3, 2, 1, 0};
    for (int q = 0; q < 8; ++q)
      apply_mode(c, L, AM_GSC, cur, other(L, cur), L.r, nullptr, order[q], nullptr);
    return cur;
  }
  // coefficient slot clamped to MAX_NU-1: only block-Jacobi (step-invariant
  // coefficients) may run more steps than that (beta-doubling)
  const int slot = step < MAX_NU ? step : MAX_NU - 1;
  if (tiled(L.d, AM_SMOOTH)) {
    double* out = other(L, cur);
    c->launches += launch_apply_tile(L.d, AM_SMOOTH, cur, nullptr, L.r, L.dv, out, slot, nullptr,
                                     c->st);
    return out;
  }
  if (gathered(L.d, AM_SMOOTH)) {
    double* out = other(L, cur);
    c->launches += launch_apply_gather(L.d, AM_SMOOTH, cur, nullptr, L.r, L.dv, out, slot, c->st);
    return out;
  }
  apply_mode(c, L, AM_SMOOTH, cur, other(L, cur), L.r, L.dv,
             slot | (dfx ? STEP_D_FROM_X : 0) | (nod ? STEP_NO_D_STORE : 0), zpart);
  return cur;
}

// smoothing steps on level li: V(nu, nu), times 2 per coarser level with the
// paper's beta = 2 schedule
static inline int nu_at(const Ctx* c, int nu, int li) { return c->sm.nu_doubling ? nu << li : nu; }

// res = L.r - A cur into the other work vector; returns it
static inline double* residual(Ctx* c, HostLevel& L, const double* cur) {
  double* res = other(L, cur);
  apply_mode(c, L, AM_RESID, cur, res, L.r, nullptr, 0, nullptr);
  return res;
}

// is level li+1 the gather level (li the last partitioned level)?
static inline bool gathers(const Ctx* c, int li) { return partitioned(c) && li + 1 == c->Lg; }

// rc = Q_{k-1} res from level li into level li+1 (Eqs. 3.5 / 3.6); with do_lc,
// also step 3 (e_I += A_II^-1 res_I, Eq. 3.11) on level li.  At the gather level
// the result goes into this rank's block (lgl), then every rank's block is
// all-gathered into the replicated level Lg.
static void restrict_level(Ctx* c, int li, const double* res, double* e, bool do_lc, double* rc,
                           bool fuse) {
  HostLevel& L = c->lev[li];
  const bool gat = gathers(c, li);
  HostLevel& C = gat ? c->lgl : c->lev[li + 1];
  double* rcl = gat ? c->lgl.r : rc;
  if (gat) fuse = false;
  if (L.kind == KIND_H) {
    c->launches += launch_lc_restrict(L.d, res, e, L.KIIinv, L.Rm, L.cbuf, do_lc, true, c->st);
    c->launches += launch_restrict_edges(L.d, C.d, res, L.cbuf, rcl, fuse, C.e, C.dv, c->st);
    if (C.d.imask) {
      c->launches += launch_restrict_halo_pack(C.d, L.cbuf, c->hsend, c->st);
      halo_exchange(c, C.d, itf_stride(C.d), 2);
      c->launches += launch_restrict_halo_finish(C.d, rcl, c->hsend, c->hrecv, fuse, C.e, C.dv,
                                                 c->st);
    }
  } else {
    c->launches += launch_p_restrict(L.d, C.d, c->refdev.Jp, res, rcl, fuse, C.e, C.dv, c->st);
  }
  if (gat) {
    const LevelDev& B = c->lgl.d;
    comm_fail(c, c->comm->allgather(c->lgl.r, c->gall, (size_t)B.ndof, c->st));
    c->launches += launch_gather_vec(c->lev[c->Lg].d, B.nx, B.ny, c->px, c->py, B.ndof, c->gall,
                                     rc, c->st);
  }
}

// e += I_k ec (Eqs. 3.3 / 3.4) from level li+1 into level li
static void prolong_level(Ctx* c, int li, const double* ec, double* e) {
  HostLevel& L = c->lev[li];
  const bool gat = gathers(c, li);
  HostLevel& C = gat ? c->lgl : c->lev[li + 1];
  const double* ecl = ec;
  if (gat) {   // this rank's block of the replicated coarse correction
    const LevelDev& G = c->lev[c->Lg].d;
    c->launches += launch_scatter_vec(C.d, C.d.ox, C.d.oy, G.nx, G.ny, ec, c->lgl.e, c->st);
    ecl = c->lgl.e;
  }
  if (L.kind == KIND_H) {
    c->launches += launch_prolong_macro(L.d, C.d, ecl, L.Pm, e, c->st);   // (interface edges included)
  } else {
    c->launches += launch_p_prolong(L.d, c->refdev.Jp, ecl, e, c->st);
  }
}

// V-cycle B_k (Algorithm 1) on level li with input L.r; returns the vector holding
// the result (L.e or L.w, see smooth_step).
// `first_done`: the first pre-smoothing step (from e = 0) was fused into the
// restriction kernel of the finer level.  Step 3 (local correction) and the
// restriction share one residual: Q_{k-1} A_k T_k = 0, so Q(r - A e2) equals
// Q(r - A e1).
// `zpart` (fine level, pcg_zdot): the last post-smoothing step also leaves the partial sums
// of r . z (z = its new iterate) in zpart
static double* vcycle_level(Ctx* c, int li, bool first_done, double* zpart = nullptr) {
  NvtxRange nv(level_range_name(li));
  HostLevel& L = c->lev[li];
  const int nlev = (int)c->lev.size();
  const bool tail_ok = c->sm.kind != MG_SMOOTH_LUSGS;   // the tail kernels have no LU-SGS
  if (tail_ok && c->tail_dense && li == c->tail_start) {   // this level and every coarser one: e = B_tail r
    c->launches += launch_tail_dense(c->tfidx, c->nft, c->Bt, L.r, L.e, c->st);
    return L.e;
  }
  if (tail_ok && c->tail_vcycle && li == c->tail_start) {   // this level and every coarser one: one launch
    TailParams& T = c->tail;
    T.nu_pre = nu_at(c, c->sm.nu_pre, li);
    T.nu_post = nu_at(c, c->sm.nu_post, li);
    T.nu_doubling = c->sm.nu_doubling;
    T.first_fused = first_done ? 1 : 0;
    for (int k = 0; k < T.nlev; ++k) T.lev[k].d = c->lev[c->tail_start + k].d;   // smoother kind
    c->launches += launch_coarse_tail(T, c->st);
    return L.e;
  }
  if (li == nlev - 1) {
    c->launches += launch_coarse_solve(L.d, c->fidx, c->nf, c->A1inv, L.r, L.e, c->st);
    return L.e;
  }
  const int nu_pre = nu_at(c, c->sm.nu_pre, li), nu_post = nu_at(c, c->sm.nu_post, li);
  int s0 = 0;
  if (nu_pre > 0 && c->sm.kind != MG_SMOOTH_LUSGS) {
    if (!first_done) c->launches += launch_smooth_first(L.d, L.r, L.e, L.dv, c->st);
    s0 = 1;
  } else {
    c->launches += launch_zero(L.e, L.d.ndof, c->st);
  }
  double* cur = L.e;
  const bool dok = dfx_ok(c, li);
  for (int s = s0; s < nu_pre; ++s)
    cur = smooth_step(c, L, s, cur, s == 1 && s0 == 1 && dok, s == nu_pre - 1 && dok);
  HostLevel& C = c->lev[li + 1];
  const bool fuse = (li + 1 < nlev - 1) && nu_at(c, c->sm.nu_pre, li + 1) > 0 &&
                    c->sm.kind != MG_SMOOTH_LUSGS &&
                    !(c->tail_dense && li + 1 == c->tail_start) && !gathers(c, li);
  if (L.kind == KIND_P && L.d.orb && L.d.imask == 0 && !L.clist && !gathers(c, li) &&
      !partitioned(c) && C.d.orb && C.d.p == 1) {
    // residual and p-restriction in one pair of passes: the colour-1 epilogue restricts
    // each edge's residual r - A e1 (Eq. 3.6 with the P1 injection J_p) instead of storing it
    c->launches += launch_resid_prestrict(L.d, C.d, c->refdev.Jp, cur, other(L, cur), L.r, C.r, fuse,
                                          C.e, dfx_ok(c, li + 1) ? nullptr : C.dv, c->st);
  } else {
    double* res = residual(c, L, cur);  // r - A e1
    restrict_level(c, li, res, cur, true, C.r, fuse);
  }
  const double* ec = vcycle_level(c, li + 1, fuse);
  int s1 = 0;
  if (nu_post > 0 && L.kind == KIND_P && L.d.orb && L.d.imask == 0 && !L.clist &&
      !gathers(c, li) && !partitioned(c) && c->sm.kind != MG_SMOOTH_LUSGS &&
      !tiled(L.d, AM_SMOOTH)) {
    // the p-prolongation folded into the first post-smoothing step's colour-0 pass
    c->launches += launch_w0_prolong(L.d, c->refdev.Jp, ec, cur, other(L, cur), c->st);
    c->launches += launch_apply(L.d, 1, AM_SMOOTH, cur, other(L, cur), L.r, L.dv,
                                nu_post == 1 && dok ? STEP_NO_D_STORE : 0, nullptr, true, c->st);
    s1 = 1;
  } else if (nu_post > 0 && L.kind == KIND_H && L.d.orb && L.d.p == 1 && L.d.imask == 0 &&
             !L.clist && !gathers(c, li) && !partitioned(c) && c->sm.kind != MG_SMOOTH_LUSGS &&
             !tiled(L.d, AM_SMOOTH) && !gathered(L.d, AM_SMOOTH) && env_or("MGDTN_W0H", 1) != 0) {
    // the h-prolongation (Eqs. 3.3 / 3.4) folded into the first post-smoothing step's
    // colour-0 pass of the P1 orbit level (AM_W0H; config 5: the 4096^2 P1 level)
    c->launches += launch_w0_hprolong(L.d, ec, L.Pm, cur, other(L, cur), c->st);
    c->launches += launch_apply(L.d, 1, AM_SMOOTH, cur, other(L, cur), L.r, L.dv,
                                nu_post == 1 && dok ? STEP_NO_D_STORE : 0, nullptr, true, c->st);
    s1 = 1;
  } else {
    prolong_level(c, li, ec, cur);
  }
  for (int s = s1; s < nu_post; ++s)
    cur = smooth_step(c, L, s, cur, false, s == nu_post - 1 && dok, s == nu_post - 1 ? zpart : nullptr);
  return cur;
}

// ---------------------------------------------------------------- setup
// everything of mg_setup_dtn after the input copies (reads Kc / tauc / methc only), on c->st
static int setup_body(Ctx* c) {
  cudaStream_t st = c->st;
  HostLevel& F = c->lev[0];
  // (MG_OPT_KEEP_FINE_MAPS: the maps mg_debug_set_element_dtn wrote stay; test hook)
  if (!c->keep_fine_maps)
    c->launches += launch_local_dtn(F.d, c->refdev, F.h, c->Kc, c->methc, c->tauc, c->err, st);
  const int nlev = (int)c->lev.size();
  const int numax = MAX_NU;   // coefficients for any step count (mg_smooth may exceed nu)
  // Chebyshev: lambda_max of D_B^-1 A_k by power iteration (Q11), v <- D^-1 A v in
  // place (colour-1 epilogue AM_DINV), no per-step normalisation.  A level's
  // iteration needs only that level's operator and edge blocks: on one GPU it is
  // forked onto its own stream (own scratch) as soon as they exist, so it overlaps
  // the coarsening of the levels below (MGDTN_SETUP_STREAMS=0: in sequence).
  // A level's whole smoother setup (edge blocks, their packed copy, the coefficients or
  // the Chebyshev power iteration) needs only that level's operator: on one GPU it is
  // forked onto its own stream as soon as the operator exists, so the main stream goes
  // straight on to the next coarsening (the critical path is then the coarsening chain
  // and the tail).  Tail levels stay on the main stream (k_tail_lmax / k_tail_basis
  // read their blocks).  MGDTN_SETUP_STREAMS=0: everything in sequence.
  const bool cheb = c->sm.kind == MG_SMOOTH_CHEBYSHEV;
  const bool fork = !partitioned(c) && env_or("MGDTN_SETUP_STREAMS", 1) != 0;
  auto in_tail = [&](int li) { return c->tail_start >= 0 && li >= c->tail_start; };
  auto is_pow = [&](int li) {
    return cheb && li < nlev - 1 && !(c->tail_lmax && in_tail(li));
  };
  auto forked = [&](int li) { return fork && li < nlev - 1 && !in_tail(li); };
  int npow = 0;
  for (int li = 0; li < nlev - 1; ++li) npow += forked(li) ? 1 : 0;
  if (fork && (int)c->side.size() < npow) return fail(c, MG_ERR_STATE, "side streams missing");
  int q = 0;   // forked levels so far
  auto power_iteration = [&](int li) -> int {   // on c->st
    HostLevel& L = c->lev[li];
    double* part = forked(li) ? L.lpart : c->part;
    double* sc = forked(li) ? L.lpart + c->npart : c->sscal;
    c->launches += launch_pow_init(L.d, L.e, c->st);
    for (int it = 0; it < c->sm.lmax_iters; ++it) {
      const bool last = it + 1 == c->sm.lmax_iters;
      apply_mode(c, L, AM_DINV, L.e, L.w, nullptr, nullptr, 0, last ? part : nullptr);
    }
    reduce_scal(c, part, apply_parts(L, AM_DINV), sc, 7, 0);   // v.Dv
    apply_full(c, L, L.e, L.w, part);
    reduce_scal(c, part, apply_parts(L, AM_APPLY), sc, 8, 0);  // v.Av
    c->launches += launch_lmax_finish(sc, c->sm.lmax_safety, c->sm.cheb_ratio, numax, L.lam,
                                      L.d.coef, c->st);
    return MG_OK;
  };
  auto smoother_setup = [&](int li) -> int {   // level li's operator is complete on st
    HostLevel& L = c->lev[li];
    const bool fk = forked(li);
    if (fk) {
      CK(cudaEventRecord(c->fork_evs[q], st));
      c->st = c->side[q];
      CK(cudaStreamWaitEvent(c->st, c->fork_evs[q], 0));
    }
    L.d.smoother = c->sm.kind;
    c->launches += launch_edge_blocks(L.d, c->err, c->st);
    if (L.d.imask) {   // interface edge blocks: D_e = D_own + D_remote, then inverted
      c->launches += launch_eblk_pack(L.d, c->hsend, c->st);
      halo_exchange(c, L.d, eblk_stride(L.d), L.d.k1 * L.d.k1);
      c->launches += launch_eblk_finish(L.d, c->hrecv, c->err, c->st);
    }
    if (!c->ns) c->launches += launch_dinv_pack(L.d, c->st);
    if (!cheb) c->launches += launch_set_bj_coef(c->sm.omega, L.d.coef, c->st);
    if (is_pow(li)) RC(power_iteration(li));
    if (fk) {
      CK(cudaEventRecord(c->side_ev[q], c->st));
      c->st = st;
      ++q;
    }
    return MG_OK;
  };
  for (int li = 0; li < nlev; ++li) {
    HostLevel& L = c->lev[li];
    // orbit storage (R9): symmetrise the level's maps and write their orbit records
    // before anything reads them
    c->launches += launch_orbit_pack(L.d, st);
    // smoother setup of level li (its operator is complete on st)
    if (li < nlev - 1) RC(smoother_setup(li));
    if (li + 1 >= nlev) break;
    // coarsening li -> li + 1
    HostLevel& C = c->lev[li + 1];
    if (L.kind == KIND_P) {
      c->launches += launch_p_coarsen(L.d, C.d, c->refdev.Jp, st);
      c->launches += launch_project_const(C.d, st);   // R10
    } else if (gathers(c, li)) {
      // gather level: this rank's macros' coarse DtN maps, all-gathered into the
      // replicated level (every rank then builds the coarser levels redundantly)
      HostLevel& B = c->lgl;   // dense output: the block's element count may be odd
      c->launches += launch_agglomerate(L.d, B.d, L.KIIinv, L.Pm, c->err, st, c->sden);
      comm_fail(c, c->comm->allgather(c->sden, c->sall, (size_t)B.d.ne * 64, st));
      c->launches += launch_gather_S(C.d, B.d.nx, B.d.ny, c->px, c->sall, st);
      c->launches += launch_project_const(C.d, st);   // R10 (same on every rank)
    } else {
      c->launches += launch_agglomerate(L.d, C.d, L.KIIinv, L.Pm, c->err, st, nullptr,
                                        c->ns ? L.Rm : nullptr);
      c->launches += launch_project_const(C.d, st);   // R10
    }
  }
  if (c->sm.kind == MG_SMOOTH_CHEBYSHEV && c->tail_lmax && c->tail_start >= 0 &&
      c->tail_start < nlev - 1) {   // (overlaps the forked power iterations)
    TailParams& T = c->tail;
    for (int k = 0; k < T.nlev; ++k) T.lev[k].d = c->lev[c->tail_start + k].d;
    c->launches += launch_tail_lmax(T, c->sm.lmax_iters, c->sm.lmax_safety, c->sm.cheb_ratio,
                                    numax, c->part, st);
  }
  c->lev.back().d.smoother = c->sm.kind;
  c->launches += launch_coarse_assemble_factor(c->lev.back().d, c->fpos, c->nf, c->A1, c->A1inv,
                                               c->err, st);
  // the tabulated tail needs only the tail levels (their coefficients come from
  // k_tail_lmax / block-Jacobi on this stream): it also overlaps the forked iterations
  auto tail_basis = [&]() {
    TailParams& T = c->tail;
    T.nu_pre = nu_at(c, c->sm.nu_pre, c->tail_start);
    T.nu_post = nu_at(c, c->sm.nu_post, c->tail_start);
    T.nu_doubling = c->sm.nu_doubling;
    T.first_fused = 0;
    for (int k = 0; k < T.nlev; ++k) T.lev[k].d = c->lev[c->tail_start + k].d;
    c->launches += launch_tail_basis(T, c->tfidx, c->nft, c->Bt, st);
  };
  const bool use_basis = c->tail_dense && c->sm.kind != MG_SMOOTH_LUSGS;
  const bool basis_early = use_basis && (c->tail_lmax || c->sm.kind == MG_SMOOTH_BLOCK_JACOBI);
  if (basis_early) tail_basis();
  if (fork)   // join
    for (int k = 0; k < q; ++k) CK(cudaStreamWaitEvent(st, c->side_ev[k], 0));
  CK(cudaGetLastError());
  // e / w / d vectors must hold 0 on dOmega: zero them once
  for (auto& L : c->lev) {
    CK(cudaMemsetAsync(L.e, 0, L.d.ndof * sizeof(double), st));
    CK(cudaMemsetAsync(L.w, 0, L.d.ndof * sizeof(double), st));
    CK(cudaMemsetAsync(L.dv, 0, L.d.ndof * sizeof(double), st));
    CK(cudaMemsetAsync(L.r, 0, L.d.ndof * sizeof(double), st));
  }
  if (partitioned(c)) {
    CK(cudaMemsetAsync(c->lgl.r, 0, c->lgl.d.ndof * sizeof(double), st));
    CK(cudaMemsetAsync(c->lgl.e, 0, c->lgl.d.ndof * sizeof(double), st));
  }
  if (use_basis && !basis_early) tail_basis();
  CK(cudaGetLastError());
  return MG_OK;
}

static bool same_smoother(const mg_smoother_cfg& a, const mg_smoother_cfg& b) {
  return a.kind == b.kind && a.nu_pre == b.nu_pre && a.nu_post == b.nu_post &&
         a.omega == b.omega && a.cheb_ratio == b.cheb_ratio && a.lmax_iters == b.lmax_iters &&
         a.lmax_safety == b.lmax_safety && a.nu_doubling == b.nu_doubling;
}

// mg_setup_dtn: copy the element data, then the setup body -- replayed from a CUDA
// graph on one GPU (its ~300 launches cost one graph launch of host time; the forked
// smoother setups become parallel graph branches), eager otherwise
static int setup_impl(Ctx* c, const double* K, const int8_t* method, const double* tau) {
  NvtxRange nv("mg/setup");
  cudaStream_t st = c->st;
  CK(cudaMemsetAsync(c->err, 0, sizeof(DevError), st));
  HostLevel& F = c->lev[0];
  const int64_t ne = F.d.ne;
  CK(cudaMemcpyAsync(c->Kc, K, ne * sizeof(double), cudaMemcpyDeviceToDevice, st));
  CK(cudaMemcpyAsync(c->tauc, tau, ne * sizeof(double), cudaMemcpyDeviceToDevice, st));
  CK(cudaMemcpyAsync(c->methc, method, ne * sizeof(int8_t), cudaMemcpyDeviceToDevice, st));
  if (!partitioned(c)) {   // side streams of the forked smoother setups (created outside capture)
    const int need = (int)c->lev.size();
    while ((int)c->side.size() < need) {
      cudaStream_t sx;
      cudaEvent_t ex, fx;
      CK(cudaStreamCreateWithFlags(&sx, cudaStreamNonBlocking));
      CK(cudaEventCreateWithFlags(&ex, cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&fx, cudaEventDisableTiming));
      c->side.push_back(sx);
      c->side_ev.push_back(ex);
      c->fork_evs.push_back(fx);
    }
  }
  const bool graph = c->use_graphs && !partitioned(c) && st != nullptr &&
                     env_or("MGDTN_SETUP_GRAPH", 1) != 0;
  if (graph) {
    if (c->gU && !same_smoother(c->gU_sm, c->sm)) {
      cudaGraphExecDestroy(c->gU);
      c->gU = nullptr;
    }
    if (!c->gU) {
      const long long l0 = c->launches;
      CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
      const int rc = setup_body(c);
      c->st = st;
      cudaGraph_t g = nullptr;
      const cudaError_t e = cudaStreamEndCapture(st, &g);
      c->nU = c->launches - l0;
      c->launches = l0;
      if (rc != MG_OK) {
        if (g) cudaGraphDestroy(g);
        return rc;
      }
      CK(e);
      const cudaError_t e2 = cudaGraphInstantiate(&c->gU, g, 0);
      cudaGraphDestroy(g);
      CK(e2);
      c->gU_sm = c->sm;
    }
    CK(cudaGraphLaunch(c->gU, st));
    c->launches += c->nU;
  } else {
    RC(setup_body(c));
  }
  RC(check_device_error(c));
  c->setup_done = true;
  return MG_OK;
}

// ---------------------------------------------------------------- PCG
// scal: [0] rz, [1] pAp, [2] rr, [3] alpha, [4] beta, [5] gg
// the fine level's first pre-smoothing step folded into the PCG update (k_pcg_update_sf):
// orbit fine level (D_e^-1 orbits), a pre-smoothing step, not LU-SGS, and the fine level
// runs the launch-per-step V-cycle (not the tabulated / single-launch tail)
static bool pcg_sf(const Ctx* c) {
  const HostLevel& F = c->lev[0];
  return F.d.orb && c->sm.kind != MG_SMOOTH_LUSGS && c->sm.nu_pre > 0 && c->tail_start != 0 &&
         c->lev.size() > 1;
}

// the direction update p = z + beta p folded into the colour-0 pass of the next PCG apply
// (AM_W0U): one-GPU orbit fine level whose apply is the pair of colour passes.  Config 5:
// removes k_pcg_pupdate (0.77 ms, 4.0 GB) for a heavier colour-0 pass
static bool pcg_w0u(const Ctx* c) {
  const HostLevel& F = c->lev[0];
  return F.d.orb && !F.d.imask && !F.clist && !partitioned(c) && !tiled(F.d, AM_APPLY) &&
         !gathered(F.d, AM_APPLY) && env_or("MGDTN_W0U", 1) != 0;
}

static void pcg_iter_A(Ctx* c) {  // Ap, alpha, x/r update, rr
  HostLevel& F = c->lev[0];
  const int vg = vec_grid(F.d.ndof);
  if (c->pu_pending) {   // p = z + beta p in the colour-0 pass, then the colour-1 pass
    c->pu_pending = false;
    c->launches += launch_w0_update(F.d, c->zp, c->scal, c->pv, c->ap, c->st);
    c->launches += launch_apply(F.d, 1, AM_APPLY, c->pv, c->ap, nullptr, nullptr, 0, c->part, true,
                                c->st);
  } else {
    apply_full(c, F, c->pv, c->ap, c->part);
  }
  reduce_scal(c, c->part, apply_parts(F, AM_APPLY), c->scal, 1, 1);
  if (pcg_sf(c)) {
    const int64_t nb = (F.d.nedge + 127) / 128;
    const int g = (int)(nb < 148 * 8 ? nb : 148 * 8);
    c->launches += launch_pcg_update_sf(F.d, c->x, F.r, c->pv, c->ap, c->scal, c->part, g, F.e,
                                        dfx_ok(c, 0) ? nullptr : F.dv, c->st);
    reduce_scal(c, c->part, g, c->scal, 2, 0);
    return;
  }
  c->launches += launch_pcg_update(c->x, F.r, c->pv, c->ap, c->scal, F.d.ndof, c->part, vg, c->st,
                                   &F.d);
  reduce_scal(c, c->part, vg, c->scal, 2, 0);
}

// (r.z stays a separate k_dot pass: folding it into the last fine smoothing pass
// (SMOOTH + DOT epilogue) cost that pass 0.53 ms against k_dot's 0.38 ms at config 5,
// register pressure; profiles/r02_c5_iteration_launches.txt)
// r.z folded into the V-cycle's last fine smoothing step (its colour-1 epilogue holds r_e
// and the new iterate z_e of every free edge it owns): one-GPU orbit fine level run by the
// launch-per-step V-cycle, a last post-smoothing step through the pair of colour passes
static bool pcg_zdot(const Ctx* c) {
  const HostLevel& F = c->lev[0];
  return F.d.orb && !F.d.imask && !F.clist && !partitioned(c) && !tiled(F.d, AM_SMOOTH) &&
         !gathered(F.d, AM_SMOOTH) && c->sm.kind != MG_SMOOTH_LUSGS && c->sm.nu_post >= 2 &&
         c->tail_start != 0 && !c->sm.nu_doubling && env_or("MGDTN_ZDOT", 1) != 0;
}

static void pcg_iter_B(Ctx* c) {  // z = B r, beta, p update
  HostLevel& F = c->lev[0];
  const int vg = vec_grid(F.d.ndof);
  const double* z;
  if (pcg_zdot(c)) {
    z = vcycle_level(c, 0, pcg_sf(c), c->part);
    reduce_scal(c, c->part, apply_parts(F, AM_SMOOTH), c->scal, 0, 2);
  } else {
    z = vcycle_level(c, 0, pcg_sf(c));   // first step done by the update
    c->launches += launch_dot(F.r, z, F.d.ndof, c->part, vg, c->st, &F.d);
    reduce_scal(c, c->part, vg, c->scal, 0, 2);
  }
  if (pcg_w0u(c)) {   // done by the next pcg_iter_A's colour-0 pass
    c->pu_pending = true;
    c->zp = z;
    return;
  }
  c->launches += launch_pcg_pupdate(c->pv, z, c->scal, F.d.ndof, c->st);
}

// Rotated PCG loop (same kernel sequence as the textbook loop):
//   prologue: x = 0; gg = g.g; z = B r; rz = r.z; p = z; A-part; check
//   body:     B-part (z = B r, beta, p = z + beta p); A-part; check
static void pcg_prologue(Ctx* c) {
  HostLevel& F = c->lev[0];
  const int64_t n = F.d.ndof;
  const int vg = vec_grid(n);
  c->launches += launch_zero(c->x, n, c->st);
  c->launches += launch_dot(F.r, F.r, n, c->part, vg, c->st, &F.d);
  reduce_scal(c, c->part, vg, c->scal, 5, 0);
  const double* z = vcycle_level(c, 0, false);
  c->launches += launch_dot(F.r, z, n, c->part, vg, c->st, &F.d);
  reduce_scal(c, c->part, vg, c->scal, 0, 0);
  c->launches += launch_copy(c->pv, z, n, c->st);
  pcg_iter_A(c);
  c->launches += launch_pcg_check(c->scal, c->ist, c->dhist, HIST_CAP, c->cond, c->st);
}

static void pcg_body(Ctx* c) {
  pcg_iter_B(c);
  pcg_iter_A(c);
  c->launches += launch_pcg_check(c->scal, c->ist, c->dhist, HIST_CAP, c->cond, c->st);
}

// One graph for the whole solve: the prologue, then a conditional WHILE node
// whose body is one PCG iteration; k_pcg_check sets the loop condition on the
// device, so the host synchronises once per solve instead of once per iteration.
static int capture_solve(Ctx* c) {
  cudaGraph_t g = nullptr;
  CK(cudaGraphCreate(&g, 0));
  CK(cudaGraphConditionalHandleCreate(&c->cond, g, 0, cudaGraphCondAssignDefault));
  const long long l0 = c->launches;
  CK(cudaStreamBeginCaptureToGraph(c->st, g, nullptr, nullptr, 0,
                                   cudaStreamCaptureModeThreadLocal));
  pcg_prologue(c);
  c->nPro = c->launches - l0;
  cudaStreamCaptureStatus cs;
  const cudaGraphNode_t* deps = nullptr;
  size_t nd = 0;
  cudaError_t e = cudaStreamGetCaptureInfo(c->st, &cs, nullptr, nullptr, &deps, &nd);
  std::vector<cudaGraphNode_t> dv(deps, deps + (e == cudaSuccess ? nd : 0));
  cudaGraph_t gc = nullptr;
  cudaError_t e2 = cudaStreamEndCapture(c->st, &gc);
  c->launches = l0;
  CK(e);
  CK(e2);
  cudaGraphNodeParams cp = {};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = c->cond;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  cudaGraphNode_t cn;
  CK(cudaGraphAddNode(&cn, g, dv.data(), dv.size(), &cp));
  cudaGraph_t body = cp.conditional.phGraph_out[0];
  CK(cudaStreamBeginCaptureToGraph(c->st, body, nullptr, nullptr, 0,
                                   cudaStreamCaptureModeThreadLocal));
  pcg_body(c);
  c->nBody = c->launches - l0;
  c->launches = l0;
  CK(cudaStreamEndCapture(c->st, &body));
  e = cudaGraphInstantiate(&c->gS, g, 0);
  cudaGraphDestroy(g);
  CK(e);
  return MG_OK;
}

static int pcg_impl(Ctx* c, const double* g, double* lambda, double rtol, int maxit,
                    int* iters_out, double* relres_out, int* status_out, double* hist) {
  HostLevel& F = c->lev[0];
  cudaStream_t st = c->st;
  const int64_t n = F.d.ndof;
  const int vg = vec_grid(n);
  const long long l0 = c->launches;
  if (c->st == nullptr) c->use_graphs = false;   // legacy stream cannot be captured
  c->pu_pending = false;
  c->launches += launch_copy_masked(F.d, F.r, g, st);
  int status = MG_MAXIT, it = 0;
  double rel = 0.0;
  if (c->use_graphs && maxit < HIST_CAP && !partitioned(c)) {
    if (!c->gS) RC(capture_solve(c));
    c->launches += launch_pcg_init(c->ist, c->scal, rtol, maxit, st);
    CK(cudaGraphLaunch(c->gS, st));
    CK(cudaMemcpyAsync(c->pinned, c->ist, 2 * sizeof(int), cudaMemcpyDeviceToHost, st));
    RC(sync_st(c, st));
    int hs[2];
    std::memcpy(hs, c->pinned, sizeof(hs));
    it = hs[0];
    status = hs[1];
    c->launches += c->nPro + (it > 1 ? (long long)(it - 1) * c->nBody : 0);
    std::vector<double> hv(it + 1);
    CK(cudaMemcpyAsync(hv.data(), c->dhist, (it + 1) * sizeof(double), cudaMemcpyDeviceToHost,
                       st));
    if (it == 0) {   // g = 0: lambda = 0
      CK(cudaMemsetAsync(lambda, 0, n * sizeof(double), st));
    } else {
      c->launches += launch_copy(lambda, c->x, n, st);
    }
    CK(cudaGetLastError());
    RC(sync_st(c, st));
    rel = hv[it];
    if (hist) std::memcpy(hist, hv.data(), (it + 1) * sizeof(double));
    if (iters_out) *iters_out = it;
    if (relres_out) *relres_out = rel;
    if (status_out) *status_out = status;
    c->last_solve_launches = c->launches - l0;
    return MG_OK;
  }
  // eager host-driven loop (use_graphs off, legacy stream, or maxit >= HIST_CAP):
  // the same kernel sequence, with a host round trip per iteration
  c->launches += launch_zero(c->x, n, st);
  c->launches += launch_dot(F.r, F.r, n, c->part, vg, st, &F.d);
  reduce_scal(c, c->part, vg, c->scal, 5, 0);
  CK(cudaMemcpyAsync(c->pinned, c->scal, 8 * sizeof(double), cudaMemcpyDeviceToHost, st));
  RC(sync_st(c, st));
  const double gg = c->pinned[5];
  if (hist) hist[0] = gg > 0 ? 1.0 : 0.0;
  if (!(gg > 0.0)) {   // g = 0 -> lambda = 0 in 0 iterations
    CK(cudaMemsetAsync(lambda, 0, n * sizeof(double), st));
    RC(sync_st(c, st));
    if (iters_out) *iters_out = 0;
    if (relres_out) *relres_out = 0.0;
    if (status_out) *status_out = MG_CONVERGED;
    c->last_solve_launches = c->launches - l0;
    return MG_OK;
  }
  // z = B r ; rz = r.z ; p = z
  const double* z = vcycle_level(c, 0, false);
  c->launches += launch_dot(F.r, z, n, c->part, vg, st, &F.d);
  reduce_scal(c, c->part, vg, c->scal, 0, 0);
  c->launches += launch_copy(c->pv, z, n, st);
  CK(cudaGetLastError());
  // Partitioned over NCCL with graphs on: every iteration's ~150 launches -- the V-cycle,
  // the halo send / recv groups, the all-reduced PCG scalars -- are captured once (NCCL
  // collectives are stream-capturable) and replayed as ONE graph launch; the host then
  // waits (polling NCCL's error state) and reads the two scalars of the stop test.
  const bool gpart = partitioned(c) && c->use_graphs && c->comm && c->comm->capturable() &&
                     st != nullptr;
  auto capture = [&](bool withB, cudaGraphExec_t* out, long long* nk) -> int {
    cudaGraph_t g = nullptr;
    const long long l0g = c->launches;
    CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    if (withB) pcg_iter_B(c);
    pcg_iter_A(c);
    cudaMemcpyAsync(c->pinned, c->scal, 8 * sizeof(double), cudaMemcpyDeviceToHost, st);
    const cudaError_t e = cudaStreamEndCapture(st, &g);
    *nk = c->launches - l0g;
    c->launches = l0g;
    if (c->comm_rc) {
      if (g) cudaGraphDestroy(g);
      return c->comm_rc;
    }
    CK(e);
    const cudaError_t e2 = cudaGraphInstantiate(out, g, 0);
    cudaGraphDestroy(g);
    CK(e2);
    return MG_OK;
  };
  if (gpart && !c->gPA) RC(capture(false, &c->gPA, &c->nPA));
  if (gpart && !c->gPBA) RC(capture(true, &c->gPBA, &c->nPBA));
  for (it = 1; it <= maxit; ++it) {
    NvtxRange nv_it("mg/pcg/iteration");
    if (gpart) {
      CK(cudaGraphLaunch(it == 1 ? c->gPA : c->gPBA, st));
      c->launches += it == 1 ? c->nPA : c->nPBA;
    } else {
      pcg_iter_A(c);
      CK(cudaMemcpyAsync(c->pinned, c->scal, 8 * sizeof(double), cudaMemcpyDeviceToHost, st));
    }
    RC(sync_st(c, st));
    const double pAp = c->pinned[1], rr = c->pinned[2];
    rel = std::sqrt(rr / gg);
    if (hist) hist[it] = rel;
    if (!(pAp > 0.0) || !std::isfinite(rr)) {
      status = MG_BREAKDOWN;
      break;
    }
    if (rel <= rtol) {
      status = MG_CONVERGED;
      break;
    }
    if (rel > 1e6) {
      status = MG_DIVERGED;
      break;
    }
    if (it == maxit) break;
    if (!gpart) pcg_iter_B(c);
  }
  if (it > maxit) it = maxit;
  c->launches += launch_copy(lambda, c->x, n, st);
  CK(cudaGetLastError());
  RC(sync_st(c, st));
  if (iters_out) *iters_out = it;
  if (relres_out) *relres_out = rel;
  if (status_out) *status_out = status;
  c->last_solve_launches = c->launches - l0;
  return MG_OK;
}

// ---------------------------------------------------------------- MG as a solver, GMRES
// host-driven drivers of the paper's own Krylov setting (PAPER.md:937-939,
// 1008-1018): every step is a library kernel; the host holds the scalars.
static double gdot(Ctx* c, const double* a, const double* b) {
  HostLevel& F = c->lev[0];
  const int vg = vec_grid(F.d.ndof);
  c->launches += launch_dot(a, b, F.d.ndof, c->part, vg, c->st, &F.d);
  reduce_scal(c, c->part, vg, c->scal, 12, 0);
  cudaMemcpyAsync(c->pinned, c->scal + 12, sizeof(double), cudaMemcpyDeviceToHost, c->st);
  cudaStreamSynchronize(c->st);
  return c->pinned[0];
}

// B_N F.r: the V-cycle's fixed kernel sequence, replayed from a CUDA graph captured on
// first use (one GPU, graphs on); eager launches otherwise.  Returns the vector that
// holds the result (fixed by the captured sequence).
static const double* run_vcycle(Ctx* c) {
  if (!c->use_graphs || partitioned(c) || c->st == nullptr) return vcycle_level(c, 0, false);
  if (!c->gV) {
    cudaGraph_t g = nullptr;
    const long long l0 = c->launches;
    if (cudaStreamBeginCapture(c->st, cudaStreamCaptureModeThreadLocal) != cudaSuccess)
      return vcycle_level(c, 0, false);
    c->vres = vcycle_level(c, 0, false);
    c->nV = c->launches - l0;
    c->launches = l0;
    if (cudaStreamEndCapture(c->st, &g) != cudaSuccess || !g ||
        cudaGraphInstantiate(&c->gV, g, 0) != cudaSuccess) {
      if (g) cudaGraphDestroy(g);
      c->gV = nullptr;
      cudaGetLastError();
      return vcycle_level(c, 0, false);
    }
    cudaGraphDestroy(g);
  }
  cudaGraphLaunch(c->gV, c->st);
  c->launches += c->nV;
  return c->vres;
}

// out = B_N v: one V-cycle of Algorithm 1 from e = 0
static void precond(Ctx* c, const double* v, double* out) {
  HostLevel& F = c->lev[0];
  c->launches += launch_copy_masked(F.d, F.r, v, c->st);
  const double* z = run_vcycle(c);
  c->launches += launch_copy(out, z, F.d.ndof, c->st);
}

// lambda^{i+1} = lambda^i + B_N (g - A lambda^i), lambda^0 = 0,
// until ||g - A lambda|| <= tol ||g||
static int mgsolve_impl(Ctx* c, const double* g, double* x, double tol, int maxit, int* iters,
                        double* relres, int* status, double* hist) {
  HostLevel& F = c->lev[0];
  const int64_t n = F.d.ndof;
  double* gb = c->gbuf;   // masked g
  double* r = c->pv;
  c->launches += launch_copy_masked(F.d, gb, g, c->st);
  c->launches += launch_zero(x, n, c->st);
  c->launches += launch_copy(r, gb, n, c->st);
  const double gn = std::sqrt(gdot(c, gb, gb));
  int st = MG_MAXIT, it = 0;
  double rel = gn > 0 ? 1.0 : 0.0;
  if (hist) hist[0] = rel;
  if (!(gn > 0)) st = MG_CONVERGED;
  for (it = 1; it <= maxit && st != MG_CONVERGED; ++it) {
    precond(c, r, c->ap);
    c->launches += launch_add(x, c->ap, n, c->st);
    apply_full(c, F, x, c->ap, nullptr);
    c->launches += launch_axpby(1.0, gb, -1.0, c->ap, r, n, c->st);
    rel = std::sqrt(gdot(c, r, r)) / gn;
    if (hist) hist[it] = rel;
    if (rel <= tol) {
      st = MG_CONVERGED;
      break;
    }
    if (!std::isfinite(rel) || rel > 1e6) {
      st = MG_DIVERGED;
      break;
    }
  }
  if (it > maxit) it = maxit;
  CK(cudaGetLastError());
  *iters = gn > 0 ? it : 0;
  *relres = rel;
  *status = st;
  return c->comm_rc ? c->comm_rc : MG_OK;
}

// Left-preconditioned full GMRES: Arnoldi on B_N A from
// v_0 = B_N g / ||B_N g||, modified Gram-Schmidt, Givens least squares; stops on
// the true residual ||g - A lambda_j|| <= tol ||g||.
// V: caller-provided device basis [(maxit+1)][ndof].
static int gmres_impl(Ctx* c, const double* g, double* x, double tol, int maxit, double* V,
                      int* iters, double* relres, int* status, double* hist) {
  HostLevel& F = c->lev[0];
  const int64_t n = F.d.ndof;
  double* gb = c->gbuf;
  c->launches += launch_copy_masked(F.d, gb, g, c->st);
  c->launches += launch_zero(x, n, c->st);
  const double gn = std::sqrt(gdot(c, gb, gb));
  *iters = 0;
  *relres = 0.0;
  *status = MG_CONVERGED;
  if (hist) hist[0] = gn > 0 ? 1.0 : 0.0;
  if (!(gn > 0)) return MG_OK;
  auto Vj = [&](int j) { return V + (int64_t)j * n; };
  precond(c, gb, Vj(0));
  const double beta = std::sqrt(gdot(c, Vj(0), Vj(0)));
  c->launches += launch_axpby(1.0 / beta, Vj(0), 0.0, Vj(0), Vj(0), n, c->st);
  std::vector<double> H((size_t)(maxit + 1) * maxit, 0.0), cs(maxit), sn(maxit), rhs(maxit + 1, 0.0);
  auto h = [&](int i, int j) -> double& { return H[(size_t)i * maxit + j]; };
  rhs[0] = beta;
  int st = MG_MAXIT, j = 0;
  double rel = 1.0;
  // one GPU: the Hessenberg column stays on the device through the Gram-Schmidt
  // sweep (k_axpy_dev / k_scale_rsqrt) and comes back with one copy per step;
  // x = V y is one k_combine.  Partitioned: dots all-reduced through the host.
  const bool dev_mgs = !partitioned(c) && maxit + 2 <= HIST_CAP / 2;
  double* Hd = c->dhist;                  // column j of H (H[j+1][j] as ||w||^2)
  double* yd = c->dhist + HIST_CAP / 2;   // least-squares coefficients
  const int vg = vec_grid(n);
  std::vector<double> hcol(maxit + 2);
  for (j = 0; j < maxit; ++j) {
    apply_full(c, F, Vj(j), c->ap, nullptr);
    precond(c, c->ap, Vj(j + 1));
    double hn;
    if (dev_mgs) {
      for (int i = 0; i <= j; ++i) {   // modified Gram-Schmidt
        c->launches += launch_dot(Vj(j + 1), Vj(i), n, c->part, vg, c->st, &F.d);
        c->launches += launch_reduce(c->part, vg, Hd, i, 0, nullptr, c->st);
        c->launches += launch_axpy_dev(Hd + i, -1.0, Vj(i), Vj(j + 1), n, c->st);
      }
      c->launches += launch_dot(Vj(j + 1), Vj(j + 1), n, c->part, vg, c->st, &F.d);
      c->launches += launch_reduce(c->part, vg, Hd, j + 1, 0, nullptr, c->st);
      c->launches += launch_scale_rsqrt(Hd + j + 1, Vj(j + 1), n, c->st);
      CK(cudaMemcpyAsync(hcol.data(), Hd, (j + 2) * sizeof(double), cudaMemcpyDeviceToHost,
                         c->st));
      RC(sync_st(c, c->st));
      for (int i = 0; i <= j; ++i) h(i, j) = hcol[i];
      hn = std::sqrt(hcol[j + 1]);
    } else {
      for (int i = 0; i <= j; ++i) {   // modified Gram-Schmidt
        h(i, j) = gdot(c, Vj(j + 1), Vj(i));
        c->launches += launch_axpby(-h(i, j), Vj(i), 1.0, Vj(j + 1), Vj(j + 1), n, c->st);
      }
      hn = std::sqrt(gdot(c, Vj(j + 1), Vj(j + 1)));
      if (hn > 0) c->launches += launch_axpby(1.0 / hn, Vj(j + 1), 0.0, Vj(j + 1), Vj(j + 1), n, c->st);
    }
    h(j + 1, j) = hn;
    // least squares min || beta e1 - H y || by Givens rotations on a copy of column j
    std::vector<double> col(j + 2);
    for (int i = 0; i <= j + 1; ++i) col[i] = h(i, j);
    for (int i = 0; i < j; ++i) {
      const double t = cs[i] * col[i] + sn[i] * col[i + 1];
      col[i + 1] = -sn[i] * col[i] + cs[i] * col[i + 1];
      col[i] = t;
    }
    const double rr = std::hypot(col[j], col[j + 1]);
    cs[j] = rr > 0 ? col[j] / rr : 1.0;
    sn[j] = rr > 0 ? col[j + 1] / rr : 0.0;
    col[j] = rr;
    col[j + 1] = 0.0;
    for (int i = 0; i <= j; ++i) h(i, j) = col[i];   // R factor, column j
    rhs[j + 1] = -sn[j] * rhs[j];
    rhs[j] = cs[j] * rhs[j];
    std::vector<double> y(j + 1);
    for (int i = j; i >= 0; --i) {
      double s = rhs[i];
      for (int k = i + 1; k <= j; ++k) s -= h(i, k) * y[k];
      y[i] = s / h(i, i);
    }
    // x = V y and the true residual
    if (dev_mgs) {
      CK(cudaMemcpyAsync(yd, y.data(), (j + 1) * sizeof(double), cudaMemcpyHostToDevice, c->st));
      c->launches += launch_combine(x, V, n, yd, j + 1, c->st);
    } else {
      c->launches += launch_zero(x, n, c->st);
      for (int i = 0; i <= j; ++i) c->launches += launch_axpby(y[i], Vj(i), 1.0, x, x, n, c->st);
    }
    apply_full(c, F, x, c->ap, nullptr);
    c->launches += launch_axpby(1.0, gb, -1.0, c->ap, c->pv, n, c->st);
    rel = std::sqrt(gdot(c, c->pv, c->pv)) / gn;
    if (hist) hist[j + 1] = rel;
    if (rel <= tol || hn == 0.0) {
      st = MG_CONVERGED;
      ++j;
      break;
    }
    if (!std::isfinite(rel)) {
      st = MG_BREAKDOWN;
      ++j;
      break;
    }
  }
  CK(cudaGetLastError());
  *iters = j > maxit ? maxit : j;
  *relres = rel;
  *status = st;
  return c->comm_rc ? c->comm_rc : MG_OK;
}

static int rhs_impl(Ctx* c, const double* f_qp, double f_const, const double* gD_qp, double* g,
                    double* lambda_bc) {
  HostLevel& F = c->lev[0];
  cudaStream_t st = c->st;
  const int64_t n = F.d.ndof;
  CK(cudaMemsetAsync(c->lamD, 0, n * sizeof(double), st));
  if (gD_qp) c->launches += launch_dirichlet(F.d, c->refdev, gD_qp, c->lamD, st);
  CK(cudaMemsetAsync(g, 0, n * sizeof(double), st));
  c->launches += launch_local_rhs(F.d, c->refdev, F.h, c->Kc, c->methc, c->tauc, f_qp, f_const,
                                  gD_qp ? c->lamD : nullptr, g, c->err, st);
  if (F.d.imask) {   // g = sum_T G_T^T b_T: interface edges sum both ranks' elements
    c->launches += launch_itf_pack(F.d, g, c->hsend, st);
    halo_exchange(c, F.d, itf_stride(F.d), F.d.k1);
    c->launches += launch_itf_epilogue(F.d, AM_APPLY, nullptr, g, nullptr, nullptr, 0, c->hrecv,
                                       nullptr, st);
  }
  if (lambda_bc)
    CK(cudaMemcpyAsync(lambda_bc, c->lamD, n * sizeof(double), cudaMemcpyDeviceToDevice, st));
  CK(cudaGetLastError());
  return MG_OK;
}

static HostLevel* level_of(Ctx* c, int level) {
  const int N = (int)c->lev.size();
  if (level < 1 || level > N) return nullptr;
  return &c->lev[N - level];
}

}  // namespace mgdtn

using namespace mgdtn;

// ============================================================================ C ABI
extern "C" {

}  // extern "C"

namespace mgdtn {
// Level structure (host only).  One GPU: finest (order p), the p-level (P1,
// same mesh) if p > 1, then 2x2 agglomeration while both sides stay divisible
// by 4.  Partitioned: the same global
// sequence of levels; each rank holds its px x py element block of every level
// down to the gather level Lg -- the first level whose global element count is
// <= gather_ne, or whose blocks could not be agglomerated again, or the coarsest
// -- and every level from Lg down is replicated on all ranks.
static int build_levels(Ctx* c, const mg_quad_mesh* mesh, int p, int n_h_levels,
                        const mg_partition* part) {
  const int nx = mesh->nx, ny = mesh->ny;
  const int nranks = part ? part->nranks : 1;
  if (nranks > 1) {
    if (part->px < 1 || part->py < 1 || part->px * part->py != nranks || part->rank < 0 ||
        part->rank >= nranks)
      return fail(c, MG_ERR_ARG, "partition: px * py must equal nranks, 0 <= rank < nranks");
    if (nx % part->px || ny % part->py || ((nx / part->px) & 1) || ((ny / part->py) & 1))
      return fail(c, MG_ERR_SHAPE, "partition: element blocks must have even sides");
    c->nranks = nranks;
    c->rank = part->rank;
    c->px = part->px;
    c->py = part->py;
    c->rx = c->rank % c->px;
    c->ry = c->rank / c->px;
    c->nbr[0] = c->ry > 0 ? c->rank - c->px : -1;
    c->nbr[1] = c->rx < c->px - 1 ? c->rank + 1 : -1;
    c->nbr[2] = c->ry < c->py - 1 ? c->rank + c->px : -1;
    c->nbr[3] = c->rx > 0 ? c->rank - 1 : -1;
  }
  int dmask = 15;
  for (int f = 0; f < 4; ++f)
    if (c->nbr[f] >= 0) dmask &= ~(1 << f);
  const int imask = 15 & ~dmask;
  const int64_t gather_ne = (part && part->gather_ne > 0) ? part->gather_ne : 16384;
  auto local = [&](HostLevel& L, int gx, int gy) {   // this rank's block of a gx x gy level
    LevelDev& d = L.d;
    d.dmask = dmask;
    d.imask = imask;
    d.ox = c->rx * d.nx;
    d.oy = c->ry * d.ny;
    d.gnx = gx;
    d.gny = gy;
  };
  int gx = nx, gy = ny;
  int cx = nx / c->px, cy = ny / c->py;
  double h = mesh->h;
  HostLevel top;
  init_level(top, cx, cy, p, h, KIND_COARSEST);
  if (partitioned(c)) local(top, gx, gy);
  c->lev.push_back(top);
  if (p > 1) {
    c->lev.back().kind = KIND_P;
    HostLevel L1;
    init_level(L1, cx, cy, 1, h, KIND_COARSEST);
    if (partitioned(c)) local(L1, gx, gy);
    c->lev.push_back(L1);
  }
  int nh = 0;
  while (gx > 2 && gy > 2 && (gx % 4 == 0) && (gy % 4 == 0) &&
         (n_h_levels <= 0 || nh < n_h_levels)) {
    c->lev.back().kind = KIND_H;
    const int ngx = gx / 2, ngy = gy / 2;
    h *= 2;
    HostLevel L;
    if (partitioned(c) && c->Lg < 0) {
      const int ncx = cx / 2, ncy = cy / 2;
      const bool more = ngx > 2 && ngy > 2 && (ngx % 4 == 0) && (ngy % 4 == 0) &&
                        (n_h_levels <= 0 || nh + 1 < n_h_levels);
      const bool stay = more && (int64_t)ngx * ngy > gather_ne && ncx % 2 == 0 && ncy % 2 == 0;
      if (stay) {
        init_level(L, ncx, ncy, 1, h, KIND_COARSEST);
        local(L, ngx, ngy);
        cx = ncx;
        cy = ncy;
      } else {   // gather: this rank's block of the new level + the replicated level
        init_level(c->lgl, ncx, ncy, 1, h, KIND_COARSEST);
        local(c->lgl, ngx, ngy);
        init_level(L, ngx, ngy, 1, h, KIND_COARSEST);
        c->Lg = (int)c->lev.size();
      }
    } else {
      init_level(L, ngx, ngy, 1, h, KIND_COARSEST);
    }
    c->lev.push_back(L);
    gx = ngx;
    gy = ngy;
    ++nh;
  }
  if (partitioned(c) && c->Lg < 0)
    return fail(c, MG_ERR_SHAPE, "partition: the hierarchy needs at least one 2x2 coarsening");
  const LevelDev& d1 = c->lev.back().d;
  c->nf = (int)(((int64_t)d1.nx * (d1.ny - 1) + (int64_t)(d1.nx - 1) * d1.ny) * d1.k1);
  if (c->nf > 4096) return fail(c, MG_ERR_SHAPE, "coarsest level too large for the dense solve");
  return MG_OK;
}
}  // namespace mgdtn

extern "C" {

int mg_build_hierarchy(const mg_quad_mesh* mesh, int32_t p, int32_t n_h_levels,
                       const mg_partition* part, void* cuda_stream, void** out_ctx) {
  return mg_build_hierarchy_ex(mesh, p, n_h_levels, part, 0, cuda_stream, out_ctx);
}

int mg_build_hierarchy_ex(const mg_quad_mesh* mesh, int32_t p, int32_t n_h_levels,
                          const mg_partition* part, int32_t flags, void* cuda_stream,
                          void** out_ctx) {
  if (!mesh || !out_ctx) return MG_ERR_ARG;
  if (flags & ~MG_BUILD_NONSYMMETRIC) return MG_ERR_ARG;
  const bool ns = (flags & MG_BUILD_NONSYMMETRIC) != 0;
  if (ns && part && part->nranks > 1) return MG_ERR_UNSUPPORTED;
  *out_ctx = nullptr;
  if (p < 1 || p > 4) return MG_ERR_ARG;
  const int nx = mesh->nx, ny = mesh->ny;
  if (nx < 2 || ny < 2 || (nx & 1) || (ny & 1) || !(mesh->h > 0)) return MG_ERR_SHAPE;
  Ctx* c = new Ctx();
  c->mesh = *mesh;
  c->p = p;
  c->st = reinterpret_cast<cudaStream_t>(cuda_stream);
  try {
    c->ref = build_ref_tables(p);
  } catch (const std::exception&) {
    delete c;
    return MG_ERR_ARG;
  }
  const RefTables& T = c->ref;
  c->ref_doubles = T.G.size() + T.F.size() + T.P.size() + T.E.size() + T.W.size() + T.H.size() +
                   T.LN.size() + T.Nl.size() + T.fq.size() + T.ew.size() + T.H1inv.size() +
                   T.Jp.size();
  for (int k = 0; k < 2; ++k)
    c->ref_doubles += T.pen[k].lam.size() + T.pen[k].mu.size() + T.pen[k].At.size() +
                      T.pen[k].Bk.size() + T.pen[k].fqT.size() + T.pen[k].Tt.size();
  c->ref_doubles += T.vq.size() + T.wq.size() + T.L.size() + T.N.size();
  int rc = build_levels(c, mesh, p, n_h_levels, part);
  if (rc != MG_OK) {
    delete c;
    return rc;
  }
  c->ns = ns;
  for (auto& L : c->lev) {   // full element-map storage on every level
    L.d.ns = ns ? 1 : 0;
    if (ns) L.d.npk = L.d.m * L.d.m;
  }
  if (partitioned(c)) {   // the communicator: loopback hub (tests) or NCCL (one process per GPU)
    if (part->loopback) {
      c->comm = make_loopback_comm(static_cast<LoopbackHub*>(part->loopback), c->rank);
    } else {
      if (!part->nccl_id) {
        delete c;
        return MG_ERR_ARG;
      }
      int dev = 0;
      cudaGetDevice(&dev);
      std::string err;
      c->comm = make_nccl_comm(part->nccl_id, c->rank, c->nranks, dev, err);
      if (!c->comm) {
        delete c;
        return MG_ERR_NCCL;
      }
    }
    // PCG: host-driven loop; over NCCL each iteration is replayed from a captured graph
    // (the loopback hub synchronises its virtual ranks on the host: eager launches)
    if (cudaStreamCreateWithFlags(&c->cst, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->evB, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->evC, cudaEventDisableTiming) != cudaSuccess) {
      delete c->comm;
      delete c;
      return MG_ERR_CUDA;
    }
  }
  plan_tail(c);
  plan_tail_dense(c);
  plan_gather(c);
  // orbit storage (R9, d4.cuh): the finest level and its p-coarsened P1 level hold
  // D4-invariant element maps (uniform squares, scalar K per element)
  if (!c->ns) {
    c->lev[0].d.orb = 1;
    if (c->lev[0].kind == KIND_P) c->lev[1].d.orb = 1;
  }
  layout(c);   // host only: no CUDA call until mg_bind_workspace
  *out_ctx = c;
  return MG_OK;
}

int mg_partition_plan(const mg_quad_mesh* mesh, int32_t p, int32_t n_h_levels,
                      const mg_partition* part, int32_t max_levels, int32_t* nlevels,
                      int32_t* gather_level, int32_t* info) {
  if (!mesh || !part || !nlevels || !gather_level || !info || max_levels < 1) return MG_ERR_ARG;
  if (p < 1 || p > 4) return MG_ERR_ARG;
  Ctx c;
  int rc = build_levels(&c, mesh, p, n_h_levels, part);
  if (rc != MG_OK) return rc;
  const int N = (int)c.lev.size();
  *nlevels = N;
  *gather_level = c.Lg < 0 ? 0 : N - c.Lg;   // paper numbering of the first replicated level
  for (int k = 0; k < N && k < max_levels; ++k) {
    const LevelDev& d = c.lev[N - 1 - k].d;   // info[k] = level k+1 (paper numbering)
    int32_t* o = info + 8 * k;
    o[0] = d.nx; o[1] = d.ny; o[2] = d.ox; o[3] = d.oy;
    o[4] = d.gnx; o[5] = d.gny; o[6] = d.dmask; o[7] = d.imask;
  }
  return MG_OK;
}

int mg_partition_side_edges(const mg_quad_mesh* mesh, int32_t p, int32_t n_h_levels,
                            const mg_partition* part, int32_t level, int32_t side,
                            int64_t* global_edges, int32_t* count) {
  if (!mesh || !part || !count || side < 0 || side > 3) return MG_ERR_ARG;
  Ctx c;
  int rc = build_levels(&c, mesh, p, n_h_levels, part);
  if (rc != MG_OK) return rc;
  const int N = (int)c.lev.size();
  if (level < 1 || level > N) return MG_ERR_ARG;
  const LevelDev& d = c.lev[N - level].d;
  if (!((d.imask >> side) & 1)) {
    *count = 0;
    return MG_OK;
  }
  const int n = side_len(d.nx, d.ny, side);
  *count = n;
  if (global_edges)
    for (int q = 0; q < n; ++q) global_edges[q] = global_edge(d, side_edge(d.nx, d.ny, side, q));
  return MG_OK;
}

int mg_get_nccl_unique_id(uint8_t out[128]) {
  if (!out) return MG_ERR_ARG;
  std::string err;
  return nccl_unique_id(out, err) == 0 ? MG_OK : MG_ERR_NCCL;
}

void* mg_loopback_create(int32_t nranks) { return nranks >= 1 ? loopback_create(nranks) : nullptr; }
void mg_loopback_destroy(void* hub) { loopback_destroy(static_cast<LoopbackHub*>(hub)); }
void mg_loopback_abort(void* hub) { loopback_abort(static_cast<LoopbackHub*>(hub)); }

int mg_workspace_bytes(const void* ctx, size_t* bytes) {
  const Ctx* c = static_cast<const Ctx*>(ctx);
  if (!c || !bytes) return MG_ERR_ARG;
  *bytes = c->ws_need;
  return MG_OK;
}

int mg_bind_workspace(void* ctx, void* dev_ptr, size_t bytes) {
  Ctx* c = static_cast<Ctx*>(ctx);
  if (!c || !dev_ptr) return MG_ERR_ARG;
  if (bytes < c->ws_need) return fail(c, MG_ERR_WORKSPACE, "workspace too small");
  if (reinterpret_cast<uintptr_t>(dev_ptr) & 255)
    return fail(c, MG_ERR_WORKSPACE, "workspace must be 256-byte aligned");
  drop_graphs(c);
  if (!c->pinned) CK(cudaMallocHost(&c->pinned, 16 * sizeof(double)));
  c->ws = static_cast<char*>(dev_ptr);
  c->ws_bytes = bytes;
  c->setup_done = false;
  bind_pointers(c);
  fill_tail(c);
  CK(cudaMemsetAsync(c->ws, 0, c->ws_need, c->st));
  return upload_static(c);
}

int mg_setup_dtn(void* ctx, const double* K, const int8_t* method, const double* tau,
                 const mg_smoother_cfg* smoother) {
  Ctx* c = static_cast<Ctx*>(ctx);
  if (!c) return MG_ERR_ARG;
  if (!c->ws) return fail(c, MG_ERR_WORKSPACE, "no workspace bound");
  if (!K || !method || !tau || !smoother) return fail(c, MG_ERR_ARG, "NULL argument");
  mg_smoother_cfg sm = *smoother;
  if (sm.kind != MG_SMOOTH_BLOCK_JACOBI && sm.kind != MG_SMOOTH_CHEBYSHEV &&
      sm.kind != MG_SMOOTH_LUSGS)
    return fail(c, MG_ERR_ARG, "unknown smoother kind");
  if (sm.kind == MG_SMOOTH_LUSGS && partitioned(c))
    return fail(c, MG_ERR_UNSUPPORTED, "LU-SGS on a partitioned context");
  if (c->ns && sm.kind != MG_SMOOTH_BLOCK_JACOBI)
    return fail(c, MG_ERR_UNSUPPORTED,
                "nonsymmetric context: block-Jacobi only (Chebyshev needs a real spectrum)");
  if (sm.nu_pre < 0 || sm.nu_post < 0 || sm.nu_pre > MAX_NU || sm.nu_post > MAX_NU)
    return fail(c, MG_ERR_ARG, "nu out of range (0..8)");
  if (!(sm.omega > 0)) sm.omega = 1.0;
  if (!(sm.cheb_ratio > 1)) sm.cheb_ratio = 30.0;
  if (sm.lmax_iters <= 0) sm.lmax_iters = 20;
  if (!(sm.lmax_safety > 0)) sm.lmax_safety = 1.05;
  if (sm.nu_doubling && sm.kind == MG_SMOOTH_CHEBYSHEV)
    return fail(c, MG_ERR_ARG, "nu_doubling needs block-Jacobi or LU-SGS");
  if (sm.nu_pre != c->sm.nu_pre || sm.nu_post != c->sm.nu_post || sm.kind != c->sm.kind ||
      sm.nu_doubling != c->sm.nu_doubling)
    drop_graphs(c);
  c->sm = sm;
  c->setup_done = false;
  return setup_impl(c, K, method, tau);
}

int mg_assemble_rhs(void* ctx, const double* f_qp, double f_const, const double* gD_qp,
                    double* g, double* lambda_bc) {
  Ctx* c = static_cast<Ctx*>(ctx);
  if (!c || !g) return MG_ERR_ARG;
  if (!c->setup_done) return fail(c, MG_ERR_STATE, "mg_setup_dtn must precede mg_assemble_rhs");
  return rhs_impl(c, f_qp, f_const, gD_qp, g, lambda_bc);
}

int mg_apply(void* ctx, int32_t level, const double* x, double* y) {
  Ctx* c = static_cast<Ctx*>(ctx);
  if (!c || !x || !y || x == y) return MG_ERR_ARG;
  if (!c->setup_done) return fail(c, MG_ERR_STATE, "setup first");
  HostLevel* L = level_of(c, level);
  if (!L) return fail(c, MG_ERR_ARG, "level out of range");
  apply_full(c, *L, x, y, nullptr);
  CK(cudaGetLastError());
  return MG_OK;
}

int mg_vcycle(void* ctx, const double* r, double* z) {
  Ctx* c = static_cast<Ctx*>(ctx);
  if (!c || !r || !z) return MG_ERR_ARG;
  if (!c->setup_done) return fail(c, MG_ERR_STATE, "setup first");
  HostLevel& F = c->lev[0];
  c->launches += launch_copy_masked(F.d, F.r, r, c->st);
  const double* zr = run_vcycle(c);
  c->launches += launch_copy(z, zr, F.d.ndof, c->st);
  CK(cudaGetLastError());
  return MG_OK;
}

int mg_smooth(void* ctx, int32_t level, const double* r, double* e, int32_t nsteps) {
  Ctx* c = static_cast<Ctx*>(ctx);
  if (!c || !r || !e || nsteps < 0 || nsteps > MAX_NU) return MG_ERR_ARG;
  if (!c->setup_done) return fail(c, MG_ERR_STATE, "setup first");
  HostLevel* L = level_of(c, level);
  if (!L || L == &c->lev.back()) return fail(c, MG_ERR_ARG, "no smoother on this level");
  c->launches += launch_copy_masked(L->d, L->r, r, c->st);
  c->launches += launch_copy_masked(L->d, L->e, e, c->st);
  double* cur = L->e;
  for (int s = 0; s < nsteps; ++s) cur = smooth_step(c, *L, s, cur);
  c->launches += launch_copy(e, cur, L->d.ndof, c->st);
  CK(cudaGetLastError());
  return MG_OK;
}

int mg_local_correct(void* ctx, int32_t level, const double* res, double* e) {
  Ctx* c = static_cast<Ctx*>(ctx);
  if (!c || !res || !e) return MG_ERR_ARG;
  if (!c->setup_done) return fail(c, MG_ERR_STATE, "setup first");
  HostLevel* L = level_of(c, level);
  if (!L || L->kind != KIND_H) return fail(c, MG_ERR_ARG, "level has no interior dofs");
  c->launches += launch_lc_restrict(L->d, res, e, L->KIIinv, L->Pm, L->cbuf, true, false, c->st);
  CK(cudaGetLastError());
  return MG_OK;
}

int mg_restrict(void* ctx, int32_t level, const double* res, double* rc) {
  Ctx* c = static_cast<Ctx*>(ctx);
  if (!c || !res || !rc) return MG_ERR_ARG;
  if (!c->setup_done) return fail(c, MG_ERR_STATE, "setup first");
  HostLevel* L = level_of(c, level);
  if (!L || L->kind == KIND_COARSEST) return fail(c, MG_ERR_ARG, "no coarser level");
  const int li = (int)(L - &c->lev[0]);
  restrict_level(c, li, res, nullptr, false, rc, false);
  CK(cudaGetLastError());
  return c->comm_rc ? c->comm_rc : MG_OK;
}

int mg_prolong(void* ctx, int32_t level, const double* ec, double* e) {
  Ctx* c = static_cast<Ctx*>(ctx);
  if (!c || !ec || !e) return MG_ERR_ARG;
  if (!c->setup_done) return fail(c, MG_ERR_STATE, "setup first");
  HostLevel* L = level_of(c, level);
  if (!L || L->kind == KIND_COARSEST) return fail(c, MG_ERR_ARG, "no coarser level");
  const int li = (int)(L - &c->lev[0]);
  prolong_level(c, li, ec, e);
  CK(cudaGetLastError());
  return c->comm_rc ? c->comm_rc : MG_OK;
}

int mg_pcg_solve(void* ctx, const double* g, double* lambda, double rtol, int32_t maxit,
                 int32_t* iters, double* relres, int32_t* solve_status, double* resid_hist) {
  Ctx* c = static_cast<Ctx*>(ctx);
  if (!c || !g || !lambda || maxit < 1 || !(rtol > 0)) return MG_ERR_ARG;
  if (!c->setup_done) return fail(c, MG_ERR_STATE, "setup first");
  if (c->ns)
    return fail(c, MG_ERR_UNSUPPORTED,
                "PCG needs a symmetric operator: use mg_gmres_solve / mg_mg_solve");
  int it = 0, stt = 0;
  double rel = 0;
  RC(pcg_impl(c, g, lambda, rtol, maxit, &it, &rel, &stt, resid_hist));
  if (iters) *iters = it;
  if (relres) *relres = rel;
  if (solve_status) *solve_status = stt;
  return MG_OK;
}

int mg_mg_solve(void* ctx, const double* g, double* lambda, double tol, int32_t maxit,
                int32_t* iters, double* relres, int32_t* solve_status, double* resid_hist) {
  Ctx* c = static_cast<Ctx*>(ctx);
  if (!c || !g || !lambda || maxit < 1 || !(tol > 0)) return MG_ERR_ARG;
  if (!c->setup_done) return fail(c, MG_ERR_STATE, "setup first");
  int it = 0, st = 0;
  double rel = 0;
  RC(mgsolve_impl(c, g, lambda, tol, maxit, &it, &rel, &st, resid_hist));
  if (iters) *iters = it;
  if (relres) *relres = rel;
  if (solve_status) *solve_status = st;
  return MG_OK;
}

int mg_gmres_solve(void* ctx, const double* g, double* lambda, double tol, int32_t maxit,
                   double* basis, int32_t* iters, double* relres, int32_t* solve_status,
                   double* resid_hist) {
  Ctx* c = static_cast<Ctx*>(ctx);
  if (!c || !g || !lambda || !basis || maxit < 1 || !(tol > 0)) return MG_ERR_ARG;
  if (!c->setup_done) return fail(c, MG_ERR_STATE, "setup first");
  int it = 0, st = 0;
  double rel = 0;
  RC(gmres_impl(c, g, lambda, tol, maxit, basis, &it, &rel, &st, resid_hist));
  if (iters) *iters = it;
  if (relres) *relres = rel;
  if (solve_status) *solve_status = st;
  return MG_OK;
}

int mg_staging_bytes(const void* ctx, int32_t with_f, int32_t with_gD, size_t* bytes) {
  const Ctx* c = static_cast<const Ctx*>(ctx);
  if (!c || !bytes) return MG_ERR_ARG;
  const LevelDev& d = c->lev[0].d;
  const int nq = c->p + 4;
  size_t b = 0;
  b += align_up(d.ne * sizeof(double)) * 2 + align_up(d.ne);                 // K, tau, method
  b += align_up(d.ndof * sizeof(double)) * 2;                                // g, lambda
  if (with_f) b += align_up((size_t)d.ne * nq * nq * sizeof(double));
  if (with_gD) b += align_up((size_t)(2 * d.nx + 2 * d.ny) * nq * sizeof(double));
  *bytes = b;
  return MG_OK;
}

int mg_bind_staging(void* ctx, void* dev_ptr, size_t bytes) {
  Ctx* c = static_cast<Ctx*>(ctx);
  if (!c || !dev_ptr) return MG_ERR_ARG;
  if (reinterpret_cast<uintptr_t>(dev_ptr) & 255)
    return fail(c, MG_ERR_WORKSPACE, "staging must be 256-byte aligned");
  c->stg = static_cast<char*>(dev_ptr);
  c->stg_bytes = bytes;
  return MG_OK;
}

int mg_solve_host(void* ctx, const double* K_host, const int8_t* method_host,
                  const double* tau_host, const double* f_qp_host, double f_const,
                  const double* gD_qp_host, const mg_smoother_cfg* smoother, double rtol,
                  int32_t maxit, double* lambda_host, int32_t* iters, double* relres,
                  int32_t* solve_status) {
  Ctx* c = static_cast<Ctx*>(ctx);
  if (!c || !K_host || !method_host || !tau_host || !lambda_host || !smoother) return MG_ERR_ARG;
  if (c->ns) return fail(c, MG_ERR_UNSUPPORTED, "mg_solve_host runs PCG: symmetric contexts only");
  size_t need = 0;
  mg_staging_bytes(c, f_qp_host != nullptr, gD_qp_host != nullptr, &need);
  if (!c->stg || c->stg_bytes < need) return fail(c, MG_ERR_WORKSPACE, "staging not bound / too small");
  const LevelDev& d = c->lev[0].d;
  const int nq = c->p + 4;
  char* b = c->stg;
  size_t o = 0;
  auto take = [&](size_t bytes) {
    char* p = b + o;
    o += align_up(bytes);
    return p;
  };
  double* Kd = reinterpret_cast<double*>(take(d.ne * sizeof(double)));
  double* taud = reinterpret_cast<double*>(take(d.ne * sizeof(double)));
  int8_t* md = reinterpret_cast<int8_t*>(take(d.ne));
  double* gd = reinterpret_cast<double*>(take(d.ndof * sizeof(double)));
  double* lamd = reinterpret_cast<double*>(take(d.ndof * sizeof(double)));
  double* fd = f_qp_host ? reinterpret_cast<double*>(take((size_t)d.ne * nq * nq * sizeof(double)))
                         : nullptr;
  double* gDd = gD_qp_host
                    ? reinterpret_cast<double*>(take((size_t)(2 * d.nx + 2 * d.ny) * nq * sizeof(double)))
                    : nullptr;
  cudaStream_t st = c->st;
  CK(cudaMemcpyAsync(Kd, K_host, d.ne * sizeof(double), cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(taud, tau_host, d.ne * sizeof(double), cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(md, method_host, d.ne, cudaMemcpyHostToDevice, st));
  // f / g_D samples (the bulk of the upload) on the copy stream, overlapped with the
  // setup; it starts after everything already queued on st (staging reuse)
  const bool side_copy = (fd || gDd) && st != nullptr;
  if (side_copy) {
    if (!c->copy_st) {
      CK(cudaStreamCreateWithFlags(&c->copy_st, cudaStreamNonBlocking));
      CK(cudaEventCreateWithFlags(&c->copy_ev0, cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&c->copy_ev1, cudaEventDisableTiming));
    }
    CK(cudaEventRecord(c->copy_ev0, st));
    CK(cudaStreamWaitEvent(c->copy_st, c->copy_ev0, 0));
  }
  cudaStream_t cst = side_copy ? c->copy_st : st;
  if (fd)
    CK(cudaMemcpyAsync(fd, f_qp_host, (size_t)d.ne * nq * nq * sizeof(double),
                       cudaMemcpyHostToDevice, cst));
  if (gDd)
    CK(cudaMemcpyAsync(gDd, gD_qp_host, (size_t)(2 * d.nx + 2 * d.ny) * nq * sizeof(double),
                       cudaMemcpyHostToDevice, cst));
  if (side_copy) CK(cudaEventRecord(c->copy_ev1, c->copy_st));
  const int rs = mg_setup_dtn(c, Kd, md, taud, smoother);
  if (side_copy) CK(cudaStreamWaitEvent(st, c->copy_ev1, 0));
  RC(rs);
  RC(rhs_impl(c, fd, f_const, gDd, gd, nullptr));
  int it = 0, stt = 0;
  double rel = 0;
  RC(pcg_impl(c, gd, lamd, rtol, maxit, &it, &rel, &stt, nullptr));
  // full trace: free part + Dirichlet values (c->lamD is 0 off dOmega, lamd is 0 on it)
  c->launches += launch_add(lamd, c->lamD, d.ndof, st);
  CK(cudaMemcpyAsync(lambda_host, lamd, d.ndof * sizeof(double), cudaMemcpyDeviceToHost, st));
  RC(sync_st(c, st));
  if (iters) *iters = it;
  if (relres) *relres = rel;
  if (solve_status) *solve_status = stt;
  return MG_OK;
}

int mg_recover_volume(void* ctx, const double* lambda_full, const double* f_qp, double f_const,
                      double* q_out, const double* q_exact_qp, double* l2_err) {
  Ctx* c = static_cast<Ctx*>(ctx);
  if (!c || !lambda_full || !q_out) return MG_ERR_ARG;
  if (!c->setup_done) return fail(c, MG_ERR_STATE, "mg_setup_dtn must precede mg_recover_volume");
  HostLevel& F = c->lev[0];
  int grid = 0;
  c->launches += launch_recover(F.d, c->refdev, F.h, c->Kc, c->methc, c->tauc, lambda_full, f_qp,
                                f_const, q_out, q_exact_qp, c->part, &grid, c->st);
  if (q_exact_qp && l2_err) {
    reduce_scal(c, c->part, grid, c->sscal, 6, 0);   // sum over elements (and ranks)
    CK(cudaMemcpyAsync(c->pinned, c->sscal + 6, sizeof(double), cudaMemcpyDeviceToHost, c->st));
    RC(sync_st(c, c->st));
    *l2_err = std::sqrt(c->pinned[0]);
  }
  CK(cudaGetLastError());
  return c->comm_rc ? c->comm_rc : MG_OK;
}

int mg_num_levels(const void* ctx, int32_t* nlevels) {
  const Ctx* c = static_cast<const Ctx*>(ctx);
  if (!c || !nlevels) return MG_ERR_ARG;
  *nlevels = (int32_t)c->lev.size();
  return MG_OK;
}

int mg_level_info(const void* ctx, int32_t level, int32_t* nx, int32_t* ny, int32_t* p,
                  int64_t* ndof) {
  Ctx* c = const_cast<Ctx*>(static_cast<const Ctx*>(ctx));
  if (!c) return MG_ERR_ARG;
  HostLevel* L = level_of(c, level);
  if (!L) return MG_ERR_ARG;
  if (nx) *nx = L->d.nx;
  if (ny) *ny = L->d.ny;
  if (p) *p = L->d.p;
  if (ndof) *ndof = L->d.ndof;
  return MG_OK;
}

int mg_copy_element_dtn(const void* ctx, int32_t level, double* dst) {
  Ctx* c = const_cast<Ctx*>(static_cast<const Ctx*>(ctx));
  if (!c || !dst) return MG_ERR_ARG;
  if (!c->ws) return fail(c, MG_ERR_WORKSPACE, "no workspace bound");
  HostLevel* L = level_of(c, level);
  if (!L) return MG_ERR_ARG;
  c->launches += launch_packed_to_dense(L->d, dst, c->st);
  CK(cudaGetLastError());
  return MG_OK;
}

int mg_gather_element_dtn(const void* ctx, int32_t level, const int64_t* elems, int64_t n,
                          double* dst) {
  Ctx* c = const_cast<Ctx*>(static_cast<const Ctx*>(ctx));
  if (!c || !elems || !dst || n < 0) return MG_ERR_ARG;
  if (!c->ws) return fail(c, MG_ERR_WORKSPACE, "no workspace bound");
  HostLevel* L = level_of(c, level);
  if (!L) return MG_ERR_ARG;
  if (n == 0) return MG_OK;
  c->launches += launch_gather_dense(L->d, elems, n, dst, c->st);
  CK(cudaGetLastError());
  return MG_OK;
}

int mg_debug_set_element_dtn(void* ctx, int32_t level, const double* src) {
  Ctx* c = static_cast<Ctx*>(ctx);
  if (!c || !src) return MG_ERR_ARG;
  if (!c->ws) return fail(c, MG_ERR_WORKSPACE, "no workspace bound");
  HostLevel* L = level_of(c, level);
  if (!L) return MG_ERR_ARG;
  c->launches += launch_dense_to_packed(L->d, src, c->st);
  c->launches += launch_orbit_pack(L->d, c->st);
  CK(cudaGetLastError());
  // the apply kernels prefetch S_T before their dependency wait (PDL): make the
  // new S_T complete before any later launch
  RC(sync_st(c, c->st));
  return MG_OK;
}

int mg_level_lambda_max(const void* ctx, int32_t level, double* lam) {
  Ctx* c = const_cast<Ctx*>(static_cast<const Ctx*>(ctx));
  if (!c || !lam) return MG_ERR_ARG;
  HostLevel* L = level_of(c, level);
  if (!L) return MG_ERR_ARG;
  *lam = 0.0;
  if (c->sm.kind != MG_SMOOTH_CHEBYSHEV || L == &c->lev.back()) return MG_OK;
  CK(cudaMemcpyAsync(lam, L->lam, sizeof(double), cudaMemcpyDeviceToHost, c->st));
  RC(sync_st(c, c->st));
  return MG_OK;
}

int mg_last_launch_count(const void* ctx, int64_t* launches) {
  const Ctx* c = static_cast<const Ctx*>(ctx);
  if (!c || !launches) return MG_ERR_ARG;
  *launches = c->last_solve_launches;
  return MG_OK;
}

int mg_total_launch_count(const void* ctx, int64_t* launches) {
  const Ctx* c = static_cast<const Ctx*>(ctx);
  if (!c || !launches) return MG_ERR_ARG;
  *launches = c->launches;
  return MG_OK;
}

int mg_check_invariants(void* ctx, double* report) {
  Ctx* c = static_cast<Ctx*>(ctx);
  if (!c || !report) return MG_ERR_ARG;
  if (!c->setup_done) return fail(c, MG_ERR_STATE, "setup first");
  cudaStream_t st = c->st;
  double* out = c->part;   // [0] worst constant-mode ratio, [1] non-finite count
  CK(cudaMemsetAsync(out, 0, 2 * sizeof(double), st));
  const int nlev = (int)c->lev.size();
  for (int li = 0; li < nlev; ++li) {
    const HostLevel& L = c->lev[li];
    c->launches += launch_check_maps(L.d, out, st);
    if (li < nlev - 1)
      c->launches += launch_check_finite(L.d.Dinv, L.d.nedge * L.d.k1 * L.d.k1, out, st);
    if (L.d.orb) {
      c->launches += launch_check_finite(L.d.So, (int64_t)2 * L.d.nchunk * d4_norb(L.d.p) * 32, out, st);
      c->launches += launch_check_finite(L.d.Dso, L.d.nedge * d4_ncs(L.d.p), out, st);
    }
  }
  c->launches += launch_check_finite(c->A1inv, (int64_t)c->nf * c->nf, out, st);
  CK(cudaMemcpyAsync(c->pinned, out, 2 * sizeof(double), cudaMemcpyDeviceToHost, st));
  RC(sync_st(c, st));
  report[0] = c->pinned[0];
  report[1] = c->pinned[1];
  report[2] = -1.0;
  report[3] = 0.0;
  // the two-colour apply against an atomic scatter on the finest level (one GPU)
  if (!partitioned(c) && !c->ns) {
    HostLevel& F = c->lev[0];
    const int64_t n = F.d.ndof;
    const int vg = vec_grid(n);
    c->launches += launch_pow_init(F.d, c->pv, st);   // deterministic v_i = 1 + (i mod 7)/7
    apply_full(c, F, c->pv, c->ap, nullptr);
    CK(cudaMemsetAsync(F.w, 0, n * sizeof(double), st));
    c->launches += launch_apply_atomic(F.d, c->pv, F.w, st);
    c->launches += launch_axpby(1.0, F.w, -1.0, c->ap, F.w, n, st);   // w = atomic - coloured
    c->launches += launch_dot(F.w, F.w, n, c->part, vg, st);
    c->launches += launch_reduce(c->part, vg, c->sscal, 10, 0, nullptr, st);
    c->launches += launch_dot(c->ap, c->ap, n, c->part, vg, st);
    c->launches += launch_reduce(c->part, vg, c->sscal, 11, 0, nullptr, st);
    CK(cudaMemsetAsync(F.w, 0, n * sizeof(double), st));   // the work vector holds 0 on dOmega
    CK(cudaMemcpyAsync(c->pinned, c->sscal + 10, 2 * sizeof(double), cudaMemcpyDeviceToHost, st));
    RC(sync_st(c, st));
    report[2] = c->pinned[1] > 0 ? std::sqrt(c->pinned[0] / c->pinned[1]) : 0.0;
  }
  CK(cudaGetLastError());
  if (report[1] > 0) return fail(c, MG_ERR_STATE, "invariants: non-finite entries in the hierarchy");
  if (report[0] > 1e-12)
    return fail(c, MG_ERR_STATE, "invariants: an element map does not annihilate constants");
  if (report[2] > 1e-13)
    return fail(c, MG_ERR_STATE, "invariants: coloured apply differs from the atomic scatter");
  return MG_OK;
}

int mg_set_option(void* ctx, int32_t key, int64_t value) {
  Ctx* c = static_cast<Ctx*>(ctx);
  if (!c) return MG_ERR_ARG;
  if (key == MG_OPT_SWEEP) {
    if (value < -1 || value > 1) return fail(c, MG_ERR_ARG, "MG_OPT_SWEEP: -1, 0 or 1");
    for (auto& L : c->lev) L.d.sweep = (int)value;
  } else if (key == MG_OPT_COMM_TIMEOUT_MS) {
    if (value < 1) return fail(c, MG_ERR_ARG, "MG_OPT_COMM_TIMEOUT_MS must be >= 1");
    c->comm_timeout_s = (double)value * 1e-3;
    return MG_OK;
  } else if (key == MG_OPT_GATHER_NE) {
    if (value < 0) return fail(c, MG_ERR_ARG, "MG_OPT_GATHER_NE must be >= 0");
    c->gather_ne = value;
    plan_gather(c);
  } else if (key == MG_OPT_KEEP_FINE_MAPS) {
    if (value < 0 || value > 1) return fail(c, MG_ERR_ARG, "MG_OPT_KEEP_FINE_MAPS: 0 or 1");
    c->keep_fine_maps = value != 0;
  } else if (key == MG_OPT_APPLY_GRID_CAP) {
    if (value < 0 || value > (1 << 20)) return fail(c, MG_ERR_ARG, "MG_OPT_APPLY_GRID_CAP out of range");
    for (auto& L : c->lev) L.d.grid_cap = (int)value;
  } else {
    return fail(c, MG_ERR_ARG, "unknown option");
  }
  drop_graphs(c);   // (the tail kernels copy the level descriptors at every launch)
  return MG_OK;
}

int mg_set_use_graphs(void* ctx, int32_t on) {
  Ctx* c = static_cast<Ctx*>(ctx);
  if (!c) return MG_ERR_ARG;
  c->use_graphs = on != 0;
  return MG_OK;
}

const char* mg_last_error(const void* ctx) {
  const Ctx* c = static_cast<const Ctx*>(ctx);
  return c ? c->last_err.c_str() : "null context";
}

int64_t mg_last_error_index(const void* ctx) {
  const Ctx* c = static_cast<const Ctx*>(ctx);
  return c ? c->last_idx : -1;
}

void mg_destroy(void* ctx) {
  Ctx* c = static_cast<Ctx*>(ctx);
  if (!c) return;
  drop_graphs(c);
  delete c->comm;
  for (auto sx : c->side) cudaStreamDestroy(sx);
  for (auto ex : c->side_ev) cudaEventDestroy(ex);
  for (auto ex : c->fork_evs) cudaEventDestroy(ex);
  if (c->copy_st) cudaStreamDestroy(c->copy_st);
  if (c->cst) cudaStreamDestroy(c->cst);
  if (c->evB) cudaEventDestroy(c->evB);
  if (c->evC) cudaEventDestroy(c->evC);
  if (c->copy_ev0) cudaEventDestroy(c->copy_ev0);
  if (c->copy_ev1) cudaEventDestroy(c->copy_ev1);
  if (c->pinned) cudaFreeHost(c->pinned);
  delete c;
}

}  // extern "C"
