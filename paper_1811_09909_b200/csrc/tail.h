// Parameters of the cluster-resident coarse tail of the V-cycle (k_coarse.cu).
#pragma once
#include "kernels.cuh"

namespace mgdtn {

constexpr int MAX_TAIL = 16;

struct TailLevel {
  LevelDev d;
  double *r, *e, *w, *dv;        // level vectors (r input, e output of B_k)
  double *KIIinv, *Pm, *cbuf;    // per-macro A_II^-1, P_M, restriction buffer (h-levels)
  double* lam;                   // Chebyshev lambda_max estimate (device scalar)
};

struct TailParams {
  int nlev;              // levels in the tail; lev[nlev-1] is the coarsest (direct solve)
  int smem_doubles;      // k_coarse_tail: shared-memory copies of every tail vector (0 = off)
  int nu_pre, nu_post;   // at the top tail level; x 2 per coarser level if nu_doubling
  int nu_doubling;        // beta = 2 smoothing-step doubling
  int first_fused;       // lev[0]'s first pre-smoothing step was done by the upstream restriction
  const int* fidx;       // coarsest free-dof map and explicit inverse
  int nf;
  const double* A1inv;
  TailLevel lev[MAX_TAIL];
};

int launch_coarse_tail(const TailParams& P, cudaStream_t st);
// B_tail as a dense matrix (setup): column j = the tail V-cycle applied to the
// unit vector on free dof tfidx[j] of the top tail level; Bt row-major [nf][nf]
int launch_tail_basis(const TailParams& P, const int* tfidx, int nf, double* Bt, cudaStream_t st);
// e = B_tail r on the top tail level's free dofs (warp per row, deterministic)
int launch_tail_dense(const int* tfidx, int nf, const double* Bt, const double* r, double* e,
                      cudaStream_t st);
// Chebyshev lambda_max (Q11) of every tail level but the coarsest, one launch;
// part: >= cluster-size doubles of scratch.
int launch_tail_lmax(const TailParams& P, int iters, double safety, double ratio, int nu_max,
                     double* part, cudaStream_t st);
int tail_cluster_size();

}  // namespace mgdtn
