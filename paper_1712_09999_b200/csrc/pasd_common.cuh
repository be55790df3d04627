// pasd_common.cuh — shared device-side types of the B200 PASD solver.
//
// Every mode-n operation of the reference works on the mode-n unfolding
// (tensor.cpp:98-127).  Instead of materialising unfoldings we view the
// first-index-fastest tensor, for mode n, as a 3-way array (inner, I_n, outer)
// with inner = prod_{l<n} I_l and outer = prod_{l>n} I_l: entry (p, i, q) sits
// at p + inner*i + inner*I_n*q and is element (i, kappa = p + inner*q) of the
// unfolding.  All per-mode kernels are written against that view, so any
// order N (<= PASD_MAX_ORDER) is supported without copies.
#pragma once
#include <cstdint>

#define PASD_MAX_ORDER 8
#define PASD_MAX_RANK 64

namespace pasd {

// Per-mode geometry and device pointers (passed by value to kernels).
struct ModeDev {
  int64_t inner;    // prod of lower dims
  int64_t I;        // I_n
  int64_t outer;    // prod of higher dims
  int64_t J;        // inner * outer = S / I_n (unfolding columns)
  int64_t Ifull;    // full I_n: leading dimension of U, UM, Wt (== I unless the mode is slab-sharded)
  int64_t ioff;     // offset of local index 0 within [0, Ifull) (slab begin for the sharded mode)
  int R;            // R_n
  int mode;         // 0-based
  double lambda;    // lambda_n (SVT weight)
  // State (all column-major where matrices):
  double* U;        // I x R   current basis U_n
  double* UM;       // I x R   U_n * M_n (refold operator)
  double* M;        // R x R   SVT map: V_n = M_n * A_n
  double* A;        // inner x R x outer: A_n = U_n^T G_(n), kappa-major per r
  double* Wt;       // I x R   Wtilde_n = G_(n)^{next} A_n^T
  double* Wpart;    // [nkc][I][R] partial Wtilde
  double* Gram;     // R x R   A_n A_n^T
  double* Gpart;    // [nkc][R][R] partial Gram
  double* sig;      // R       singular values of A_n (from the Gram eigen-solve)
  double* P;        // R x R   eigenvectors of Gram_n (left singular vectors of A_n); warm start
  double* Qp;       // R x R   right rotation of the last Procrustes solve; warm start
  double* gpart;    // [nkc * nib] partial ||G||_F^2 of the W pass
  double* scratch;  // 3 x I x R scratch for the polar solve
  int nkc_w;        // kappa chunks of the W pass
  int nib_w;        // i blocks of the W pass
  int nkc_g;        // kappa chunks of the Gram pass
  int refine_ok;    // A_n complete on this rank (not a slab partial): the SVT may refine from A_n
};

// Scalars of the device-resident ADMM loop (read by every kernel so that an
// iteration can be replayed from a CUDA graph without host involvement).
struct Ctl {
  double mu;             // penalty for the running iteration (pasd.cpp:169)
  double mu_used_last;   // mu used by the last completed iteration
  double rho, mu_max, eps;
  int iter;              // completed iterations
  int maxiter;
  int done;              // 1 = loop finished (converged, maxiter or NaN)
  int converged;
  int nan_flag;
  int ecur;              // index of the current E buffer (double buffering)
  int fixed_iters;
  int order;
  double resid[PASD_MAX_ORDER];
  double gnorm2[PASD_MAX_ORDER];   // ||G_n^{next}||_F^2 for the degenerate test
  double vnorm2[PASD_MAX_ORDER];   // ||V_n||_F^2 = sum_i (sigma_i - tau)_+^2
  double nuclear[PASD_MAX_ORDER];  // ||V_n||_* = sum_i (sigma_i - tau)_+
  int keep[PASD_MAX_ORDER];        // SVT rank kept
  int degenerate[PASD_MAX_ORDER];  // last Procrustes took the degenerate branch
  int polar_rank[PASD_MAX_ORDER];  // numerical rank of W in the last Procrustes
};

}  // namespace pasd
