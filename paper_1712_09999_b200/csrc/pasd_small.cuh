// pasd_small.cuh — the r x r solves of one PASD iteration, one CTA per mode.
//
// The reference runs LAPACK dgesdd twice per mode and iteration
// (linops.cpp:62 via svt, linops.cpp:83, and procrustes, linops.cpp:98-103).
// Both reduce to R_n x R_n symmetric eigenproblems:
//   * SVT:  A_n = U_n^T G_(n) (R x J).  eig(A A^T) = P diag(sigma^2) P^T, so
//           SVT_tau(A) = P diag((sigma-tau)_+/sigma) P^T A = M_n A_n  (the
//           kept set is sigma_i > tau strictly, linops.cpp:85).
//   * Procrustes: W = G V^T (I x R).  polar(W) = u v^T of its thin SVD.  We
//           take two Gram/Jacobi passes (eig(W^T W) -> rotate -> re-Gram) so
//           small singular directions are resolved to working accuracy, and
//           complete numerically-null directions deterministically from the
//           previous basis (the reference inherits dgesdd's rounding-noise
//           completion there; any orthonormal completion is a valid polar
//           factor — see DESIGN.md "parity floor").
// Eigenproblems use a CTA-parallel cyclic Jacobi (round-robin ordering, R/2
// disjoint rotations per step) in shared memory.
#pragma once
#include <cooperative_groups.h>

#include "pasd_kernels.cuh"

namespace pasd {

#ifndef PASD_SMALL_THREADS
#define PASD_SMALL_THREADS 512
#endif
constexpr int kSmallThreads = PASD_SMALL_THREADS;

// Shared-memory workspace of one small-solve CTA (dynamic smem).
struct SmallWs {
  int Rp, ld;
  double* S;    // Rp x ld   working matrix (row-major)
  double* V;    // Rp x ld   eigenvectors / rotations
  double* Q;    // Rp x ld   accumulated rotation / misc
  double* Z;    // Rp x ld   misc
  double* T64;  // 64 x ld   row staging of the tall-skinny products
  double* cs;   // Rp/2
  double* sn;   // Rp/2
  double* lam;  // Rp
  double* red;  // 32
  double* cl;   // Rp + 8  vector partials of the cluster reductions (read remotely)
  int* pq;      // Rp
  int* perm;    // Rp
};

__host__ __device__ inline size_t small_ws_bytes(int R) {
  const int Rp = R + (R & 1);
  const int ld = Rp + 1;
  return sizeof(double) * (4 * (size_t)Rp * ld + 64 * (size_t)ld + Rp + Rp + 32 + Rp + 8) +
         sizeof(int) * (2 * (size_t)Rp) + 64;
}

__device__ inline SmallWs make_ws(int R, void* base) {
  SmallWs w;
  w.Rp = R + (R & 1);
  w.ld = w.Rp + 1;
  double* d = reinterpret_cast<double*>(base);
  const size_t mat = (size_t)w.Rp * w.ld;
  w.S = d;
  w.V = d + mat;
  w.Q = d + 2 * mat;
  w.Z = d + 3 * mat;
  w.T64 = d + 4 * mat;
  w.cs = w.T64 + 64 * (size_t)w.ld;
  w.sn = w.cs + w.Rp / 2;
  w.lam = w.sn + w.Rp / 2;
  w.red = w.lam + w.Rp;
  w.cl = w.red + 32;
  w.pq = reinterpret_cast<int*>(w.cl + w.Rp + 8);
  w.perm = w.pq + w.Rp;
  return w;
}

#ifndef PASD_POLAR_ONEPASS
#define PASD_POLAR_ONEPASS 1e-3  // max relative off-diagonal of (W Qp)^T (W Qp) for the one-pass Procrustes
#endif
#ifndef PASD_JACOBI_QUAD
#define PASD_JACOBI_QUAD 1e-10
#endif

__device__ __forceinline__ int rr_pos(int m, int round, int Rp) {
  return m == 0 ? 0 : 1 + (m - 1 + round) % (Rp - 1);
}

// Cyclic parallel Jacobi on the symmetric n x n matrix in ws.S (row-major, ld).
// On exit diag(S) holds eigenvalues, ws.V (row-major) the eigenvectors as
// columns: S_in = V diag V^T.  Then sorts eigenpairs descending into
// lam[0..n) and the columns of V.
__device__ void cta_jacobi_eig(SmallWs& ws, int n, int tag = 0) {
  const int Rp = ws.Rp, ld = ws.ld, tid = threadIdx.x, nt = blockDim.x;
  double* S = ws.S;
  double* V = ws.V;
  // pad odd n with an isolated zero row/column
  for (int idx = tid; idx < Rp * Rp; idx += nt) {
    const int r = idx / Rp, c = idx % Rp;
    if (r >= n || c >= n) S[r * ld + c] = 0.0;
    V[r * ld + c] = (r == c) ? 1.0 : 0.0;
  }
  __syncthreads();
  const int npairs = Rp / 2;
  // this thread's block items (ja, jb) and V items (pair j, row k), fixed for the call
  constexpr int JB_MAX = (PASD_MAX_RANK / 2 * PASD_MAX_RANK / 2 + kSmallThreads - 1) / kSmallThreads;
  constexpr int JV_MAX = (PASD_MAX_RANK / 2 * PASD_MAX_RANK + kSmallThreads - 1) / kSmallThreads;
  int bja[JB_MAX], bjb[JB_MAX], vj[JV_MAX], vk[JV_MAX];
#pragma unroll
  for (int u = 0; u < JB_MAX; ++u) {
    const int bidx = tid + u * nt;
    bja[u] = bidx < npairs * npairs ? bidx / npairs : -1;
    bjb[u] = bidx < npairs * npairs ? bidx % npairs : 0;
  }
#pragma unroll
  for (int u = 0; u < JV_MAX; ++u) {
    const int idx = tid + u * nt;
    vj[u] = idx < npairs * Rp ? idx / Rp : -1;
    vk[u] = idx < npairs * Rp ? idx % Rp : 0;
  }
  __shared__ int rotated, big;
  for (int sweep = 0; sweep < 30 && Rp > 1; ++sweep) {
    if (tid == 0) rotated = big = 0;
    __syncthreads();
    for (int round = 0; round < Rp - 1; ++round) {
      for (int j = tid; j < npairs; j += nt) {
        const int a = rr_pos(j, round, Rp), b = rr_pos(Rp - 1 - j, round, Rp);
        const int p = a < b ? a : b, q = a < b ? b : a;
        const double apq = S[p * ld + q];
        const double app = S[p * ld + p], aqq = S[q * ld + q];
        double c = 1.0, s = 0.0;
        // Skip rotations below rounding level (relative-accuracy criterion for
        // symmetric PSD Jacobi); a sweep without rotations terminates.
        if (fabs(apq) > 2.2e-16 * sqrt(fabs(app) * fabs(aqq)) && fabs(apq) > 1e-300) {
          const double zeta = (aqq - app) / (2.0 * apq);
          const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
          c = 1.0 / sqrt(1.0 + t * t);
          s = t * c;
          rotated = 1;
          if (fabs(apq) > PASD_JACOBI_QUAD * sqrt(fabs(app) * fabs(aqq))) big = 1;
        }
        ws.cs[j] = c;
        ws.sn[j] = s;
        ws.pq[2 * j] = p;
        ws.pq[2 * j + 1] = q;
      }
      __syncthreads();
      // Apply the round's disjoint rotations: S <- J^T S J block by block (the
      // 2 x 2 block of pairs (ja, jb) depends only on itself; rows first, then
      // columns, the same operation order as separate row and column passes)
      // and V <- V J.  One barrier per round instead of two.  Work items are
      // assigned once per call (no integer divisions inside the rounds).
#pragma unroll
      for (int u = 0; u < JB_MAX; ++u) {
        if (bja[u] < 0) continue;
        const int ja = bja[u], jb = bjb[u];
        const double sa = ws.sn[ja], sb = ws.sn[jb];
        if (sa == 0.0 && sb == 0.0) continue;
        const double ca = ws.cs[ja], cb = ws.cs[jb];
        const int pa = ws.pq[2 * ja], qa = ws.pq[2 * ja + 1], pb = ws.pq[2 * jb], qb = ws.pq[2 * jb + 1];
        double a00 = S[pa * ld + pb], a01 = S[pa * ld + qb], a10 = S[qa * ld + pb], a11 = S[qa * ld + qb];
        if (sa != 0.0) {  // rows pa, qa
          const double r00 = ca * a00 - sa * a10, r10 = sa * a00 + ca * a10;
          const double r01 = ca * a01 - sa * a11, r11 = sa * a01 + ca * a11;
          a00 = r00; a10 = r10; a01 = r01; a11 = r11;
        }
        if (sb != 0.0) {  // columns pb, qb
          const double c00 = cb * a00 - sb * a01, c01 = sb * a00 + cb * a01;
          const double c10 = cb * a10 - sb * a11, c11 = sb * a10 + cb * a11;
          a00 = c00; a01 = c01; a10 = c10; a11 = c11;
        }
        S[pa * ld + pb] = a00;
        S[pa * ld + qb] = a01;
        S[qa * ld + pb] = a10;
        S[qa * ld + qb] = a11;
      }
#pragma unroll
      for (int u = 0; u < JV_MAX; ++u) {  // columns p, q of V
        if (vj[u] < 0) continue;
        const int j = vj[u], k = vk[u];
        const double s = ws.sn[j];
        if (s == 0.0) continue;
        const int p = ws.pq[2 * j], q = ws.pq[2 * j + 1];
        const double c = ws.cs[j];
        const double va = V[k * ld + p], vb = V[k * ld + q];
        V[k * ld + p] = c * va - s * vb;
        V[k * ld + q] = s * va + c * vb;
      }
      __syncthreads();
    }
    // Converged: no rotation at all, or only rotations so small (relative
    // off-diagonal <= PASD_JACOBI_QUAD) that the quadratic convergence of the
    // cyclic sweep leaves nothing above the rounding threshold for another one
    // (saves the confirming sweep).
    if (rotated == 0 || big == 0) {
#ifdef PASD_DEBUG_SWEEPS
      if (tid == 0) printf("jacobi n=%d block=%d tag=%d sweeps=%d\n", n, blockIdx.x, tag, sweep + 1);
#endif
      break;
    }
    __syncthreads();
  }
  // sort descending (stable on index): perm[rank] = j
  for (int j = tid; j < n; j += nt) {
    const double lj = S[j * ld + j];
    int rank = 0;
    for (int i = 0; i < n; ++i) {
      const double li = S[i * ld + i];
      rank += (li > lj) || (li == lj && i < j);
    }
    ws.perm[rank] = j;
  }
  __syncthreads();
  for (int j = tid; j < n; j += nt) ws.lam[j] = S[ws.perm[j] * ld + ws.perm[j]];
  // sorted eigenvectors into Z (row-major, column j = eigenvector j), then back to V
  for (int idx = tid; idx < n * n; idx += nt) {
    const int r = idx / n, j = idx % n;
    ws.Z[r * ld + j] = V[r * ld + ws.perm[j]];
  }
  __syncthreads();
  for (int idx = tid; idx < n * n; idx += nt) {
    const int r = idx / n, j = idx % n;
    V[r * ld + j] = ws.Z[r * ld + j];
  }
  __syncthreads();
}

// Warm start: load the previous rotation Pg (R x R, global column-major) into
// ws.Q and replace S by Q^T S Q (uses ws.Z).  After cta_jacobi_eig, call
// cta_warm_finish to turn the Jacobi rotation V into Q V.
__device__ void cta_warm_start(SmallWs& ws, int R, const double* Pg) {
  const int tid = threadIdx.x, nt = blockDim.x, ld = ws.ld;
  for (int idx = tid; idx < R * R; idx += nt) ws.Q[(idx % R) * ld + idx / R] = Pg[idx];
  __syncthreads();
  for (int idx = tid; idx < R * R; idx += nt) {  // Z = S Q
    const int r = idx / R, c = idx % R;
    double a = 0.0;
    for (int k = 0; k < R; ++k) a = fma(ws.S[r * ld + k], ws.Q[k * ld + c], a);
    ws.Z[r * ld + c] = a;
  }
  __syncthreads();
  for (int idx = tid; idx < R * R; idx += nt) {  // S = Q^T Z
    const int r = idx / R, c = idx % R;
    double a = 0.0;
    for (int k = 0; k < R; ++k) a = fma(ws.Q[k * ld + r], ws.Z[k * ld + c], a);
    ws.S[r * ld + c] = a;
  }
  __syncthreads();
  for (int idx = tid; idx < R * R; idx += nt) {  // exact symmetry
    const int r = idx / R, c = idx % R;
    if (r < c) {
      const double v = 0.5 * (ws.S[r * ld + c] + ws.S[c * ld + r]);
      ws.S[r * ld + c] = v;
      ws.S[c * ld + r] = v;
    }
  }
  __syncthreads();
}

__device__ void cta_warm_finish(SmallWs& ws, int R) {  // V <- Q V
  const int tid = threadIdx.x, nt = blockDim.x, ld = ws.ld;
  for (int idx = tid; idx < R * R; idx += nt) {
    const int r = idx / R, c = idx % R;
    double a = 0.0;
    for (int k = 0; k < R; ++k) a = fma(ws.Q[r * ld + k], ws.V[k * ld + c], a);
    ws.Z[r * ld + c] = a;
  }
  __syncthreads();
  for (int idx = tid; idx < R * R; idx += nt) ws.V[(idx / R) * ld + idx % R] = ws.Z[(idx / R) * ld + idx % R];
  __syncthreads();
}

// out(R x R2, smem row-major ld) = X^T Y with X (I x R), Y (I x R2) global column-major.
// Rows of X and Y stream through shared memory in 32-row chunks; each thread
// owns up to GT_MAX output entries (tid, tid + nt, ...) in registers, so the
// FMA chains of different entries interleave (the small solves are latency
// bound).  Per entry the sum still runs over i in ascending order from 0.
constexpr int GT_MAX = (PASD_MAX_RANK * PASD_MAX_RANK + kSmallThreads - 1) / kSmallThreads;
// X, Y: `I` rows with column stride ldg (a row block of an ldg-row matrix).
__device__ void cta_gram_tn(const double* X, const double* Y, int64_t I, int64_t ldg, int R, int R2, double* out,
                            int ld, double* stage /* 2 x 32 x ld */) {
  const int tid = threadIdx.x, nt = blockDim.x;
  const int ne = R * R2;
  double* Xs = stage;
  double* Ys = stage + 32 * ld;
  double acc[GT_MAX];
  int ro[GT_MAX], so[GT_MAX];
#pragma unroll
  for (int e = 0; e < GT_MAX; ++e) {
    const int idx = tid + e * nt;
    acc[e] = 0.0;
    ro[e] = idx < ne ? idx / R2 : 0;
    so[e] = idx < ne ? idx % R2 : 0;
  }
  for (int64_t i0 = 0; i0 < I; i0 += 32) {
    const int ic = (int)imin64(32, I - i0);
    for (int idx = tid; idx < 32 * R; idx += nt) {
      const int il = idx % 32, r = idx / 32;
      Xs[il * ld + r] = il < ic ? X[i0 + il + ldg * r] : 0.0;
    }
    for (int idx = tid; idx < 32 * R2; idx += nt) {
      const int il = idx % 32, r = idx / 32;
      Ys[il * ld + r] = il < ic ? Y[i0 + il + ldg * r] : 0.0;
    }
    __syncthreads();
    for (int il = 0; il < ic; ++il) {
#pragma unroll
      for (int e = 0; e < GT_MAX; ++e)
        if (tid + e * nt < ne) acc[e] = fma(Xs[il * ld + ro[e]], Ys[il * ld + so[e]], acc[e]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int e = 0; e < GT_MAX; ++e)
    if (tid + e * nt < ne) out[ro[e] * ld + so[e]] = acc[e];
  __syncthreads();
}

// out (I x R2, col-major) = X (I x R, col-major) B (R x R2, smem row-major, ld).
// 64-row chunks of X are staged in shared memory with coalesced loads; thread
// (q = tid % 16, column group tid / 16) forms the 4 rows q, q+16, q+32, q+48
// of up to MN_MAXC columns c, c + nt/16, ... (16 independent accumulators;
// each X value is reused across its columns, each B value across its rows).
// The sum over r runs in index order from 0 (same result as an unstaged loop).
// `stage`: 64 x ld doubles.
constexpr int MN_MAXC = (PASD_MAX_RANK + kSmallThreads / 16 - 1) / (kSmallThreads / 16);
// X and out: `I` rows with column stride ldg.
__device__ void cta_mul_nn(const double* X, int64_t I, int64_t ldg, int R, const double* B, int ld, int R2,
                           double* out, double* stage) {
  const int tid = threadIdx.x, nt = blockDim.x;
  const int q = tid & 15, cg = tid >> 4, ncg = nt >> 4;
  for (int64_t i0 = 0; i0 < I; i0 += 64) {
    const int ic = (int)imin64(64, I - i0);
    for (int idx = tid; idx < 64 * R; idx += nt) {
      const int il = idx & 63, r = idx >> 6;
      stage[il * ld + r] = il < ic ? X[i0 + il + ldg * r] : 0.0;
    }
    __syncthreads();
    double a[MN_MAXC][4];
#pragma unroll
    for (int k = 0; k < MN_MAXC; ++k) a[k][0] = a[k][1] = a[k][2] = a[k][3] = 0.0;
    for (int r = 0; r < R; ++r) {
      const double x0 = stage[q * ld + r], x1 = stage[(q + 16) * ld + r];
      const double x2 = stage[(q + 32) * ld + r], x3 = stage[(q + 48) * ld + r];
#pragma unroll
      for (int k = 0; k < MN_MAXC; ++k) {
        const int c = cg + k * ncg;
        if (c < R2) {
          const double b = B[r * ld + c];
          a[k][0] = fma(x0, b, a[k][0]);
          a[k][1] = fma(x1, b, a[k][1]);
          a[k][2] = fma(x2, b, a[k][2]);
          a[k][3] = fma(x3, b, a[k][3]);
        }
      }
    }
#pragma unroll
    for (int k = 0; k < MN_MAXC; ++k) {
      const int c = cg + k * ncg;
      if (c < R2) {
        double* o = out + i0 + ldg * c;
        if (q < ic) o[q] = a[k][0];
        if (q + 16 < ic) o[q + 16] = a[k][1];
        if (q + 32 < ic) o[q + 32] = a[k][2];
        if (q + 48 < ic) o[q + 48] = a[k][3];
      }
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// Cluster-parallel small solves.  Each mode is one thread-block cluster of
// kSmallCluster CTAs (one per SM).  The tall-skinny I_n x R products run on
// row blocks (CTA c owns rows [lo, hi)); R x R Gram matrices and column norms
// are reduced through distributed shared memory in cluster-rank order, so every
// CTA holds bit-identical totals and runs the same R x R Jacobi redundantly
// (no broadcast needed, results independent of the cluster size only up to
// the summation order of the partials).
#ifndef PASD_SMALL_CLUSTER
#define PASD_SMALL_CLUSTER 8
#endif
constexpr int kSmallCluster = PASD_SMALL_CLUSTER;

struct RowBlock {
  int64_t lo, rows;
};
__device__ inline RowBlock row_block(int64_t I, int crank) {
  const int64_t chunk = (I + kSmallCluster - 1) / kSmallCluster;
  const int64_t lo = imin64(I, chunk * crank), hi = imin64(I, lo + chunk);
  return {lo, hi - lo};
}

// dst[r * ld + c] = sum over cluster ranks (in rank order) of src[r * ld + c]
// (src: this CTA's partial in shared memory).  Ends with a cluster barrier, so
// src may be reused afterwards.
__device__ void cluster_sum_mat(const double* src, double* dst, int R, int R2, int ld) {
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  cl.sync();  // every partial written
  for (int idx = threadIdx.x; idx < R * R2; idx += blockDim.x) {
    const int r = idx / R2, c = idx - r * R2;
    double a = 0.0;
    for (int q = 0; q < kSmallCluster; ++q) a += cl.map_shared_rank(src, q)[r * ld + c];
    dst[r * ld + c] = a;
  }
  cl.sync();  // every remote read done
}

// ---------------------------------------------------------------------------
// Refinement of numerically unresolved small singular values of A (R x J).
// sigma_i^2 from eig(A A^T) carry an absolute error ~eps sigma_1^2, so a
// sigma_i below ~1e-5 sigma_1 is not resolved by the Gram; when the SVT
// threshold is that small too (late iterations: tau = lambda/mu with mu -> 1e10)
// the keep test sigma > tau (linops.cpp:85) and the factor (sigma - tau)/sigma
// would act on rounding noise where dgesdd on A itself resolves them.  The last
// k eigenvectors P_s (R x k) are refined from A: B = P_s^T A (k x J) has rows
// sigma_i v_i^T + O(eps sigma_1), so eig(B B^T) (k x k, Jacobi) gives them to
// relative accuracy ~eps sigma_1 / sigma_i.  Every CTA of the cluster forms the
// partial B B^T of its column block, the partials are summed through DSMEM in
// rank order (bit-identical on every CTA) and each CTA runs the same k x k
// Jacobi.  On entry ws.V / ws.lam hold the first pass (descending); on exit the
// refined ones.  Uses ws.Q, ws.Z, ws.T64.
__device__ void svt_refine_small(SmallWs& ws, const ModeDev& m, int R, int k, int crank) {
  const int tid = threadIdx.x, nt = blockDim.x, ld = ws.ld, r0 = R - k;
  // P (first pass) -> Q; first-pass eigenvalues of the kept-large part -> T64 row 63
  for (int idx = tid; idx < R * R; idx += nt) ws.Q[(idx / R) * ld + idx % R] = ws.V[(idx / R) * ld + idx % R];
  __syncthreads();
  double* lam_saved = ws.T64 + 63 * ld;
  for (int j = tid; j < R; j += nt) lam_saved[j] = ws.lam[j];
  // this CTA's columns of A
  const int64_t chunk = (m.J + kSmallCluster - 1) / kSmallCluster;
  const int64_t c_lo = imin64(m.J, chunk * crank), c_hi = imin64(m.J, c_lo + chunk);
  constexpr int KE = (PASD_MAX_RANK * (PASD_MAX_RANK + 1) / 2 + kSmallThreads - 1) / kSmallThreads;
  const int ne = k * (k + 1) / 2;
  double acc[KE];
  int ea[KE], eb[KE];
#pragma unroll
  for (int e = 0; e < KE; ++e) {
    acc[e] = 0.0;
    int lin = tid + e * nt, a = 0;
    if (lin < ne) {
      while (lin >= k - a) {
        lin -= k - a;
        ++a;
      }
      ea[e] = a;
      eb[e] = a + lin;
    } else {
      ea[e] = -1;
      eb[e] = 0;
    }
  }
  // 31 columns per chunk: A columns in T64 rows 0..30, their B = P_s^T a in rows 31..61
  for (int64_t c0 = c_lo; c0 < c_hi; c0 += 31) {
    const int nc = (int)imin64(31, c_hi - c0);
    __syncthreads();
    for (int idx = tid; idx < 31 * R; idx += nt) {
      const int c = idx % 31, r = idx / 31;
      ws.T64[c * ld + r] = c < nc ? m.A[a_offset(m, c0 + c, r)] : 0.0;
    }
    __syncthreads();
    for (int idx = tid; idx < 31 * k; idx += nt) {
      const int c = idx / k, a = idx - c * k;
      double b = 0.0;
      for (int r = 0; r < R; ++r) b = fma(ws.Q[r * ld + r0 + a], ws.T64[c * ld + r], b);
      ws.T64[(31 + c) * ld + a] = b;
    }
    __syncthreads();
#pragma unroll
    for (int e = 0; e < KE; ++e) {
      if (ea[e] < 0) continue;
      for (int c = 0; c < nc; ++c) acc[e] = fma(ws.T64[(31 + c) * ld + ea[e]], ws.T64[(31 + c) * ld + eb[e]], acc[e]);
    }
  }
  __syncthreads();
#pragma unroll
  for (int e = 0; e < KE; ++e)
    if (ea[e] >= 0) {
      ws.Z[ea[e] * ld + eb[e]] = acc[e];
      ws.Z[eb[e] * ld + ea[e]] = acc[e];
    }
  cluster_sum_mat(ws.Z, ws.S, k, k, ld);  // S = B B^T (k x k), identical on every CTA
  __syncthreads();
  cta_jacobi_eig(ws, k, 2);  // ws.V (k x k), ws.lam[0..k) descending
  // V_final = [P_large, P_s V_s]; lam_final = [lam_large, lam_s]
  for (int idx = tid; idx < R * R; idx += nt) {
    const int r = idx / R, c = idx % R;
    double v;
    if (c < r0) {
      v = ws.Q[r * ld + c];
    } else {
      v = 0.0;
      for (int a = 0; a < k; ++a) v = fma(ws.Q[r * ld + r0 + a], ws.V[a * ld + (c - r0)], v);
    }
    ws.Z[r * ld + c] = v;
  }
  __syncthreads();
  for (int j = tid; j < R; j += nt) {
    const double l = j < r0 ? lam_saved[j] : ws.lam[j - r0];
    lam_saved[j] = l;
  }
  __syncthreads();
  for (int idx = tid; idx < R * R; idx += nt) ws.V[(idx / R) * ld + idx % R] = ws.Z[(idx / R) * ld + idx % R];
  for (int j = tid; j < R; j += nt) ws.lam[j] = lam_saved[j];
  __syncthreads();
}

// ---------------------------------------------------------------------------
// SVT factor: M_n = P diag(f) P^T, f_i = (sigma_i - tau)/sigma_i for sigma_i > tau.
// SVT of mode n from its reduced Gram (every CTA of the mode's cluster; rank 0
// publishes sig, M, P and the keep / vnorm2 / nuclear scalars, each CTA forms
// its rows of UM = U M).
__device__ void svt_mode(const ModeDev& m, int n, Ctl* ctl, double* smem, int crank) {
  const int R = m.R, tid = threadIdx.x, nt = blockDim.x;
  SmallWs ws = make_ws(R, smem);
  const int ld = ws.ld;
  const bool lead = crank == 0;
  // Gram_n (reduced over chunks by k_gram_reduce, and over ranks when sharded)
  for (int idx = tid; idx < R * R; idx += nt) ws.S[(idx / R) * ld + idx % R] = m.Gram[idx];
  __syncthreads();
  cta_warm_start(ws, R, m.P);  // previous eigenvectors: Gram changes slowly between iterations
  cooperative_groups::this_cluster().sync();  // every CTA has read m.P before rank 0 rewrites it
  cta_jacobi_eig(ws, R, 1);
  cta_warm_finish(ws, R);
  const double tau = __ddiv_rn(m.lambda, ctl->mu);  // lambda / mu (pasd.cpp:77)
  {
    __shared__ int ksmall;
    if (tid == 0) {
      // unresolved: lambda_i < 1e-10 lambda_1 (sigma_i < 1e-5 sigma_1), and only
      // when the threshold is down there too (tau < 1e-5 sigma_1)
      const double l1 = ws.lam[0];
      int k = 0;
      if (m.refine_ok && l1 > 0.0 && tau * tau < 1e-10 * l1)
        while (k < R - 1 && ws.lam[R - 1 - k] < 1e-10 * l1) ++k;
      ksmall = k;
    }
    __syncthreads();
    if (ksmall > 0) svt_refine_small(ws, m, R, ksmall, crank);
  }
  if (tid == 0) {
    int keep = 0;
    double vn2 = 0.0, nuc = 0.0;
    for (int j = 0; j < R; ++j) {
      const double sg = sqrt(fmax(ws.lam[j], 0.0));
      ws.lam[j] = sg;
      if (lead) m.sig[j] = sg;
    }
    while (keep < R && ws.lam[keep] > tau) ++keep;  // linops.cpp:84-86
    for (int j = 0; j < R; ++j) {
      double f = 0.0;
      if (j < keep) {
        const double sh = ws.lam[j] - tau;
        f = sh / ws.lam[j];
        vn2 += sh * sh;
        nuc += sh;
      }
      ws.Q[j] = f;  // row 0 of Q holds f_j
    }
    if (lead) {
      ctl->keep[n] = keep;
      ctl->vnorm2[n] = vn2;
      ctl->nuclear[n] = nuc;
    }
  }
  __syncthreads();
  // M = P diag(f) P^T  -> S (row-major) and global m.M (column-major == same, symmetric)
  for (int idx = tid; idx < R * R; idx += nt) {
    const int r = idx / R, s = idx % R;
    double a = 0.0;
    for (int j = 0; j < R; ++j) a = fma(ws.V[r * ld + j] * ws.Q[j], ws.V[s * ld + j], a);
    ws.Z[r * ld + s] = a;
  }
  __syncthreads();
  for (int idx = tid; idx < R * R; idx += nt) {
    const int r = idx / R, s = idx % R;
    // symmetrise exactly
    const double a = 0.5 * (ws.Z[r * ld + s] + ws.Z[s * ld + r]);
    ws.S[r * ld + s] = a;
    if (lead) {
      m.M[r + R * s] = a;
      m.P[r + R * s] = ws.V[r * ld + s];
    }
  }
  __syncthreads();
  // UM = U * M on this CTA's rows
  const RowBlock rb = row_block(m.Ifull, crank);
  if (rb.rows > 0) cta_mul_nn(m.U + rb.lo, rb.rows, m.Ifull, R, ws.S, ld, R, m.UM + rb.lo, ws.T64);
}

__global__ void __cluster_dims__(kSmallCluster, 1, 1) __launch_bounds__(kSmallThreads)
    k_svt(const ModePack* __restrict__ mp, Ctl* ctl, int mode0 = 0) {
  if (ctl->done) return;
  extern __shared__ double smem[];
  const int crank = (int)cooperative_groups::this_cluster().block_rank();
  const int n = mode0 + blockIdx.x / kSmallCluster;  // mode0: per-mode launches
  svt_mode(mp->m[n], n, ctl, smem, crank);
}

// ---------------------------------------------------------------------------
// Procrustes: U_n <- polar(Wt_n M_n) unless degenerate (linops.cpp:93-104).
__global__ void __cluster_dims__(kSmallCluster, 1, 1) __launch_bounds__(kSmallThreads)
    k_polar(const ModePack* __restrict__ mp, Ctl* ctl, int mode0 = 0) {
  if (ctl->done) return;
  extern __shared__ double smem[];
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  const int crank = (int)cl.block_rank();
  const bool lead = crank == 0;
  const int n = mode0 + blockIdx.x / kSmallCluster;  // mode0: per-mode launches
  const ModeDev& m = mp->m[n];
  const int R = m.R, tid = threadIdx.x, nt = blockDim.x;
  const int64_t I = m.Ifull, IR = I * R;
  SmallWs ws = make_ws(R, smem);
  const int ld = ws.ld;
  double* Wt = m.Wt;                // I x R: G^{next} A^T, reduced by the pass that produced it
  double* X = m.scratch + IR;       // I x R
  double* X2 = m.scratch + 2 * IR;  // I x R
  const RowBlock rb = row_block(I, crank);
  const int64_t lo = rb.lo, rows = rb.rows;
  const double g2 = ctl->gnorm2[n];  // ||G_n^{next}||_F^2
  // 2. W = Wt M  (M in S), this CTA's rows; ||W||_F^2 over the cluster
  for (int idx = tid; idx < R * R; idx += nt) ws.S[(idx / R) * ld + idx % R] = m.M[(idx / R) + R * (idx % R)];
  __syncthreads();
  if (rows > 0) cta_mul_nn(Wt + lo, rows, I, R, ws.S, ld, R, X + lo, ws.T64);
  double w2 = 0.0;
  for (int64_t idx = tid; idx < rows * R; idx += nt) {
    const double v = X[lo + (idx % rows) + I * (idx / rows)];
    w2 += v * v;
  }
  w2 = block_reduce(w2, AddOp(), ws.red);
  if (tid == 0) ws.cl[0] = w2;
  cluster_sum_mat(ws.cl, ws.lam, 1, 1, 1);
  w2 = ws.lam[0];
  const double gnorm = sqrt(g2), vnorm = sqrt(ctl->vnorm2[n]);
  const double scale = fmax(1.0, gnorm * vnorm);  // linops.cpp:99
  if (sqrt(w2) <= 1e-14 * scale) {                // linops.cpp:100-101 -> keep U (pasd.cpp:70-74)
    if (lead && tid == 0) { ctl->degenerate[n] = 1; ctl->polar_rank[n] = 0; }
    return;  // uniform over the cluster (identical w2)
  }
  // 3'. One pass from the previous rotation: X2 = W Qp, C = X2^T X2.  In the
  //     steady state W's right singular vectors move little between iterations,
  //     so C is nearly diagonal and a single relative-accuracy Jacobi on it
  //     resolves every direction (the role of the two-pass scheme below).  When
  //     C is not nearly diagonal (transitions), fall back to the two passes.
  bool onepass = false;
  if (PASD_POLAR_ONEPASS > 0.0) {
    for (int idx = tid; idx < R * R; idx += nt) ws.Q[(idx % R) * ld + idx / R] = m.Qp[idx];
    __syncthreads();
    if (rows > 0) {
      cta_mul_nn(X + lo, rows, I, R, ws.Q, ld, R, X2 + lo, ws.T64);
      cta_gram_tn(X2 + lo, X2 + lo, rows, I, R, R, ws.Z, ld, ws.T64);
    } else {
      for (int idx = tid; idx < R * R; idx += nt) ws.Z[(idx / R) * ld + idx % R] = 0.0;
    }
    cluster_sum_mat(ws.Z, ws.S, R, R, ld);
    double off = 0.0;  // max |C_ij| / sqrt(C_ii C_jj), i < j (identical in every CTA)
    for (int idx = tid; idx < R * R; idx += nt) {
      const int r = idx / R, c = idx % R;
      if (r < c) {
        const double d = sqrt(fabs(ws.S[r * ld + r]) * fabs(ws.S[c * ld + c]));
        const double v = fabs(ws.S[r * ld + c]);
        off = fmax(off, d > 0.0 ? v / d : (v > 0.0 ? 1.0 : 0.0));
      }
    }
    off = block_reduce(off, MaxOp(), ws.red);
    if (off <= PASD_POLAR_ONEPASS) {
      onepass = true;
      cta_jacobi_eig(ws, R, 3);
      if (rows > 0) cta_mul_nn(X2 + lo, rows, I, R, ws.V, ld, R, X + lo, ws.T64);
      for (int idx = tid; idx < R * R; idx += nt) {  // Q = Qp V
        const int r = idx / R, s = idx % R;
        double a = 0.0;
        for (int j = 0; j < R; ++j) a = fma(ws.Q[r * ld + j], ws.V[j * ld + s], a);
        ws.Z[r * ld + s] = a;
      }
      __syncthreads();
      for (int idx = tid; idx < R * R; idx += nt) ws.Q[(idx / R) * ld + idx % R] = ws.Z[(idx / R) * ld + idx % R];
      __syncthreads();
    }
  }
  if (!onepass) {
    // 3. first Gram/Jacobi pass: C = W^T W = Q1 L Q1^T ; X2 = W Q1
    if (rows > 0) {
      cta_gram_tn(X + lo, X + lo, rows, I, R, R, ws.Z, ld, ws.T64);
    } else {
      for (int idx = tid; idx < R * R; idx += nt) ws.Z[(idx / R) * ld + idx % R] = 0.0;
    }
    cluster_sum_mat(ws.Z, ws.S, R, R, ld);
    cta_warm_start(ws, R, m.Qp);  // previous right rotation
    cta_jacobi_eig(ws, R, 2);
    cta_warm_finish(ws, R);
    for (int idx = tid; idx < R * R; idx += nt) ws.Q[(idx / R) * ld + idx % R] = ws.V[(idx / R) * ld + idx % R];
    __syncthreads();
    if (rows > 0) cta_mul_nn(X + lo, rows, I, R, ws.Q, ld, R, X2 + lo, ws.T64);
    // 4. second pass on the rotated columns: C2 = X2^T X2 = Q2 L2 Q2^T ; X = X2 Q2 ; Q = Q1 Q2
    if (rows > 0) {
      cta_gram_tn(X2 + lo, X2 + lo, rows, I, R, R, ws.Z, ld, ws.T64);
    } else {
      for (int idx = tid; idx < R * R; idx += nt) ws.Z[(idx / R) * ld + idx % R] = 0.0;
    }
    cluster_sum_mat(ws.Z, ws.S, R, R, ld);
    cta_jacobi_eig(ws, R, 3);
    if (rows > 0) cta_mul_nn(X2 + lo, rows, I, R, ws.V, ld, R, X + lo, ws.T64);
    for (int idx = tid; idx < R * R; idx += nt) {
      const int r = idx / R, s = idx % R;
      double a = 0.0;
      for (int j = 0; j < R; ++j) a = fma(ws.Q[r * ld + j], ws.V[j * ld + s], a);
      ws.Z[r * ld + s] = a;
    }
    __syncthreads();
    for (int idx = tid; idx < R * R; idx += nt) ws.Q[(idx / R) * ld + idx % R] = ws.Z[(idx / R) * ld + idx % R];
    __syncthreads();
  }
  // 5. column norms sigma_j of X (sorted descending by the Jacobi pass): one
  //    warp per column over this CTA's rows, then the cluster sum
  for (int j = tid >> 5; j < R; j += nt >> 5) {
    const int lane = tid & 31;
    double a = 0.0;
    for (int64_t i = lane; i < rows; i += 32) a = fma(X[lo + i + I * j], X[lo + i + I * j], a);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
    if (lane == 0) ws.cl[j] = a;
  }
  cluster_sum_mat(ws.cl, ws.lam, 1, R, R);
  for (int j = tid; j < R; j += nt) ws.lam[j] = sqrt(ws.lam[j]);
  __syncthreads();
  const double smax = ws.lam[0] > 0.0 ? ws.lam[0] : 1.0;
  int k = 0;
  while (k < R && ws.lam[k] > 1e-12 * smax) ++k;
  if (lead && tid == 0) { ctl->degenerate[n] = 0; ctl->polar_rank[n] = k; }
  // U_tilde columns j < k: X[:, j] / sigma_j   (this CTA's rows, in place)
  for (int64_t idx = tid; idx < rows * k; idx += nt) {
    const int j = (int)(idx / rows);
    const int64_t i = lo + idx % rows;
    X[i + I * j] = X[i + I * j] / ws.lam[j];
  }
  __syncthreads();
  if (k < R) {
    // The completion (transition iterations only) works on whole columns: rank 0
    // runs it on all I rows while the cluster waits.
    cl.sync();  // every CTA's rows of X, X2 written
    if (lead) {
      // 6. completion of the numerically null directions Q[:, k:].
      //    Candidates: Wt Q[:, k:] = G^{next} A_prev^T Q_null (one subspace-
      //    iteration step of G G^T on the sub-threshold directions), projected
      //    off range(Ut) and symmetrically orthonormalised (polar).  If those are
      //    ill-conditioned (e.g. at the first non-degenerate step), fall back to
      //    the previous basis U_prev Q[:, k:] (for k = 0 that reproduces the
      //    reference's keep-U rule, pasd.cpp:70-74).
      const int mcols = R - k;
      double* B = X2;  // I x mcols
      double* Tm = Wt;  // I x mcols temp (Wt is consumed by attempt 0)
      for (int attempt = 0; attempt < 2; ++attempt) {
        const double* src = attempt == 0 ? Wt : m.U;
        for (int64_t idx = tid; idx < I * mcols; idx += nt) {
          const int64_t i = idx % I;
          const int c = (int)(idx / I);
          double a = 0.0;
          for (int r = 0; r < R; ++r) a = fma(src[i + I * r], ws.Q[r * ld + k + c], a);
          B[idx] = a;
        }
        __syncthreads();
        for (int pass = 0; pass < 2 && k > 0; ++pass) {
          cta_gram_tn(X, B, I, I, k, mcols, ws.S, ld, ws.T64);  // S (k x mcols) = Ut^T B
          for (int64_t idx = tid; idx < I * mcols; idx += nt) {
            const int64_t i = idx % I;
            const int c = (int)(idx / I);
            double a = B[idx];
            for (int j = 0; j < k; ++j) a = fma(-X[i + I * j], ws.S[j * ld + c], a);
            B[idx] = a;
          }
          __syncthreads();
        }
        cta_gram_tn(B, B, I, I, mcols, mcols, ws.S, ld, ws.T64);
        cta_jacobi_eig(ws, mcols, 4);
        const bool ok = ws.lam[0] > 0.0 && ws.lam[mcols - 1] >= 1e-8 * ws.lam[0];
        if (!ok && attempt == 0) continue;
        // two symmetric-orthonormalisation passes: Y <- Y (Y^T Y)^{-1/2}
        for (int pass = 0; pass < 2; ++pass) {
          const double* in = pass == 0 ? B : Tm;
          double* outp = pass == 0 ? Tm : X + I * k;
          if (pass == 1) {
            cta_gram_tn(Tm, Tm, I, I, mcols, mcols, ws.S, ld, ws.T64);
            cta_jacobi_eig(ws, mcols, 5);
          }
          for (int idx = tid; idx < mcols * mcols; idx += nt) {
            const int r = idx / mcols, c = idx % mcols;
            double a = 0.0;
            for (int j = 0; j < mcols; ++j) {
              const double l = ws.lam[j];
              const double inv = l > 1e-280 ? 1.0 / sqrt(l) : 0.0;
              a = fma(ws.V[r * ld + j] * inv, ws.V[c * ld + j], a);
            }
            ws.Z[r * ld + c] = a;
          }
          __syncthreads();
          for (int64_t idx = tid; idx < I * mcols; idx += nt) {
            const int64_t i = idx % I;
            const int c = (int)(idx / I);
            double a = 0.0;
            for (int j = 0; j < mcols; ++j) a = fma(in[i + I * j], ws.Z[j * ld + c], a);
            outp[i + I * c] = a;
          }
          __syncthreads();
        }
        break;
      }
    }
    cl.sync();  // completed columns visible to every CTA
  }
  // 7. U = Ut Q^T on this CTA's rows ; rank 0 keeps Q as the next warm start
  for (int idx = tid; idx < R * R; idx += nt) {
    const int r = idx / R, s = idx % R;
    ws.S[r * ld + s] = ws.Q[s * ld + r];
    if (lead) m.Qp[r + R * s] = ws.Q[r * ld + s];
  }
  __syncthreads();
  if (rows > 0) cta_mul_nn(X + lo, rows, I, R, ws.S, ld, R, m.U + lo, ws.T64);
}

}  // namespace pasd
