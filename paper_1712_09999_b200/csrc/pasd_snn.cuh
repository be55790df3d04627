// pasd_snn.cuh — the SNN / HoRPCA full-SVT ADMM baseline on the device
// (tenrec::snn_recover, proj/src/baselines.cpp:37-143; SnnConfig,
// proj/include/tenrec/baselines.hpp:9-20), included by pasd_solver.cu.
//
// Per iteration (baselines.cpp:61-125), every mode reading the previous E:
//   G_n = (T - E) + Y_n/mu                       (:66-70)
//   Z_n = fold_n(SVT_{lambda_n inv_mu}(unfold_n(G_n)))   (:71-74, full SVT of the I_n x J_n unfolding)
//   E   = soft(sum_n ((T - Z_n) + Y_n/mu) / N, 1/(mu N))  (:77-91)
//   Y_n += mu ((T - Z_n) - E), resid_n = max |.|, NaN guard (:93-112)
//   mu schedule / history / stop rule as pasd_recover (:113-123)
// The full SVT reduces to the I_n x I_n eigenproblem of the Gram G G^T:
// eig = P diag(sigma^2) P^T, SVT_tau(G) = P diag((sigma - tau)_+ / sigma) P^T G
// = M_n G (kept set sigma > tau strictly, linops.cpp:85), applied as a mode-n
// product in place of the stored G_n.  Kernels per iteration:
//   k_snn_gram    G_n (into Z_n's buffer) + per-block Gram partials, all modes
//   k_snn_reduce  fixed-order sum of the partials (deterministic)
//   k_snn_eig     cyclic Jacobi on the Gram in shared memory (one CTA per
//                 mode), M_n, kept rank, sum (sigma - tau)_+
//   k_snn_apply   Z_n = M_n x_n G_n in place (panels of 32 unfolding columns)
//   k_snn_update  E / Y / residual partials in the reference's operation order
//   k_finish      (pasd_kernels.cuh)
// Limits of this build: the Gram side I_n <= 112 and I_n <= prod_{m != n} I_m
// (the eigenproblem lives in one CTA's shared memory) -- SPEC.md's SNN runs
// (30^3, 40-80^3, 12^4) and the 100^3 BASELINE config fit.
#pragma once

namespace {

constexpr int kSnnMaxSide = 112;
constexpr int kSnnPanel = 32;
constexpr int kSnnThreads = 256;
constexpr int kSnnEigThreads = 1024;

struct SnnMode {
  int64_t inner, I, outer, J;
  double lambda;
  double* Z;      // S: G_n, then Z_n (in place)
  double* Gpart;  // [nblk][I * I]
  double* Gram;   // I x I
  double* M;      // I x I  SVT map
  int nblk;
};
struct SnnPack {
  int order;
  SnnMode m[PASD_MAX_ORDER];
  double* Y[PASD_MAX_ORDER];
};

// 4 x 4 tiles of the upper triangle: linear index -> (ti, tj), ti <= tj.
__device__ __forceinline__ void upper_tile(int lin, int nt, int& ti, int& tj) {
  ti = 0;
  while (lin >= nt - ti) {
    lin -= nt - ti;
    ++ti;
  }
  tj = ti + lin;
}

// G_n = (T - E) + Y_n * inv_mu (baselines.cpp:66-70) for panels of 32 unfolding
// columns, stored to Z_n's buffer, and per-block Gram partials G G^T (upper
// 4 x 4 tiles, 2 per thread).  grid = (max nblk, N).
__global__ void __launch_bounds__(kSnnThreads) k_snn_gram(const SnnPack* __restrict__ pk, const double* __restrict__ T,
                                                          const double* E0, const double* E1, const Ctl* ctl) {
  if (ctl->done) return;
  const int n = blockIdx.y;
  const SnnMode& m = pk->m[n];
  if ((int)blockIdx.x >= m.nblk) return;
  __shared__ double panel[kSnnMaxSide][kSnnPanel + 1];
  const double* __restrict__ E = ctl->ecur ? E1 : E0;
  const double* __restrict__ Y = pk->Y[n];
  const double inv_mu = __ddiv_rn(1.0, ctl->mu);
  const int I = (int)m.I, nt4 = (I + 3) / 4, ntiles = nt4 * (nt4 + 1) / 2;
  const int tid = threadIdx.x;
  int ti[2], tj[2];
  double acc[2][16];
#pragma unroll
  for (int s = 0; s < 2; ++s) {
    const int lin = tid + s * kSnnThreads;
    if (lin < ntiles)
      upper_tile(lin, nt4, ti[s], tj[s]);
    else
      ti[s] = tj[s] = -1;
#pragma unroll
    for (int k = 0; k < 16; ++k) acc[s][k] = 0.0;
  }
  const int64_t nchunks = (m.J + kSnnPanel - 1) / kSnnPanel;
  for (int64_t c = blockIdx.x; c < nchunks; c += m.nblk) {
    const int64_t j0 = c * kSnnPanel;
    // contiguous direction first: i when inner == 1 (mode 1), else the column
    for (int idx = tid; idx < nt4 * 4 * kSnnPanel; idx += kSnnThreads) {
      int i, jj;
      if (m.inner == 1) {
        i = idx % (nt4 * 4);
        jj = idx / (nt4 * 4);
      } else {
        jj = idx % kSnnPanel;
        i = idx / kSnnPanel;
      }
      const int64_t j = j0 + jj;
      double g = 0.0;
      if (i < I && j < m.J) {
        const int64_t q = j / m.inner, p = j - q * m.inner;
        const int64_t off = p + m.inner * (i + m.I * q);
        g = g_elem(T[off], E[off], Y[off], inv_mu);
        m.Z[off] = g;
      }
      panel[i][jj] = g;
    }
    __syncthreads();
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      if (ti[s] < 0) continue;
      for (int jj = 0; jj < kSnnPanel; ++jj) {
        double a[4], b[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          a[k] = panel[4 * ti[s] + k][jj];
          b[k] = panel[4 * tj[s] + k][jj];
        }
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
          for (int q = 0; q < 4; ++q) acc[s][4 * r + q] = fma(a[r], b[q], acc[s][4 * r + q]);
      }
    }
    __syncthreads();
  }
  double* out = m.Gpart + (int64_t)blockIdx.x * I * I;
#pragma unroll
  for (int s = 0; s < 2; ++s) {
    if (ti[s] < 0) continue;
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int ii = 4 * ti[s] + r, jj = 4 * tj[s] + q;
        if (ii < I && jj < I && ii <= jj) out[ii + (int64_t)I * jj] = acc[s][4 * r + q];
      }
  }
}

// Gram_n = sum of the block partials in block order (upper), mirrored.  grid = (64, N)
__global__ void k_snn_reduce(const SnnPack* __restrict__ pk, const Ctl* ctl) {
  if (ctl->done) return;
  const SnnMode& m = pk->m[blockIdx.y];
  const int I = (int)m.I;
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < I * I; idx += gridDim.x * blockDim.x) {
    const int r = idx % I, c = idx / I;
    if (r > c) continue;
    double s = 0.0;
    for (int b = 0; b < m.nblk; ++b) s += m.Gpart[(int64_t)b * I * I + idx];
    m.Gram[idx] = s;
    m.Gram[c + I * r] = s;
  }
}

__host__ __device__ inline size_t snn_eig_smem(int I) {
  const int Ip = I + (I & 1), ld = Ip + 1;
  return sizeof(double) * (2 * (size_t)Ip * ld + 2 * (size_t)(Ip / 2 + 1) + (size_t)(Ip + 2)) +
         sizeof(int) * (2 * (size_t)(Ip / 2 + 1));
}

// eig(Gram_n) by a cyclic parallel Jacobi in shared memory (round-robin pairs,
// n/2 disjoint rotations per round, rotations accumulated into V), then the SVT
// map M = V diag(f) V^T with f = (sigma - tau)/sigma on the kept set
// sigma > tau = lambda_n * inv_mu (baselines.cpp:73, linops.cpp:85).  One CTA
// per mode; S and V take 2 I (I + 1) doubles (204 KB at I = 112).
__global__ void __launch_bounds__(kSnnEigThreads) k_snn_eig(const SnnPack* __restrict__ pk, Ctl* ctl) {
  if (ctl->done) return;
  extern __shared__ double sm[];
  const int n = blockIdx.x;
  const SnnMode& m = pk->m[n];
  const int I = (int)m.I, Ip = I + (I & 1), ld = Ip + 1, tid = threadIdx.x, nt = blockDim.x;
  const int npairs = Ip / 2;
  double* S = sm;
  double* V = S + (size_t)Ip * ld;
  double* cs = V + (size_t)Ip * ld;
  double* sn = cs + (npairs + 1);
  double* f = sn + (npairs + 1);
  int* pq = reinterpret_cast<int*>(f + (Ip + 2));
  __shared__ int rotated, big;
  for (int idx = tid; idx < Ip * Ip; idx += nt) {  // odd I: an isolated zero row / column
    const int r = idx / Ip, c = idx % Ip;
    S[r * ld + c] = (r < I && c < I) ? m.Gram[r + I * c] : 0.0;
    V[r * ld + c] = (r == c) ? 1.0 : 0.0;
  }
  __syncthreads();
  for (int sweep = 0; sweep < 40 && Ip > 1; ++sweep) {
    if (tid == 0) rotated = big = 0;
    __syncthreads();
    for (int round = 0; round < Ip - 1; ++round) {
      for (int j = tid; j < npairs; j += nt) {
        const int a = j == 0 ? 0 : 1 + (j - 1 + round) % (Ip - 1);
        const int jb = Ip - 1 - j;
        const int b = jb == 0 ? 0 : 1 + (jb - 1 + round) % (Ip - 1);
        const int p = a < b ? a : b, q = a < b ? b : a;
        const double apq = S[p * ld + q], app = S[p * ld + p], aqq = S[q * ld + q];
        double c = 1.0, s = 0.0;
        if (fabs(apq) > 2.2e-16 * sqrt(fabs(app) * fabs(aqq)) && fabs(apq) > 1e-300) {
          const double zeta = (aqq - app) / (2.0 * apq);
          const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
          c = 1.0 / sqrt(1.0 + t * t);
          s = t * c;
          rotated = 1;
          if (fabs(apq) > 1e-10 * sqrt(fabs(app) * fabs(aqq))) big = 1;
        }
        cs[j] = c;
        sn[j] = s;
        pq[2 * j] = p;
        pq[2 * j + 1] = q;
      }
      __syncthreads();
      // S <- J^T S J on 2 x 2 blocks of pairs (ja, jb); V <- V J
      for (int idx = tid; idx < npairs * npairs; idx += nt) {
        const int ja = idx / npairs, jb = idx - ja * npairs;
        const double sa = sn[ja], sb = sn[jb];
        if (sa == 0.0 && sb == 0.0) continue;
        const double ca = cs[ja], cb = cs[jb];
        const int pa = pq[2 * ja], qa = pq[2 * ja + 1], pb = pq[2 * jb], qb = pq[2 * jb + 1];
        double a00 = S[pa * ld + pb], a01 = S[pa * ld + qb], a10 = S[qa * ld + pb], a11 = S[qa * ld + qb];
        if (sa != 0.0) {
          const double r00 = ca * a00 - sa * a10, r10 = sa * a00 + ca * a10;
          const double r01 = ca * a01 - sa * a11, r11 = sa * a01 + ca * a11;
          a00 = r00; a10 = r10; a01 = r01; a11 = r11;
        }
        if (sb != 0.0) {
          const double c00 = cb * a00 - sb * a01, c01 = sb * a00 + cb * a01;
          const double c10 = cb * a10 - sb * a11, c11 = sb * a10 + cb * a11;
          a00 = c00; a01 = c01; a10 = c10; a11 = c11;
        }
        S[pa * ld + pb] = a00;
        S[pa * ld + qb] = a01;
        S[qa * ld + pb] = a10;
        S[qa * ld + qb] = a11;
      }
      for (int idx = tid; idx < npairs * Ip; idx += nt) {
        const int j = idx / Ip, k = idx - j * Ip;
        const double s = sn[j];
        if (s == 0.0) continue;
        const int p = pq[2 * j], q = pq[2 * j + 1];
        const double c = cs[j];
        const double va = V[k * ld + p], vb = V[k * ld + q];
        V[k * ld + p] = c * va - s * vb;
        V[k * ld + q] = s * va + c * vb;
      }
      __syncthreads();
    }
    if (rotated == 0 || big == 0) break;  // quadratic convergence: nothing left above rounding
    __syncthreads();
  }
  const double tau = __dmul_rn(m.lambda, __ddiv_rn(1.0, ctl->mu));  // config.lambdas[n] * inv_mu (baselines.cpp:73)
  for (int i = tid; i < Ip; i += nt) {
    const double lam = S[i * ld + i];
    const double sig = lam > 0.0 ? sqrt(lam) : 0.0;
    const bool keep = i < I && sig > tau;
    f[i] = keep ? (sig - tau) / sig : 0.0;
    S[i * ld + i] = keep ? sig - tau : 0.0;  // (sigma - tau)_+
  }
  __syncthreads();
  if (tid == 0) {  // kept rank and nuclear norm sum (sigma - tau)_+, in index order
    int keep = 0;
    double nuc = 0.0;
    for (int i = 0; i < I; ++i) {
      const double v = S[i * ld + i];
      if (v > 0.0) {
        ++keep;
        nuc += v;
      }
    }
    ctl->keep[n] = keep;
    ctl->nuclear[n] = nuc;
  }
  for (int idx = tid; idx < I * I; idx += nt) {  // M = V diag(f) V^T (column-major)
    const int r = idx % I, c = idx / I;
    double s = 0.0;
    for (int k = 0; k < I; ++k) s = fma(V[r * ld + k] * f[k], V[c * ld + k], s);
    m.M[idx] = s;
  }
}

// Z_n = M_n x_n G_n in place over panels of 32 unfolding columns.  grid = (max nblk, N)
__global__ void __launch_bounds__(kSnnThreads) k_snn_apply(const SnnPack* __restrict__ pk, const Ctl* ctl) {
  if (ctl->done) return;
  extern __shared__ double sm[];
  const int n = blockIdx.y;
  const SnnMode& m = pk->m[n];
  if ((int)blockIdx.x >= m.nblk) return;
  const int I = (int)m.I, tid = threadIdx.x;
  double* Ms = sm;                       // I x I row-major: Ms[i * I + k] = M[i, k]
  double* pan = sm + (size_t)I * I;      // [I][33]
  for (int idx = tid; idx < I * I; idx += kSnnThreads) Ms[(idx % I) * I + idx / I] = m.M[idx];
  const int jj = tid & 31, r0 = tid >> 5;  // column of the panel, first row (rows r0 + 8 k)
  constexpr int RMAX = kSnnMaxSide / 8;
  const int64_t nchunks = (m.J + kSnnPanel - 1) / kSnnPanel;
  for (int64_t c = blockIdx.x; c < nchunks; c += m.nblk) {
    const int64_t j0 = c * kSnnPanel;
    __syncthreads();
    for (int idx = tid; idx < I * kSnnPanel; idx += kSnnThreads) {
      int i, cc;
      if (m.inner == 1) {
        i = idx % I;
        cc = idx / I;
      } else {
        cc = idx % kSnnPanel;
        i = idx / kSnnPanel;
      }
      const int64_t j = j0 + cc;
      double g = 0.0;
      if (j < m.J) {
        const int64_t q = j / m.inner, p = j - q * m.inner;
        g = m.Z[p + m.inner * (i + m.I * q)];
      }
      pan[i * (kSnnPanel + 1) + cc] = g;
    }
    __syncthreads();
    double acc[RMAX];
#pragma unroll
    for (int k = 0; k < RMAX; ++k) acc[k] = 0.0;
    for (int k = 0; k < I; ++k) {
      const double g = pan[k * (kSnnPanel + 1) + jj];
#pragma unroll
      for (int u = 0; u < RMAX; ++u) {
        const int i = r0 + 8 * u;
        if (i < I) acc[u] = fma(Ms[i * I + k], g, acc[u]);
      }
    }
    const int64_t j = j0 + jj;
    if (j < m.J) {
      const int64_t q = j / m.inner, p = j - q * m.inner;
#pragma unroll
      for (int u = 0; u < RMAX; ++u) {
        const int i = r0 + 8 * u;
        if (i < I) m.Z[p + m.inner * (i + m.I * q)] = acc[u];
      }
    }
  }
}

// E / Y / residual partials (baselines.cpp:77-112), the reference's operation
// order with round-to-nearest intrinsics.
__global__ void __launch_bounds__(kThreads) k_snn_update(const SnnPack* __restrict__ pk, const double* __restrict__ T,
                                                         double* E0, double* E1, double* resid_part, int* bad_part,
                                                         int64_t S, const Ctl* ctl) {
  if (ctl->done) return;
  __shared__ double red[32];
  __shared__ int redi[32];
  const int N = pk->order;
  double* __restrict__ Enew = ctl->ecur ? E0 : E1;
  const double mu = ctl->mu;
  const double inv_mu = __ddiv_rn(1.0, mu);
  const double dn = (double)N;
  const double inv_n = __ddiv_rn(1.0, dn);
  const double tau = __ddiv_rn(1.0, __dmul_rn(mu, dn));
  double worst[PASD_MAX_ORDER];
  for (int n = 0; n < PASD_MAX_ORDER; ++n) worst[n] = 0.0;
  int bad = 0;
  for (int64_t idx = (int64_t)blockIdx.x * kThreads + threadIdx.x; idx < S; idx += (int64_t)gridDim.x * kThreads) {
    const double t = T[idx];
    double zt[PASD_MAX_ORDER], yv[PASD_MAX_ORDER];
    double h = 0.0;
    for (int n = 0; n < N; ++n) {
      zt[n] = __dsub_rn(t, pk->m[n].Z[idx]);
      yv[n] = pk->Y[n][idx];
      h = __dadd_rn(h, __dadd_rn(zt[n], __dmul_rn(yv[n], inv_mu)));  // baselines.cpp:84
    }
    const double e = soft(__dmul_rn(h, inv_n), tau);  // baselines.cpp:90
    Enew[idx] = e;
    for (int n = 0; n < N; ++n) {
      const double r = __dsub_rn(zt[n], e);                // baselines.cpp:103
      pk->Y[n][idx] = __dadd_rn(yv[n], __dmul_rn(mu, r));  // baselines.cpp:104
      const double a = fabs(r);
      if (a > worst[n]) worst[n] = a;
      bad |= !isfinite(r);
    }
  }
  for (int n = 0; n < N; ++n) {
    const double w = block_reduce(worst[n], MaxOp(), red);
    if (threadIdx.x == 0) resid_part[(int64_t)blockIdx.x * PASD_MAX_ORDER + n] = w;
  }
  const int b = block_reduce(bad, OrOp(), redi);
  if (threadIdx.x == 0) bad_part[blockIdx.x] = b;
}

__global__ void k_snn_init(SnnPack* pk, Ctl* ctl, double mu0, double rho, double mu_max, double eps, int maxiter,
                           int fixed) {
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    ctl->mu = mu0;
    ctl->mu_used_last = mu0;
    ctl->rho = rho;
    ctl->mu_max = mu_max;
    ctl->eps = eps;
    ctl->iter = 0;
    ctl->maxiter = maxiter;
    ctl->done = 0;
    ctl->converged = 0;
    ctl->nan_flag = 0;
    ctl->ecur = 0;
    ctl->fixed_iters = fixed;
    ctl->order = pk->order;
    for (int n = 0; n < PASD_MAX_ORDER; ++n) {
      ctl->resid[n] = CUDART_INF;
      ctl->nuclear[n] = 0.0;
      ctl->keep[n] = 0;
    }
  }
}

// SnnConfig::validate (baselines.cpp:12-29), same messages.
void snn_validate(const pasd_options* o) {
  if (!o) fail(PASD_ERR_ARGUMENT, "config: null options");
  if (o->order < 1 || !o->dims) fail(PASD_ERR_ARGUMENT, "tensor order must be at least 1");
  const int N = o->order;
  dims_product(std::vector<int64_t>(o->dims, o->dims + N));
  if (!o->lambdas) fail(PASD_ERR_ARGUMENT, "config: expected " + std::to_string(N) + " lambdas, got 0");
  for (int n = 0; n < N; ++n)
    if (!(o->lambdas[n] > 0.0) || !std::isfinite(o->lambdas[n]))
      fail(PASD_ERR_ARGUMENT, "config: lambda of mode " + std::to_string(n + 1) + " must be positive");
  if (!(o->mu0 > 0.0) || !(o->mu_max >= o->mu0) || !(o->rho > 1.0) || !(o->eps > 0.0) || o->maxiter < 1)
    fail(PASD_ERR_ARGUMENT, "config: invalid penalty schedule or stopping parameters");
  if (o->output_weights)
    for (int n = 0; n < N; ++n)
      if (!(o->output_weights[n] > 0.0)) fail(PASD_ERR_ARGUMENT, "config: output weights must be positive");
  if (N > PASD_MAX_ORDER)
    fail(PASD_ERR_ARGUMENT, "pasd_b200: order " + std::to_string(N) + " exceeds the supported maximum " +
                                std::to_string(PASD_MAX_ORDER));
}

struct SnnRun {
  int N = 0;
  int64_t S = 0;
  std::vector<int64_t> dims;
  cudaStream_t st = nullptr;
  std::vector<void*> owned;
  double *T = nullptr, *E[2] = {nullptr, nullptr};
  SnnPack h{};
  SnnPack* d = nullptr;
  Ctl* ctl = nullptr;
  Ctl* hctl = nullptr;
  double* hist = nullptr;
  double* resid_part = nullptr;
  int* bad_part = nullptr;
  int nblk_upd = 0, max_nblk = 1;
  size_t eig_smem = 0, apply_smem = 0;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  template <class U>
  U* alloc(size_t n) {
    U* p = dalloc<U>(n);
    owned.push_back(p);
    return p;
  }
  ~SnnRun() {
    if (exec) cudaGraphExecDestroy(exec);
    if (graph) cudaGraphDestroy(graph);
    for (void* p : owned) dfree(p);
    if (hctl) cudaFreeHost(hctl);
    if (st) cudaStreamDestroy(st);
  }
  void launch_iteration() {
    k_snn_gram<<<dim3(max_nblk, N), kSnnThreads, 0, st>>>(d, T, E[0], E[1], ctl);
    k_snn_reduce<<<dim3(64, N), 256, 0, st>>>(d, ctl);
    k_snn_eig<<<N, kSnnEigThreads, eig_smem, st>>>(d, ctl);
    k_snn_apply<<<dim3(max_nblk, N), kSnnThreads, apply_smem, st>>>(d, ctl);
    k_snn_update<<<nblk_upd, kThreads, 0, st>>>(d, T, E[0], E[1], resid_part, bad_part, S, ctl);
    k_finish<<<1, kThreads, 0, st>>>(ctl, resid_part, bad_part, nblk_upd, hist, nullptr);
    CK(cudaGetLastError());
  }
};

void snn_recover_device(const double* t, const pasd_options* o, pasd_outputs* out, pasd_observer_fn obs, void* user) {
  snn_validate(o);
  if (!t || !out) fail(PASD_ERR_ARGUMENT, "pasd_b200: null argument");
  SnnRun r;
  r.N = o->order;
  r.dims.assign(o->dims, o->dims + r.N);
  r.S = dims_product(r.dims);
  for (int n = 0; n < r.N; ++n) {
    const int64_t I = r.dims[n];
    if (I > kSnnMaxSide || I > r.S / I)
      fail(PASD_ERR_ARGUMENT, "pasd_b200: snn supports unfoldings with I_n <= " + std::to_string(kSnnMaxSide) +
                                  " and I_n <= prod of the other dimensions (mode " + std::to_string(n + 1) +
                                  ": " + std::to_string(I) + ")");
  }
  for (int64_t i = 0; i < r.S; ++i)
    if (!std::isfinite(t[i])) fail(PASD_ERR_ARGUMENT, "snn: input tensor contains non-finite entries");  // :41-42
  CK(cudaSetDevice(o->device));
  CK(cudaStreamCreateWithFlags(&r.st, cudaStreamNonBlocking));
  const int64_t S = r.S;
  int sms = 148;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, o->device));
  r.T = r.alloc<double>(S);
  r.E[0] = r.alloc<double>(S);
  r.E[1] = r.alloc<double>(S);
  CK(cudaMemcpyAsync(r.T, t, S * sizeof(double), cudaMemcpyHostToDevice, r.st));
  CK(cudaMemsetAsync(r.E[0], 0, S * sizeof(double), r.st));
  CK(cudaMemsetAsync(r.E[1], 0, S * sizeof(double), r.st));
  r.h.order = r.N;
  int maxI = 1;
  for (int n = 0; n < r.N; ++n) {
    SnnMode& m = r.h.m[n];
    m.I = r.dims[n];
    m.inner = 1;
    for (int l = 0; l < n; ++l) m.inner *= r.dims[l];
    m.outer = S / (m.inner * m.I);
    m.J = S / m.I;
    m.lambda = o->lambdas[n];
    const int64_t nchunks = (m.J + kSnnPanel - 1) / kSnnPanel;
    m.nblk = (int)std::max<int64_t>(1, std::min<int64_t>(nchunks, 2 * sms / r.N + 1));
    r.max_nblk = std::max(r.max_nblk, m.nblk);
    m.Z = r.alloc<double>(S);
    m.Gpart = r.alloc<double>((size_t)m.nblk * m.I * m.I);
    m.Gram = r.alloc<double>(m.I * m.I);
    m.M = r.alloc<double>(m.I * m.I);
    r.h.Y[n] = r.alloc<double>(S);
    CK(cudaMemsetAsync(r.h.Y[n], 0, S * sizeof(double), r.st));
    CK(cudaMemsetAsync(m.Z, 0, S * sizeof(double), r.st));
    maxI = std::max<int>(maxI, (int)m.I);
  }
  r.d = r.alloc<SnnPack>(1);
  CK(cudaMemcpyAsync(r.d, &r.h, sizeof(SnnPack), cudaMemcpyHostToDevice, r.st));
  r.ctl = r.alloc<Ctl>(1);
  CK(cudaMallocHost(&r.hctl, sizeof(Ctl)));
  r.hist = r.alloc<double>(std::max(1, o->maxiter));
  r.nblk_upd = (int)std::max<int64_t>(1, std::min<int64_t>((S + kThreads - 1) / kThreads, (int64_t)sms * 8));
  r.resid_part = r.alloc<double>((size_t)r.nblk_upd * PASD_MAX_ORDER);
  r.bad_part = r.alloc<int>(r.nblk_upd);
  r.eig_smem = snn_eig_smem(kSnnMaxSide);
  r.apply_smem = sizeof(double) * ((size_t)maxI * maxI + (size_t)maxI * (kSnnPanel + 1));
  ensure_smem_attr<k_snn_eig>(snn_eig_smem(kSnnMaxSide));
  ensure_smem_attr<k_snn_apply>(sizeof(double) * ((size_t)kSnnMaxSide * kSnnMaxSide + kSnnMaxSide * (kSnnPanel + 1)));
  k_snn_init<<<16, 256, 0, r.st>>>(r.d, r.ctl, o->mu0, o->rho, o->mu_max, o->eps, o->maxiter,
                                   (o->flags & PASD_FLAG_FIXED_ITERS) ? 1 : 0);
  CK(cudaGetLastError());
  // one iteration = 6 kernels, captured once and replayed (observer: every iteration)
  CK(cudaStreamBeginCapture(r.st, cudaStreamCaptureModeThreadLocal));
  r.launch_iteration();
  CK(cudaStreamEndCapture(r.st, &r.graph));
  CK(cudaGraphInstantiate(&r.exec, r.graph, 0));
  const int poll = obs ? 1 : (o->poll_every > 0 ? o->poll_every : 8);
  std::vector<double> he, hz, hy;
  int launched = 0;
  while (launched < o->maxiter) {
    const int chunk = std::min(poll, o->maxiter - launched);
    for (int k = 0; k < chunk; ++k) CK(cudaGraphLaunch(r.exec, r.st));
    launched += chunk;
    CK(cudaMemcpyAsync(r.hctl, r.ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, r.st));
    CK(cudaStreamSynchronize(r.st));
    const Ctl& c = *r.hctl;
    if (c.nan_flag)  // baselines.cpp:115-116
      fail(PASD_ERR_NUMERICAL, "snn: non-finite iterate at iteration " + std::to_string(c.iter));
    if (obs) {  // IterationView{iter, mu_used, mu_next, resid, e, z, y, nullptr, nullptr} (baselines.cpp:124-125)
      he.resize(S);
      hz.resize((size_t)S * r.N);
      hy.resize((size_t)S * r.N);
      CK(cudaMemcpyAsync(he.data(), r.E[c.ecur], S * sizeof(double), cudaMemcpyDeviceToHost, r.st));
      std::vector<const double*> zp, yp;
      for (int n = 0; n < r.N; ++n) {
        CK(cudaMemcpyAsync(hz.data() + (size_t)n * S, r.h.m[n].Z, S * sizeof(double), cudaMemcpyDeviceToHost, r.st));
        CK(cudaMemcpyAsync(hy.data() + (size_t)n * S, r.h.Y[n], S * sizeof(double), cudaMemcpyDeviceToHost, r.st));
        zp.push_back(hz.data() + (size_t)n * S);
        yp.push_back(hy.data() + (size_t)n * S);
      }
      CK(cudaStreamSynchronize(r.st));
      pasd_iteration_view view{c.iter, c.mu_used_last, c.mu, c.resid, he.data(), zp.data(), yp.data(), nullptr,
                               nullptr};
      obs(&view, user);
    }
    if (c.done) break;
  }
  const Ctl c = *r.hctl;
  out->iters = c.iter;
  out->converged = c.converged;
  if (out->residual_history && c.iter > 0)
    CK(cudaMemcpyAsync(out->residual_history, r.hist, c.iter * sizeof(double), cudaMemcpyDeviceToHost, r.st));
  if (out->final_residuals)
    for (int n = 0; n < r.N; ++n) out->final_residuals[n] = c.resid[n];
  const double* e = r.E[c.ecur];
  // X = weighted mean of Z_n (recovery.cpp:7-25), Z_n, Y_n; no Y-hat / certificate
  // (snn_recover leaves them empty, baselines.cpp:128-141)
  double wsum = 0.0;
  for (int n = 0; n < r.N; ++n) wsum += o->output_weights ? o->output_weights[n] : o->lambdas[n];
  double* xbuf = nullptr;
  if (out->x) {
    xbuf = r.alloc<double>(S);
    for (int n = 0; n < r.N; ++n) {
      const double w = o->output_weights ? o->output_weights[n] : o->lambdas[n];
      k_accum_x<<<1184, 256, 0, r.st>>>(xbuf, r.h.m[n].Z, w / wsum, n == 0, S);
    }
    CK(cudaMemcpyAsync(out->x, xbuf, S * sizeof(double), cudaMemcpyDeviceToHost, r.st));
  }
  if (out->e) CK(cudaMemcpyAsync(out->e, e, S * sizeof(double), cudaMemcpyDeviceToHost, r.st));
  for (int n = 0; n < r.N; ++n) {
    if (out->z && out->z[n])
      CK(cudaMemcpyAsync(out->z[n], r.h.m[n].Z, S * sizeof(double), cudaMemcpyDeviceToHost, r.st));
    if (out->y && out->y[n])
      CK(cudaMemcpyAsync(out->y[n], r.h.Y[n], S * sizeof(double), cudaMemcpyDeviceToHost, r.st));
  }
  // objective = ||E||_1 + sum_n lambda_n ||unfold_n(Z_n)||_*  (baselines.cpp:131-134); the nuclear
  // norm of Z_n = SVT output is sum (sigma - tau)_+ of its last SVT
  double* stats = r.alloc<double>(2 * 2048);
  k_abs_stats<<<1184, 256, 0, r.st>>>(e, S, stats, stats + 2048);
  std::vector<double> sums(1184);
  CK(cudaMemcpyAsync(sums.data(), stats, 1184 * sizeof(double), cudaMemcpyDeviceToHost, r.st));
  CK(cudaStreamSynchronize(r.st));
  double obj = 0.0;
  for (double v : sums) obj += v;
  for (int n = 0; n < r.N; ++n) obj += o->lambdas[n] * c.nuclear[n];
  out->objective = obj;
  out->has_certificate = 0;
  out->cert_epsilon_hat = out->cert_c = out->cert_bound = 0.0;
}

}  // namespace

extern "C" int pasd_b200_snn_recover(const double* t, const pasd_options* opt, pasd_outputs* out,
                                     pasd_observer_fn observer, void* user, char* errbuf, size_t errlen) {
  return guarded_call(errbuf, errlen, [&] { snn_recover_device(t, opt, out, observer, user); });
}
