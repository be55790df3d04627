// pasd_spec.cuh — the spec-shaped half of the reference header API on the device
// (included by pasd_solver.cu after the linops ABI, whose helpers it reuses).
//
//   pasd_g_matrix            pasd.hpp:43-45, pasd.cpp:82-97    -> pasd_b200_g_matrix
//   update_u                 pasd.hpp:47-49, pasd.cpp:99-103   -> pasd_b200_update_u
//   update_v                 pasd.hpp:51-54, pasd.cpp:105-109  -> pasd_b200_update_v
//   update_e                 pasd.hpp:56-58, pasd.cpp:111-130  -> pasd_b200_update_e
//   suboptimality_certificate pasd.hpp:68-70, pasd.cpp:277-309 -> pasd_b200_certificate
//
// The reference has no in-tree callers for these (they exist for unit tests,
// SURVEY 4); here they are host-buffer-in / host-buffer-out entry points built
// from device kernels -- the G formation and the E shrink use the solver's
// round-to-nearest elementwise order, the SVT and Procrustes are the solver's
// own small solves (k_svt, k_polar).  Not a hot path: no graphs, no streams.
#pragma once

namespace {

// G_n = unfold_n((T - E) + Y * inv_mu), I_n x J_n column-major (pasd.cpp:91-96,
// unfold index map tensor.cpp:98-113).
__global__ void k_g_unfold(const double* __restrict__ T, const double* __restrict__ E, const double* __restrict__ Y,
                           double inv_mu, int64_t inner, int64_t I, int64_t S, double* __restrict__ G) {
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < S; idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t rest = idx / inner;
    const int64_t p = idx - rest * inner;
    const int64_t q = rest / I;
    const int64_t i = rest - q * I;
    G[i + I * (p + inner * q)] = g_elem(T[idx], E[idx], Y[idx], inv_mu);
  }
}

// A = U^T G (R x J column-major) for U (I x R), G (I x J): one thread per entry.
__global__ void k_ut_g(const double* __restrict__ U, const double* __restrict__ G, int64_t I, int R, int64_t J,
                       double* __restrict__ A) {
  const int64_t total = (int64_t)R * J;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(idx % R);
    const int64_t j = idx / R;
    const double* u = U + I * r;
    const double* g = G + I * j;
    double acc = 0.0;
    for (int64_t i = 0; i < I; ++i) acc = fma(u[i], g[i], acc);
    A[idx] = acc;
  }
}

struct SpecMode {
  int64_t inner, I;
  int R;
  const double* U;  // I x R
  const double* V;  // R x J (unfolding column order)
  const double* Y;  // S
};
struct SpecPack {
  int order;
  SpecMode m[PASD_MAX_ORDER];
};

// E = shrink(mean_n((T - Z_n) + Y_n / mu), 1 / (mu N)) with Z_n = fold(U_n V_n)
// (pasd.cpp:111-130): acc from 0.0 in mode order, then soft(acc * inv_n, tau).
__global__ void k_update_e(const SpecPack p, const double* __restrict__ T, double inv_mu, double inv_n, double tau,
                           int64_t S, double* __restrict__ E) {
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < S; idx += (int64_t)gridDim.x * blockDim.x) {
    double acc = 0.0;
    const double t = T[idx];
    for (int n = 0; n < p.order; ++n) {
      const SpecMode& m = p.m[n];
      const int64_t rest = idx / m.inner;
      const int64_t pp = idx - rest * m.inner;
      const int64_t q = rest / m.I;
      const int64_t i = rest - q * m.I;
      const double* v = m.V + (int64_t)m.R * (pp + m.inner * q);
      double z = 0.0;
      for (int r = 0; r < m.R; ++r) z = fma(m.U[i + m.I * r], v[r], z);
      acc = __dadd_rn(acc, __dadd_rn(__dsub_rn(t, z), __dmul_rn(m.Y[idx], inv_mu)));
    }
    const double x = __dmul_rn(acc, inv_n);
    E[idx] = x > tau ? __dsub_rn(x, tau) : (x < -tau ? __dadd_rn(x, tau) : 0.0);  // linops.hpp:37-43
  }
}

// acc_i = sum_n (Y_n - Yhat_n) from 0.0 in mode order (pasd.cpp:287-292).
__global__ void k_cert_acc(const double* const* __restrict__ y, const double* const* __restrict__ yh, int order,
                           int64_t S, double* __restrict__ acc) {
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < S; idx += (int64_t)gridDim.x * blockDim.x) {
    double a = 0.0;
    for (int n = 0; n < order; ++n) a = __dadd_rn(a, __dsub_rn(y[n][idx], yh[n][idx]));
    acc[idx] = a;
  }
}

struct SpecTensors {
  std::vector<int64_t> dims;
  int64_t S = 0;
};

SpecTensors spec_dims(int32_t order, const int64_t* dims) {
  if (order < 1 || !dims) fail(PASD_ERR_ARGUMENT, "tensor order must be at least 1");
  SpecTensors st;
  st.dims.assign(dims, dims + order);
  st.S = dims_product(st.dims);
  return st;
}

void check_mode(const std::vector<int64_t>& dims, int32_t mode) {  // tensor.cpp:133-137
  if (mode < 1 || mode > (int32_t)dims.size())
    fail(PASD_ERR_ARGUMENT, "mode " + std::to_string(mode) + " out of range 1.." + std::to_string(dims.size()));
}

void check_mu(double mu) {
  if (!(mu > 0.0) || !std::isfinite(mu)) fail(PASD_ERR_ARGUMENT, "pasd_b200: mu must be a positive finite number");
}

double* upload(TmpDev& t, const double* h, int64_t n) {
  double* d = t.alloc<double>((size_t)std::max<int64_t>(n, 1));
  CK(cudaMemcpy(d, h, sizeof(double) * n, cudaMemcpyHostToDevice));
  return d;
}

constexpr int kSpecBlocks = 1184;

// Device G_n of a host state (the shared first step of update_u / update_v).
double* spec_g_device(TmpDev& tmp, const SpecTensors& st, const double* t, const double* e, const double* y, double mu,
                      int32_t mode) {
  check_mode(st.dims, mode);
  check_mu(mu);
  const double* dt = upload(tmp, t, st.S);
  const double* de = upload(tmp, e, st.S);
  const double* dy = upload(tmp, y, st.S);
  double* g = tmp.alloc<double>((size_t)st.S);
  int64_t inner = 1;
  for (int l = 0; l < mode - 1; ++l) inner *= st.dims[l];
  k_g_unfold<<<kSpecBlocks, 256>>>(dt, de, dy, 1.0 / mu, inner, st.dims[mode - 1], st.S, g);  // inv_mu = 1.0 / mu
  CK(cudaGetLastError());
  return g;
}

void spec_g_matrix(int32_t order, const int64_t* dims, const double* t, const double* e, const double* y, double mu,
                   int32_t mode, double* g_out, int device) {
  if (!t || !e || !y || !g_out) fail(PASD_ERR_ARGUMENT, "pasd_b200: null argument");
  const SpecTensors st = spec_dims(order, dims);
  CK(cudaSetDevice(device));
  TmpDev tmp;
  const double* g = spec_g_device(tmp, st, t, e, y, mu, mode);
  CK(cudaMemcpy(g_out, g, sizeof(double) * st.S, cudaMemcpyDeviceToHost));
}

// update_u = update_u_from(G_n, V_n, U_n): procrustes or keep U_n (pasd.cpp:70-74, 99-103).
void spec_update_u(int32_t order, const int64_t* dims, const double* t, const double* e, const double* y, double mu,
                   int32_t mode, int64_t rank, const double* u_prev, const double* v, double* u_out, int32_t* degenerate,
                   int device) {
  if (!t || !e || !y || !u_prev || !v || !u_out) fail(PASD_ERR_ARGUMENT, "pasd_b200: null argument");
  const SpecTensors st = spec_dims(order, dims);
  check_mode(st.dims, mode);
  const int64_t I = st.dims[mode - 1], J = st.S / I;
  if (rank < 1) fail(PASD_ERR_ARGUMENT, "config: rank of mode " + std::to_string(mode) + " must be positive");
  CK(cudaSetDevice(device));
  TmpDev tmp;
  const double* g = spec_g_device(tmp, st, t, e, y, mu, mode);
  int32_t deg = 0, rk = 0;
  device_procrustes(g, I, J, v, rank, u_prev, u_out, &deg, &rk, device, /*g_is_device=*/true);
  if (deg) std::memcpy(u_out, u_prev, sizeof(double) * I * rank);  // keep the previous basis
  if (degenerate) *degenerate = deg;
}

// update_v = svt(U_n^T G_n, lambda / mu) (pasd.cpp:76-78, 105-109).
void spec_update_v(int32_t order, const int64_t* dims, const double* t, const double* e, const double* y, double mu,
                   int32_t mode, int64_t rank, const double* u, double lambda, double* v_out, int32_t* kept,
                   int device) {
  if (!t || !e || !y || !u || !v_out) fail(PASD_ERR_ARGUMENT, "pasd_b200: null argument");
  const SpecTensors st = spec_dims(order, dims);
  check_mode(st.dims, mode);
  const int64_t I = st.dims[mode - 1], J = st.S / I;
  if (rank < 1) fail(PASD_ERR_ARGUMENT, "config: rank of mode " + std::to_string(mode) + " must be positive");
  CK(cudaSetDevice(device));
  TmpDev tmp;
  const double* g = spec_g_device(tmp, st, t, e, y, mu, mode);
  const double* du = upload(tmp, u, I * rank);
  double* a = tmp.alloc<double>((size_t)(rank * J));
  k_ut_g<<<kSpecBlocks, 256>>>(du, g, I, (int)rank, J, a);
  CK(cudaGetLastError());
  device_svt(a, rank, J, lambda / mu, v_out, kept, device, /*m_is_device=*/true);
}

void spec_update_e(int32_t order, const int64_t* dims, const int64_t* ranks, const double* t, const double* const* u,
                   const double* const* v, const double* const* y, double mu, double* e_out, int device) {
  if (!t || !u || !v || !y || !ranks || !e_out) fail(PASD_ERR_ARGUMENT, "pasd_b200: null argument");
  const SpecTensors st = spec_dims(order, dims);
  if (order > PASD_MAX_ORDER) fail(PASD_ERR_ARGUMENT, "pasd_b200: order exceeds the supported maximum");
  check_mu(mu);
  CK(cudaSetDevice(device));
  TmpDev tmp;
  SpecPack p{};
  p.order = order;
  int64_t inner = 1;
  for (int n = 0; n < order; ++n) {
    const int64_t I = st.dims[n], J = st.S / I, R = ranks[n];
    if (R < 1 || R > I)
      fail(PASD_ERR_ARGUMENT, "config: rank " + std::to_string(R) + " exceeds dimension " + std::to_string(I) +
                                  " in mode " + std::to_string(n + 1));
    if (!u[n] || !v[n] || !y[n]) fail(PASD_ERR_ARGUMENT, "pasd_b200: null argument");
    p.m[n] = SpecMode{inner, I, (int)R, upload(tmp, u[n], I * R), upload(tmp, v[n], R * J), upload(tmp, y[n], st.S)};
    inner *= I;
  }
  const double* dt = upload(tmp, t, st.S);
  double* de = tmp.alloc<double>((size_t)st.S);
  const double inv_n = 1.0 / (double)order;          // pasd.cpp:125
  const double tau = 1.0 / (mu * (double)order);     // pasd.cpp:126
  k_update_e<<<kSpecBlocks, 256>>>(p, dt, 1.0 / mu, inv_n, tau, st.S, de);
  CK(cudaGetLastError());
  CK(cudaMemcpy(e_out, de, sizeof(double) * st.S, cudaMemcpyDeviceToHost));
}

// suboptimality_certificate (pasd.cpp:277-309), reductions on the device.
void spec_certificate(const double* t, const pasd_options* o, int32_t iters, int32_t converged,
                      const double* const* y, const double* const* y_hat, double* eps_hat_out, double* c_out,
                      double* bound_out) {
  if (!o || !t) fail(PASD_ERR_ARGUMENT, "pasd_b200: null argument");
  validate_options(o);
  if (!converged) fail(PASD_ERR_STATE, "certificate requires a converged result");      // pasd.cpp:279-280
  if (!y || !y_hat) fail(PASD_ERR_STATE, "certificate requires the final multipliers");  // pasd.cpp:282-283
  const int N = o->order;
  for (int n = 0; n < N; ++n)
    if (!y[n] || !y_hat[n]) fail(PASD_ERR_STATE, "certificate requires the final multipliers");
  const SpecTensors st = spec_dims(N, o->dims);
  CK(cudaSetDevice(o->device));
  TmpDev tmp;
  std::vector<const double*> dy(N), dh(N);
  for (int n = 0; n < N; ++n) {
    dy[n] = upload(tmp, y[n], st.S);
    dh[n] = upload(tmp, y_hat[n], st.S);
  }
  const double** py = tmp.alloc<const double*>(N);
  const double** ph = tmp.alloc<const double*>(N);
  CK(cudaMemcpy(py, dy.data(), sizeof(double*) * N, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(ph, dh.data(), sizeof(double*) * N, cudaMemcpyHostToDevice));
  double* acc = tmp.alloc<double>((size_t)st.S);
  k_cert_acc<<<kSpecBlocks, 256>>>(py, ph, N, st.S, acc);
  const double* dt = upload(tmp, t, st.S);
  double* part = tmp.alloc<double>(4 * kSpecBlocks);
  std::vector<double> sums(kSpecBlocks), maxs(kSpecBlocks);
  auto stats = [&](const double* x, double* sum, double* mx) {
    k_abs_stats<<<kSpecBlocks, 256>>>(x, st.S, part, part + 2 * kSpecBlocks);
    CK(cudaGetLastError());
    CK(cudaMemcpy(sums.data(), part, sizeof(double) * kSpecBlocks, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(maxs.data(), part + 2 * kSpecBlocks, sizeof(double) * kSpecBlocks, cudaMemcpyDeviceToHost));
    double a = 0.0, m = 0.0;
    for (int b = 0; b < kSpecBlocks; ++b) {
      a += sums[b];
      m = std::max(m, maxs[b]);
    }
    if (sum) *sum = a;
    if (mx) *mx = m;
  };
  double eps_hat = 0.0, tl1 = 0.0;
  stats(acc, nullptr, &eps_hat);
  stats(dt, &tl1, nullptr);
  const int k_star = iters - 1;
  const double rho = o->rho;
  const double geom = rho * (1.0 + rho) / (rho - 1.0) + 0.5 / std::pow(rho, k_star);
  double dim_sum = 0.0, lam_term = 0.0;
  for (int n = 0; n < N; ++n) {
    dim_sum += (double)st.S;
    lam_term += o->lambdas[n] * (double)st.S * o->eps;
  }
  const double nn = (double)N;
  const double c = dim_sum * geom / (o->mu0 * nn * nn) + tl1;
  if (eps_hat_out) *eps_hat_out = eps_hat;
  if (c_out) *c_out = c;
  if (bound_out) *bound_out = c * eps_hat + lam_term;
}

// unfold_n(T), I_n x J_n column-major (tensor.cpp:98-113).
__global__ void k_unfold(const double* __restrict__ T, int64_t inner, int64_t I, int64_t S, double* __restrict__ G) {
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < S; idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t rest = idx / inner;
    const int64_t p = idx - rest * inner;
    const int64_t q = rest / I;
    const int64_t i = rest - q * I;
    G[i + I * (p + inner * q)] = T[idx];
  }
}

// Gaussian test matrix for the range finder (counter-based: splitmix64 of the
// index, Box-Muller).  Any full-rank draw serves; the seed is fixed.
__global__ void k_gauss(double* __restrict__ out, int64_t n, uint64_t seed) {
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < n; idx += (int64_t)gridDim.x * blockDim.x) {
    uint64_t x = seed + 0x9e3779b97f4a7c15ULL * (uint64_t)(2 * idx + 1);
    auto mix = [](uint64_t z) {
      z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
      z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
      return z ^ (z >> 31);
    };
    const uint64_t a = mix(x), b = mix(x + 0x9e3779b97f4a7c15ULL);
    const double u1 = ((double)((a >> 11) + 1)) * 0x1.0p-53, u2 = (double)(b >> 11) * 0x1.0p-53;
    out[idx] = sqrt(-2.0 * log(u1)) * cospi(2.0 * u2);
  }
}

// nuclear_norm(unfold(t, mode)) (linops.cpp:74-76 on tensor.cpp:139-146) on the
// device for unfoldings of numerical rank <= PASD_MAX_RANK: a Gaussian range
// finder (W = Z Omega^T, Omega: R' x J) through the Procrustes solve's two-pass
// Jacobi gives an orthonormal basis Q of range(Z) with the numerical rank k
// (singular values above 1e-12 sigma_1 of W); the singular values of Z are then
// those of the full-row-rank k x J matrix Q^T Z (Gram + Jacobi, k_svt).  Fails
// (ArgumentError) when ||Q^T Z||_F falls short of ||Z||_F, i.e. when the rank
// exceeds PASD_MAX_RANK.
double spec_nuclear_unfold(const double* t, int32_t order, const int64_t* dims, int32_t mode, int device) {
  if (!t) fail(PASD_ERR_ARGUMENT, "pasd_b200: null argument");
  const SpecTensors st = spec_dims(order, dims);
  check_mode(st.dims, mode);
  const int64_t I = st.dims[mode - 1], J = st.S / I;
  CK(cudaSetDevice(device));
  TmpDev tmp;
  const double* dt = upload(tmp, t, st.S);
  double* z = tmp.alloc<double>((size_t)st.S);
  int64_t inner = 1;
  for (int l = 0; l < mode - 1; ++l) inner *= st.dims[l];
  k_unfold<<<kSpecBlocks, 256>>>(dt, inner, I, st.S, z);
  const int Rp = (int)std::min<int64_t>({I, J, (int64_t)PASD_MAX_RANK});
  double* om = tmp.alloc<double>((size_t)(Rp * J));
  k_gauss<<<kSpecBlocks, 256>>>(om, Rp * J, 0x5eed5eedULL);
  double* xl = tmp.alloc<double>((size_t)(I * Rp));
  int32_t deg = 0, k = 0;
  device_procrustes(z, I, J, om, Rp, nullptr, nullptr, &deg, &k, device, true, true, xl);
  if (deg || k == 0) return 0.0;
  double* a = tmp.alloc<double>((size_t)(k * J));
  k_ut_g<<<kSpecBlocks, 256>>>(xl, z, I, k, J, a);
  CK(cudaGetLastError());
  std::vector<double> sig((size_t)k);
  device_svt(a, k, J, 1e-300, nullptr, nullptr, device, true, sig.data());
  double nuc = 0.0, s2 = 0.0;
  for (double v : sig) {
    nuc += v;
    s2 += v * v;
  }
  // ||Z||_F^2 against the captured energy
  double* part = tmp.alloc<double>(4 * kSpecBlocks);
  k_sumsq<<<1, 1024>>>(z, st.S, part);
  double z2 = 0.0;
  CK(cudaMemcpy(&z2, part, sizeof(double), cudaMemcpyDeviceToHost));
  if (k == Rp && Rp < std::min(I, J) && s2 < z2 * (1.0 - 1e-9))
    fail(PASD_ERR_ARGUMENT, "pasd_b200: nuclear_norm: mode-" + std::to_string(mode) + " unfolding has rank above " +
                                std::to_string(PASD_MAX_RANK));
  return nuc;
}

}  // namespace

extern "C" {

int pasd_b200_nuclear_norm_unfold(const double* t, int32_t order, const int64_t* dims, int32_t mode, double* out,
                                  int32_t device, char* errbuf, size_t errlen) {
  return guarded_call(errbuf, errlen, [&] {
    if (!out) fail(PASD_ERR_ARGUMENT, "pasd_b200: null argument");
    *out = spec_nuclear_unfold(t, order, dims, mode, device);
  });
}

int pasd_b200_g_matrix(int32_t order, const int64_t* dims, const double* t, const double* e, const double* y, double mu,
                       int32_t mode, double* g_out, int32_t device, char* errbuf, size_t errlen) {
  return guarded_call(errbuf, errlen, [&] { spec_g_matrix(order, dims, t, e, y, mu, mode, g_out, device); });
}

int pasd_b200_update_u(int32_t order, const int64_t* dims, const double* t, const double* e, const double* y,
                       double mu, int32_t mode, int64_t rank, const double* u_prev, const double* v, double* u_out,
                       int32_t* degenerate, int32_t device, char* errbuf, size_t errlen) {
  return guarded_call(errbuf, errlen, [&] {
    spec_update_u(order, dims, t, e, y, mu, mode, rank, u_prev, v, u_out, degenerate, device);
  });
}

int pasd_b200_update_v(int32_t order, const int64_t* dims, const double* t, const double* e, const double* y,
                       double mu, int32_t mode, int64_t rank, const double* u, double lambda, double* v_out,
                       int32_t* kept, int32_t device, char* errbuf, size_t errlen) {
  return guarded_call(errbuf, errlen, [&] {
    spec_update_v(order, dims, t, e, y, mu, mode, rank, u, lambda, v_out, kept, device);
  });
}

int pasd_b200_update_e(int32_t order, const int64_t* dims, const int64_t* ranks, const double* t,
                       const double* const* u, const double* const* v, const double* const* y, double mu,
                       double* e_out, int32_t device, char* errbuf, size_t errlen) {
  return guarded_call(errbuf, errlen, [&] { spec_update_e(order, dims, ranks, t, u, v, y, mu, e_out, device); });
}

int pasd_b200_certificate(const double* t, const pasd_options* opt, int32_t iters, int32_t converged,
                          const double* const* y, const double* const* y_hat, double* epsilon_hat, double* c,
                          double* bound, char* errbuf, size_t errlen) {
  return guarded_call(errbuf, errlen, [&] {
    spec_certificate(t, opt, iters, converged, y, y_hat, epsilon_hat, c, bound);
  });
}

}  // extern "C"
