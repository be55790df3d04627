// tenrec_b200/pasd.hpp — header-only C++ drop-in for the reference solver API
// (proj/include/tenrec/{pasd,recovery,tensor,errors}.hpp) over the C-ABI of
// include/pasd_b200.h.
//
//   tenrec::pasd_recover(t, config, observer)     (pasd.hpp:65-66)
//   -> tenrec_b200::pasd_recover(t, config, observer)
//
// Same option names and defaults (PasdConfig, pasd.hpp:8-27), same result
// layout (RecoveryResult, recovery.hpp:20-34), same exception types and
// messages (errors.hpp:9-30).  The reference's Eigen types are replaced by a
// minimal column-major Matrix and a first-index-fastest DenseTensor because
// Eigen is not a dependency of this build; `data()` layouts are identical.
#pragma once

#include <algorithm>
#include <cstdint>
#include <functional>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "../pasd_b200.h"

namespace tenrec_b200 {

using Index = std::int64_t;

// errors.hpp:9-30
class ArgumentError : public std::invalid_argument { using std::invalid_argument::invalid_argument; };
class IoError : public std::runtime_error { using std::runtime_error::runtime_error; };
class NumericalError : public std::runtime_error { using std::runtime_error::runtime_error; };
class StateError : public std::logic_error { using std::logic_error::logic_error; };
class DeviceError : public std::runtime_error { using std::runtime_error::runtime_error; };

// Column-major dense matrix (tensor.hpp:14-15).
struct Matrix {
  Index rows_ = 0, cols_ = 0;
  std::vector<double> data_;
  Matrix() = default;
  Matrix(Index r, Index c) : rows_(r), cols_(c), data_(static_cast<std::size_t>(r * c), 0.0) {}
  Index rows() const { return rows_; }
  Index cols() const { return cols_; }
  double* data() { return data_.data(); }
  const double* data() const { return data_.data(); }
  double& operator()(Index i, Index j) { return data_[static_cast<std::size_t>(i + rows_ * j)]; }
  double operator()(Index i, Index j) const { return data_[static_cast<std::size_t>(i + rows_ * j)]; }
};

// Dense N-order tensor, first index fastest (tensor.hpp:21-70).
class DenseTensor {
 public:
  DenseTensor() = default;
  static DenseTensor zeros(std::vector<Index> dims) {
    DenseTensor t;
    Index n = 1;
    for (Index d : dims) n *= d;
    t.dims_ = std::move(dims);
    t.data_.assign(static_cast<std::size_t>(n), 0.0);
    return t;
  }
  static DenseTensor from_data(std::vector<Index> dims, std::vector<double> data) {
    DenseTensor t;
    t.dims_ = std::move(dims);
    t.data_ = std::move(data);
    return t;
  }
  Index order() const { return static_cast<Index>(dims_.size()); }
  const std::vector<Index>& dims() const { return dims_; }
  Index dim(Index mode) const { return dims_[static_cast<std::size_t>(mode - 1)]; }
  Index size() const { return static_cast<Index>(data_.size()); }
  double* data() { return data_.data(); }
  const double* data() const { return data_.data(); }
  std::vector<double>& values() { return data_; }
  const std::vector<double>& values() const { return data_; }
  double operator[](Index i) const { return data_[static_cast<std::size_t>(i)]; }
  double& operator[](Index i) { return data_[static_cast<std::size_t>(i)]; }

 private:
  std::vector<Index> dims_;
  std::vector<double> data_;
};

// recovery.hpp:14-34
struct Certificate {
  double epsilon_hat = 0.0;
  double c = 0.0;
  double bound = 0.0;
};

struct RecoveryResult {
  DenseTensor x;
  DenseTensor e;
  std::vector<DenseTensor> z;
  int iters = 0;
  bool converged = false;
  std::vector<double> residual_history;
  std::vector<double> final_residuals;
  double objective = 0.0;
  std::optional<Certificate> certificate;
  std::vector<DenseTensor> y;
  std::vector<DenseTensor> y_hat;
};

// recovery.hpp:38-50: the same members, typed.  The referenced objects are
// host copies owned by the callback frame and valid only during the call
// (pasd.cpp:241-242).
struct IterationView {
  int iter = 0;        // 1-based count of completed iterations
  double mu_used = 0;  // penalty used by this iteration's updates
  double mu_next = 0;  // penalty after the schedule step
  const std::vector<double>& residual_inf;
  const DenseTensor& e;
  const std::vector<DenseTensor>& z;
  const std::vector<DenseTensor>& y;
  const std::vector<Matrix>* u = nullptr;  // I_n x R_n
  const std::vector<Matrix>* v = nullptr;  // R_n x J_n (unfolding column order)
};
using IterationObserver = std::function<void(const IterationView&)>;

// pasd.hpp:33-41
struct PasdState {
  std::vector<Matrix> u;
  std::vector<Matrix> v;
  DenseTensor e;
  std::vector<DenseTensor> y;
  std::vector<DenseTensor> y_hat;
  double mu = 0.0;
  int iter = 0;
};

// pasd.hpp:8-27
struct PasdConfig {
  std::vector<double> lambdas;
  std::vector<Index> ranks;
  double mu0 = 1e-4;
  double mu_max = 1e10;
  double rho = 1.1;
  double eps = 1e-5;
  int maxiter = 1000;
  std::vector<double> output_weights;
  int device = 0;  // placement (no reference analogue)
  bool fp32 = false;  // PASD_FLAG_FP32: float32 element storage, fp64 arithmetic (no reference analogue)

  const std::vector<double>& alphas() const { return output_weights.empty() ? lambdas : output_weights; }

  pasd_options to_c(const std::vector<Index>& dims) const {
    pasd_options o{};
    o.order = static_cast<int32_t>(dims.size());
    o.dims = dims.data();
    o.ranks = ranks.data();
    o.lambdas = lambdas.data();
    o.output_weights = output_weights.empty() ? nullptr : output_weights.data();
    o.mu0 = mu0;
    o.mu_max = mu_max;
    o.rho = rho;
    o.eps = eps;
    o.maxiter = maxiter;
    o.device = device;
    o.flags = fp32 ? PASD_FLAG_FP32 : PASD_FLAG_NONE;
    o.poll_every = 0;
    return o;
  }

  void validate(const std::vector<Index>& dims) const;                      // pasd.cpp:12-49
  static std::vector<double> default_lambdas(const std::vector<Index>& dims);  // pasd.cpp:51-60
  static Index default_rank_bound(Index target_rank);                        // pasd.cpp:62-66
};

namespace detail {
[[noreturn]] inline void rethrow(int rc, const char* msg) {
  switch (rc) {
    case PASD_ERR_ARGUMENT: throw ArgumentError(msg);
    case PASD_ERR_IO: throw IoError(msg);
    case PASD_ERR_NUMERICAL: throw NumericalError(msg);
    case PASD_ERR_STATE: throw StateError(msg);
    default: throw DeviceError(msg);
  }
}
inline void check(int rc, const char* msg) {
  if (rc != PASD_OK) rethrow(rc, msg);
}
inline void count_checks(const PasdConfig& c, std::size_t n) {
  if (c.lambdas.size() != n)
    throw ArgumentError("config: expected " + std::to_string(n) + " lambdas, got " + std::to_string(c.lambdas.size()));
  if (c.ranks.size() != n)
    throw ArgumentError("config: expected " + std::to_string(n) + " ranks, got " + std::to_string(c.ranks.size()));
  if (!c.output_weights.empty() && c.output_weights.size() != n)
    throw ArgumentError("config: expected " + std::to_string(n) + " output weights");
}
}  // namespace detail

inline void PasdConfig::validate(const std::vector<Index>& dims) const {
  detail::count_checks(*this, dims.size());
  pasd_options o = to_c(dims);
  char err[1024] = {0};
  detail::check(pasd_b200_validate(&o, err, sizeof(err)), err);
}

inline std::vector<double> PasdConfig::default_lambdas(const std::vector<Index>& dims) {
  std::vector<double> out(dims.size());
  char err[1024] = {0};
  detail::check(pasd_b200_default_lambdas(static_cast<int32_t>(dims.size()), dims.data(), out.data(), err,
                                          sizeof(err)),
                err);
  return out;
}

inline Index PasdConfig::default_rank_bound(Index target_rank) {
  int64_t out = 0;
  char err[1024] = {0};
  detail::check(pasd_b200_default_rank_bound(target_rank, &out, err, sizeof(err)), err);
  return out;
}

// Drop-in for tenrec::pasd_recover (pasd.hpp:65-66).
inline RecoveryResult pasd_recover(const DenseTensor& t, const PasdConfig& config,
                                   const IterationObserver& observer = {}) {
  const std::vector<Index>& dims = t.dims();
  detail::count_checks(config, dims.size());
  const std::size_t n = dims.size();
  pasd_options o = config.to_c(dims);
  RecoveryResult res;
  res.x = DenseTensor::zeros(dims);
  res.e = DenseTensor::zeros(dims);
  res.z.assign(n, DenseTensor::zeros(dims));
  res.y.assign(n, DenseTensor::zeros(dims));
  res.y_hat.assign(n, DenseTensor::zeros(dims));
  std::vector<double*> zp(n), yp(n), hp(n);
  for (std::size_t k = 0; k < n; ++k) {
    zp[k] = res.z[k].data();
    yp[k] = res.y[k].data();
    hp[k] = res.y_hat[k].data();
  }
  res.residual_history.assign(static_cast<std::size_t>(config.maxiter > 0 ? config.maxiter : 1), 0.0);
  res.final_residuals.assign(n, 0.0);
  pasd_outputs out{};
  out.x = res.x.data();
  out.e = res.e.data();
  out.z = zp.data();
  out.y = yp.data();
  out.y_hat = hp.data();
  out.residual_history = res.residual_history.data();
  out.final_residuals = res.final_residuals.data();
  struct Ctx {
    const IterationObserver* obs;
    const std::vector<Index>* dims;
    const std::vector<Index>* ranks;
  } ctx{&observer, &dims, &config.ranks};
  pasd_observer_fn fn = nullptr;
  if (observer) {
    fn = [](const pasd_iteration_view* v, void* user) {
      auto* c = static_cast<Ctx*>(user);
      const std::vector<Index>& d = *c->dims;
      const std::size_t N = d.size();
      Index S = 1;
      for (Index x : d) S *= x;
      auto tensor = [&](const double* p) { return DenseTensor::from_data(d, std::vector<double>(p, p + S)); };
      std::vector<double> resid(v->residual_inf, v->residual_inf + N);
      const DenseTensor e = tensor(v->e);
      std::vector<DenseTensor> z, y;
      std::vector<Matrix> u, vv;
      for (std::size_t k = 0; k < N; ++k) {
        z.push_back(tensor(v->z[k]));
        y.push_back(tensor(v->y[k]));
        const Index I = d[k], R = (*c->ranks)[k], J = S / I;
        Matrix um(I, R), vm(R, J);
        std::copy(v->u[k], v->u[k] + I * R, um.data());
        std::copy(v->v[k], v->v[k] + R * J, vm.data());
        u.push_back(std::move(um));
        vv.push_back(std::move(vm));
      }
      const IterationView view{v->iter, v->mu_used, v->mu_next, resid, e, z, y, &u, &vv};
      (*c->obs)(view);
    };
  }
  char err[1024] = {0};
  detail::check(pasd_b200_recover(t.data(), &o, &out, fn, &ctx, err, sizeof(err)), err);
  res.iters = out.iters;
  res.converged = out.converged != 0;
  res.residual_history.resize(static_cast<std::size_t>(out.iters));
  res.objective = out.objective;
  if (out.has_certificate) res.certificate = Certificate{out.cert_epsilon_hat, out.cert_c, out.cert_bound};
  return res;
}

// ---- spec-shaped single-step API (pasd.hpp:43-58, 68-70) ------------------
namespace detail {
inline void check_state(const PasdState& st, const DenseTensor& t, Index mode) {
  if (mode < 1 || mode > t.order())
    throw ArgumentError("mode " + std::to_string(mode) + " out of range 1.." + std::to_string(t.order()));
  const auto n = static_cast<std::size_t>(mode - 1);
  if (st.u.size() <= n || st.v.size() <= n || st.y.size() <= n)
    throw ArgumentError("pasd_b200: state has no basis / coefficients / multiplier for mode " + std::to_string(mode));
}
}  // namespace detail

// pasd_g_matrix (pasd.cpp:82-97)
inline Matrix pasd_g_matrix(const DenseTensor& t, const DenseTensor& e, const DenseTensor& y, double mu, Index mode,
                            int device = 0) {
  if (t.dims() != e.dims() || t.dims() != y.dims()) throw ArgumentError("g_matrix: dimension mismatch");
  if (mode < 1 || mode > t.order())
    throw ArgumentError("mode " + std::to_string(mode) + " out of range 1.." + std::to_string(t.order()));
  Matrix g(t.dim(mode), t.size() / t.dim(mode));
  char err[1024] = {0};
  detail::check(pasd_b200_g_matrix(static_cast<int32_t>(t.order()), t.dims().data(), t.data(), e.data(), y.data(), mu,
                                   static_cast<int32_t>(mode), g.data(), device, err, sizeof(err)),
                err);
  return g;
}

// update_u (pasd.cpp:99-103)
inline Matrix update_u(const PasdState& state, const DenseTensor& t, Index mode, int device = 0) {
  detail::check_state(state, t, mode);
  const auto n = static_cast<std::size_t>(mode - 1);
  const Matrix& up = state.u[n];
  Matrix u(up.rows(), up.cols());
  int32_t degenerate = 0;
  char err[1024] = {0};
  detail::check(pasd_b200_update_u(static_cast<int32_t>(t.order()), t.dims().data(), t.data(), state.e.data(),
                                   state.y[n].data(), state.mu, static_cast<int32_t>(mode), up.cols(), up.data(),
                                   state.v[n].data(), u.data(), &degenerate, device, err, sizeof(err)),
                err);
  return u;
}

// update_v (pasd.cpp:105-109)
inline Matrix update_v(const PasdState& state, const DenseTensor& t, Index mode, double lambda, int device = 0) {
  detail::check_state(state, t, mode);
  const auto n = static_cast<std::size_t>(mode - 1);
  const Index R = state.u[n].cols();
  Matrix v(R, t.size() / t.dim(mode));
  int32_t kept = 0;
  char err[1024] = {0};
  detail::check(pasd_b200_update_v(static_cast<int32_t>(t.order()), t.dims().data(), t.data(), state.e.data(),
                                   state.y[n].data(), state.mu, static_cast<int32_t>(mode), R, state.u[n].data(),
                                   lambda, v.data(), &kept, device, err, sizeof(err)),
                err);
  return v;
}

// update_e (pasd.cpp:111-130)
inline DenseTensor update_e(const PasdState& state, const DenseTensor& t, int device = 0) {
  const auto N = static_cast<std::size_t>(t.order());
  if (state.u.size() != N || state.v.size() != N || state.y.size() != N)
    throw ArgumentError("pasd_b200: state needs one basis / coefficient matrix / multiplier per mode");
  std::vector<Index> ranks(N);
  std::vector<const double*> u(N), v(N), y(N);
  for (std::size_t k = 0; k < N; ++k) {
    ranks[k] = state.u[k].cols();
    u[k] = state.u[k].data();
    v[k] = state.v[k].data();
    y[k] = state.y[k].data();
  }
  DenseTensor e = DenseTensor::zeros(t.dims());
  char err[1024] = {0};
  detail::check(pasd_b200_update_e(static_cast<int32_t>(N), t.dims().data(), ranks.data(), t.data(), u.data(),
                                   v.data(), y.data(), state.mu, e.data(), device, err, sizeof(err)),
                err);
  return e;
}

// suboptimality_certificate (pasd.cpp:277-309)
inline Certificate suboptimality_certificate(const RecoveryResult& result, const DenseTensor& t,
                                             const PasdConfig& config) {
  if (!result.converged) throw StateError("certificate requires a converged result");
  const auto N = static_cast<std::size_t>(t.order());
  if (result.y.size() != N || result.y_hat.size() != N) throw StateError("certificate requires the final multipliers");
  detail::count_checks(config, N);
  pasd_options o = config.to_c(t.dims());
  std::vector<const double*> y(N), h(N);
  for (std::size_t k = 0; k < N; ++k) {
    y[k] = result.y[k].data();
    h[k] = result.y_hat[k].data();
  }
  Certificate c;
  char err[1024] = {0};
  detail::check(pasd_b200_certificate(t.data(), &o, result.iters, 1, y.data(), h.data(), &c.epsilon_hat, &c.c,
                                      &c.bound, err, sizeof(err)),
                err);
  return c;
}

// baselines.hpp:9-20 -- the SNN / HoRPCA full-SVT baseline's settings.
struct SnnConfig {
  std::vector<double> lambdas;
  double mu0 = 1e-4;
  double mu_max = 1e10;
  double rho = 1.1;
  double eps = 1e-5;
  int maxiter = 1000;
  std::vector<double> output_weights;  // empty = lambdas
  int device = 0;

  const std::vector<double>& alphas() const { return output_weights.empty() ? lambdas : output_weights; }
};

// Drop-in for tenrec::snn_recover (baselines.hpp:39-40, baselines.cpp:37-143) on the device.
// Observer views carry u = v = nullptr, as the reference's; no y_hat, no certificate.
inline RecoveryResult snn_recover(const DenseTensor& t, const SnnConfig& config,
                                  const IterationObserver& observer = {}) {
  const std::vector<Index>& dims = t.dims();
  const std::size_t n = dims.size();
  if (config.lambdas.size() != n)  // baselines.cpp:15-17
    throw ArgumentError("config: expected " + std::to_string(n) + " lambdas, got " +
                        std::to_string(config.lambdas.size()));
  if (!config.output_weights.empty() && config.output_weights.size() != n)
    throw ArgumentError("config: expected " + std::to_string(n) + " output weights");
  pasd_options o{};
  o.order = static_cast<int32_t>(n);
  o.dims = dims.data();
  o.ranks = nullptr;
  o.lambdas = config.lambdas.data();
  o.output_weights = config.output_weights.empty() ? nullptr : config.output_weights.data();
  o.mu0 = config.mu0;
  o.mu_max = config.mu_max;
  o.rho = config.rho;
  o.eps = config.eps;
  o.maxiter = config.maxiter;
  o.device = config.device;
  RecoveryResult res;
  res.x = DenseTensor::zeros(dims);
  res.e = DenseTensor::zeros(dims);
  res.z.assign(n, DenseTensor::zeros(dims));
  res.y.assign(n, DenseTensor::zeros(dims));
  std::vector<double*> zp(n), yp(n);
  for (std::size_t k = 0; k < n; ++k) {
    zp[k] = res.z[k].data();
    yp[k] = res.y[k].data();
  }
  res.residual_history.assign(static_cast<std::size_t>(config.maxiter > 0 ? config.maxiter : 1), 0.0);
  res.final_residuals.assign(n, 0.0);
  pasd_outputs out{};
  out.x = res.x.data();
  out.e = res.e.data();
  out.z = zp.data();
  out.y = yp.data();
  out.residual_history = res.residual_history.data();
  out.final_residuals = res.final_residuals.data();
  struct Ctx {
    const IterationObserver* obs;
    const std::vector<Index>* dims;
  } ctx{&observer, &dims};
  pasd_observer_fn fn = nullptr;
  if (observer) {
    fn = [](const pasd_iteration_view* v, void* user) {
      auto* c = static_cast<Ctx*>(user);
      const std::vector<Index>& d = *c->dims;
      const std::size_t N = d.size();
      Index S = 1;
      for (Index x : d) S *= x;
      auto tensor = [&](const double* p) { return DenseTensor::from_data(d, std::vector<double>(p, p + S)); };
      std::vector<double> resid(v->residual_inf, v->residual_inf + N);
      const DenseTensor e = tensor(v->e);
      std::vector<DenseTensor> z, y;
      for (std::size_t k = 0; k < N; ++k) {
        z.push_back(tensor(v->z[k]));
        y.push_back(tensor(v->y[k]));
      }
      const IterationView view{v->iter, v->mu_used, v->mu_next, resid, e, z, y, nullptr, nullptr};
      (*c->obs)(view);
    };
  }
  char err[1024] = {0};
  detail::check(pasd_b200_snn_recover(t.data(), &o, &out, fn, &ctx, err, sizeof(err)), err);
  res.iters = out.iters;
  res.converged = out.converged != 0;
  res.residual_history.resize(static_cast<std::size_t>(out.iters));
  res.objective = out.objective;
  return res;
}

}  // namespace tenrec_b200
