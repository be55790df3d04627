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

// recovery.hpp:38-50 (u/v are column-major host copies).
struct IterationView {
  int iter = 0;
  double mu_used = 0;
  double mu_next = 0;
  std::vector<double> residual_inf;
  const pasd_iteration_view* raw = nullptr;  // e, z, y, u, v pointers, valid during the callback
};
using IterationObserver = std::function<void(const IterationView&)>;

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
    o.flags = PASD_FLAG_NONE;
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
    std::size_t n;
  } ctx{&observer, n};
  pasd_observer_fn fn = nullptr;
  if (observer) {
    fn = [](const pasd_iteration_view* v, void* user) {
      auto* c = static_cast<Ctx*>(user);
      IterationView view;
      view.iter = v->iter;
      view.mu_used = v->mu_used;
      view.mu_next = v->mu_next;
      view.residual_inf.assign(v->residual_inf, v->residual_inf + c->n);
      view.raw = v;
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

}  // namespace tenrec_b200
