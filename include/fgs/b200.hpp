// fgs/b200.hpp -- C++ drop-in for the reference's hot-path interface over the
// B200 C ABI (fgs_b200.h).  Header-only; link with -lfgs_b200.
//
// Mirrors, name for name (reference: /root/reference/proj/include/fgs):
//   errors.hpp:8-49      ParameterError, RangeError, ShapeError, NumericalError, ResourceError
//   kernels.hpp:20-35    KernelFamily, KernelSpec
//   fastsum.hpp:13-23    FastsumParams (+ preset)
//   nfft.hpp:59-94       NfftPlan (forward, adjoint, forward_real)
//   fastsum.hpp:34-67    FastsumPlan (apply, scaling, output_factor, kernel_zero,
//                        coefficients, kernel_error_estimate)
//   graphop.hpp:45-97    AdjacencyOperator (degrees, apply_kernel/weight/normalized/
//                        sym_laplacian)
//   spectral.hpp:18-30   SymmetricOperatorHandle, dense_handle, adjacency_handle,
//                        laplacian_handle
//   spectral.hpp:33-79   EigenPairs, LanczosOptions, LanczosInfo, lanczos_largest,
//                        adjacency_to_laplacian, residual_norms, max_residual
//   learn.hpp            KMeansOptions, KMeansResult, kmeans, spectral_cluster,
//                        misclassification_rate(_permuted), kernel_ssl_solve,
//                        kernel_ssl_truncated, RidgeModel, krr_fit, krr_predict
//   spectral.hpp:120-140 CgStatus, CgResult
//   spectral.hpp:81-86   NystromOptions, nystrom_gaussian
//   graphop.hpp:19-22    AdjacencyBackend {Fastsum, Direct}
// The reference's call sites compile unchanged, e.g. commands.cpp:179
//   pairs = lanczos_largest(adjacency_handle(op), opts.k, lopts, &info);
// A handle made by adjacency_handle / laplacian_handle remembers its device
// operator, so lanczos_largest / residual_norms / nystrom_gaussian on it run
// device-resident (Krylov basis in HBM, fgs_lanczos_largest); any other
// handle (dense_handle, a user std::function) runs the device recurrence
// with the caller's apply per step (fgs_lanczos_largest_operator).  The
// vector types are Eigen's when FGS_B200_WITH_EIGEN is defined, else the
// minimal column-major stand-ins below (Eigen is not installed in this build
// image).
#pragma once

#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdint>
#include <functional>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "fgs_b200.h"

#ifdef FGS_B200_WITH_EIGEN
#include <Eigen/Dense>
#endif

namespace fgs {

// ---- errors.hpp ------------------------------------------------------------
class ParameterError : public std::invalid_argument {
 public:
  using std::invalid_argument::invalid_argument;
};
class RangeError : public std::invalid_argument {
 public:
  using std::invalid_argument::invalid_argument;
};
class ShapeError : public std::invalid_argument {
 public:
  using std::invalid_argument::invalid_argument;
};
class NumericalError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class ResourceError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
/// CUDA / cuFFT / NCCL runtime failure (no reference analogue).
class DeviceError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};

namespace detail {
inline void check(fgs_status s) {
  if (s == FGS_OK) return;
  const std::string msg = fgs_last_error();
  switch (s) {
    case FGS_EPARAM: throw ParameterError(msg);
    case FGS_ERANGE: throw RangeError(msg);
    case FGS_ESHAPE: throw ShapeError(msg);
    case FGS_ENUMERIC: throw NumericalError(msg);
    case FGS_ERESOURCE: throw ResourceError(msg);
    default: throw DeviceError(msg);
  }
}
}  // namespace detail

// ---- vector types ----------------------------------------------------------
#ifdef FGS_B200_WITH_EIGEN
using Eigen::MatrixXd;
using Eigen::VectorXcd;
using Eigen::VectorXd;
using Index = Eigen::Index;
#else
using Index = std::int64_t;
template <class T>
class BasicVector {
 public:
  BasicVector() = default;
  explicit BasicVector(Index n) : v_(static_cast<size_t>(n), T(0)) {}
  static BasicVector Zero(Index n) { return BasicVector(n); }
  static BasicVector Ones(Index n) {
    BasicVector r(n);
    for (auto& x : r.v_) x = T(1);
    return r;
  }
  Index size() const { return static_cast<Index>(v_.size()); }
  T& operator()(Index i) { return v_[static_cast<size_t>(i)]; }
  const T& operator()(Index i) const { return v_[static_cast<size_t>(i)]; }
  T* data() { return v_.data(); }
  const T* data() const { return v_.data(); }
  void resize(Index n) { v_.resize(static_cast<size_t>(n)); }

 private:
  std::vector<T> v_;
};
using VectorXd = BasicVector<double>;
using VectorXcd = BasicVector<std::complex<double>>;

/// Column-major dense matrix (Eigen's default layout).
class MatrixXd {
 public:
  MatrixXd() = default;
  MatrixXd(Index r, Index c) : r_(r), c_(c), a_(static_cast<size_t>(r * c), 0.0) {}
  Index rows() const { return r_; }
  Index cols() const { return c_; }
  double& operator()(Index i, Index j) { return a_[static_cast<size_t>(j * r_ + i)]; }
  double operator()(Index i, Index j) const { return a_[static_cast<size_t>(j * r_ + i)]; }
  double* data() { return a_.data(); }
  const double* data() const { return a_.data(); }
  VectorXd col(Index j) const {
    VectorXd v(r_);
    for (Index i = 0; i < r_; ++i) v(i) = (*this)(i, j);
    return v;
  }

 private:
  Index r_ = 0, c_ = 0;
  std::vector<double> a_;
};
#endif

// ---- kernels.hpp / fastsum.hpp parameters ----------------------------------
enum class KernelFamily { Gaussian, LaplacianRbf, Multiquadric, InverseMultiquadric };

struct KernelSpec {
  KernelFamily family = KernelFamily::Gaussian;
  double shape = 1.0;
  static KernelSpec gaussian(double s) { return make(KernelFamily::Gaussian, s); }
  static KernelSpec laplacian_rbf(double s) { return make(KernelFamily::LaplacianRbf, s); }
  static KernelSpec multiquadric(double c) { return make(KernelFamily::Multiquadric, c); }
  static KernelSpec inverse_multiquadric(double c) { return make(KernelFamily::InverseMultiquadric, c); }

 private:
  static KernelSpec make(KernelFamily f, double s) {  // kernels.cpp:18-22
    if (!(s > 0.0) || !(s < 1e308)) throw ParameterError("kernel shape parameter must be positive and finite");
    return KernelSpec{f, s};
  }
};

struct FastsumParams {
  int bandwidth = 32;
  int cutoff = 4;
  int smoothness = 4;
  double eps_b = 0.0;
  double oversampling = 2.0;
  static FastsumParams preset(int level, double eps_b = 0.0) {
    fgs_fastsum_params p;
    detail::check(fgs_fastsum_preset(level, eps_b, &p));
    return FastsumParams{p.bandwidth, p.cutoff, p.smoothness, p.eps_b, p.oversampling};
  }
  fgs_fastsum_params c() const { return {bandwidth, cutoff, smoothness, eps_b, oversampling}; }
};

inline double bessel_i0(double x) {
  double r;
  detail::check(fgs_bessel_i0(x, &r));
  return r;
}

// ---- NfftPlan --------------------------------------------------------------
class NfftPlan {
 public:
  NfftPlan(int dims, int bandwidth, int cutoff, const MatrixXd& nodes, double oversampling = 2.0, int device = 0)
      : n_(nodes.rows()), d_(dims), N_(bandwidth), m_(cutoff) {
    detail::check(fgs_nfft_create(dims, bandwidth, cutoff, nodes.data(), nodes.rows(), oversampling, device, &h_));
    int M = 0;
    std::int64_t F = 0;
    detail::check(fgs_nfft_info(h_, &M, &F));
    M_ = M;
    F_ = F;
  }
  ~NfftPlan() { fgs_nfft_destroy(h_); }
  NfftPlan(NfftPlan&& o) noexcept { *this = std::move(o); }
  NfftPlan& operator=(NfftPlan&& o) noexcept {
    std::swap(h_, o.h_);
    n_ = o.n_;
    d_ = o.d_;
    N_ = o.N_;
    m_ = o.m_;
    M_ = o.M_;
    F_ = o.F_;
    return *this;
  }
  NfftPlan(const NfftPlan&) = delete;
  NfftPlan& operator=(const NfftPlan&) = delete;

  int dims() const { return d_; }
  int bandwidth() const { return N_; }
  int cutoff() const { return m_; }
  Index node_count() const { return n_; }
  std::size_t coefficient_count() const { return static_cast<std::size_t>(F_); }
  int grid_size() const { return M_; }

  VectorXcd forward(const VectorXcd& fhat) const {
    VectorXcd out(n_);
    detail::check(fgs_nfft_forward(h_, reinterpret_cast<const double*>(fhat.data()), fhat.size(),
                                   reinterpret_cast<double*>(out.data())));
    return out;
  }
  VectorXcd adjoint(const VectorXcd& x) const {
    VectorXcd out(F_);
    detail::check(fgs_nfft_adjoint(h_, reinterpret_cast<const double*>(x.data()), x.size(),
                                   reinterpret_cast<double*>(out.data())));
    return out;
  }
  VectorXd forward_real(const VectorXcd& fhat) const {
    VectorXd out(n_);
    detail::check(fgs_nfft_forward_real(h_, reinterpret_cast<const double*>(fhat.data()), fhat.size(), out.data()));
    return out;
  }

 private:
  fgs_nfft_t h_ = nullptr;
  Index n_ = 0;
  int d_ = 0, N_ = 0, m_ = 0, M_ = 0;
  std::int64_t F_ = 0;
};

// ---- FastsumPlan -----------------------------------------------------------
class FastsumPlan {
 public:
  FastsumPlan(const MatrixXd& nodes, const KernelSpec& kernel, const FastsumParams& params, int device = 0)
      : n_(nodes.rows()), d_(static_cast<int>(nodes.cols())), kernel_(kernel), params_(params) {
    const fgs_fastsum_params p = params.c();
    detail::check(fgs_fastsum_create(nodes.data(), nodes.rows(), d_, static_cast<fgs_kernel>(kernel.family),
                                     kernel.shape, &p, device, &h_));
    detail::check(fgs_fastsum_info(h_, &rho_, &of_, &k0_, &scaled_shape_));
  }
  ~FastsumPlan() { fgs_fastsum_destroy(h_); }
  FastsumPlan(const FastsumPlan&) = delete;
  FastsumPlan& operator=(const FastsumPlan&) = delete;

  Index size() const { return n_; }
  int dims() const { return d_; }
  const FastsumParams& params() const { return params_; }
  const KernelSpec& kernel() const { return kernel_; }
  KernelSpec scaled_kernel() const { return KernelSpec{kernel_.family, scaled_shape_}; }
  double scaling() const { return rho_; }
  double output_factor() const { return of_; }
  double kernel_zero() const { return k0_; }
  VectorXcd coefficients() const {
    Index F = 1;
    for (int t = 0; t < d_; ++t) F *= params_.bandwidth;
    VectorXcd c(F);
    detail::check(fgs_fastsum_coefficients(h_, reinterpret_cast<double*>(c.data())));
    return c;
  }
  VectorXd apply(const VectorXd& x) const {
    VectorXd y(n_);
    detail::check(fgs_fastsum_apply(h_, x.data(), x.size(), y.data()));
    return y;
  }
  fgs_fastsum_t handle() const { return h_; }
  double kernel_error_estimate(int sample_count, std::uint64_t seed) const {
    double r;
    detail::check(fgs_fastsum_error_estimate(h_, sample_count, seed, &r));
    return r;
  }

 private:
  fgs_fastsum_t h_ = nullptr;
  Index n_ = 0;
  int d_ = 0;
  KernelSpec kernel_;
  FastsumParams params_;
  double rho_ = 1.0, of_ = 1.0, k0_ = 0.0, scaled_shape_ = 1.0;
};

// ---- AdjacencyOperator -----------------------------------------------------
// graphop.hpp:19-22: Fastsum = NFFT fast summation, Direct = exact O(n^2) sums
enum class AdjacencyBackend { Fastsum, Direct };

class AdjacencyOperator {
 public:
  AdjacencyOperator(const MatrixXd& nodes, const KernelSpec& kernel, const FastsumParams& params,
                    AdjacencyBackend backend = AdjacencyBackend::Fastsum, int device = 0)
      : n_(nodes.rows()), d_(static_cast<int>(nodes.cols())), kernel_(kernel), backend_(backend) {
    const fgs_fastsum_params p = params.c();
    std::int64_t bad = -1;
    if (backend == AdjacencyBackend::Direct)
      detail::check(fgs_adjacency_create_direct(nodes.data(), nodes.rows(), d_,
                                                static_cast<fgs_kernel>(kernel.family), kernel.shape, device, &h_,
                                                &bad));
    else
      detail::check(fgs_adjacency_create(nodes.data(), nodes.rows(), d_, static_cast<fgs_kernel>(kernel.family),
                                         kernel.shape, &p, device, &h_, &bad));
    detail::check(fgs_adjacency_info(h_, nullptr, nullptr, &k0_, nullptr, nullptr));
    degrees_ = VectorXd(n_);
    detail::check(fgs_adjacency_degrees(h_, degrees_.data()));
  }
  ~AdjacencyOperator() { fgs_adjacency_destroy(h_); }
  AdjacencyOperator(const AdjacencyOperator&) = delete;
  AdjacencyOperator& operator=(const AdjacencyOperator&) = delete;

  Index size() const { return n_; }
  int dims() const { return d_; }
  const KernelSpec& kernel() const { return kernel_; }
  AdjacencyBackend backend() const { return backend_; }
  double kernel_zero() const { return k0_; }
  const VectorXd& degrees() const { return degrees_; }
  VectorXd apply_kernel(const VectorXd& x) const { return apply(FGS_OP_KERNEL, x); }
  VectorXd apply_weight(const VectorXd& x) const { return apply(FGS_OP_WEIGHT, x); }
  VectorXd apply_normalized(const VectorXd& x) const { return apply(FGS_OP_NORMALIZED, x); }
  VectorXd apply_sym_laplacian(const VectorXd& x) const { return apply(FGS_OP_SYM_LAPLACIAN, x); }
  fgs_adjacency_t handle() const { return h_; }

 private:
  VectorXd apply(fgs_op op, const VectorXd& x) const {
    if (x.size() != n_) throw ShapeError("input length does not match operator dimension");
    VectorXd y(n_);
    detail::check(fgs_adjacency_apply(h_, op, x.data(), y.data(), 1, n_));
    return y;
  }
  fgs_adjacency_t h_ = nullptr;
  Index n_ = 0;
  int d_ = 0;
  KernelSpec kernel_;
  AdjacencyBackend backend_ = AdjacencyBackend::Fastsum;
  double k0_ = 0.0;
  VectorXd degrees_;
};

// ---- spectral.hpp ----------------------------------------------------------
struct EigenPairs {
  VectorXd values;
  MatrixXd vectors;
  Index count() const { return values.size(); }
};

struct LanczosOptions {
  int max_iter = 1000;
  double tol = 1e-12;
  std::uint64_t seed = 1;
};

struct LanczosInfo {
  int iterations = 0;
  bool converged = false;
};

/// spectral.hpp:18-22: a symmetric operator as a dimension and an apply
/// function.  `device` / `which` are set by adjacency_handle /
/// laplacian_handle (non-owning, as the reference's handles,
/// spectral.hpp:28-30) and route the solvers to the device operator.
struct SymmetricOperatorHandle {
  Index dimension = 0;
  std::function<VectorXd(const VectorXd&)> apply;
  const AdjacencyOperator* device = nullptr;
  int which = 0;  // 0: A = D^-1/2 W D^-1/2, 1: L_s = I - A
};

/// spectral.cpp:79-89: a dense symmetric matrix as an operator
inline SymmetricOperatorHandle dense_handle(MatrixXd matrix) {
  if (matrix.rows() != matrix.cols()) throw ShapeError("dense operator must be square");
  auto shared = std::make_shared<MatrixXd>(std::move(matrix));
  SymmetricOperatorHandle h;
  h.dimension = shared->rows();
  h.apply = [shared](const VectorXd& x) -> VectorXd {
    const MatrixXd& a = *shared;
    VectorXd y(a.rows());
    for (Index i = 0; i < a.rows(); ++i) y(i) = 0.0;
    for (Index j = 0; j < a.cols(); ++j)
      for (Index i = 0; i < a.rows(); ++i) y(i) += a(i, j) * x(j);
    return y;
  };
  return h;
}

/// spectral.cpp:91-96
inline SymmetricOperatorHandle adjacency_handle(const AdjacencyOperator& op) {
  SymmetricOperatorHandle h;
  h.dimension = op.size();
  h.apply = [&op](const VectorXd& x) { return op.apply_normalized(x); };
  h.device = &op;
  h.which = 0;
  return h;
}

/// spectral.cpp:98-103
inline SymmetricOperatorHandle laplacian_handle(const AdjacencyOperator& op) {
  SymmetricOperatorHandle h;
  h.dimension = op.size();
  h.apply = [&op](const VectorXd& x) { return op.apply_sym_laplacian(x); };
  h.device = &op;
  h.which = 1;
  return h;
}

namespace detail {
inline EigenPairs pairs_from(Index n, int count, const std::vector<double>& vals, const MatrixXd& vecs,
                             bool with_vectors) {
  EigenPairs out;
  out.values = VectorXd(count);
  out.vectors = MatrixXd(with_vectors ? n : 0, count);
  for (int i = 0; i < count; ++i) {
    out.values(i) = vals[static_cast<size_t>(i)];
    if (with_vectors)
      for (Index r = 0; r < n; ++r) out.vectors(r, i) = vecs(r, i);
  }
  return out;
}
inline int apply_trampoline(void* ctx, const double* x, double* y, std::int64_t n) {
  try {
    const auto& h = *static_cast<const SymmetricOperatorHandle*>(ctx);
    VectorXd xv(n);
    for (std::int64_t i = 0; i < n; ++i) xv(i) = x[i];
    const VectorXd yv = h.apply(xv);
    if (yv.size() != n) return 1;
    for (std::int64_t i = 0; i < n; ++i) y[i] = yv(i);
    return 0;
  } catch (...) {
    return 1;
  }
}
}  // namespace detail

/// spectral.cpp:141-256 on any handle: device-resident over the fast graph
/// operator when the handle came from adjacency_handle / laplacian_handle,
/// else the device recurrence with the handle's apply per step.
inline EigenPairs lanczos_largest(const SymmetricOperatorHandle& op, int k, const LanczosOptions& opts = {},
                                  LanczosInfo* info = nullptr, int device = 0) {
  if (op.dimension < 1 || (!op.apply && !op.device)) throw ParameterError("operator handle is empty");
  const Index n = op.dimension;
  std::vector<double> vals(static_cast<size_t>(k > 0 ? k : 1));
  MatrixXd vecs(n, k > 0 ? k : 1);
  int count = 0, it = 0, conv = 0;
  if (op.device)
    detail::check(fgs_lanczos_largest(op.device->handle(), op.which, k, opts.max_iter, opts.tol, opts.seed,
                                      vals.data(), vecs.data(), &count, &it, &conv));
  else
    detail::check(fgs_lanczos_largest_operator(n, &detail::apply_trampoline, const_cast<SymmetricOperatorHandle*>(&op),
                                               device, k, opts.max_iter, opts.tol, opts.seed, vals.data(),
                                               vecs.data(), &count, &it, &conv));
  if (info) {
    info->iterations = it;
    info->converged = conv != 0;
  }
  return detail::pairs_from(n, count, vals, vecs, true);
}

/// k largest eigenpairs of A = D^-1/2 W D^-1/2 (what lanczos_largest(
/// adjacency_handle(op), ...) computes in the reference, spectral.cpp:91-96).
inline EigenPairs lanczos_largest(const AdjacencyOperator& op, int k, const LanczosOptions& opts = {},
                                  LanczosInfo* info = nullptr) {
  const Index n = op.size();
  std::vector<double> vals(static_cast<size_t>(k > 0 ? k : 1));
  MatrixXd vecs(n, k > 0 ? k : 1);
  int count = 0, it = 0, conv = 0;
  detail::check(fgs_lanczos_largest(op.handle(), 0, k, opts.max_iter, opts.tol, opts.seed, vals.data(),
                                    vecs.data(), &count, &it, &conv));
  if (info) {
    info->iterations = it;
    info->converged = conv != 0;
  }
  EigenPairs out;
  out.values = VectorXd(count);
  out.vectors = MatrixXd(n, count);
  for (int i = 0; i < count; ++i) {
    out.values(i) = vals[static_cast<size_t>(i)];
    for (Index r = 0; r < n; ++r) out.vectors(r, i) = vecs(r, i);
  }
  return out;
}

/// spectral.cpp:129-139
inline EigenPairs adjacency_to_laplacian(const EigenPairs& pairs) {
  const Index k = pairs.count();
  EigenPairs out;
  out.values = VectorXd(k);
  out.vectors = MatrixXd(pairs.vectors.rows(), k);
  for (Index i = 0; i < k; ++i) {
    out.values(i) = 1.0 - pairs.values(k - 1 - i);
    for (Index r = 0; r < pairs.vectors.rows(); ++r) out.vectors(r, i) = pairs.vectors(r, k - 1 - i);
  }
  return out;
}

/// spectral.cpp:258-275: ||A v_j - lambda_j v_j||_2 per pair, A applied on
/// the device (one block apply of all pairs).
inline VectorXd residual_norms(const AdjacencyOperator& op, const EigenPairs& pairs) {
  const Index n = op.size(), k = pairs.count();
  if (k > 0 && pairs.vectors.rows() != n) throw ShapeError("eigenvector length does not match operator dimension");
  VectorXd norms(k);
  if (k == 0) return norms;
  MatrixXd av(n, k);
  detail::check(fgs_adjacency_apply(op.handle(), FGS_OP_NORMALIZED, pairs.vectors.data(), av.data(),
                                    static_cast<int>(k), n));
  for (Index j = 0; j < k; ++j) {
    double s = 0.0;
    for (Index i = 0; i < n; ++i) {
      const double r = av(i, j) - pairs.values(j) * pairs.vectors(i, j);
      s += r * r;
    }
    norms(j) = std::sqrt(s);
  }
  return norms;
}

inline double max_residual(const AdjacencyOperator& op, const EigenPairs& pairs) {
  if (pairs.count() == 0) return 0.0;
  VectorXd r = residual_norms(op, pairs);
  double m = r(0);
  for (Index j = 1; j < r.size(); ++j) m = std::max(m, r(j));
  return m;
}

/// spectral.cpp:258-269 on any handle (device block apply for the graph
/// operator's handles; the handle's apply per pair otherwise)
inline VectorXd residual_norms(const SymmetricOperatorHandle& reference, const EigenPairs& pairs) {
  if (reference.dimension < 1 || (!reference.apply && !reference.device))
    throw ParameterError("operator handle is empty");
  const Index n = reference.dimension, k = pairs.count();
  if (k > 0 && pairs.vectors.rows() != n) throw ShapeError("eigenvector length does not match operator dimension");
  VectorXd norms(k);
  if (k == 0) return norms;
  MatrixXd av(n, k);
  if (reference.device) {
    detail::check(fgs_adjacency_apply(reference.device->handle(),
                                      reference.which == 0 ? FGS_OP_NORMALIZED : FGS_OP_SYM_LAPLACIAN,
                                      pairs.vectors.data(), av.data(), static_cast<int>(k), n));
  } else {
    for (Index j = 0; j < k; ++j) {
      VectorXd v(n);
      for (Index i = 0; i < n; ++i) v(i) = pairs.vectors(i, j);
      const VectorXd y = reference.apply(v);
      if (y.size() != n) throw ShapeError("vector length does not match operator dimension");
      for (Index i = 0; i < n; ++i) av(i, j) = y(i);
    }
  }
  for (Index j = 0; j < k; ++j) {
    double s = 0.0;
    for (Index i = 0; i < n; ++i) {
      const double r = av(i, j) - pairs.values(j) * pairs.vectors(i, j);
      s += r * r;
    }
    norms(j) = std::sqrt(s);
  }
  return norms;
}

inline double max_residual(const SymmetricOperatorHandle& reference, const EigenPairs& pairs) {
  if (pairs.count() == 0) return 0.0;
  VectorXd r = residual_norms(reference, pairs);
  double m = r(0);
  for (Index j = 1; j < r.size(); ++j) m = std::max(m, r(j));
  return m;
}

// ---- spectral.hpp:81-86 Nystrom (spectral.cpp:384-444) ---------------------
struct NystromOptions {
  int k = 10;
  int L = 100;
  int M = 10;
  std::uint64_t seed = 1;
};

/// nystrom_gaussian(adjacency_handle(op), opts): the 2L operator applies run
/// as block applies on the device
inline EigenPairs nystrom_gaussian(const AdjacencyOperator& op, const NystromOptions& opts = {}) {
  const Index n = op.size();
  std::vector<double> vals(static_cast<size_t>(opts.k > 0 ? opts.k : 1));
  MatrixXd vecs(n, opts.k > 0 ? opts.k : 1);
  detail::check(fgs_nystrom_gaussian(op.handle(), opts.k, opts.L, opts.M, opts.seed, vals.data(), vecs.data()));
  EigenPairs out;
  out.values = VectorXd(opts.k);
  out.vectors = MatrixXd(n, opts.k);
  for (int i = 0; i < opts.k; ++i) {
    out.values(i) = vals[static_cast<size_t>(i)];
    for (Index r = 0; r < n; ++r) out.vectors(r, i) = vecs(r, i);
  }
  return out;
}

/// nystrom_gaussian(adjacency_handle(op), opts) as the reference's CLI calls it
/// (commands.cpp:207): device block applies of the graph operator
inline EigenPairs nystrom_gaussian(const SymmetricOperatorHandle& op, const NystromOptions& opts) {
  if (!op.device || op.which != 0)
    throw ParameterError("nystrom_gaussian runs on adjacency_handle(op) of a device AdjacencyOperator");
  return nystrom_gaussian(*op.device, opts);
}

// ---- spectral.hpp:120-140 CG, learn.hpp SSL / ridge (learn.cpp:364-445) ----
enum class CgStatus { Converged, MaxIterations, Indefinite };

struct CgResult {
  VectorXd x;
  int iterations = 0;
  CgStatus status = CgStatus::MaxIterations;
  bool converged() const { return status == CgStatus::Converged; }
};

/// (I + beta L_s) u = f by conjugate gradients on the device (beta = 0: u = f)
inline CgResult kernel_ssl_solve(const AdjacencyOperator& op, const VectorXd& f, double beta, double tol = 1e-4,
                                 int max_iter = 1000) {
  CgResult r;
  r.x = VectorXd(f.size());
  int it = 0, st = 1;
  detail::check(fgs_kernel_ssl_solve(op.handle(), f.data(), f.size(), beta, tol, max_iter, r.x.data(), &it, &st));
  r.iterations = it;
  r.status = static_cast<CgStatus>(st);
  return r;
}

/// learn.cpp:383-394: closed form in a truncated eigenbasis of A
inline VectorXd kernel_ssl_truncated(const EigenPairs& pairs, const VectorXd& f, double beta) {
  if (!(beta >= 0.0)) throw ParameterError("beta must be nonnegative");
  const Index n = f.size(), k = pairs.count();
  if (k > 0 && pairs.vectors.rows() != n) throw ShapeError("fidelity length does not match eigenvectors");
  std::vector<double> coords(static_cast<size_t>(k), 0.0);
  for (Index j = 0; j < k; ++j)
    for (Index i = 0; i < n; ++i) coords[static_cast<size_t>(j)] += pairs.vectors(i, j) * f(i);
  VectorXd out(n);
  for (Index i = 0; i < n; ++i) {
    double inside = 0.0, projected = 0.0;
    for (Index j = 0; j < k; ++j) {
      const double c = coords[static_cast<size_t>(j)];
      inside += pairs.vectors(i, j) * (c / (1.0 + beta * (1.0 - pairs.values(j))));
      projected += pairs.vectors(i, j) * c;
    }
    out(i) = inside + (f(i) - projected) / (1.0 + beta);
  }
  return out;
}

struct RidgeModel {
  MatrixXd train_nodes;
  KernelSpec kernel;
  FastsumParams params;
  double beta = 0.0;
  VectorXd alpha;
  int cg_iterations = 0;
  double cg_tol = 0.0;
};

/// (K + beta I) alpha = f by device CG over a FastsumPlan (learn.cpp:403-430)
inline RidgeModel krr_fit(const MatrixXd& train_nodes, const KernelSpec& kernel, double beta, const VectorXd& f,
                          const FastsumParams& params, double tol = 1e-6, int max_iter = 1000, int device = 0) {
  if (!(beta > 0.0)) throw ParameterError("beta must be positive");
  if (f.size() != train_nodes.rows()) throw ShapeError("target length does not match training node count");
  FastsumPlan plan(train_nodes, kernel, params, device);
  RidgeModel m;
  m.alpha = VectorXd(f.size());
  int it = 0, st = 1;
  detail::check(fgs_fastsum_ridge_solve(plan.handle(), f.data(), f.size(), beta, tol, max_iter, m.alpha.data(), &it,
                                        &st));
  if (st == 2)
    throw NumericalError("regularized Gram operator is indefinite for this kernel; solve dense regularized normal "
                         "equations instead");
  m.train_nodes = train_nodes;
  m.kernel = kernel;
  m.params = params;
  m.beta = beta;
  m.cg_iterations = it;
  m.cg_tol = tol;
  return m;
}

/// learn.cpp:432-445: one fast summation over train + query nodes
inline VectorXd krr_predict(const RidgeModel& model, const MatrixXd& query, int device = 0) {
  if (query.cols() != model.train_nodes.cols()) throw ShapeError("query dimension does not match training dimension");
  const Index nt = model.train_nodes.rows(), nq = query.rows(), d = query.cols();
  MatrixXd all(nt + nq, d);
  for (Index t = 0; t < d; ++t) {
    for (Index i = 0; i < nt; ++i) all(i, t) = model.train_nodes(i, t);
    for (Index i = 0; i < nq; ++i) all(nt + i, t) = query(i, t);
  }
  FastsumPlan plan(all, model.kernel, model.params, device);
  VectorXd masked(nt + nq);
  for (Index i = 0; i < nt + nq; ++i) masked(i) = i < nt ? model.alpha(i) : 0.0;
  const VectorXd y = plan.apply(masked);
  VectorXd out(nq);
  for (Index i = 0; i < nq; ++i) out(i) = y(nt + i);
  return out;
}

// ---- learn.hpp: k-means / spectral clustering (learn.cpp:17-167) ----------
struct KMeansOptions {
  int restarts = 10;
  int max_iter = 100;
  std::uint64_t seed = 1;
};

struct KMeansResult {
  std::vector<int> labels;
  MatrixXd centroids;  // k x d
  double wcss = 0.0;
};

inline KMeansResult kmeans(const MatrixXd& points, int k, const KMeansOptions& opts = {}, int device = 0) {
  KMeansResult r;
  r.labels.resize(static_cast<size_t>(points.rows()));
  r.centroids = MatrixXd(k > 0 ? k : 0, points.cols());
  detail::check(fgs_kmeans(points.data(), points.rows(), static_cast<int>(points.cols()), k, opts.restarts,
                           opts.max_iter, opts.seed, device, r.labels.data(), k > 0 ? r.centroids.data() : nullptr,
                           &r.wcss));
  return r;
}

inline std::vector<int> spectral_cluster(const EigenPairs& pairs, int k_clusters, const KMeansOptions& opts = {},
                                         int device = 0) {
  std::vector<int> labels(static_cast<size_t>(pairs.vectors.rows()));
  detail::check(fgs_spectral_cluster(pairs.vectors.data(), pairs.vectors.rows(),
                                     static_cast<int>(pairs.vectors.cols()), k_clusters, opts.restarts,
                                     opts.max_iter, opts.seed, device, 0, labels.data()));
  return labels;
}

inline double misclassification_rate(const std::vector<int>& predicted, const std::vector<int>& truth) {
  if (predicted.size() != truth.size()) throw ShapeError("label vectors differ in length");
  double r;
  detail::check(fgs_misclassification_rate(predicted.data(), truth.data(), static_cast<std::int64_t>(predicted.size()),
                                           0, &r));
  return r;
}

inline double misclassification_rate_permuted(const std::vector<int>& predicted, const std::vector<int>& truth) {
  if (predicted.size() != truth.size()) throw ShapeError("label vectors differ in length");
  double r;
  detail::check(fgs_misclassification_rate(predicted.data(), truth.data(), static_cast<std::int64_t>(predicted.size()),
                                           1, &r));
  return r;
}

}  // namespace fgs
