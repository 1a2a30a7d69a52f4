// ============================================================================
// eigen_shim.hpp -- TEST INFRASTRUCTURE ONLY.
//
// A minimal, eager stand-in for the subset of Eigen 3 that the reference's
// hot-path sources use (/root/reference/proj/src/{nfft,kernels,fastsum,
// graphop,spectral}.cpp and their headers), so those files compile here
// UNCHANGED (Eigen3 is absent from this image) into
// oracle/_ref/libfgsref.so by oracle/build_ref.sh.  It is not Eigen: every
// expression is evaluated immediately into a column-major owning Matrix, and
// the reductions run serially in index order, the same IEEE operations the
// oracle restatement (fgs_oracle.cpp) performs:
//   dot / squaredNorm / sum     s = 0; s += a_i * b_i, i ascending
//   A * B                       C(:, j) += A(:, k) * B(k, j), k ascending
//   normalize, v / s            division by the scalar
//   rsqrt                       1 / sqrt(x)
// Real Eigen vectorises its reductions; results differ from a real-Eigen
// build at the rounding level only.  The dense / tridiagonal symmetric
// eigensolvers and the Householder QR come from oracle/linalg.hpp (the
// oracle's own), so both sides share them bit for bit.
// Views (col, row, leftCols, rightCols, topRows, transpose, Map, Ref) are
// strided pointers into the owning storage and write through on assignment.
// ============================================================================
#pragma once

#include <algorithm>
#include <cmath>
#include <complex>
#include <cstddef>
#include <stdexcept>
#include <type_traits>
#include <utility>
#include <vector>

#include "../linalg.hpp"

namespace Eigen {

using Index = std::ptrdiff_t;
enum NoChange_t { NoChange };
enum DecompositionOptions { ComputeEigenvectors = 1, EigenvaluesOnly = 2 };
enum UpLoType { Lower = 1, Upper = 2 };

template <class S>
class Matrix;
template <class S>
class Block;
template <class S>
class ArrayRef;
template <class S>
class ArrayVal;
template <class S>
struct DiagonalWrapper;
template <class S>
struct Rowwise;

namespace internal {
template <class S>
inline S rsqrt(S x) {
  return S(1) / std::sqrt(x);
}
template <class S>
struct real_of {
  using type = double;
};
inline double real_part(double x) { return x; }
inline double real_part(const std::complex<double>& x) { return x.real(); }
inline double imag_part(double) { return 0.0; }
inline double imag_part(const std::complex<double>& x) { return x.imag(); }

// is X a dense object of this shim (has view())?
template <class X, class = void>
struct is_dense : std::false_type {};
template <class X>
struct is_dense<X, std::void_t<decltype(std::declval<const X&>().view())>> : std::true_type {};
template <class X>
inline constexpr bool is_dense_v = is_dense<std::decay_t<X>>::value;
template <class X>
using scalar_t = typename std::decay_t<decltype(std::declval<const X&>().view())>::Scalar;
}  // namespace internal

// ---- read-only interface shared by Matrix and Block (CRTP) -----------------
template <class Derived, class S>
class DenseOps {
  const Derived& self() const { return static_cast<const Derived&>(*this); }

 public:
  Block<S> col(Index j) const { Block<S> v = self().view(); return Block<S>(v.p + j * v.cs, v.r, 1, v.rs, v.cs); }
  Block<S> row(Index i) const { Block<S> v = self().view(); return Block<S>(v.p + i * v.rs, 1, v.c, v.rs, v.cs); }
  Block<S> leftCols(Index k) const { Block<S> v = self().view(); return Block<S>(v.p, v.r, k, v.rs, v.cs); }
  Block<S> rightCols(Index k) const {
    Block<S> v = self().view();
    return Block<S>(v.p + (v.c - k) * v.cs, v.r, k, v.rs, v.cs);
  }
  Block<S> topRows(Index k) const { Block<S> v = self().view(); return Block<S>(v.p, k, v.c, v.rs, v.cs); }
  Block<S> transpose() const { Block<S> v = self().view(); return Block<S>(v.p, v.c, v.r, v.cs, v.rs); }

  template <class X, class = std::enable_if_t<internal::is_dense_v<X>>>
  S dot(const X& o) const {
    Block<S> a = self().view(), b = o.view();
    if (a.size() != b.size()) throw std::invalid_argument("eigen shim: dot of different sizes");
    S s = S(0);
    for (Index i = 0; i < a.size(); ++i) s += a.lin(i) * b.lin(i);
    return s;
  }
  double squaredNorm() const {
    Block<S> a = self().view();
    double s = 0.0;
    for (Index i = 0; i < a.size(); ++i) s += std::norm(a.lin(i));
    return s;
  }
  double norm() const { return std::sqrt(squaredNorm()); }
  S sum() const {
    Block<S> a = self().view();
    S s = S(0);
    for (Index i = 0; i < a.size(); ++i) s += a.lin(i);
    return s;
  }
  S maxCoeff() const { return extreme(true, nullptr); }
  S maxCoeff(Index* at) const { return extreme(true, at); }
  S minCoeff() const { return extreme(false, nullptr); }
  S minCoeff(Index* at) const { return extreme(false, at); }

  Matrix<typename internal::real_of<S>::type> cwiseAbs() const {
    Block<S> a = self().view();
    Matrix<typename internal::real_of<S>::type> out(a.r, a.c);
    for (Index i = 0; i < a.size(); ++i) out.data()[i] = std::abs(a.lin(i));
    return out;
  }
  Matrix<typename internal::real_of<S>::type> real() const {
    Block<S> a = self().view();
    Matrix<typename internal::real_of<S>::type> out(a.r, a.c);
    for (Index i = 0; i < a.size(); ++i) out.data()[i] = internal::real_part(a.lin(i));
    return out;
  }
  Matrix<typename internal::real_of<S>::type> imag() const {
    Block<S> a = self().view();
    Matrix<typename internal::real_of<S>::type> out(a.r, a.c);
    for (Index i = 0; i < a.size(); ++i) out.data()[i] = internal::imag_part(a.lin(i));
    return out;
  }
  template <class X>
  Matrix<S> cwiseProduct(const X& o) const { return zip(o, [](S x, S y) { return x * y; }); }
  template <class X>
  Matrix<S> cwiseQuotient(const X& o) const { return zip(o, [](S x, S y) { return x / y; }); }
  Matrix<S> cwiseInverse() const { return map([](S x) { return S(1) / x; }); }
  template <class T>
  Matrix<T> cast() const {
    Block<S> a = self().view();
    Matrix<T> out(a.r, a.c);
    for (Index i = 0; i < a.size(); ++i) out.data()[i] = static_cast<T>(a.lin(i));
    return out;
  }
  Matrix<S> eval() const { return Matrix<S>(self()); }
  Matrix<S> normalized() const { Matrix<S> m(self()); m.normalize(); return m; }
  ArrayRef<S> array() const { return ArrayRef<S>(self().view()); }
  DiagonalWrapper<S> asDiagonal() const { return DiagonalWrapper<S>{Matrix<S>(self())}; }
  Rowwise<S> rowwise() const { return Rowwise<S>{self().view()}; }
  template <int Mode>
  Matrix<S> triangularView() const {
    static_assert(Mode == Upper, "eigen shim: only triangularView<Upper> is provided");
    Matrix<S> m(self());
    for (Index j = 0; j < m.cols(); ++j)
      for (Index i = j + 1; i < m.rows(); ++i) m(i, j) = S(0);
    return m;
  }

  template <class F>
  Matrix<S> map(F f) const {
    Block<S> a = self().view();
    Matrix<S> out(a.r, a.c);
    for (Index i = 0; i < a.size(); ++i) out.data()[i] = f(a.lin(i));
    return out;
  }
  template <class X, class F>
  Matrix<S> zip(const X& o, F f) const {
    Block<S> a = self().view();
    auto b = o.view();
    if (a.r != b.r || a.c != b.c) throw std::invalid_argument("eigen shim: shape mismatch");
    Matrix<S> out(a.r, a.c);
    for (Index i = 0; i < a.size(); ++i) out.data()[i] = f(a.lin(i), b.lin(i));
    return out;
  }

 private:
  S extreme(bool want_max, Index* at) const {
    Block<S> a = self().view();
    if (a.size() == 0) throw std::invalid_argument("eigen shim: extreme of an empty object");
    Index best = 0;
    for (Index i = 1; i < a.size(); ++i)  // first occurrence wins (Eigen's visitor)
      if (want_max ? (a.lin(i) > a.lin(best)) : (a.lin(i) < a.lin(best))) best = i;
    if (at) *at = best;
    return a.lin(best);
  }
};

// ---- strided view -----------------------------------------------------------
template <class S>
class Block : public DenseOps<Block<S>, S> {
 public:
  using Scalar = S;
  S* p;
  Index r, c, rs, cs;  // element (i, j) at p[i * rs + j * cs]

  Block(S* p_, Index r_, Index c_, Index rs_, Index cs_) : p(p_), r(r_), c(c_), rs(rs_), cs(cs_) {}
  Block(const Block&) = default;

  Index rows() const { return r; }
  Index cols() const { return c; }
  Index size() const { return r * c; }
  Block view() const { return *this; }
  // column-major linear index
  S& lin(Index i) const { return p[(i % r) * rs + (i / r) * cs]; }
  S& operator()(Index i, Index j) const { return p[i * rs + j * cs]; }
  S& operator()(Index i) const { return r == 1 ? p[i * cs] : lin(i); }

  Block& operator=(const Block& o) { return assign(o); }
  template <class X, class = std::enable_if_t<internal::is_dense_v<X>>>
  Block& operator=(const X& o) {
    return assign(o);
  }
  template <class X>
  Block& operator+=(const X& o) {
    Matrix<S> t(o);
    check(t);
    for (Index i = 0; i < size(); ++i) lin(i) += t.data()[i];
    return *this;
  }
  template <class X>
  Block& operator-=(const X& o) {
    Matrix<S> t(o);
    check(t);
    for (Index i = 0; i < size(); ++i) lin(i) -= t.data()[i];
    return *this;
  }
  Block& operator*=(S s) {
    for (Index i = 0; i < size(); ++i) lin(i) *= s;
    return *this;
  }
  Block& operator/=(S s) {
    for (Index i = 0; i < size(); ++i) lin(i) /= s;
    return *this;
  }

 private:
  template <class X>
  Block& assign(const X& o) {
    Matrix<S> t(o);  // evaluate first: the source may alias this view
    check(t);
    for (Index i = 0; i < size(); ++i) lin(i) = t.data()[i];
    return *this;
  }
  void check(const Matrix<S>& t) const {
    if (t.rows() != r || t.cols() != c) throw std::invalid_argument("eigen shim: block assignment shape mismatch");
  }
};

// ---- owning column-major matrix (VectorX* = n x 1) --------------------------
template <class S>
class Matrix : public DenseOps<Matrix<S>, S> {
 public:
  using Scalar = S;

  Matrix() = default;
  explicit Matrix(Index n) : r_(n), c_(1), d_(static_cast<size_t>(n)) {}
  Matrix(Index r, Index c) : r_(r), c_(c), d_(static_cast<size_t>(r * c)) {}
  Matrix(const Matrix&) = default;
  Matrix(Matrix&&) noexcept = default;
  template <class X, class = std::enable_if_t<internal::is_dense_v<X> && !std::is_same_v<std::decay_t<X>, Matrix>>>
  Matrix(const X& x) {  // NOLINT: implicit, as Eigen's expression conversions
    auto v = x.view();
    r_ = v.r;
    c_ = v.c;
    d_.resize(static_cast<size_t>(r_ * c_));
    for (Index i = 0; i < r_ * c_; ++i) d_[static_cast<size_t>(i)] = static_cast<S>(v.lin(i));
  }
  Matrix& operator=(const Matrix&) = default;
  Matrix& operator=(Matrix&&) noexcept = default;
  template <class X, class = std::enable_if_t<internal::is_dense_v<X> && !std::is_same_v<std::decay_t<X>, Matrix>>>
  Matrix& operator=(const X& x) {
    Matrix t(x);
    *this = std::move(t);
    return *this;
  }

  static Matrix Zero(Index n) { return Constant(n, S(0)); }
  static Matrix Zero(Index r, Index c) { return Constant(r, c, S(0)); }
  static Matrix Ones(Index n) { return Constant(n, S(1)); }
  static Matrix Ones(Index r, Index c) { return Constant(r, c, S(1)); }
  static Matrix Constant(Index n, S v) { Matrix m(n); std::fill(m.d_.begin(), m.d_.end(), v); return m; }
  static Matrix Constant(Index r, Index c, S v) { Matrix m(r, c); std::fill(m.d_.begin(), m.d_.end(), v); return m; }
  static Matrix Identity(Index r, Index c) {
    Matrix m = Zero(r, c);
    for (Index i = 0; i < std::min(r, c); ++i) m(i, i) = S(1);
    return m;
  }
  static Matrix Identity(Index n) { return Identity(n, n); }

  Index rows() const { return r_; }
  Index cols() const { return c_; }
  Index size() const { return r_ * c_; }
  S* data() { return d_.data(); }
  const S* data() const { return d_.data(); }
  Block<S> view() const { return Block<S>(const_cast<S*>(d_.data()), r_, c_, 1, r_); }
  S& operator()(Index i, Index j) { return d_[static_cast<size_t>(j * r_ + i)]; }
  const S& operator()(Index i, Index j) const { return d_[static_cast<size_t>(j * r_ + i)]; }
  S& operator()(Index i) { return d_[static_cast<size_t>(i)]; }
  const S& operator()(Index i) const { return d_[static_cast<size_t>(i)]; }
  S& operator[](Index i) { return d_[static_cast<size_t>(i)]; }
  const S& operator[](Index i) const { return d_[static_cast<size_t>(i)]; }

  void resize(Index n) { resize(n, 1); }
  void resize(Index r, Index c) {
    r_ = r;
    c_ = c;
    d_.assign(static_cast<size_t>(r * c), S(0));
  }
  void conservativeResize(Index n) {  // vectors: keep the leading entries
    d_.resize(static_cast<size_t>(n), S(0));
    r_ = n;
    c_ = 1;
  }
  void conservativeResize(NoChange_t, Index c) {  // keep the leading columns
    d_.resize(static_cast<size_t>(r_ * c), S(0));
    c_ = c;
  }
  void setZero() { std::fill(d_.begin(), d_.end(), S(0)); }
  void normalize() { *this /= static_cast<S>(this->norm()); }
  Matrix& noalias() { return *this; }

  template <class X>
  Matrix& operator+=(const X& o) {
    Matrix t(o);
    check(t);
    for (size_t i = 0; i < d_.size(); ++i) d_[i] += t.d_[i];
    return *this;
  }
  template <class X>
  Matrix& operator-=(const X& o) {
    Matrix t(o);
    check(t);
    for (size_t i = 0; i < d_.size(); ++i) d_[i] -= t.d_[i];
    return *this;
  }
  Matrix& operator*=(S s) {
    for (S& v : d_) v *= s;
    return *this;
  }
  Matrix& operator/=(S s) {
    for (S& v : d_) v /= s;
    return *this;
  }

 private:
  void check(const Matrix& t) const {
    if (t.r_ != r_ || t.c_ != c_) throw std::invalid_argument("eigen shim: shape mismatch");
  }
  Index r_ = 0, c_ = 0;
  std::vector<S> d_;
};

// ---- arrays (coefficient-wise views / results) ------------------------------
template <class S>
class ArrayVal {
 public:
  Matrix<S> m;
  Block<S> view() const { return m.view(); }
  Matrix<S> matrix() const { return m; }
  ArrayVal rsqrt() const { return ArrayVal{m.map([](S x) { return internal::rsqrt(x); })}; }
  ArrayVal sqrt() const { return ArrayVal{m.map([](S x) { return std::sqrt(x); })}; }
  ArrayVal abs() const { return ArrayVal{m.map([](S x) { return std::abs(x); })}; }
  ArrayVal inverse() const { return ArrayVal{m.map([](S x) { return S(1) / x; })}; }
};

template <class S>
class ArrayRef {
 public:
  explicit ArrayRef(Block<S> v_) : v(v_) {}
  Block<S> v;
  Block<S> view() const { return v; }
  Matrix<S> matrix() const { return Matrix<S>(v); }
  ArrayVal<S> rsqrt() const { return ArrayVal<S>{Matrix<S>(v)}.rsqrt(); }
  ArrayVal<S> sqrt() const { return ArrayVal<S>{Matrix<S>(v)}.sqrt(); }
  ArrayVal<S> abs() const { return ArrayVal<S>{Matrix<S>(v)}.abs(); }
  ArrayVal<S> inverse() const { return ArrayVal<S>{Matrix<S>(v)}.inverse(); }
  template <class X>
  ArrayRef& operator*=(const X& o) {  // coefficient-wise product in place
    Matrix<S> t(o);
    for (Index i = 0; i < v.size(); ++i) v.lin(i) *= t.data()[i];
    return *this;
  }
  template <class X>
  ArrayRef& operator/=(const X& o) {
    Matrix<S> t(o);
    for (Index i = 0; i < v.size(); ++i) v.lin(i) /= t.data()[i];
    return *this;
  }
  ArrayRef& operator*=(S s) {
    v *= s;
    return *this;
  }
};

template <class S>
struct DiagonalWrapper {
  Matrix<S> diag;
};

template <class S>
struct Rowwise {
  Block<S> v;
  Matrix<typename internal::real_of<S>::type> norm() const {
    Matrix<typename internal::real_of<S>::type> out(v.r);
    for (Index i = 0; i < v.r; ++i) {
      double s = 0.0;
      for (Index j = 0; j < v.c; ++j) s += std::norm(v(i, j));
      out(i) = std::sqrt(s);
    }
    return out;
  }
  Matrix<S> sum() const {
    Matrix<S> out(v.r);
    for (Index i = 0; i < v.r; ++i) {
      S s = S(0);
      for (Index j = 0; j < v.c; ++j) s += v(i, j);
      out(i) = s;
    }
    return out;
  }
};

// ---- Map / Ref ---------------------------------------------------------------
template <class T>
class Map;
template <class S>
class Map<const Matrix<S>> : public Block<S> {
 public:
  Map(const S* p, Index n) : Block<S>(const_cast<S*>(p), n, 1, 1, n) {}
  Map(const S* p, Index r, Index c) : Block<S>(const_cast<S*>(p), r, c, 1, r) {}
};
template <class S>
class Map<Matrix<S>> : public Block<S> {
 public:
  Map(S* p, Index n) : Block<S>(p, n, 1, 1, n) {}
  Map(S* p, Index r, Index c) : Block<S>(p, r, c, 1, r) {}
  using Block<S>::operator=;
};

template <class T>
class Ref;
template <class S>
class Ref<const Matrix<S>> : public Block<S> {
 public:
  Ref(const Matrix<S>& m) : Block<S>(m.view()) {}  // NOLINT: implicit, as Eigen::Ref
  Ref(const Block<S>& b) : Block<S>(b) {}           // NOLINT
};

// ---- arithmetic --------------------------------------------------------------
template <class X, class Y, class = std::enable_if_t<internal::is_dense_v<X> && internal::is_dense_v<Y>>>
Matrix<internal::scalar_t<X>> operator+(const X& a, const Y& b) {
  using S = internal::scalar_t<X>;
  return Matrix<S>(a).zip(b, [](S x, S y) { return x + y; });
}
template <class X, class Y, class = std::enable_if_t<internal::is_dense_v<X> && internal::is_dense_v<Y>>>
Matrix<internal::scalar_t<X>> operator-(const X& a, const Y& b) {
  using S = internal::scalar_t<X>;
  return Matrix<S>(a).zip(b, [](S x, S y) { return x - y; });
}
template <class X, class = std::enable_if_t<internal::is_dense_v<X>>>
Matrix<internal::scalar_t<X>> operator-(const X& a) {
  using S = internal::scalar_t<X>;
  return Matrix<S>(a).map([](S x) { return -x; });
}
template <class X, class T, class = std::enable_if_t<internal::is_dense_v<X> && std::is_arithmetic_v<T>>>
Matrix<internal::scalar_t<X>> operator*(T s, const X& a) {
  using S = internal::scalar_t<X>;
  const S ss = static_cast<S>(s);
  return Matrix<S>(a).map([ss](S x) { return ss * x; });
}
template <class X, class T, class = std::enable_if_t<internal::is_dense_v<X> && std::is_arithmetic_v<T>>>
Matrix<internal::scalar_t<X>> operator*(const X& a, T s) {
  using S = internal::scalar_t<X>;
  const S ss = static_cast<S>(s);
  return Matrix<S>(a).map([ss](S x) { return x * ss; });
}
template <class X, class T, class = std::enable_if_t<internal::is_dense_v<X> && std::is_arithmetic_v<T>>>
Matrix<internal::scalar_t<X>> operator/(const X& a, T s) {
  using S = internal::scalar_t<X>;
  const S ss = static_cast<S>(s);
  return Matrix<S>(a).map([ss](S x) { return x / ss; });
}

// matrix product C = A B: C(:, j) += A(:, k) B(k, j), k ascending
template <class X, class Y, class = std::enable_if_t<internal::is_dense_v<X> && internal::is_dense_v<Y>>>
Matrix<internal::scalar_t<X>> operator*(const X& a_, const Y& b_) {
  using S = internal::scalar_t<X>;
  const Block<S> a = a_.view();
  const auto b = b_.view();
  if (a.c != b.r) throw std::invalid_argument("eigen shim: product shape mismatch");
  Matrix<S> out = Matrix<S>::Zero(a.r, b.c);
  for (Index j = 0; j < b.c; ++j)
    for (Index k = 0; k < a.c; ++k) {
      const S bkj = b(k, j);
      for (Index i = 0; i < a.r; ++i) out(i, j) += a(i, k) * bkj;
    }
  return out;
}

// diagonal products: diag(d) A scales rows, A diag(d) scales columns
template <class S, class X, class = std::enable_if_t<internal::is_dense_v<X>>>
Matrix<S> operator*(const DiagonalWrapper<S>& dw, const X& a_) {
  Matrix<S> out(a_);
  for (Index j = 0; j < out.cols(); ++j)
    for (Index i = 0; i < out.rows(); ++i) out(i, j) = dw.diag(i) * out(i, j);
  return out;
}
template <class S, class X, class = std::enable_if_t<internal::is_dense_v<X>>>
Matrix<S> operator*(const X& a_, const DiagonalWrapper<S>& dw) {
  Matrix<S> out(a_);
  for (Index j = 0; j < out.cols(); ++j)
    for (Index i = 0; i < out.rows(); ++i) out(i, j) = out(i, j) * dw.diag(j);
  return out;
}

using MatrixXd = Matrix<double>;
using VectorXd = Matrix<double>;
using VectorXcd = Matrix<std::complex<double>>;
using MatrixXcd = Matrix<std::complex<double>>;

// ---- decompositions (oracle/linalg.hpp) --------------------------------------
namespace internal {
inline orc_linalg::Mat to_mat(const MatrixXd& a) {
  orc_linalg::Mat m(a.rows(), a.cols());
  std::copy(a.data(), a.data() + a.size(), m.a.begin());
  return m;
}
inline MatrixXd from_mat(const orc_linalg::Mat& m) {
  MatrixXd a(m.rows, m.cols);
  std::copy(m.a.begin(), m.a.end(), a.data());
  return a;
}
}  // namespace internal

template <class MatrixType>
class SelfAdjointEigenSolver {
 public:
  SelfAdjointEigenSolver() = default;
  explicit SelfAdjointEigenSolver(const MatrixXd& a, int = ComputeEigenvectors) { compute(a); }
  SelfAdjointEigenSolver& compute(const MatrixXd& a, int = ComputeEigenvectors) {
    std::vector<double> vals;
    orc_linalg::Mat vecs;
    orc_linalg::dense_sym_eig(internal::to_mat(a), vals, vecs);
    values_ = MatrixXd(static_cast<Index>(vals.size()));
    std::copy(vals.begin(), vals.end(), values_.data());
    vectors_ = internal::from_mat(vecs);
    return *this;
  }
  template <class D, class E>
  SelfAdjointEigenSolver& computeFromTridiagonal(const D& diag, const E& sub, int = ComputeEigenvectors) {
    const Index m = diag.size();
    std::vector<double> dv(static_cast<size_t>(m)), sv(static_cast<size_t>(std::max<Index>(m - 1, 0)));
    for (Index i = 0; i < m; ++i) dv[static_cast<size_t>(i)] = diag(i);
    for (Index i = 0; i + 1 < m; ++i) sv[static_cast<size_t>(i)] = sub(i);
    std::vector<double> z;
    orc_linalg::tridiag_eig(static_cast<int>(m), dv, sv, z);
    values_ = MatrixXd(m);
    std::copy(dv.begin(), dv.end(), values_.data());
    vectors_ = MatrixXd(m, m);
    std::copy(z.begin(), z.end(), vectors_.data());
    return *this;
  }
  const MatrixXd& eigenvalues() const { return values_; }
  const MatrixXd& eigenvectors() const { return vectors_; }

 private:
  MatrixXd values_, vectors_;
};

// Q of a HouseholderQR; only Q * Identity(rows, k <= cols) (the thin factor)
// is used by the reference (spectral.cpp:316,404,429)
struct HouseholderThinQ {
  MatrixXd q;  // rows x min(rows, cols)
};
template <class X, class = std::enable_if_t<internal::is_dense_v<X>>>
MatrixXd operator*(const HouseholderThinQ& h, const X& b_) {
  const MatrixXd b(b_);
  if (b.rows() != h.q.rows() || b.cols() > h.q.cols())
    throw std::invalid_argument("eigen shim: householderQ() supports Q * Identity(rows, k) only");
  for (Index j = 0; j < b.cols(); ++j)
    for (Index i = 0; i < b.rows(); ++i)
      if (b(i, j) != (i == j ? 1.0 : 0.0))
        throw std::invalid_argument("eigen shim: householderQ() supports Q * Identity(rows, k) only");
  return MatrixXd(h.q.leftCols(b.cols()));
}

template <class MatrixType>
class HouseholderQR {
 public:
  explicit HouseholderQR(const MatrixXd& a) {
    orc_linalg::Mat Q, R;
    orc_linalg::householder_qr(internal::to_mat(a), Q, R);
    q_.q = internal::from_mat(Q);
    // matrixQR(): R in the upper triangle of the leading rows (the
    // Householder vectors Eigen keeps below the diagonal are not used)
    qr_ = MatrixXd::Zero(a.rows(), a.cols());
    for (Index j = 0; j < a.cols(); ++j)
      for (Index i = 0; i <= std::min<Index>(j, a.rows() - 1); ++i) qr_(i, j) = R(i, j);
  }
  const HouseholderThinQ& householderQ() const { return q_; }
  const MatrixXd& matrixQR() const { return qr_; }

 private:
  HouseholderThinQ q_;
  MatrixXd qr_;
};

}  // namespace Eigen
