// hostmath.hpp -- plan-time host math of the product (kernel catalog, the
// regularised kernel K_R, the Kaiser-Bessel deconvolution).  These run once
// per plan; the per-apply work is all on the device (kernels.cuh).
#pragma once

#include <cmath>
#include <complex>
#include <cstdint>
#include <numbers>
#include <random>
#include <string>
#include <vector>

#include "common.cuh"

namespace fgsb {

constexpr double kPi = std::numbers::pi;

struct KernelSpec {
  int family = FGS_GAUSSIAN;
  double shape = 1.0;
};

inline void check_spec(const KernelSpec& s) {  // kernels.cpp:24-27
  if (!(s.shape > 0.0) || !std::isfinite(s.shape))
    fail(FGS_EPARAM, "kernel shape parameter must be positive and finite");
  if (s.family < FGS_GAUSSIAN || s.family > FGS_INV_MULTIQUADRIC) fail(FGS_EPARAM, "unknown kernel family");
}

// Modified Bessel I0 by its positive power series (nfft.cpp:60-69).
inline double i0_series(double x) {
  const double q = 0.25 * x * x;
  double term = 1.0, sum = 1.0;
  for (int k = 1; k < 1000; ++k) {
    term *= q / (static_cast<double>(k) * k);
    sum += term;
    if (term < sum * 1e-17) break;
  }
  return sum;
}

// Radial kernel value (kernels.cpp:79-93).
inline double kernel_value(const KernelSpec& s, double r) {
  check_spec(s);
  if (!(r >= 0.0)) fail(FGS_ERANGE, "kernel radius must be nonnegative");
  switch (s.family) {
    case FGS_GAUSSIAN: return std::exp(-(r * r) / (s.shape * s.shape));
    case FGS_LAPLACIAN_RBF: return std::exp(-r / s.shape);
    case FGS_MULTIQUADRIC: return std::sqrt(r * r + s.shape * s.shape);
    default: return 1.0 / std::sqrt(r * r + s.shape * s.shape);
  }
}

// K^(j)(r0), j < count, through exact Taylor recurrences (kernels.cpp:29-52,
// 95-128).
inline std::vector<double> kernel_derivatives(const KernelSpec& s, double r0, int count) {
  check_spec(s);
  if (!(r0 >= 0.0)) fail(FGS_ERANGE, "kernel radius must be nonnegative");
  if (count < 1 || count > 16) fail(FGS_EPARAM, "derivative count must lie in [1, 16]");
  std::vector<double> w(static_cast<size_t>(count));
  auto exp_rec = [&](double g0, double g1, double g2) {
    w[0] = std::exp(g0);
    for (int k = 1; k < count; ++k) {
      double acc = g1 * w[k - 1];
      if (k >= 2) acc += 2.0 * g2 * w[k - 2];
      w[k] = acc / k;
    }
  };
  auto pow_rec = [&](double u0, double u1, double u2, double alpha) {
    w[0] = std::pow(u0, alpha);
    for (int k = 1; k < count; ++k) {
      double acc = ((alpha + 1.0) * 1.0 - k) * u1 * w[k - 1];
      if (k >= 2) acc += ((alpha + 1.0) * 2.0 - k) * u2 * w[k - 2];
      w[k] = acc / (k * u0);
    }
  };
  const double c2 = s.shape * s.shape;
  switch (s.family) {
    case FGS_GAUSSIAN: exp_rec(-r0 * r0 / c2, -2.0 * r0 / c2, -1.0 / c2); break;
    case FGS_LAPLACIAN_RBF: exp_rec(-r0 / s.shape, -1.0 / s.shape, 0.0); break;
    case FGS_MULTIQUADRIC: pow_rec(r0 * r0 + c2, 2.0 * r0, 1.0, 0.5); break;
    default: pow_rec(r0 * r0 + c2, 2.0 * r0, 1.0, -0.5); break;
  }
  double fact = 1.0;
  for (int j = 0; j < count; ++j) {
    if (j > 0) fact *= j;
    w[j] *= fact;
  }
  return w;
}

// Hermite blend of K across [1/2 - eps_b, 1/2] (kernels.cpp:163-238): value
// and first p-1 derivatives match at the inner radius, derivatives 1..p
// vanish at 1/2; solved in s = (r - mid)/h by forward substitution.
struct Blend {
  double mid = 0.0, h = 1.0;
  std::vector<double> c{0.0};
  double operator()(double r) const {
    const double s = (r - mid) / h;
    double acc = 0.0;
    for (int k = static_cast<int>(c.size()) - 1; k >= 0; --k) acc = acc * s + c[static_cast<size_t>(k)];
    return acc;
  }
};

inline Blend make_blend(const KernelSpec& spec, double eps_b, int p) {
  check_spec(spec);
  if (!(eps_b > 0.0) || !(eps_b < 0.5)) fail(FGS_EPARAM, "blend width must lie in (0, 1/2)");
  if (p < 1 || p > 8) fail(FGS_EPARAM, "smoothness order must lie in [1, 8]");
  const double a = 0.5 - eps_b;
  Blend out;
  out.mid = 0.5 * (a + 0.5);
  out.h = 0.5 * eps_b;
  const double h = out.h;
  const std::vector<double> der = kernel_derivatives(spec, a, p);
  std::vector<double> q(static_cast<size_t>(std::max(p - 1, 1)), 0.0);
  double hp = h;
  for (int i = 0; i + 1 < p; ++i) {
    double rhs = hp * der[static_cast<size_t>(i + 1)];
    hp *= h;
    for (int j = 0; j < i; ++j) {
      double binom = 1.0, fall = 1.0, fact = 1.0;
      for (int t = 0; t < i - j; ++t) binom = binom * (i - t) / (t + 1.0);
      for (int t = 0; t < i - j; ++t) fall *= p - t;
      for (int t = 2; t <= j; ++t) fact *= t;
      rhs -= q[static_cast<size_t>(j)] * binom * fall * std::pow(-2.0, p - i + j) * fact;
    }
    double fi = 1.0;
    for (int t = 2; t <= i; ++t) fi *= t;
    q[static_cast<size_t>(i)] = rhs / (std::pow(-2.0, p) * fi);
  }
  // (s - 1)^p in monomials
  std::vector<double> left(static_cast<size_t>(p + 1), 0.0);
  left[0] = 1.0;
  for (int t = 0; t < p; ++t) {
    std::vector<double> nx(static_cast<size_t>(p + 1), 0.0);
    for (int k = 0; k <= t; ++k) {
      nx[static_cast<size_t>(k + 1)] += left[static_cast<size_t>(k)];
      nx[static_cast<size_t>(k)] -= left[static_cast<size_t>(k)];
    }
    left.swap(nx);
  }
  // sum_j q_j (s + 1)^j
  std::vector<double> right(static_cast<size_t>(p > 1 ? p - 1 : 1), 0.0);
  right[0] = p > 1 ? q[0] : 0.0;
  for (int j = 1; j + 1 < p; ++j) {
    double binom = 1.0;
    for (int k = 0; k <= j; ++k) {
      right[static_cast<size_t>(k)] += q[static_cast<size_t>(j)] * binom;
      binom = binom * (j - k) / (k + 1.0);
    }
  }
  std::vector<double> u(static_cast<size_t>(2 * p - 1), 0.0);
  for (size_t ka = 0; ka <= static_cast<size_t>(p); ++ka)
    for (size_t kb = 0; kb < right.size(); ++kb)
      if (ka + kb < u.size()) u[ka + kb] += left[ka] * right[kb];
  // integrate from s = -1 with P(-1) = K(a)
  std::vector<double> c(static_cast<size_t>(2 * p), 0.0);
  for (size_t k = 0; k < u.size(); ++k) c[k + 1] = u[k] / static_cast<double>(k + 1);
  double at_m1 = 0.0, sp = -1.0;
  for (size_t k = 1; k < c.size(); ++k) {
    at_m1 += c[k] * sp;
    sp = -sp;
  }
  c[0] = der[0] - at_m1;
  size_t last = c.size() - 1;
  while (last > 0 && c[last] == 0.0) --last;
  c.resize(last + 1);
  out.c = std::move(c);
  return out;
}

// Regularised kernel K_R (kernels.cpp:240-260).
struct RegKernel {
  KernelSpec spec;
  double eps_b = 0.0;
  int p = 1;
  Blend blend;
  double tail = 0.0;
  RegKernel() = default;
  RegKernel(const KernelSpec& s, double e, int pp) : spec(s), eps_b(e), p(pp) {
    check_spec(s);
    if (!(e >= 0.0) || !(e < 0.5)) fail(FGS_EPARAM, "blend width must lie in [0, 1/2)");
    if (pp < 1 || pp > 8) fail(FGS_EPARAM, "smoothness order must lie in [1, 8]");
    if (eps_b > 0.0) {
      blend = make_blend(s, e, pp);
      tail = blend(0.5);
    } else {
      tail = kernel_value(s, 0.5);
    }
  }
  double operator()(double r) const {
    if (eps_b == 0.0) return kernel_value(spec, std::min(r, 0.5));
    if (r <= 0.5 - eps_b) return kernel_value(spec, r);
    if (r <= 0.5) return blend(r);
    return tail;
  }
};

}  // namespace fgsb
