// ============================================================================
// fgs_oracle.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A serial CPU restatement of the reference's NFFT fast-summation hot path
// (reference: /root/reference/proj, the `fgs` C++20 library).  It exists so
// that tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
// arm can CHECK the B200 product against the reference algorithm.  Nothing in
// the product (paper_1808_04580_b200/) links, loads or calls this file.
//
// Why a restatement: the reference's own build needs Eigen3, FFTW3, libpng
// and vendored doctest/CLI11/json, none of which is in this image (SURVEY.md
// §8c).  Every function below cites the reference file:line it follows.  The
// two third-party arithmetic pieces live in oracle/linalg.hpp (self-written
// FFT for FFTW3; implicit-QL / Householder eigen and QR solvers for Eigen3).
// Parity pin: the reference's OWN hot-path sources (nfft.cpp, kernels.cpp,
// fastsum.cpp, graphop.cpp, spectral.cpp) ARE compiled here, unchanged,
// against shim Eigen/FFTW headers built on the same linalg.hpp
// (oracle/build_ref.sh -> oracle/_ref/libfgsref.so), and
// tests/test_ref_pin.py requires this restatement to reproduce that binary
// BIT FOR BIT on every hot-path entry (NFFT forward/adjoint, b-hat for all
// kernel families, fastsum, degrees, the four graph operators on all five
// BASELINE configurations, Lanczos incl. Ritz vectors, dense Lanczos, error
// classes and the failing node).  tests/test_oracle_*.py additionally run the
// reference's known-answer tests (test_nfft.cpp, test_kernels.cpp,
// test_fastsum.cpp, test_graphop.cpp, test_spectral.cpp, acceptance.cpp) and
// check the FFT against numpy.fft.
//
// Build: oracle/build_oracle.sh -> oracle/liboracle.so (g++ -O3
// -ffp-contract=off, matching the reference's default x86-64 Release flags,
// which emit no FMA).
// ============================================================================
#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdint>
#include <cstring>
#include <functional>
#include <limits>
#include <memory>
#include <numbers>
#include <numeric>
#include <random>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "linalg.hpp"

namespace orc {

using orc_linalg::Mat;
using orc_linalg::dense_sym_eig;
using orc_linalg::fft_line;
using orc_linalg::fft_nd;
using orc_linalg::householder_qr;
using orc_linalg::tridiag_eig;
using cd = std::complex<double>;
constexpr double kPi = std::numbers::pi;
constexpr double kEps = std::numeric_limits<double>::epsilon();

// Status codes, 1:1 with the reference exception classes (errors.hpp:8-49).
enum Status { S_OK = 0, S_PARAM = 1, S_RANGE = 2, S_SHAPE = 3, S_NUMERIC = 4, S_RESOURCE = 5 };

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] void fail(int code, const std::string& msg) { throw Error(code, msg); }

// Host threads of the NFFT loops (orc_set_threads; default 1 = the serial
// reference order, which tests/test_ref_pin.py pins bit for bit).  With more
// threads the taps and the gather are split over points (results unchanged)
// and the spread goes into per-thread grids summed in thread order (a fixed
// order, but a different rounding of the grid sums than the serial loop):
// used only to make full-size GPU parity checks (C4/C5) affordable.
int g_threads = 1;

template <class F>
void parallel_ranges(int64_t n, F&& fn) {  // fn(thread, lo, hi)
  const int T = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(g_threads, n / 1024)));
  if (T <= 1) {
    fn(0, int64_t{0}, n);
    return;
  }
  std::vector<std::thread> pool;
  std::vector<std::exception_ptr> errs(static_cast<size_t>(T));
  for (int t = 0; t < T; ++t)
    pool.emplace_back([&, t] {
      try {
        fn(t, n * t / T, n * (t + 1) / T);
      } catch (...) {
        errs[static_cast<size_t>(t)] = std::current_exception();
      }
    });
  for (auto& th : pool) th.join();
  for (auto& e : errs)
    if (e) std::rethrow_exception(e);
}

size_t ipow(size_t base, int e) {  // nfft.cpp:53-57
  size_t r = 1;
  while (e-- > 0) r *= base;
  return r;
}

// ---------------------------------------------------------------------------
// NFFT  (nfft.hpp:19-94, nfft.cpp)
// ---------------------------------------------------------------------------
double bessel_i0(double x) {  // nfft.cpp:60-69
  double q = 0.25 * x * x;
  double term = 1.0, sum = 1.0;
  for (int k = 1; k < 1000; ++k) {
    term *= q / (static_cast<double>(k) * k);
    sum += term;
    if (term < sum * 1e-17) break;
  }
  return sum;
}

void validate_common(int d, int N, const Mat& nodes) {  // nfft.cpp:33-50
  if (d < 1 || d > 3) fail(S_PARAM, "dims must be 1, 2, or 3, got " + std::to_string(d));
  if (N < 2 || N % 2 != 0) fail(S_PARAM, "bandwidth must be even and >= 2, got " + std::to_string(N));
  if (nodes.cols != d)
    fail(S_SHAPE, "nodes have " + std::to_string(nodes.cols) + " columns, expected " + std::to_string(d));
  if (nodes.rows == 0) fail(S_SHAPE, "node set is empty");
  for (int64_t j = 0; j < nodes.rows; ++j)
    for (int t = 0; t < d; ++t) {
      double v = nodes(j, t);
      if (!(v >= -0.5 && v < 0.5))
        fail(S_RANGE, "node " + std::to_string(j) + " component " + std::to_string(t) + " = " +
                         std::to_string(v) + " outside [-1/2, 1/2)");
    }
}

// FrequencyIndexSet::component (nfft.cpp:78-83)
int freq_component(int d, int N, size_t flat, int dim) {
  size_t stride = ipow(static_cast<size_t>(N), d - 1 - dim);
  return static_cast<int>((flat / stride) % static_cast<size_t>(N)) - N / 2;
}

// direct_ndft / direct_adjoint_ndft (nfft.cpp:85-125)
std::vector<cd> direct_ndft(int d, int N, const Mat& nodes, const std::vector<cd>& fhat) {
  validate_common(d, N, nodes);
  size_t F = ipow(static_cast<size_t>(N), d);
  if (fhat.size() != F) fail(S_SHAPE, "coefficient vector has wrong length");
  std::vector<cd> out(static_cast<size_t>(nodes.rows), 0.0);
  for (int64_t j = 0; j < nodes.rows; ++j) {
    cd acc = 0.0;
    for (size_t f = 0; f < F; ++f) {
      double phase = 0.0;
      for (int t = 0; t < d; ++t) phase += freq_component(d, N, f, t) * nodes(j, t);
      acc += fhat[f] * std::polar(1.0, 2.0 * kPi * phase);
    }
    out[static_cast<size_t>(j)] = acc;
  }
  return out;
}

std::vector<cd> direct_adjoint_ndft(int d, int N, const Mat& nodes, const std::vector<cd>& x) {
  validate_common(d, N, nodes);
  size_t F = ipow(static_cast<size_t>(N), d);
  if (static_cast<int64_t>(x.size()) != nodes.rows) fail(S_SHAPE, "input vector length does not match node count");
  std::vector<cd> out(F, 0.0);
  for (size_t f = 0; f < F; ++f) {
    cd acc = 0.0;
    for (int64_t j = 0; j < nodes.rows; ++j) {
      double phase = 0.0;
      for (int t = 0; t < d; ++t) phase += freq_component(d, N, f, t) * nodes(j, t);
      acc += x[static_cast<size_t>(j)] * std::polar(1.0, -2.0 * kPi * phase);
    }
    out[f] = acc;
  }
  return out;
}

// NfftPlan::Impl (nfft.cpp:127-388, 402-438)
struct Nfft {
  int d = 0, N = 0, m = 0, M = 0;
  double b = 0.0;
  int64_t n = 0;
  size_t grid_total = 0, coeff_total = 0;
  std::vector<double> deconv;  // indexed by l + N/2
  int taps = 0;
  std::vector<double> w;  // [n][d][taps]
  std::vector<int> idx;   // [n][d][taps]
  mutable std::vector<cd> grid_in, grid_out;

  double window(double diff) const {  // nfft.cpp:161-169
    double arg = static_cast<double>(m) * m - (M * diff) * (M * diff);
    if (arg <= 0.0) return b / kPi;
    double t = std::sqrt(arg);
    if (t < 1e-8) return (b + b * b * b * t * t / 6.0) / kPi;
    return std::sinh(b * t) / (kPi * t);
  }
  int wrap_freq(int l) const { return (l + M) % M; }  // nfft.cpp:171

  Nfft(int dims, int bandwidth, int cutoff, const Mat& nodes, double oversampling) {
    validate_common(dims, bandwidth, nodes);  // nfft.cpp:328-335
    if (cutoff < 1 || cutoff > 32) fail(S_PARAM, "cutoff must lie in [1, 32], got " + std::to_string(cutoff));
    if (!(oversampling >= 1.0)) fail(S_PARAM, "oversampling factor must be >= 1");
    d = dims;
    N = bandwidth;
    m = cutoff;
    n = nodes.rows;
    coeff_total = ipow(static_cast<size_t>(N), d);
    M = 2 * static_cast<int>(std::ceil(oversampling * bandwidth / 2.0));  // nfft.cpp:343
    grid_total = ipow(static_cast<size_t>(M), d);
    b = kPi * (2.0 - static_cast<double>(N) / M);  // nfft.cpp:347
    deconv.resize(static_cast<size_t>(N));         // nfft.cpp:349-354
    for (int a = 0; a < N; ++a) {
      double l = a - N / 2;
      double arg = b * b - std::pow(2.0 * kPi * l / M, 2);
      deconv[static_cast<size_t>(a)] = 1.0 / bessel_i0(m * std::sqrt(std::max(arg, 0.0)));
    }
    taps = 2 * m;  // nfft.cpp:356-369
    w.resize(static_cast<size_t>(n) * d * taps);
    idx.resize(static_cast<size_t>(n) * d * taps);
    parallel_ranges(n, [&](int, int64_t lo, int64_t hi) {
      for (int64_t j = lo; j < hi; ++j)
        for (int t = 0; t < d; ++t) {
          double v = nodes(j, t);
          int u0 = static_cast<int>(std::ceil(v * M - m));
          size_t base = (static_cast<size_t>(j) * d + t) * taps;
          for (int a = 0; a < taps; ++a) {
            int u = u0 + a;
            w[base + a] = window(v - static_cast<double>(u) / M);
            idx[base + a] = ((u % M) + M) % M;
          }
        }
    });
    grid_in.assign(grid_total, 0.0);
    grid_out.assign(grid_total, 0.0);
  }

  void place_coefficients(const std::vector<cd>& fhat, cd* grid) const {  // nfft.cpp:174-213
    std::fill(grid, grid + grid_total, cd(0.0));
    const int half = N / 2;
    if (d == 1) {
      for (int a = 0; a < N; ++a) grid[wrap_freq(a - half)] = fhat[a] * deconv[a];
    } else if (d == 2) {
      size_t f = 0;
      for (int a = 0; a < N; ++a) {
        size_t ga = static_cast<size_t>(wrap_freq(a - half)) * M;
        for (int c = 0; c < N; ++c, ++f)
          grid[ga + wrap_freq(c - half)] = fhat[f] * (deconv[a] * deconv[c]);
      }
    } else {
      size_t f = 0;
      for (int a = 0; a < N; ++a) {
        size_t ga = static_cast<size_t>(wrap_freq(a - half)) * M * M;
        for (int c = 0; c < N; ++c) {
          size_t gc = ga + static_cast<size_t>(wrap_freq(c - half)) * M;
          double dac = deconv[a] * deconv[c];
          for (int e = 0; e < N; ++e, ++f) grid[gc + wrap_freq(e - half)] = fhat[f] * (dac * deconv[e]);
        }
      }
    }
  }

  void extract_coefficients(const cd* grid, std::vector<cd>& out) const {  // nfft.cpp:216-250
    const int half = N / 2;
    out.resize(coeff_total);
    if (d == 1) {
      for (int a = 0; a < N; ++a) out[a] = grid[wrap_freq(a - half)] * deconv[a];
    } else if (d == 2) {
      size_t f = 0;
      for (int a = 0; a < N; ++a) {
        size_t ga = static_cast<size_t>(wrap_freq(a - half)) * M;
        for (int c = 0; c < N; ++c, ++f) out[f] = grid[ga + wrap_freq(c - half)] * (deconv[a] * deconv[c]);
      }
    } else {
      size_t f = 0;
      for (int a = 0; a < N; ++a) {
        size_t ga = static_cast<size_t>(wrap_freq(a - half)) * M * M;
        for (int c = 0; c < N; ++c) {
          size_t gc = ga + static_cast<size_t>(wrap_freq(c - half)) * M;
          double dac = deconv[a] * deconv[c];
          for (int e = 0; e < N; ++e, ++f) out[f] = grid[gc + wrap_freq(e - half)] * (dac * deconv[e]);
        }
      }
    }
  }

  cd gather(const cd* grid, int64_t j) const {  // nfft.cpp:252-287
    const double* wj = &w[static_cast<size_t>(j) * d * taps];
    const int* ij = &idx[static_cast<size_t>(j) * d * taps];
    cd acc = 0.0;
    if (d == 1) {
      for (int a = 0; a < taps; ++a) acc += wj[a] * grid[ij[a]];
    } else if (d == 2) {
      for (int a = 0; a < taps; ++a) {
        size_t ra = static_cast<size_t>(ij[a]) * M;
        cd row = 0.0;
        for (int c = 0; c < taps; ++c) row += wj[taps + c] * grid[ra + ij[taps + c]];
        acc += wj[a] * row;
      }
    } else {
      for (int a = 0; a < taps; ++a) {
        size_t ra = static_cast<size_t>(ij[a]) * M * M;
        cd plane = 0.0;
        for (int c = 0; c < taps; ++c) {
          size_t rc = ra + static_cast<size_t>(ij[taps + c]) * M;
          cd row = 0.0;
          for (int e = 0; e < taps; ++e) row += wj[2 * taps + e] * grid[rc + ij[2 * taps + e]];
          plane += wj[taps + c] * row;
        }
        acc += wj[a] * plane;
      }
    }
    return acc;
  }

  void spread(cd xj, int64_t j, cd* grid) const {  // nfft.cpp:289-325
    const double* wj = &w[static_cast<size_t>(j) * d * taps];
    const int* ij = &idx[static_cast<size_t>(j) * d * taps];
    if (d == 1) {
      for (int a = 0; a < taps; ++a) grid[ij[a]] += xj * wj[a];
    } else if (d == 2) {
      for (int a = 0; a < taps; ++a) {
        size_t ra = static_cast<size_t>(ij[a]) * M;
        cd va = xj * wj[a];
        for (int c = 0; c < taps; ++c) grid[ra + ij[taps + c]] += va * wj[taps + c];
      }
    } else {
      for (int a = 0; a < taps; ++a) {
        size_t ra = static_cast<size_t>(ij[a]) * M * M;
        cd va = xj * wj[a];
        for (int c = 0; c < taps; ++c) {
          size_t rc = ra + static_cast<size_t>(ij[taps + c]) * M;
          cd vc = va * wj[taps + c];
          for (int e = 0; e < taps; ++e) grid[rc + ij[2 * taps + e]] += vc * wj[2 * taps + e];
        }
      }
    }
  }

  std::vector<cd> forward(const std::vector<cd>& fhat) const {  // nfft.cpp:402-413
    if (fhat.size() != coeff_total) fail(S_SHAPE, "coefficient vector has wrong length");
    place_coefficients(fhat, grid_in.data());
    grid_out = grid_in;
    fft_nd(grid_out.data(), d, M, +1, g_threads);  // FFTW_BACKWARD
    std::vector<cd> result(static_cast<size_t>(n));
    parallel_ranges(n, [&](int, int64_t lo, int64_t hi) {
      for (int64_t j = lo; j < hi; ++j) result[static_cast<size_t>(j)] = gather(grid_out.data(), j);
    });
    return result;
  }

  std::vector<cd> adjoint(const std::vector<cd>& x) const {  // nfft.cpp:415-427
    if (static_cast<int64_t>(x.size()) != n) fail(S_SHAPE, "input vector length does not match node count");
    std::fill(grid_in.begin(), grid_in.end(), cd(0.0));
    if (g_threads <= 1 || n < 2048) {
      for (int64_t j = 0; j < n; ++j) spread(x[static_cast<size_t>(j)], j, grid_in.data());
    } else {
      std::vector<std::vector<cd>> part(static_cast<size_t>(g_threads));
      parallel_ranges(n, [&](int t, int64_t lo, int64_t hi) {
        part[static_cast<size_t>(t)].assign(grid_total, cd(0.0));
        for (int64_t j = lo; j < hi; ++j) spread(x[static_cast<size_t>(j)], j, part[static_cast<size_t>(t)].data());
      });
      for (auto& g : part)
        if (!g.empty())
          for (size_t i = 0; i < grid_total; ++i) grid_in[i] += g[i];
    }
    grid_out = grid_in;
    fft_nd(grid_out.data(), d, M, -1, g_threads);  // FFTW_FORWARD
    std::vector<cd> result;
    extract_coefficients(grid_out.data(), result);
    return result;
  }

  std::vector<double> forward_real(const std::vector<cd>& fhat) const {  // nfft.cpp:429-438
    std::vector<cd> z = forward(fhat);
    std::vector<double> re(z.size());
    for (size_t i = 0; i < z.size(); ++i) re[i] = z[i].real();
    return re;
  }
};

// ---------------------------------------------------------------------------
// Kernels  (kernels.hpp:15-123, kernels.cpp)
// ---------------------------------------------------------------------------
enum Family { GAUSSIAN = 0, LAPLACIAN_RBF = 1, MULTIQUADRIC = 2, INV_MULTIQUADRIC = 3 };
struct KernelSpec {
  int family = GAUSSIAN;
  double shape = 1.0;
};

void validate_spec(const KernelSpec& s) {  // kernels.cpp:24-27
  if (!(s.shape > 0.0) || !std::isfinite(s.shape)) fail(S_PARAM, "kernel shape parameter must be positive and finite");
  if (s.family < 0 || s.family > 3) fail(S_PARAM, "unknown kernel family");
}

double eval_kernel(const KernelSpec& spec, double r) {  // kernels.cpp:79-93
  validate_spec(spec);
  if (!(r >= 0.0)) fail(S_RANGE, "kernel radius must be nonnegative");
  switch (spec.family) {
    case GAUSSIAN: return std::exp(-(r * r) / (spec.shape * spec.shape));
    case LAPLACIAN_RBF: return std::exp(-r / spec.shape);
    case MULTIQUADRIC: return std::sqrt(r * r + spec.shape * spec.shape);
    default: return 1.0 / std::sqrt(r * r + spec.shape * spec.shape);
  }
}

std::vector<double> exp_series(double g0, double g1, double g2, int count) {  // kernels.cpp:29-39
  std::vector<double> w(static_cast<size_t>(count));
  w[0] = std::exp(g0);
  for (int k = 1; k < count; ++k) {
    double acc = g1 * w[k - 1];
    if (k >= 2) acc += 2.0 * g2 * w[k - 2];
    w[k] = acc / k;
  }
  return w;
}

std::vector<double> pow_series(double u0, double u1, double u2, double alpha, int count) {  // kernels.cpp:41-52
  std::vector<double> w(static_cast<size_t>(count));
  w[0] = std::pow(u0, alpha);
  for (int k = 1; k < count; ++k) {
    double acc = ((alpha + 1.0) * 1.0 - k) * u1 * w[k - 1];
    if (k >= 2) acc += ((alpha + 1.0) * 2.0 - k) * u2 * w[k - 2];
    w[k] = acc / (k * u0);
  }
  return w;
}

std::vector<double> kernel_radial_derivatives(const KernelSpec& spec, double r0, int count) {  // kernels.cpp:95-128
  validate_spec(spec);
  if (!(r0 >= 0.0)) fail(S_RANGE, "kernel radius must be nonnegative");
  if (count < 1 || count > 16) fail(S_PARAM, "derivative count must lie in [1, 16]");
  std::vector<double> series;
  switch (spec.family) {
    case GAUSSIAN: {
      double s2 = spec.shape * spec.shape;
      series = exp_series(-r0 * r0 / s2, -2.0 * r0 / s2, -1.0 / s2, count);
      break;
    }
    case LAPLACIAN_RBF: series = exp_series(-r0 / spec.shape, -1.0 / spec.shape, 0.0, count); break;
    case MULTIQUADRIC: series = pow_series(r0 * r0 + spec.shape * spec.shape, 2.0 * r0, 1.0, 0.5, count); break;
    default: series = pow_series(r0 * r0 + spec.shape * spec.shape, 2.0 * r0, 1.0, -0.5, count); break;
  }
  double factorial = 1.0;
  for (int j = 0; j < count; ++j) {
    if (j > 0) factorial *= j;
    series[j] *= factorial;
  }
  return series;
}

struct Polynomial {  // kernels.cpp:130-161
  double center = 0.0, scale = 1.0;
  std::vector<double> coeffs{0.0};
  Polynomial() = default;
  Polynomial(double c, double s, std::vector<double> k) : center(c), scale(s), coeffs(std::move(k)) {
    if (!(scale > 0.0)) fail(S_PARAM, "polynomial scale must be positive");
    if (coeffs.empty()) fail(S_PARAM, "polynomial needs coefficients");
    size_t last = coeffs.size() - 1;
    while (last > 0 && coeffs[last] == 0.0) --last;
    coeffs.resize(last + 1);
  }
  double value(double r) const {
    double s = (r - center) / scale;
    double acc = 0.0;
    for (int64_t k = static_cast<int64_t>(coeffs.size()) - 1; k >= 0; --k) acc = acc * s + coeffs[k];
    return acc;
  }
  double derivative(double r, int order) const {
    if (order < 0) fail(S_PARAM, "derivative order must be nonnegative");
    std::vector<double> c = coeffs;
    for (int o = 0; o < order; ++o) {
      if (c.size() == 1) return 0.0;
      std::vector<double> next(c.size() - 1);
      for (size_t k = 1; k < c.size(); ++k) next[k - 1] = static_cast<double>(k) * c[k];
      c = std::move(next);
    }
    double s = (r - center) / scale;
    double acc = 0.0;
    for (int64_t k = static_cast<int64_t>(c.size()) - 1; k >= 0; --k) acc = acc * s + c[k];
    return acc / std::pow(scale, order);
  }
};

Polynomial two_point_taylor(const KernelSpec& spec, double eps_b, int p) {  // kernels.cpp:163-238
  validate_spec(spec);
  if (!(eps_b > 0.0) || !(eps_b < 0.5)) fail(S_PARAM, "blend width must lie in (0, 1/2)");
  if (p < 1 || p > 8) fail(S_PARAM, "smoothness order must lie in [1, 8]");
  const double a = 0.5 - eps_b;
  const double mid = 0.5 * (a + 0.5);
  const double h = 0.5 * eps_b;
  std::vector<double> derivs = kernel_radial_derivatives(spec, a, p);
  std::vector<double> q(static_cast<size_t>(std::max(p - 1, 1)), 0.0);
  double hpow = h;
  for (int i = 0; i + 1 < p; ++i) {
    double rhs = hpow * derivs[i + 1];
    hpow *= h;
    for (int j = 0; j < i; ++j) {
      double binom = 1.0;
      for (int t = 0; t < i - j; ++t) binom = binom * (i - t) / (t + 1.0);
      double fall = 1.0;
      for (int t = 0; t < i - j; ++t) fall *= p - t;
      double fact = 1.0;
      for (int t = 2; t <= j; ++t) fact *= t;
      rhs -= q[j] * binom * fall * std::pow(-2.0, p - i + j) * fact;
    }
    double fact_i = 1.0;
    for (int t = 2; t <= i; ++t) fact_i *= t;
    q[i] = rhs / (std::pow(-2.0, p) * fact_i);
  }
  std::vector<double> left(static_cast<size_t>(p + 1), 0.0);
  left[0] = 1.0;
  for (int t = 0; t < p; ++t) {
    std::vector<double> next(static_cast<size_t>(p + 1), 0.0);
    for (int k = 0; k <= t; ++k) {
      next[k + 1] += left[k];
      next[k] -= left[k];
    }
    left = next;
  }
  std::vector<double> u(static_cast<size_t>(2 * p - 1), 0.0);
  std::vector<double> right(static_cast<size_t>(p - 1 > 0 ? p - 1 : 1), 0.0);
  right[0] = p > 1 ? q[0] : 0.0;
  for (int j = 1; j + 1 < p; ++j) {
    double binom = 1.0;
    for (int k = 0; k <= j; ++k) {
      right[k] += q[j] * binom;
      binom = binom * (j - k) / (k + 1.0);
    }
  }
  for (size_t ka = 0; ka <= static_cast<size_t>(p); ++ka)
    for (size_t kb = 0; kb < right.size(); ++kb)
      if (ka + kb < u.size()) u[ka + kb] += left[ka] * right[kb];
  std::vector<double> coeffs(static_cast<size_t>(2 * p), 0.0);
  for (size_t k = 0; k < u.size(); ++k) coeffs[k + 1] = u[k] / static_cast<double>(k + 1);
  double at_minus1 = 0.0, spow = -1.0;
  for (size_t k = 1; k < coeffs.size(); ++k) {
    at_minus1 += coeffs[k] * spow;
    spow = -spow;
  }
  coeffs[0] = derivs[0] - at_minus1;
  return Polynomial(mid, h, coeffs);
}

struct RegularizedKernel {  // kernels.cpp:240-264
  KernelSpec spec;
  double eps_b = 0.0;
  int p = 1;
  Polynomial blend;
  double tail = 0.0;
  RegularizedKernel() = default;
  RegularizedKernel(const KernelSpec& s, double e, int pp) : spec(s), eps_b(e), p(pp) {
    validate_spec(s);
    if (!(e >= 0.0) || !(e < 0.5)) fail(S_PARAM, "blend width must lie in [0, 1/2)");
    if (pp < 1 || pp > 8) fail(S_PARAM, "smoothness order must lie in [1, 8]");
    if (eps_b > 0.0) {
      blend = two_point_taylor(s, e, pp);
      tail = blend.value(0.5);
    } else {
      tail = eval_kernel(s, 0.5);
    }
  }
  double value(double r) const {
    if (!(r >= 0.0)) fail(S_RANGE, "kernel radius must be nonnegative");
    if (eps_b == 0.0) return eval_kernel(spec, std::min(r, 0.5));
    if (r <= 0.5 - eps_b) return eval_kernel(spec, r);
    if (r <= 0.5) return blend.value(r);
    return tail;
  }
  double value_at(const double* y, int d) const {  // y.norm(): sqrt of squaredNorm
    double s = 0.0;
    for (int t = 0; t < d; ++t) s += y[t] * y[t];
    return value(std::sqrt(s));
  }
};

// kernel_fourier_coefficients (kernels.cpp:266-335): returns bhat in
// FrequencyIndexSet order.
std::vector<cd> kernel_fourier_coefficients(const RegularizedKernel& kernel, int dims, int N) {
  if (dims < 1 || dims > 3) fail(S_PARAM, "dims must be 1, 2, or 3");
  if (N < 2 || N % 2 != 0) fail(S_PARAM, "bandwidth must be even and >= 2");
  const int half = N / 2;
  size_t total = ipow(static_cast<size_t>(N), dims);
  std::vector<cd> buf(total);
  double y[3];
  int idx[3] = {0, 0, 0};
  for (size_t flat = 0; flat < total; ++flat) {
    size_t rest = flat;
    for (int t = dims - 1; t >= 0; --t) {
      idx[t] = static_cast<int>(rest % N);
      rest /= N;
    }
    for (int t = 0; t < dims; ++t) y[t] = static_cast<double>(idx[t] - half) / N;
    buf[flat] = cd(kernel.value_at(y, dims), 0.0);
  }
  fft_nd(buf.data(), dims, N, -1);  // FFTW_FORWARD
  std::vector<cd> result(total);
  const double norm = 1.0 / static_cast<double>(total);
  for (size_t flat = 0; flat < total; ++flat) {
    size_t rest = flat;
    int lsum = 0;
    size_t bin = 0;
    for (int t = dims - 1; t >= 0; --t) {
      int a = static_cast<int>(rest % N);
      rest /= N;
      int l = a - half;
      lsum += l;
      size_t stride = 1;
      for (int q = t + 1; q < dims; ++q) stride *= static_cast<size_t>(N);
      bin += static_cast<size_t>((l + N) % N) * stride;
    }
    double sign = (lsum % 2 == 0) ? 1.0 : -1.0;
    result[flat] = buf[bin] * (sign * norm);
  }
  return result;
}

cd trig_polynomial_value(const std::vector<cd>& coeffs, int d, int N, const double* y) {  // kernels.cpp:337-367
  std::vector<cd> phase(static_cast<size_t>(d) * N);
  for (int t = 0; t < d; ++t)
    for (int a = 0; a < N; ++a) phase[static_cast<size_t>(t) * N + a] = std::polar(1.0, 2.0 * kPi * (a - N / 2) * y[t]);
  cd acc = 0.0;
  size_t flat = 0;
  if (d == 1) {
    for (int a = 0; a < N; ++a, ++flat) acc += coeffs[flat] * phase[a];
  } else if (d == 2) {
    for (int a = 0; a < N; ++a)
      for (int c = 0; c < N; ++c, ++flat) acc += coeffs[flat] * (phase[a] * phase[N + c]);
  } else {
    for (int a = 0; a < N; ++a)
      for (int c = 0; c < N; ++c) {
        cd pac = phase[a] * phase[N + c];
        for (int e = 0; e < N; ++e, ++flat) acc += coeffs[flat] * (pac * phase[2 * N + e]);
      }
  }
  return acc;
}

double kernel_approx_error(const RegularizedKernel& kernel, const std::vector<cd>& coeffs, int d, int N,
                           int sample_count, uint64_t seed) {  // kernels.cpp:369-396
  if (sample_count < 1) fail(S_PARAM, "sample count must be positive");
  const double radius = 0.5 - kernel.eps_b;
  std::mt19937_64 rng(seed);
  std::normal_distribution<double> gauss;
  std::uniform_real_distribution<double> unif(0.0, 1.0);
  double worst = 0.0;
  double y[3];
  for (int s = 0; s < sample_count; ++s) {
    double norm2 = 0.0;
    for (int t = 0; t < d; ++t) {
      y[t] = gauss(rng);
      norm2 += y[t] * y[t];
    }
    double len = std::sqrt(norm2);
    double r = radius * std::pow(unif(rng), 1.0 / d);
    if (len > 0.0)
      for (int t = 0; t < d; ++t) y[t] *= r / len;
    else
      for (int t = 0; t < d; ++t) y[t] = 0.0;
    double yn = 0.0;
    for (int t = 0; t < d; ++t) yn += y[t] * y[t];
    double err = std::abs(eval_kernel(kernel.spec, std::sqrt(yn)) - trig_polynomial_value(coeffs, d, N, y).real());
    worst = std::max(worst, err);
  }
  return worst;
}

// ---------------------------------------------------------------------------
// Fast summation  (fastsum.hpp:13-75, fastsum.cpp)
// ---------------------------------------------------------------------------
struct Params {
  int N = 32, m = 4, p = 4;
  double eps_b = 0.0, oversampling = 2.0;
};

void validate_params(const Params& p) {  // fastsum.cpp:25-36
  if (p.N < 2 || p.N % 2 != 0) fail(S_PARAM, "bandwidth must be even and >= 2");
  if (p.m < 1 || p.m > 32) fail(S_PARAM, "cutoff must lie in [1, 32]");
  if (p.p < 1 || p.p > 8) fail(S_PARAM, "smoothness order must lie in [1, 8]");
  if (!(p.eps_b >= 0.0) || !(p.eps_b < 0.5)) fail(S_PARAM, "blend width must lie in [0, 1/2)");
  if (!(p.oversampling >= 1.0)) fail(S_PARAM, "oversampling factor must be >= 1");
}

struct Fastsum {
  Mat nodes;
  Params params;
  KernelSpec kernel, scaled;
  double rho = 1.0, out_factor = 1.0, k0 = 0.0;
  RegularizedKernel reg;
  std::vector<cd> coeffs;
  std::unique_ptr<Nfft> nfft;

  Fastsum(const Mat& nodes_, const KernelSpec& k, const Params& p) {  // fastsum.cpp:69-92
    validate_params(p);
    if (nodes_.rows == 0) fail(S_SHAPE, "node set is empty");
    if (nodes_.cols < 1 || nodes_.cols > 3) fail(S_SHAPE, "nodes must have 1, 2, or 3 columns");
    validate_spec(k);
    const double radius = 0.25 - 0.5 * p.eps_b;
    if (!(radius > 0.0)) fail(S_PARAM, "blend width leaves no node radius");
    double maxnorm = 0.0;
    for (int64_t j = 0; j < nodes_.rows; ++j) {
      double s = 0.0;
      for (int64_t t = 0; t < nodes_.cols; ++t) s += nodes_(j, t) * nodes_(j, t);
      double nrm = std::sqrt(s);
      if (j == 0 || nrm > maxnorm) maxnorm = nrm;
    }
    rho = (maxnorm > radius) ? radius / maxnorm : 1.0;
    scaled = k;
    scaled.shape = k.shape * rho;
    out_factor = 1.0;
    if (k.family == MULTIQUADRIC) out_factor = 1.0 / rho;
    if (k.family == INV_MULTIQUADRIC) out_factor = rho;
    nodes = nodes_;
    params = p;
    kernel = k;
    k0 = eval_kernel(k, 0.0);
    reg = RegularizedKernel(scaled, p.eps_b, p.p);
    const int d = static_cast<int>(nodes.cols);
    coeffs = kernel_fourier_coefficients(reg, d, p.N);
    Mat sn(nodes.rows, nodes.cols);
    for (size_t i = 0; i < sn.a.size(); ++i) sn.a[i] = rho * nodes.a[i];
    nfft = std::make_unique<Nfft>(d, p.N, p.m, sn, p.oversampling);
  }

  std::vector<double> apply(const double* x, int64_t len) const {  // fastsum.cpp:111-118
    if (len != nodes.rows) fail(S_SHAPE, "input vector length does not match node count");
    std::vector<cd> xc(static_cast<size_t>(len));
    for (int64_t i = 0; i < len; ++i) xc[static_cast<size_t>(i)] = cd(x[i], 0.0);
    std::vector<cd> spectrum = nfft->adjoint(xc);
    for (size_t i = 0; i < spectrum.size(); ++i) spectrum[i] *= coeffs[i];
    std::vector<double> re = nfft->forward_real(spectrum);
    for (double& v : re) v = out_factor * v;
    return re;
  }

  double kernel_error_estimate(int sample_count, uint64_t seed) const {  // fastsum.cpp:120-124
    return std::abs(out_factor) * kernel_approx_error(reg, coeffs, static_cast<int>(nodes.cols), params.N,
                                                     sample_count, seed);
  }
};

std::vector<double> direct_apply(const Mat& nodes, const KernelSpec& kernel, const double* x, int64_t len) {
  // fastsum.cpp:126-139
  if (len != nodes.rows) fail(S_SHAPE, "input vector length does not match node count");
  const int64_t n = nodes.rows;
  std::vector<double> out(static_cast<size_t>(n), 0.0);
  for (int64_t j = 0; j < n; ++j) {
    double acc = 0.0;
    for (int64_t i = 0; i < n; ++i) {
      double s = 0.0;
      for (int64_t t = 0; t < nodes.cols; ++t) {
        double df = nodes(j, t) - nodes(i, t);
        s += df * df;
      }
      acc += eval_kernel(kernel, std::sqrt(s)) * x[i];
    }
    out[static_cast<size_t>(j)] = acc;
  }
  return out;
}

// ---------------------------------------------------------------------------
// Graph operator  (graphop.hpp:45-97, graphop.cpp:36-103)
// ---------------------------------------------------------------------------
struct Adjacency {
  Mat nodes;
  KernelSpec kernel;
  bool direct = false;
  std::unique_ptr<Fastsum> plan;
  double k0 = 0.0;
  std::vector<double> degrees, inv_sqrt;
  int64_t bad_node = -1;

  std::vector<double> apply_kernel(const double* x, int64_t len) const {  // graphop.cpp:28-33
    if (len != nodes.rows) fail(S_SHAPE, "input length does not match operator dimension");
    if (plan) return plan->apply(x, len);
    return direct_apply(nodes, kernel, x, len);
  }

  Adjacency(const Mat& nodes_, const KernelSpec& k, const Params& p, bool direct_backend) {  // graphop.cpp:36-67
    if (nodes_.rows < 2) fail(S_SHAPE, "adjacency operator needs at least two nodes");
    if (nodes_.cols < 1 || nodes_.cols > 3) fail(S_PARAM, "node dimension must be 1, 2, or 3");
    nodes = nodes_;
    kernel = k;
    direct = direct_backend;
    if (!direct) plan = std::make_unique<Fastsum>(nodes_, k, p);
    k0 = eval_kernel(k, 0.0);
    const int64_t n = nodes.rows;
    std::vector<double> ones(static_cast<size_t>(n), 1.0);
    degrees = apply_kernel(ones.data(), n);
    for (double& v : degrees) v = v - k0;
    for (int64_t j = 0; j < n; ++j)
      if (!(degrees[static_cast<size_t>(j)] > 0.0)) {
        bad_node = j;
        fail(S_NUMERIC, "computed degree of node " + std::to_string(j) + " is not positive (" +
                           std::to_string(degrees[static_cast<size_t>(j)]) +
                           "); increase the fast-summation bandwidth/cutoff or widen the kernel");
      }
    inv_sqrt.resize(static_cast<size_t>(n));
    for (int64_t j = 0; j < n; ++j) inv_sqrt[static_cast<size_t>(j)] = 1.0 / std::sqrt(degrees[static_cast<size_t>(j)]);
  }

  std::vector<double> apply_weight(const double* x, int64_t len) const {  // graphop.cpp:90-93
    std::vector<double> y = apply_kernel(x, len);
    for (int64_t i = 0; i < len; ++i) y[static_cast<size_t>(i)] -= k0 * x[i];
    return y;
  }

  std::vector<double> apply_normalized(const double* x, int64_t len) const {  // graphop.cpp:95-99
    if (len != nodes.rows) fail(S_SHAPE, "input length does not match operator dimension");
    std::vector<double> scaled(static_cast<size_t>(len));
    for (int64_t i = 0; i < len; ++i) scaled[static_cast<size_t>(i)] = inv_sqrt[static_cast<size_t>(i)] * x[i];
    std::vector<double> weighted = apply_kernel(scaled.data(), len);
    for (int64_t i = 0; i < len; ++i)
      weighted[static_cast<size_t>(i)] = inv_sqrt[static_cast<size_t>(i)] *
                                         (weighted[static_cast<size_t>(i)] - k0 * scaled[static_cast<size_t>(i)]);
    return weighted;
  }

  std::vector<double> apply_sym_laplacian(const double* x, int64_t len) const {  // graphop.cpp:101-103
    std::vector<double> a = apply_normalized(x, len);
    for (int64_t i = 0; i < len; ++i) a[static_cast<size_t>(i)] = x[i] - a[static_cast<size_t>(i)];
    return a;
  }
};

// ---------------------------------------------------------------------------
// Lanczos  (spectral.cpp:59-75, 105-139, 141-256)
// ---------------------------------------------------------------------------
using ApplyFn = std::function<std::vector<double>(const std::vector<double>&)>;

struct EigenPairs {
  std::vector<double> values;  // k
  Mat vectors;                 // n x k
};

EigenPairs make_eigenpairs(const std::vector<double>& values, const Mat& vectors) {  // spectral.cpp:105-127
  if (static_cast<int64_t>(values.size()) != vectors.cols) fail(S_SHAPE, "eigenvalue count does not match eigenvector columns");
  const int64_t k = static_cast<int64_t>(values.size());
  std::vector<int64_t> order(static_cast<size_t>(k));
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int64_t a, int64_t b) { return values[a] > values[b]; });
  EigenPairs pairs;
  pairs.values.resize(static_cast<size_t>(k));
  pairs.vectors = Mat(vectors.rows, k);
  for (int64_t i = 0; i < k; ++i) {
    pairs.values[i] = values[order[i]];
    const double* src = vectors.col(order[i]);
    int64_t at = 0;
    double best = -1.0;
    for (int64_t r = 0; r < vectors.rows; ++r)
      if (std::abs(src[r]) > best) {
        best = std::abs(src[r]);
        at = r;
      }
    double sgn = (vectors.rows > 0 && src[at] < 0.0) ? -1.0 : 1.0;
    for (int64_t r = 0; r < vectors.rows; ++r) pairs.vectors(r, i) = sgn * src[r];
  }
  return pairs;
}

double dot(const double* a, const double* b, int64_t n) {
  double s = 0.0;
  for (int64_t i = 0; i < n; ++i) s += a[i] * b[i];
  return s;
}
double norm2(const double* a, int64_t n) { return std::sqrt(dot(a, a, n)); }

// z -= Q(:, 0:m) * (Q(:, 0:m)^T z)
void cgs_pass(const Mat& basis, int m, std::vector<double>& z) {
  const int64_t n = basis.rows;
  std::vector<double> h(static_cast<size_t>(m));
  for (int j = 0; j < m; ++j) h[j] = dot(basis.col(j), z.data(), n);
  std::vector<double> qh(static_cast<size_t>(n), 0.0);
  for (int j = 0; j < m; ++j) {
    const double* q = basis.col(j);
    for (int64_t i = 0; i < n; ++i) qh[i] += q[i] * h[j];
  }
  for (int64_t i = 0; i < n; ++i) z[i] -= qh[i];
}

bool random_orthogonal(std::mt19937_64& rng, const Mat& basis, int m, std::vector<double>& out) {  // spectral.cpp:59-75
  std::uniform_real_distribution<double> unif(-1.0, 1.0);
  const int64_t n = basis.rows;
  for (int attempt = 0; attempt < 8; ++attempt) {
    std::vector<double> v(static_cast<size_t>(n));
    for (int64_t i = 0; i < n; ++i) v[i] = unif(rng);
    for (int pass = 0; pass < 2; ++pass) cgs_pass(basis, m, v);
    double nv = norm2(v.data(), n);
    if (nv > 1e-8) {
      out.resize(static_cast<size_t>(n));
      for (int64_t i = 0; i < n; ++i) out[i] = v[i] / nv;
      return true;
    }
  }
  return false;
}

struct LanczosOut {
  EigenPairs pairs;
  int iterations = 0;
  bool converged = false;
};

LanczosOut lanczos_largest(int64_t n, const ApplyFn& apply, int k, int max_iter, double tol, uint64_t seed) {
  if (n < 1) fail(S_PARAM, "operator handle is empty");
  if (k < 1) fail(S_PARAM, "at least one eigenpair must be requested");
  if (k > n) fail(S_PARAM, "requested pairs must not exceed the operator dimension");
  if (max_iter < 1) fail(S_PARAM, "max_iter must be positive");
  if (!(tol > 0.0)) fail(S_PARAM, "tolerance must be positive");

  std::mt19937_64 rng(seed);  // spectral.cpp:152-156
  std::uniform_real_distribution<double> unif(-1.0, 1.0);
  std::vector<double> start(static_cast<size_t>(n));
  for (int64_t i = 0; i < n; ++i) start[i] = unif(rng);
  double sn = norm2(start.data(), n);
  for (double& v : start) v /= sn;

  int64_t cap = std::min<int64_t>(n, 64);
  Mat basis(n, cap);
  std::copy(start.begin(), start.end(), basis.col(0));
  std::vector<double> alphas, betas;
  std::vector<double> tri_vals, tri_vecs;
  int tri_size = 0;
  double scale = 0.0;
  bool converged = false;
  int iterations = 0;
  int next_check = k;

  auto solve_tridiagonal = [&](int m) {
    tri_vals.assign(alphas.begin(), alphas.begin() + m);
    std::vector<double> sub(betas.begin(), betas.begin() + (m - 1));
    tridiag_eig(m, tri_vals, sub, tri_vecs);
    tri_size = m;
  };

  while (true) {  // spectral.cpp:181-239
    const int64_t cur = static_cast<int64_t>(alphas.size());
    std::vector<double> qcur(basis.col(cur), basis.col(cur) + n);
    std::vector<double> z = apply(qcur);
    if (static_cast<int64_t>(z.size()) != n) fail(S_SHAPE, "vector length does not match operator dimension");
    ++iterations;
    const int m = static_cast<int>(alphas.size()) + 1;
    double alpha = dot(basis.col(m - 1), z.data(), n);
    alphas.push_back(alpha);
    for (int64_t i = 0; i < n; ++i) z[i] -= alpha * basis(i, m - 1);
    const double beta_prev = m >= 2 ? betas[static_cast<size_t>(m - 2)] : 0.0;
    if (m >= 2)
      for (int64_t i = 0; i < n; ++i) z[i] -= beta_prev * basis(i, m - 2);
    for (int pass = 0; pass < 2; ++pass) cgs_pass(basis, m, z);
    double beta = norm2(z.data(), n);
    scale = std::max(scale, std::abs(alpha) + beta + beta_prev);

    const bool last = iterations >= max_iter || m == static_cast<int>(n);
    if (m >= k && (m >= next_check || last)) {
      solve_tridiagonal(m);
      bool all_small = true;
      for (int i = 0; i < k && all_small; ++i) {
        double theta = tri_vals[m - 1 - i];
        double estimate = beta * std::abs(tri_vecs[static_cast<size_t>(m - 1 - i) * m + (m - 1)]);
        double threshold = tol * std::max(std::abs(theta), kEps * std::max(scale, 1.0));
        if (estimate > threshold) all_small = false;
      }
      if (all_small) {
        converged = true;
        break;
      }
      next_check = m + std::max(8, m / 8);
    }
    if (iterations >= max_iter) break;
    if (m == static_cast<int>(n)) {
      converged = true;
      break;
    }
    if (m == basis.cols) {  // conservativeResize keeps the leading columns
      Mat bigger(n, std::min<int64_t>(n, basis.cols * 2));
      std::copy(basis.a.begin(), basis.a.end(), bigger.a.begin());
      basis = std::move(bigger);
    }
    if (beta > 1e-14 * std::max(scale, 1.0)) {
      betas.push_back(beta);
      for (int64_t i = 0; i < n; ++i) basis(i, m) = z[i] / beta;
    } else {
      std::vector<double> next;
      if (!random_orthogonal(rng, basis, m, next)) {
        converged = true;
        break;
      }
      betas.push_back(0.0);
      std::copy(next.begin(), next.end(), basis.col(m));
    }
  }

  const int m = static_cast<int>(alphas.size());  // spectral.cpp:241-255
  if (tri_size != m) solve_tridiagonal(m);
  const int wanted = std::min(k, m);
  std::vector<double> values(static_cast<size_t>(wanted));
  Mat vectors(n, wanted);
  for (int i = 0; i < wanted; ++i) {
    values[i] = tri_vals[m - 1 - i];
    const double* s = &tri_vecs[static_cast<size_t>(m - 1 - i) * m];
    double* v = vectors.col(i);
    for (int j = 0; j < m; ++j) {
      const double* q = basis.col(j);
      double sj = s[j];
      for (int64_t r = 0; r < n; ++r) v[r] += q[r] * sj;
    }
  }
  LanczosOut out;
  out.pairs = make_eigenpairs(values, vectors);
  out.iterations = iterations;
  out.converged = converged;
  return out;
}

thread_local std::string g_last_error;

// ---------------------------------------------------------------------------
// cg_solve (spectral.cpp:446-495): status 0 converged, 1 max iterations,
// 2 indefinite.  Serial dot products (Eigen's are vectorised: rounding-level
// difference only).
// ---------------------------------------------------------------------------
double dotv(const std::vector<double>& a, const std::vector<double>& b) {
  double s = 0.0;
  for (size_t i = 0; i < a.size(); ++i) s += a[i] * b[i];
  return s;
}

int cg_serial(const ApplyFn& op, const std::vector<double>& b, double tol, int max_iter, std::vector<double>& x,
              int* iterations) {
  if (!(tol > 0.0)) fail(S_PARAM, "tolerance must be positive");
  if (max_iter < 1) fail(S_PARAM, "max_iter must be positive");
  const size_t n = b.size();
  x.assign(n, 0.0);
  *iterations = 0;
  const double bn = std::sqrt(dotv(b, b));
  if (bn == 0.0) return 0;
  std::vector<double> r = b, p = r;
  double rs = dotv(r, r);
  for (int it = 1; it <= max_iter; ++it) {
    const std::vector<double> ap = op(p);
    const double curv = dotv(p, ap);
    *iterations = it;
    if (!(curv > 0.0)) return 2;
    const double step = rs / curv;
    for (size_t i = 0; i < n; ++i) x[i] += step * p[i];
    for (size_t i = 0; i < n; ++i) r[i] -= step * ap[i];
    double rs_next = dotv(r, r);
    if (std::sqrt(rs_next) <= tol * bn) {
      const std::vector<double> ax = op(x);
      std::vector<double> tr(n);
      for (size_t i = 0; i < n; ++i) tr[i] = b[i] - ax[i];
      if (std::sqrt(dotv(tr, tr)) <= tol * bn) return 0;
      r = tr;
      rs_next = dotv(r, r);
      p = r;
      rs = rs_next;
      continue;
    }
    for (size_t i = 0; i < n; ++i) p[i] = r[i] + (rs_next / rs) * p[i];
    rs = rs_next;
  }
  return 1;
}

// ---------------------------------------------------------------------------
// nystrom_gaussian (spectral.cpp:384-444).  Dense helpers standing in for
// Eigen: Householder QR with Eigen's makeHouseholder convention (beta =
// -sign(x0)|x|), Q formed explicitly (thin); the symmetric eigensolver is
// Householder tridiagonalisation followed by the implicit-QL tridiag_eig,
// ascending as SelfAdjointEigenSolver.
// ---------------------------------------------------------------------------
// spectral.cpp:384-444 over any operator
void nystrom_gaussian_serial(int64_t n, const ApplyFn& op, int k, int L, int M, uint64_t seed, std::vector<double>& values,
                             Mat& vectors) {
  if (k < 1 || M < k || L < M || L > n) fail(S_PARAM, "need 1 <= k <= M <= L <= n");
  std::mt19937_64 rng(seed);
  std::normal_distribution<double> gauss;
  Mat probes(n, L);
  for (int64_t c = 0; c < L; ++c)
    for (int64_t r = 0; r < n; ++r) probes(r, c) = gauss(rng);
  Mat sketch(n, L);
  for (int64_t c = 0; c < L; ++c) {
    std::vector<double> x(probes.col(c), probes.col(c) + n);
    const std::vector<double> y = op(x);
    std::copy(y.begin(), y.end(), sketch.col(c));
  }
  Mat q, r;
  householder_qr(sketch, q, r);
  Mat b1(n, L);
  for (int64_t c = 0; c < L; ++c) {
    std::vector<double> x(q.col(c), q.col(c) + n);
    const std::vector<double> y = op(x);
    std::copy(y.begin(), y.end(), b1.col(c));
  }
  Mat b2(L, L);
  for (int64_t j = 0; j < L; ++j)
    for (int64_t i = 0; i < L; ++i) {
      double acc = 0.0;
      for (int64_t t = 0; t < n; ++t) acc += q(t, i) * b1(t, j);
      b2(i, j) = acc;
    }
  Mat b2s(L, L);
  for (int64_t j = 0; j < L; ++j)
    for (int64_t i = 0; i < L; ++i) b2s(i, j) = 0.5 * (b2(i, j) + b2(j, i));
  std::vector<double> ev;
  Mat evec;
  dense_sym_eig(b2s, ev, evec);
  int positives = 0;
  for (double v : ev) positives += v > 0.0;
  if (positives < M)
    fail(S_NUMERIC, "sketch captured fewer than the requested number of positive eigenvalues; increase the sketch size");
  std::vector<double> sigma(static_cast<size_t>(M));
  Mat um(L, M);
  for (int i = 0; i < M; ++i) {
    sigma[static_cast<size_t>(i)] = ev[static_cast<size_t>(L - 1 - i)];
    for (int64_t t = 0; t < L; ++t) um(t, i) = evec(t, L - 1 - i);
  }
  Mat bu(n, M);
  for (int64_t j = 0; j < M; ++j)
    for (int64_t i = 0; i < n; ++i) {
      double acc = 0.0;
      for (int64_t t = 0; t < L; ++t) acc += b1(i, t) * um(t, j);
      bu(i, j) = acc;
    }
  Mat qh, rh;
  householder_qr(bu, qh, rh);
  Mat mid(M, M);
  for (int64_t i = 0; i < M; ++i)
    for (int64_t j = 0; j < M; ++j) {
      double acc = 0.0;
      for (int64_t t = 0; t < M; ++t) acc += rh(i, t) / sigma[static_cast<size_t>(t)] * rh(j, t);
      mid(i, j) = acc;
    }
  Mat mids(M, M);
  for (int64_t j = 0; j < M; ++j)
    for (int64_t i = 0; i < M; ++i) mids(i, j) = 0.5 * (mid(i, j) + mid(j, i));
  std::vector<double> mv;
  Mat mvec;
  dense_sym_eig(mids, mv, mvec);
  values.assign(static_cast<size_t>(k), 0.0);
  Mat raw(n, k);
  for (int i = 0; i < k; ++i) {
    values[static_cast<size_t>(i)] = mv[static_cast<size_t>(M - 1 - i)];
    for (int64_t row = 0; row < n; ++row) {
      double acc = 0.0;
      for (int64_t t = 0; t < M; ++t) acc += qh(row, t) * mvec(t, M - 1 - i);
      raw(row, i) = acc;
    }
  }
  vectors = raw;
}

// ---------------------------------------------------------------------------
// k-means and spectral clustering (learn.cpp:17-167), label metrics
// (learn.cpp:441-486).  Points column-major n x dim (Eigen's MatrixXd).
// Row squared norms are left-to-right sums of squares (Eigen's scalar redux
// over a strided row); dist2.sum() is a serial sum here (Eigen vectorizes
// that one -- an ulp-level difference that only matters on exact ties of
// the k-means++ target).
// ---------------------------------------------------------------------------
struct KMeansRun {
  std::vector<int> labels;
  std::vector<double> centroids;  // k x dim column-major
  double wcss = 0.0;
};

double km_dist2(const Mat& pts, int64_t i, const std::vector<double>& cen, int k, int c) {
  double s = 0.0;
  for (int64_t t = 0; t < pts.cols; ++t) {
    const double df = pts(i, t) - cen[static_cast<size_t>(t * k + c)];
    s += df * df;
  }
  return s;
}

// learn.cpp:30-75
std::vector<double> km_plus_plus(const Mat& pts, int k, std::mt19937_64& rng) {
  const int64_t n = pts.rows, dim = pts.cols;
  std::uniform_int_distribution<int64_t> any(0, n - 1);
  std::uniform_real_distribution<double> unif(0.0, 1.0);
  std::vector<double> cen(static_cast<size_t>(k * dim));
  std::vector<bool> chosen(static_cast<size_t>(n), false);
  auto take = [&](int c, int64_t i) {
    for (int64_t t = 0; t < dim; ++t) cen[static_cast<size_t>(t * k + c)] = pts(i, t);
    chosen[static_cast<size_t>(i)] = true;
  };
  take(0, any(rng));
  std::vector<double> d2(static_cast<size_t>(n));
  for (int64_t i = 0; i < n; ++i) d2[static_cast<size_t>(i)] = km_dist2(pts, i, cen, k, 0);
  for (int c = 1; c < k; ++c) {
    double total = 0.0;
    for (double v : d2) total += v;
    int64_t pick = -1;
    if (total > 0.0) {
      const double target = unif(rng) * total;
      double running = 0.0;
      for (int64_t i = 0; i < n; ++i) {
        running += d2[static_cast<size_t>(i)];
        if (running >= target) {
          pick = i;
          break;
        }
      }
      if (pick < 0) pick = n - 1;
    } else {  // every remaining distance is zero: uniform among the unchosen
      std::vector<int64_t> open;
      for (int64_t i = 0; i < n; ++i)
        if (!chosen[static_cast<size_t>(i)]) open.push_back(i);
      if (open.empty())
        pick = any(rng);
      else
        pick = open[std::uniform_int_distribution<size_t>(0, open.size() - 1)(rng)];
    }
    take(c, pick);
    for (int64_t i = 0; i < n; ++i)
      d2[static_cast<size_t>(i)] = std::min(d2[static_cast<size_t>(i)], km_dist2(pts, i, cen, k, c));
  }
  return cen;
}

// learn.cpp:77-136
KMeansRun km_lloyd(const Mat& pts, int k, int max_iter, std::mt19937_64& rng) {
  const int64_t n = pts.rows, dim = pts.cols;
  KMeansRun r;
  r.centroids = km_plus_plus(pts, k, rng);
  r.labels.assign(static_cast<size_t>(n), -1);
  for (int iter = 0; iter < max_iter; ++iter) {
    bool changed = false;
    for (int64_t i = 0; i < n; ++i) {
      int best = 0;
      double bd = km_dist2(pts, i, r.centroids, k, 0);
      for (int c = 1; c < k; ++c) {
        const double dc = km_dist2(pts, i, r.centroids, k, c);
        if (dc < bd) {
          bd = dc;
          best = c;
        }
      }
      if (best != r.labels[static_cast<size_t>(i)]) {
        r.labels[static_cast<size_t>(i)] = best;
        changed = true;
      }
    }
    std::vector<int64_t> counts(static_cast<size_t>(k), 0);
    std::vector<double> sums(static_cast<size_t>(k * dim), 0.0);
    for (int64_t i = 0; i < n; ++i) {
      const int c = r.labels[static_cast<size_t>(i)];
      for (int64_t t = 0; t < dim; ++t) sums[static_cast<size_t>(t * k + c)] += pts(i, t);
      ++counts[static_cast<size_t>(c)];
    }
    for (int c = 0; c < k; ++c) {
      if (counts[static_cast<size_t>(c)] > 0) {
        for (int64_t t = 0; t < dim; ++t)
          r.centroids[static_cast<size_t>(t * k + c)] =
              sums[static_cast<size_t>(t * k + c)] / static_cast<double>(counts[static_cast<size_t>(c)]);
      } else {  // empty cluster: re-seed at the point farthest from its centroid
        int64_t far = 0;
        double fd = -1.0;
        for (int64_t i = 0; i < n; ++i) {
          const double dd = km_dist2(pts, i, r.centroids, k, r.labels[static_cast<size_t>(i)]);
          if (dd > fd) {
            fd = dd;
            far = i;
          }
        }
        for (int64_t t = 0; t < dim; ++t) r.centroids[static_cast<size_t>(t * k + c)] = pts(far, t);
        r.labels[static_cast<size_t>(far)] = c;
        changed = true;
      }
    }
    if (!changed) break;
  }
  r.wcss = 0.0;
  for (int64_t i = 0; i < n; ++i) r.wcss += km_dist2(pts, i, r.centroids, k, r.labels[static_cast<size_t>(i)]);
  return r;
}

// learn.cpp:140-155
KMeansRun km_kmeans(const Mat& pts, int k, int restarts, int max_iter, uint64_t seed) {
  if (pts.rows < 1) fail(S_SHAPE, "k-means needs at least one point");
  if (k < 1 || k > pts.rows) fail(S_PARAM, "cluster count must lie in [1, point count]");
  if (restarts < 1 || max_iter < 1) fail(S_PARAM, "restarts and max_iter must be positive");
  std::mt19937_64 rng(seed);
  KMeansRun best;
  best.wcss = std::numeric_limits<double>::infinity();
  for (int a = 0; a < restarts; ++a) {
    KMeansRun run = km_lloyd(pts, k, max_iter, rng);
    if (run.wcss < best.wcss) best = std::move(run);
  }
  return best;
}

// learn.cpp:157-167: unit-normalised rows of the eigenvectors, then k-means
Mat km_normalized_rows(const double* vectors, int64_t n, int kv) {
  Mat rows(n, kv);
  std::copy(vectors, vectors + n * kv, rows.a.begin());
  for (int64_t i = 0; i < n; ++i) {
    double s = 0.0;
    for (int t = 0; t < kv; ++t) s += rows(i, t) * rows(i, t);
    const double norm = std::sqrt(s);
    if (norm > 0.0)
      for (int t = 0; t < kv; ++t) rows(i, t) /= norm;
  }
  return rows;
}

// learn.cpp:441-486
double km_misclassification(const int* pred, const int* truth, int64_t n, bool permuted) {
  if (n == 0) return 0.0;
  if (!permuted) {
    int64_t wrong = 0;
    for (int64_t i = 0; i < n; ++i) wrong += pred[i] != truth[i];
    return static_cast<double>(wrong) / static_cast<double>(n);
  }
  int classes = 0;
  for (int64_t i = 0; i < n; ++i) {
    if (pred[i] < 0 || truth[i] < 0) fail(S_RANGE, "labels must be nonnegative");
    classes = std::max(classes, std::max(pred[i], truth[i]) + 1);
  }
  if (classes > 8) fail(S_PARAM, "permutation matching supports at most 8 classes");
  std::vector<int64_t> cnt(static_cast<size_t>(classes * classes), 0);
  for (int64_t i = 0; i < n; ++i) ++cnt[static_cast<size_t>(pred[i] * classes + truth[i])];
  std::vector<int> map(static_cast<size_t>(classes));
  for (int c = 0; c < classes; ++c) map[static_cast<size_t>(c)] = c;
  int64_t best = 0;
  do {
    int64_t matched = 0;
    for (int p = 0; p < classes; ++p) matched += cnt[static_cast<size_t>(p * classes + map[static_cast<size_t>(p)])];
    best = std::max(best, matched);
  } while (std::next_permutation(map.begin(), map.end()));
  return 1.0 - static_cast<double>(best) / static_cast<double>(n);
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    g_last_error.clear();
    return S_OK;
  } catch (const Error& e) {
    g_last_error = e.what();
    return e.code;
  } catch (const std::bad_alloc&) {
    g_last_error = "out of memory";
    return S_RESOURCE;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return S_NUMERIC;
  }
}

Mat make_mat(const double* colmajor, int64_t rows, int64_t cols) {
  Mat m(rows, cols);
  if (rows * cols > 0) std::memcpy(m.a.data(), colmajor, sizeof(double) * static_cast<size_t>(rows * cols));
  return m;
}

std::vector<cd> make_cvec(const double* interleaved, int64_t len) {
  std::vector<cd> v(static_cast<size_t>(len));
  for (int64_t i = 0; i < len; ++i) v[static_cast<size_t>(i)] = cd(interleaved[2 * i], interleaved[2 * i + 1]);
  return v;
}

void store_cvec(const std::vector<cd>& v, double* interleaved) {
  for (size_t i = 0; i < v.size(); ++i) {
    interleaved[2 * i] = v[i].real();
    interleaved[2 * i + 1] = v[i].imag();
  }
}

}  // namespace orc

// ============================================================================
// C ABI for the Python test harness (oracle/oracle.py).  Complex vectors are
// interleaved (re, im) doubles; matrices column-major.
// ============================================================================
using namespace orc;

extern "C" {

const char* orc_last_error(void) { return g_last_error.c_str(); }

// host threads of the NFFT loops (see g_threads); returns the previous value
int orc_set_threads(int threads) {
  const int old = g_threads;
  g_threads = std::max(1, threads);
  return old;
}

double orc_bessel_i0(double x) { return bessel_i0(x); }
double orc_std_bessel_i0(double x) { return std::cyl_bessel_i(0.0, x); }

int orc_fft(double* data, int d, int M, int sign) {
  return guarded([&] {
    size_t total = ipow(static_cast<size_t>(M), d);
    std::vector<cd> v = make_cvec(data, static_cast<int64_t>(total));
    fft_nd(v.data(), d, M, sign);
    store_cvec(v, data);
  });
}

int orc_freq_component(int d, int N, int64_t flat, int dim, int* out) {
  return guarded([&] {
    if (d < 1 || d > 3) fail(S_PARAM, "dims must be 1, 2, or 3");
    if (N < 2 || N % 2 != 0) fail(S_PARAM, "bandwidth must be even and >= 2");
    size_t size = ipow(static_cast<size_t>(N), d);
    if (flat < 0 || static_cast<size_t>(flat) >= size) fail(S_RANGE, "flat index out of range");
    if (dim < 0 || dim >= d) fail(S_RANGE, "dimension out of range");
    *out = freq_component(d, N, static_cast<size_t>(flat), dim);
  });
}

int orc_direct_ndft(int d, int N, const double* nodes, int64_t n, const double* fhat, double* out) {
  return guarded([&] {
    Mat nd = make_mat(nodes, n, d);
    size_t F = ipow(static_cast<size_t>(N), d);
    store_cvec(direct_ndft(d, N, nd, make_cvec(fhat, static_cast<int64_t>(F))), out);
  });
}

int orc_direct_adjoint_ndft(int d, int N, const double* nodes, int64_t n, const double* x, double* out) {
  return guarded([&] {
    Mat nd = make_mat(nodes, n, d);
    store_cvec(direct_adjoint_ndft(d, N, nd, make_cvec(x, n)), out);
  });
}

// NFFT plan handle
int orc_nfft_create(int d, int N, int m, const double* nodes, int64_t n, double oversampling, void** out) {
  return guarded([&] {
    Mat nd = make_mat(nodes, n, d);
    *out = new Nfft(d, N, m, nd, oversampling);
  });
}
void orc_nfft_destroy(void* h) { delete static_cast<Nfft*>(h); }
int orc_nfft_info(void* h, int* M, int64_t* coeffs) {
  return guarded([&] {
    auto* p = static_cast<Nfft*>(h);
    *M = p->M;
    *coeffs = static_cast<int64_t>(p->coeff_total);
  });
}
int orc_nfft_forward(void* h, const double* fhat, int64_t len, double* out) {
  return guarded([&] {
    auto* p = static_cast<Nfft*>(h);
    store_cvec(p->forward(make_cvec(fhat, len)), out);
  });
}
int orc_nfft_adjoint(void* h, const double* x, int64_t len, double* out) {
  return guarded([&] {
    auto* p = static_cast<Nfft*>(h);
    store_cvec(p->adjoint(make_cvec(x, len)), out);
  });
}
int orc_nfft_forward_real(void* h, const double* fhat, int64_t len, double* out) {
  return guarded([&] {
    auto* p = static_cast<Nfft*>(h);
    std::vector<double> r = p->forward_real(make_cvec(fhat, len));
    std::copy(r.begin(), r.end(), out);
  });
}
// taps / wrapped indices of node j (for cross-checking the device plan)
int orc_nfft_taps(void* h, double* w, int* idx) {
  return guarded([&] {
    auto* p = static_cast<Nfft*>(h);
    std::copy(p->w.begin(), p->w.end(), w);
    std::copy(p->idx.begin(), p->idx.end(), idx);
  });
}
int orc_nfft_deconv(void* h, double* out) {
  return guarded([&] {
    auto* p = static_cast<Nfft*>(h);
    std::copy(p->deconv.begin(), p->deconv.end(), out);
  });
}

int orc_eval_kernel(int family, double shape, double r, double* out) {
  return guarded([&] { *out = eval_kernel(KernelSpec{family, shape}, r); });
}
int orc_kernel_radial_derivatives(int family, double shape, double r0, int count, double* out) {
  return guarded([&] {
    std::vector<double> v = kernel_radial_derivatives(KernelSpec{family, shape}, r0, count);
    std::copy(v.begin(), v.end(), out);
  });
}
// two_point_taylor: returns center, scale and coefficient count (<= 2p)
int orc_two_point_taylor(int family, double shape, double eps_b, int p, double* center, double* scale,
                         double* coeffs, int* count) {
  return guarded([&] {
    Polynomial t = two_point_taylor(KernelSpec{family, shape}, eps_b, p);
    *center = t.center;
    *scale = t.scale;
    *count = static_cast<int>(t.coeffs.size());
    std::copy(t.coeffs.begin(), t.coeffs.end(), coeffs);
  });
}
int orc_regularized_value(int family, double shape, double eps_b, int p, const double* r, int64_t count,
                          double* out) {
  return guarded([&] {
    RegularizedKernel reg(KernelSpec{family, shape}, eps_b, p);
    for (int64_t i = 0; i < count; ++i) out[i] = reg.value(r[i]);
  });
}
int orc_kernel_coefficients(int family, double shape, double eps_b, int p, int d, int N, double* out) {
  return guarded([&] {
    RegularizedKernel reg(KernelSpec{family, shape}, eps_b, p);
    store_cvec(kernel_fourier_coefficients(reg, d, N), out);
  });
}
int orc_trig_polynomial_value(const double* coeffs, int d, int N, const double* y, double* out) {
  return guarded([&] {
    std::vector<cd> c = make_cvec(coeffs, static_cast<int64_t>(ipow(static_cast<size_t>(N), d)));
    cd v = trig_polynomial_value(c, d, N, y);
    out[0] = v.real();
    out[1] = v.imag();
  });
}

// Fastsum plan handle
int orc_fastsum_create(const double* nodes, int64_t n, int d, int family, double shape, int N, int m, int p,
                       double eps_b, double oversampling, void** out) {
  return guarded([&] {
    Mat nd = make_mat(nodes, n, d);
    Params pr{N, m, p, eps_b, oversampling};
    *out = new Fastsum(nd, KernelSpec{family, shape}, pr);
  });
}
void orc_fastsum_destroy(void* h) { delete static_cast<Fastsum*>(h); }
int orc_fastsum_apply(void* h, const double* x, int64_t len, double* y) {
  return guarded([&] {
    std::vector<double> r = static_cast<Fastsum*>(h)->apply(x, len);
    std::copy(r.begin(), r.end(), y);
  });
}
int orc_fastsum_info(void* h, double* rho, double* out_factor, double* k0, double* scaled_shape) {
  return guarded([&] {
    auto* f = static_cast<Fastsum*>(h);
    *rho = f->rho;
    *out_factor = f->out_factor;
    *k0 = f->k0;
    *scaled_shape = f->scaled.shape;
  });
}
int orc_fastsum_coefficients(void* h, double* out) {
  return guarded([&] { store_cvec(static_cast<Fastsum*>(h)->coeffs, out); });
}
int orc_fastsum_error_estimate(void* h, int samples, uint64_t seed, double* out) {
  return guarded([&] { *out = static_cast<Fastsum*>(h)->kernel_error_estimate(samples, seed); });
}
int orc_direct_apply(const double* nodes, int64_t n, int d, int family, double shape, const double* x, double* y) {
  return guarded([&] {
    Mat nd = make_mat(nodes, n, d);
    std::vector<double> r = direct_apply(nd, KernelSpec{family, shape}, x, n);
    std::copy(r.begin(), r.end(), y);
  });
}

// Adjacency operator handle.  op: 0 kernel, 1 weight, 2 normalized, 3 sym laplacian
int orc_adjacency_create(const double* nodes, int64_t n, int d, int family, double shape, int N, int m, int p,
                         double eps_b, double oversampling, int direct, void** out, int64_t* bad_node) {
  Adjacency* holder = nullptr;
  int st = guarded([&] {
    Mat nd = make_mat(nodes, n, d);
    Params pr{N, m, p, eps_b, oversampling};
    try {
      holder = new Adjacency(nd, KernelSpec{family, shape}, pr, direct != 0);
    } catch (const Error& e) {
      // the constructor names the node in the message; recover the index
      if (e.code == S_NUMERIC && bad_node) {
        std::string msg = e.what();
        auto pos = msg.find("node ");
        if (pos != std::string::npos) *bad_node = std::stoll(msg.substr(pos + 5));
      }
      throw;
    }
  });
  *out = holder;
  return st;
}
void orc_adjacency_destroy(void* h) { delete static_cast<Adjacency*>(h); }
int orc_adjacency_apply(void* h, int op, const double* x, int64_t len, double* y) {
  return guarded([&] {
    auto* a = static_cast<Adjacency*>(h);
    std::vector<double> r;
    switch (op) {
      case 0: r = a->apply_kernel(x, len); break;
      case 1: r = a->apply_weight(x, len); break;
      case 2: r = a->apply_normalized(x, len); break;
      case 3: r = a->apply_sym_laplacian(x, len); break;
      default: fail(S_PARAM, "unknown operator");
    }
    std::copy(r.begin(), r.end(), y);
  });
}
int orc_adjacency_degrees(void* h, double* out) {
  return guarded([&] {
    auto* a = static_cast<Adjacency*>(h);
    std::copy(a->degrees.begin(), a->degrees.end(), out);
  });
}

// Lanczos over the adjacency operator (which: 0 = A via apply_normalized,
// 1 = L_s via apply_sym_laplacian) or over a dense column-major matrix.
static int lanczos_common(int64_t n, const ApplyFn& fn, int k, int max_iter, double tol, uint64_t seed,
                          double* values, double* vectors, int* count, int* iterations, int* converged) {
  return guarded([&] {
    LanczosOut r = lanczos_largest(n, fn, k, max_iter, tol, seed);
    *count = static_cast<int>(r.pairs.values.size());
    std::copy(r.pairs.values.begin(), r.pairs.values.end(), values);
    std::copy(r.pairs.vectors.a.begin(), r.pairs.vectors.a.end(), vectors);
    *iterations = r.iterations;
    *converged = r.converged ? 1 : 0;
  });
}

int orc_lanczos_adjacency(void* h, int which, int k, int max_iter, double tol, uint64_t seed, double* values,
                          double* vectors, int* count, int* iterations, int* converged) {
  auto* a = static_cast<Adjacency*>(h);
  const int64_t n = a->nodes.rows;
  ApplyFn fn = [a, which, n](const std::vector<double>& x) {
    return which == 0 ? a->apply_normalized(x.data(), n) : a->apply_sym_laplacian(x.data(), n);
  };
  return lanczos_common(n, fn, k, max_iter, tol, seed, values, vectors, count, iterations, converged);
}

int orc_lanczos_dense(const double* A, int64_t n, int k, int max_iter, double tol, uint64_t seed, double* values,
                      double* vectors, int* count, int* iterations, int* converged) {
  std::vector<double> mat(A, A + n * n);
  ApplyFn fn = [&mat, n](const std::vector<double>& x) {
    std::vector<double> y(static_cast<size_t>(n), 0.0);
    for (int64_t j = 0; j < n; ++j) {
      double xj = x[j];
      const double* c = mat.data() + j * n;
      for (int64_t i = 0; i < n; ++i) y[i] += c[i] * xj;
    }
    return y;
  };
  return lanczos_common(n, fn, k, max_iter, tol, seed, values, vectors, count, iterations, converged);
}

int orc_tridiag_eig(int m, const double* diag, const double* sub, double* values, double* vectors) {
  return guarded([&] {
    std::vector<double> dv(diag, diag + m);
    std::vector<double> sv(sub, sub + std::max(m - 1, 0));
    std::vector<double> z;
    tridiag_eig(m, dv, sv, z);
    std::copy(dv.begin(), dv.end(), values);
    std::copy(z.begin(), z.end(), vectors);
  });
}

int orc_make_eigenpairs(const double* values, const double* vectors, int64_t n, int k, double* out_values,
                        double* out_vectors) {
  return guarded([&] {
    std::vector<double> v(values, values + k);
    Mat vec = make_mat(vectors, n, k);
    EigenPairs p = make_eigenpairs(v, vec);
    std::copy(p.values.begin(), p.values.end(), out_values);
    std::copy(p.vectors.a.begin(), p.vectors.a.end(), out_vectors);
  });
}

// ---- test-input helpers mirroring the reference tests' generators --------
// test_nfft.cpp:16-27
void orc_random_nodes(int64_t n, int d, uint64_t seed, double* out) {
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> dist(-0.5, 0.5);
  for (int64_t j = 0; j < n; ++j)
    for (int t = 0; t < d; ++t) {
      double v = dist(rng);
      while (v >= 0.5) v = dist(rng);
      out[t * n + j] = v;
    }
}
// test_nfft.cpp:29-36 (interleaved complex)
void orc_random_coeffs(int64_t count, uint64_t seed, double* out) {
  std::mt19937_64 rng(seed);
  std::normal_distribution<double> dist;
  for (int64_t i = 0; i < count; ++i) {
    double re = dist(rng);
    double im = dist(rng);
    out[2 * i] = re;
    out[2 * i + 1] = im;
  }
}
// test_fastsum.cpp:14-21 / test_graphop.cpp:13-20
void orc_random_cloud(int64_t n, int d, double extent, uint64_t seed, double* out) {
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> dist(-extent, extent);
  for (int64_t j = 0; j < n; ++j)
    for (int t = 0; t < d; ++t) out[t * n + j] = dist(rng);
}
// test_fastsum.cpp:23-29
void orc_random_vector(int64_t n, uint64_t seed, double* out) {
  std::mt19937_64 rng(seed);
  std::normal_distribution<double> dist;
  for (int64_t i = 0; i < n; ++i) out[i] = dist(rng);
}


int orc_kmeans(const double* points_colmajor, int64_t n, int dim, int k, int restarts, int max_iter, uint64_t seed,
               int* labels, double* centroids, double* wcss) {
  return guarded([&] {
    if (n < 1) fail(S_SHAPE, "k-means needs at least one point");
    Mat pts(n, dim);
    std::copy(points_colmajor, points_colmajor + n * dim, pts.a.begin());
    KMeansRun r = km_kmeans(pts, k, restarts, max_iter, seed);
    std::copy(r.labels.begin(), r.labels.end(), labels);
    if (centroids) std::copy(r.centroids.begin(), r.centroids.end(), centroids);
    if (wcss) *wcss = r.wcss;
  });
}

int orc_spectral_cluster(const double* vectors_colmajor, int64_t n, int kv, int k, int restarts, int max_iter,
                         uint64_t seed, int* labels) {
  return guarded([&] {
    if (kv < k) fail(S_PARAM, "need at least as many eigenvectors as clusters");
    Mat rows = km_normalized_rows(vectors_colmajor, n, kv);
    KMeansRun r = km_kmeans(rows, k, restarts, max_iter, seed);
    std::copy(r.labels.begin(), r.labels.end(), labels);
  });
}

int orc_misclassification(const int* pred, const int* truth, int64_t n, int permuted, double* out) {
  return guarded([&] { *out = km_misclassification(pred, truth, n, permuted != 0); });
}

// test_learn.cpp:23-39 blobs(): counts[b] points N(center_b, spread^2 I)
void orc_blobs(const int* counts, int nb, const double* centers_rowmajor, int dim, double spread, uint64_t seed,
               double* out_colmajor, int* labels) {
  std::mt19937_64 rng(seed);
  std::normal_distribution<double> gauss(0.0, spread);
  int64_t total = 0;
  for (int b = 0; b < nb; ++b) total += counts[b];
  int64_t row = 0;
  for (int b = 0; b < nb; ++b)
    for (int i = 0; i < counts[b]; ++i, ++row) {
      for (int t = 0; t < dim; ++t) out_colmajor[t * total + row] = centers_rowmajor[b * dim + t] + gauss(rng);
      labels[row] = b;
    }
}

// learn.cpp:364-381 kernel_ssl_solve: (I + beta L_s) x = f
int orc_kernel_ssl_solve(void* h, const double* f, int64_t n, double beta, double tol, int max_iter, double* x,
                         int* iterations, int* status) {
  return guarded([&] {
    auto* a = static_cast<Adjacency*>(h);
    if (!(beta >= 0.0)) fail(S_PARAM, "beta must be nonnegative");
    if (n != a->nodes.rows) fail(S_SHAPE, "fidelity length does not match operator dimension");
    std::vector<double> b(f, f + n), xs;
    if (beta == 0.0) {
      std::copy(b.begin(), b.end(), x);
      *iterations = 0;
      *status = 0;
      return;
    }
    ApplyFn op = [a, beta, n](const std::vector<double>& v) {
      std::vector<double> lx = a->apply_sym_laplacian(v.data(), n);
      for (int64_t i = 0; i < n; ++i) lx[static_cast<size_t>(i)] = v[static_cast<size_t>(i)] + beta * lx[static_cast<size_t>(i)];
      return lx;
    };
    *status = cg_serial(op, b, tol, max_iter, xs, iterations);
    std::copy(xs.begin(), xs.end(), x);
  });
}

// learn.cpp:403-430 krr_fit's system: (W~ + beta I) alpha = f
int orc_fastsum_ridge_solve(void* h, const double* f, int64_t n, double beta, double tol, int max_iter, double* x,
                            int* iterations, int* status) {
  return guarded([&] {
    auto* fs = static_cast<Fastsum*>(h);
    if (!(beta > 0.0)) fail(S_PARAM, "beta must be positive");
    std::vector<double> b(f, f + n), xs;
    ApplyFn op = [fs, beta, n](const std::vector<double>& v) {
      std::vector<double> kx = fs->apply(v.data(), n);
      for (int64_t i = 0; i < n; ++i) kx[static_cast<size_t>(i)] = kx[static_cast<size_t>(i)] + beta * v[static_cast<size_t>(i)];
      return kx;
    };
    *status = cg_serial(op, b, tol, max_iter, xs, iterations);
    std::copy(xs.begin(), xs.end(), x);
  });
}

static int nystrom_out(int64_t n, const ApplyFn& fn, int k, int L, int M, uint64_t seed, double* values,
                       double* vectors) {
  return guarded([&] {
    std::vector<double> v;
    Mat vec;
    nystrom_gaussian_serial(n, fn, k, L, M, seed, v, vec);
    const EigenPairs p = make_eigenpairs(v, vec);  // spectral.cpp:105-127
    std::copy(p.values.begin(), p.values.end(), values);
    std::copy(p.vectors.a.begin(), p.vectors.a.end(), vectors);
  });
}

int orc_nystrom_dense(const double* A, int64_t n, int k, int L, int M, uint64_t seed, double* values, double* vectors) {
  std::vector<double> mat(A, A + n * n);
  ApplyFn fn = [&mat, n](const std::vector<double>& x) {
    std::vector<double> y(static_cast<size_t>(n), 0.0);
    for (int64_t j = 0; j < n; ++j) {
      const double xj = x[j];
      const double* c = mat.data() + j * n;
      for (int64_t i = 0; i < n; ++i) y[i] += c[i] * xj;
    }
    return y;
  };
  return nystrom_out(n, fn, k, L, M, seed, values, vectors);
}

int orc_nystrom_adjacency(void* h, int k, int L, int M, uint64_t seed, double* values, double* vectors) {
  auto* a = static_cast<Adjacency*>(h);
  const int64_t n = a->nodes.rows;
  ApplyFn fn = [a, n](const std::vector<double>& x) { return a->apply_normalized(x.data(), n); };
  return nystrom_out(n, fn, k, L, M, seed, values, vectors);
}

}  // extern "C"
