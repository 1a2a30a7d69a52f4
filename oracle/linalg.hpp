// ============================================================================
// linalg.hpp -- TEST INFRASTRUCTURE ONLY.
//
// The self-written stand-ins for the reference's two third-party arithmetic
// libraries, shared by the oracle restatement (fgs_oracle.cpp) and by the
// shim headers the reference's own sources are compiled against
// (oracle/shim/fftw3.h, oracle/shim/Eigen/*, build_ref.sh -> oracle/_ref):
//   * FFTW3 (fftw_plan_dft / fftw_execute_dft, nfft.cpp:379-384,409,423;
//     kernels.cpp:296-307) -> fft_nd(): radix-2 for powers of two, direct DFT
//     otherwise, FFTW's sign convention, unnormalised;
//   * Eigen3 SelfAdjointEigenSolver (computeFromTridiagonal,
//     spectral.cpp:174-179; dense, spectral.cpp:288,324,412,435,565) ->
//     tridiag_eig() / dense_sym_eig(); HouseholderQR (spectral.cpp:315,403,
//     428) -> householder_qr().
// Both sides calling the same code makes the oracle restatement and the
// reference binary agree bit for bit wherever the reference's own code does
// the same IEEE operations as the restatement.
// ============================================================================
#pragma once

#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdint>
#include <limits>
#include <numbers>
#include <stdexcept>
#include <thread>
#include <vector>

namespace orc_linalg {

using cd = std::complex<double>;
constexpr double kPi = std::numbers::pi;
constexpr double kEps = std::numeric_limits<double>::epsilon();

struct NotConverged : std::runtime_error {
  using std::runtime_error::runtime_error;
};

inline size_t ipow(size_t base, int e) {
  size_t r = 1;
  while (e-- > 0) r *= base;
  return r;
}

// Column-major dense matrix (Eigen's default storage, the layout of `nodes`).
struct Mat {
  int64_t rows = 0, cols = 0;
  std::vector<double> a;
  Mat() = default;
  Mat(int64_t r, int64_t c) : rows(r), cols(c), a(static_cast<size_t>(r * c), 0.0) {}
  double& operator()(int64_t i, int64_t j) { return a[static_cast<size_t>(j * rows + i)]; }
  double operator()(int64_t i, int64_t j) const { return a[static_cast<size_t>(j * rows + i)]; }
  double* col(int64_t j) { return a.data() + j * rows; }
  const double* col(int64_t j) const { return a.data() + j * rows; }
};

// ---------------------------------------------------------------------------
// FFT replacing FFTW (fftw_plan_dft with FFTW_FORWARD / FFTW_BACKWARD).
// ---------------------------------------------------------------------------
inline void fft_line(cd* x, int n, int sign) {
  if (n <= 1) return;
  if ((n & (n - 1)) == 0) {
    // iterative radix-2, bit-reversal then butterflies; twiddles from
    // direct cos/sin evaluation (no recurrence drift)
    for (int i = 1, j = 0; i < n; ++i) {
      int bit = n >> 1;
      for (; j & bit; bit >>= 1) j ^= bit;
      j ^= bit;
      if (i < j) std::swap(x[i], x[j]);
    }
    std::vector<cd> tw(static_cast<size_t>(n / 2));
    for (int k = 0; k < n / 2; ++k) {
      double ang = 2.0 * kPi * k / n;
      tw[static_cast<size_t>(k)] = cd(std::cos(ang), sign * std::sin(ang));
    }
    for (int len = 2; len <= n; len <<= 1) {
      int step = n / len;
      for (int i = 0; i < n; i += len)
        for (int k = 0; k < len / 2; ++k) {
          cd w = tw[static_cast<size_t>(k * step)];
          cd u = x[i + k], v = x[i + k + len / 2] * w;
          x[i + k] = u + v;
          x[i + k + len / 2] = u - v;
        }
    }
  } else {
    std::vector<cd> out(static_cast<size_t>(n));
    for (int k = 0; k < n; ++k) {
      cd acc = 0.0;
      for (int j = 0; j < n; ++j) {
        long long jk = (static_cast<long long>(j) * k) % n;
        double ang = 2.0 * kPi * static_cast<double>(jk) / n;
        acc += x[j] * cd(std::cos(ang), sign * std::sin(ang));
      }
      out[static_cast<size_t>(k)] = acc;
    }
    std::copy(out.begin(), out.end(), x);
  }
}

// d-dimensional transform of a row-major M^d array (dimension 0 slowest),
// the layout FFTW's fftw_plan_dft(d, {M,M,M}, ...) uses.
inline void fft_nd(cd* data, int d, int M, int sign, int threads = 1) {
  // every line is transformed by the same serial code, so splitting the
  // lines over threads leaves the result bit for bit unchanged
  size_t total = ipow(static_cast<size_t>(M), d);
  for (int t = 0; t < d; ++t) {
    const size_t stride = ipow(static_cast<size_t>(M), d - 1 - t);
    const size_t outer = total / (stride * M);
    const size_t lines = outer * stride;
    auto run = [&](size_t lo, size_t hi) {
      std::vector<cd> line(static_cast<size_t>(M));
      for (size_t l = lo; l < hi; ++l) {
        const size_t o = l / stride, s = l % stride;
        cd* base = data + o * stride * M + s;
        for (int k = 0; k < M; ++k) line[static_cast<size_t>(k)] = base[k * stride];
        fft_line(line.data(), M, sign);
        for (int k = 0; k < M; ++k) base[k * stride] = line[static_cast<size_t>(k)];
      }
    };
    const int T = static_cast<int>(std::min<size_t>(std::max(threads, 1), lines / 64 + 1));
    if (T <= 1) {
      run(0, lines);
    } else {
      std::vector<std::thread> pool;
      for (int q = 0; q < T; ++q) pool.emplace_back(run, lines * q / T, lines * (q + 1) / T);
      for (auto& th : pool) th.join();
    }
  }
}

// ---------------------------------------------------------------------------
// Symmetric tridiagonal eigensolver (replaces Eigen computeFromTridiagonal):
// implicit QL with Wilkinson shifts.  On return `diag` holds the eigenvalues
// ascending and z (m x m, column-major) the orthonormal eigenvectors.
// ---------------------------------------------------------------------------
inline void tridiag_eig(int m, std::vector<double>& diag, std::vector<double> sub, std::vector<double>& z) {
  z.assign(static_cast<size_t>(m) * m, 0.0);
  for (int i = 0; i < m; ++i) z[static_cast<size_t>(i) * m + i] = 1.0;
  std::vector<double> e(static_cast<size_t>(m), 0.0);
  for (int i = 0; i + 1 < m; ++i) e[i] = sub[i];
  auto Z = [&](int r, int c) -> double& { return z[static_cast<size_t>(c) * m + r]; };
  for (int l = 0; l < m; ++l) {
    int iter = 0;
    while (true) {
      int mm = l;
      for (; mm < m - 1; ++mm) {
        double dd = std::abs(diag[mm]) + std::abs(diag[mm + 1]);
        if (std::abs(e[mm]) <= kEps * dd) break;
      }
      if (mm == l) break;
      if (++iter > 60) throw NotConverged("tridiagonal eigensolver did not converge");
      double g = (diag[l + 1] - diag[l]) / (2.0 * e[l]);
      double r = std::hypot(g, 1.0);
      g = diag[mm] - diag[l] + e[l] / (g + (g >= 0.0 ? std::abs(r) : -std::abs(r)));
      double s = 1.0, c = 1.0, p = 0.0;
      int i = mm - 1;
      bool underflow = false;
      for (; i >= l; --i) {
        double f = s * e[i];
        double bb = c * e[i];
        r = std::hypot(f, g);
        e[i + 1] = r;
        if (r == 0.0) {
          diag[i + 1] -= p;
          e[mm] = 0.0;
          underflow = true;
          break;
        }
        s = f / r;
        c = g / r;
        g = diag[i + 1] - p;
        r = (diag[i] - g) * s + 2.0 * c * bb;
        p = s * r;
        diag[i + 1] = g + p;
        g = c * r - bb;
        for (int k = 0; k < m; ++k) {
          double zf = Z(k, i + 1);
          Z(k, i + 1) = s * Z(k, i) + c * zf;
          Z(k, i) = c * Z(k, i) - s * zf;
        }
      }
      if (underflow) continue;
      diag[l] -= p;
      e[l] = g;
      e[mm] = 0.0;
    }
  }
  // sort ascending (selection sort keeps the column swaps explicit)
  for (int i = 0; i < m - 1; ++i) {
    int k = i;
    for (int j = i + 1; j < m; ++j)
      if (diag[j] < diag[k]) k = j;
    if (k != i) {
      std::swap(diag[i], diag[k]);
      for (int r = 0; r < m; ++r) std::swap(Z(r, i), Z(r, k));
    }
  }
}

// thin QR of the r x c column-major A: Q (r x c) and R (c x c upper)
inline void householder_qr(const Mat& A, Mat& Q, Mat& R) {
  const int64_t r = A.rows, c = A.cols;
  Mat W = A;
  std::vector<std::vector<double>> vs;
  std::vector<double> taus;
  const int64_t steps = std::min(r, c);
  for (int64_t j = 0; j < steps; ++j) {
    double sq = 0.0;
    for (int64_t i = j + 1; i < r; ++i) sq += W(i, j) * W(i, j);
    const double c0 = W(j, j);
    std::vector<double> v(static_cast<size_t>(r - j), 0.0);
    double tau = 0.0, beta = c0;
    if (sq > 0.0) {
      beta = std::sqrt(c0 * c0 + sq);
      if (c0 >= 0.0) beta = -beta;
      v[0] = 1.0;
      for (int64_t i = j + 1; i < r; ++i) v[static_cast<size_t>(i - j)] = W(i, j) / (c0 - beta);
      tau = (beta - c0) / beta;
    } else {
      v[0] = 1.0;
    }
    W(j, j) = beta;
    for (int64_t i = j + 1; i < r; ++i) W(i, j) = 0.0;
    for (int64_t k = j + 1; k < c; ++k) {  // apply H = I - tau v v^T to the trailing columns
      double dot = 0.0;
      for (int64_t i = j; i < r; ++i) dot += v[static_cast<size_t>(i - j)] * W(i, k);
      dot *= tau;
      for (int64_t i = j; i < r; ++i) W(i, k) -= dot * v[static_cast<size_t>(i - j)];
    }
    vs.push_back(std::move(v));
    taus.push_back(tau);
  }
  R = Mat(c, c);
  for (int64_t k = 0; k < c; ++k)
    for (int64_t i = 0; i <= std::min(k, r - 1); ++i) R(i, k) = W(i, k);
  Q = Mat(r, c);  // Q = H_0 ... H_{s-1} [I; 0]
  for (int64_t k = 0; k < std::min(r, c); ++k) Q(k, k) = 1.0;
  for (int64_t j = steps - 1; j >= 0; --j) {
    const std::vector<double>& v = vs[static_cast<size_t>(j)];
    const double tau = taus[static_cast<size_t>(j)];
    for (int64_t k = 0; k < c; ++k) {
      double dot = 0.0;
      for (int64_t i = j; i < r; ++i) dot += v[static_cast<size_t>(i - j)] * Q(i, k);
      dot *= tau;
      for (int64_t i = j; i < r; ++i) Q(i, k) -= dot * v[static_cast<size_t>(i - j)];
    }
  }
}

// symmetric s x s: ascending eigenvalues, eigenvectors as columns
inline void dense_sym_eig(const Mat& A, std::vector<double>& vals, Mat& vecs) {
  const int64_t s = A.rows;
  Mat T = A, Qt(s, s);
  for (int64_t i = 0; i < s; ++i) Qt(i, i) = 1.0;
  // Householder tridiagonalisation: T <- H T H, Qt <- Qt H
  for (int64_t j = 0; j + 2 < s; ++j) {
    double sq = 0.0;
    for (int64_t i = j + 2; i < s; ++i) sq += T(i, j) * T(i, j);
    if (sq == 0.0) continue;
    const double c0 = T(j + 1, j);
    double beta = std::sqrt(c0 * c0 + sq);
    if (c0 >= 0.0) beta = -beta;
    std::vector<double> v(static_cast<size_t>(s), 0.0);
    v[static_cast<size_t>(j + 1)] = 1.0;
    for (int64_t i = j + 2; i < s; ++i) v[static_cast<size_t>(i)] = T(i, j) / (c0 - beta);
    const double tau = (beta - c0) / beta;
    for (int64_t k = 0; k < s; ++k) {  // T <- H T
      double dot = 0.0;
      for (int64_t i = j + 1; i < s; ++i) dot += v[static_cast<size_t>(i)] * T(i, k);
      dot *= tau;
      for (int64_t i = j + 1; i < s; ++i) T(i, k) -= dot * v[static_cast<size_t>(i)];
    }
    for (int64_t k = 0; k < s; ++k) {  // T <- T H, Qt <- Qt H
      double dot = 0.0, dq = 0.0;
      for (int64_t i = j + 1; i < s; ++i) {
        dot += T(k, i) * v[static_cast<size_t>(i)];
        dq += Qt(k, i) * v[static_cast<size_t>(i)];
      }
      dot *= tau;
      dq *= tau;
      for (int64_t i = j + 1; i < s; ++i) {
        T(k, i) -= dot * v[static_cast<size_t>(i)];
        Qt(k, i) -= dq * v[static_cast<size_t>(i)];
      }
    }
  }
  std::vector<double> diag(static_cast<size_t>(s)), sub(static_cast<size_t>(std::max<int64_t>(s - 1, 0)));
  for (int64_t i = 0; i < s; ++i) diag[static_cast<size_t>(i)] = T(i, i);
  for (int64_t i = 0; i + 1 < s; ++i) sub[static_cast<size_t>(i)] = T(i + 1, i);
  std::vector<double> z;
  tridiag_eig(static_cast<int>(s), diag, sub, z);
  vals = diag;
  vecs = Mat(s, s);
  for (int64_t k = 0; k < s; ++k)
    for (int64_t i = 0; i < s; ++i) {
      double acc = 0.0;
      for (int64_t t = 0; t < s; ++t) acc += Qt(i, t) * z[static_cast<size_t>(k * s + t)];
      vecs(i, k) = acc;
    }
}


}  // namespace orc_linalg
