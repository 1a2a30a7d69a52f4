// C++ drop-in smoke/parity program: the reference's own test cases
// (test_nfft.cpp:91-111, test_fastsum.cpp:93-109, test_graphop.cpp:60-73,
// test_spectral.cpp eigen conventions) written against include/fgs/b200.hpp
// exactly as a reference caller would.  Exit code = number of failures.
#include <cmath>
#include <complex>
#include <cstdio>
#include <numbers>
#include <random>

#include "fgs/b200.hpp"

using namespace fgs;

static int failures = 0;
#define CHECK(cond)                                                   \
  do {                                                                \
    if (!(cond)) {                                                    \
      ++failures;                                                     \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);     \
    }                                                                 \
  } while (0)

static MatrixXd random_nodes(int n, int d, std::uint64_t seed, double lo = -0.5, double hi = 0.5) {
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> dist(lo, hi);
  MatrixXd nodes(n, d);
  for (int j = 0; j < n; ++j)
    for (int t = 0; t < d; ++t) {
      double v = dist(rng);
      while (v >= 0.5) v = dist(rng);
      nodes(j, t) = v;
    }
  return nodes;
}

int main() {
  // NfftPlan vs the direct NDFT at m = 8 (test_nfft.cpp:91-111)
  for (int d : {1, 2, 3}) {
    const int N = 8, n = d == 3 ? 64 : 200;
    MatrixXd nodes = random_nodes(n, d, 100 * d + N);
    NfftPlan plan(d, N, 8, nodes);
    std::mt19937_64 rng(7);
    std::normal_distribution<double> g;
    VectorXcd fhat(static_cast<Index>(plan.coefficient_count()));
    double l1 = 0.0;
    for (Index i = 0; i < fhat.size(); ++i) {
      fhat(i) = {g(rng), g(rng)};
      l1 += std::abs(fhat(i));
    }
    VectorXcd fast = plan.forward(fhat);
    double worst = 0.0;
    for (int j = 0; j < n; ++j) {
      std::complex<double> acc = 0.0;
      for (Index f = 0; f < fhat.size(); ++f) {
        double phase = 0.0;
        Index rest = f;
        for (int t = d - 1; t >= 0; --t) {
          phase += static_cast<double>(rest % N - N / 2) * nodes(j, t);
          rest /= N;
        }
        acc += fhat(f) * std::polar(1.0, 2.0 * std::numbers::pi * phase);
      }
      worst = std::max(worst, std::abs(fast(j) - acc));
    }
    CHECK(worst <= 1e-12 * l1);
  }
  // FastsumPlan vs the quadratic-cost sum (test_fastsum.cpp:93-109)
  {
    const int n = 220;
    MatrixXd nodes = random_nodes(n, 3, 51, -2.0, 2.0);
    FastsumParams tight{64, 8, 8, 8.0 / 64.0, 2.0};
    FastsumPlan plan(nodes, KernelSpec::gaussian(1.5), tight);
    VectorXd x(n);
    std::mt19937_64 rng(23);
    std::normal_distribution<double> g;
    double l1 = 0.0;
    for (int i = 0; i < n; ++i) {
      x(i) = g(rng);
      l1 += std::abs(x(i));
    }
    VectorXd fast = plan.apply(x);
    double worst = 0.0;
    for (int j = 0; j < n; ++j) {
      double acc = 0.0;
      for (int i = 0; i < n; ++i) {
        double s = 0.0;
        for (int t = 0; t < 3; ++t) s += (nodes(j, t) - nodes(i, t)) * (nodes(j, t) - nodes(i, t));
        acc += std::exp(-s / (1.5 * 1.5)) * x(i);
      }
      worst = std::max(worst, std::abs(fast(j) - acc));
    }
    CHECK(worst <= l1 * (10.0 * plan.kernel_error_estimate(300, 11) + 1e-10));
    CHECK(plan.scaling() < 1.0);
  }
  // swap adjacency (test_graphop.cpp:60-73) + Lanczos conventions
  {
    MatrixXd nodes(2, 2);
    nodes(1, 0) = 0.6;
    nodes(1, 1) = 0.8;
    AdjacencyOperator op(nodes, KernelSpec::gaussian(1.0), FastsumParams::preset(3, 0.125));
    CHECK(std::abs(op.degrees()(0) - std::exp(-1.0)) <= 2e-9);
    VectorXd x(2);
    x(0) = 1.0;
    VectorXd y = op.apply_normalized(x);
    CHECK(std::abs(y(0)) <= 1e-9 && std::abs(y(1) - 1.0) <= 2e-9);
    LanczosInfo info;
    EigenPairs p = lanczos_largest(op, 2, {}, &info);
    CHECK(info.converged && info.iterations == 2);
    CHECK(std::abs(p.values(0) - 1.0) <= 1e-8 && std::abs(p.values(1) + 1.0) <= 1e-8);
    EigenPairs lap = adjacency_to_laplacian(p);
    CHECK(std::abs(lap.values(0) - 2.0) <= 1e-8 && std::abs(lap.values(1)) <= 1e-8);
  }
  // typed errors (test_nfft.cpp:193-208, test_graphop.cpp:236-240)
  {
    bool threw = false;
    try {
      NfftPlan bad(2, 7, 4, random_nodes(4, 2, 1));
    } catch (const ParameterError&) {
      threw = true;
    }
    CHECK(threw);
    threw = false;
    try {
      AdjacencyOperator one(MatrixXd(1, 2), KernelSpec::gaussian(1.0), FastsumParams::preset(1));
    } catch (const ShapeError&) {
      threw = true;
    }
    CHECK(threw);
  }
  // Direct backend, residual norms, clustering, SSL and ridge (graphop.hpp:19-22,
  // spectral.cpp:258-275, learn.cpp:17-167, 364-445)
  {
    MatrixXd pts(400, 2);
    for (int i = 0; i < 400; ++i) {
      const double cx = (i < 200) ? -0.15 : 0.15;
      pts(i, 0) = cx + 0.01 * std::sin(0.37 * i);
      pts(i, 1) = 0.01 * std::cos(0.91 * i);
    }
    const KernelSpec k = KernelSpec::gaussian(0.05);
    AdjacencyOperator fast(pts, k, FastsumParams::preset(3));
    AdjacencyOperator exact(pts, k, FastsumParams::preset(3), AdjacencyBackend::Direct);
    CHECK(exact.backend() == AdjacencyBackend::Direct);
    EigenPairs pf = lanczos_largest(fast, 2);
    EigenPairs pe = lanczos_largest(exact, 2);
    CHECK(std::abs(pf.values(0) - pe.values(0)) <= 1e-8 && std::abs(pf.values(1) - pe.values(1)) <= 1e-6);
    CHECK(max_residual(fast, pf) <= 1e-9);
    CHECK(max_residual(exact, pf) <= 1e-5);
    std::vector<int> labels = spectral_cluster(pf, 2);
    std::vector<int> truth(400);
    for (int i = 0; i < 400; ++i) truth[static_cast<size_t>(i)] = i < 200 ? 0 : 1;
    CHECK(misclassification_rate_permuted(labels, truth) == 0.0);
    KMeansResult km = kmeans(pts, 2);
    CHECK(misclassification_rate_permuted(km.labels, truth) == 0.0 && km.centroids.rows() == 2);
    VectorXd f(400);
    for (int i = 0; i < 400; ++i) f(i) = (i % 3) - 1.0;
    CgResult ssl = kernel_ssl_solve(fast, f, 10.0, 1e-10, 500);
    CHECK(ssl.converged());
    VectorXd lx = fast.apply_sym_laplacian(ssl.x);
    double rn = 0.0, fn = 0.0;
    for (int i = 0; i < 400; ++i) {
      const double r = f(i) - (ssl.x(i) + 10.0 * lx(i));
      rn += r * r;
      fn += f(i) * f(i);
    }
    CHECK(std::sqrt(rn) <= 1e-10 * std::sqrt(fn));
    RidgeModel rm = krr_fit(pts, k, 1e-2, f, FastsumParams::preset(3, 0.125), 1e-10, 500);
    VectorXd pred = krr_predict(rm, pts);
    CHECK(pred.size() == 400 && std::isfinite(pred(7)));
  }
  std::printf("dropin_test: %d failure(s)\n", failures);
  return failures;
}
