// C++ drop-in smoke/parity program: the reference's own test cases
// (test_nfft.cpp:91-111, test_fastsum.cpp:93-109, test_graphop.cpp:60-73,
// test_spectral.cpp eigen conventions) written against include/fgs/b200.hpp
// exactly as a reference caller would.  Exit code = number of failures.
#include <chrono>
#include <cmath>
#include <complex>
#include <cstdio>
#include <numbers>
#include <random>
#include <string>
#include <utility>
#include <vector>

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

// ---- the reference CLI's solve_pairs, nfft-lanczos / direct branch -------
// Stand-ins for the CLI's own types (tools/commands.cpp:26-37,61-104); the
// body between the markers is commands.cpp:171-188 VERBATIM: the reference's
// call site compiles unchanged against the drop-in header.
namespace refcli {
struct Timer {
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
  double seconds() const { return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count(); }
};
struct Report {
  std::vector<std::pair<std::string, double>> timings, metrics;
  void add_timing(const std::string& name, double s) { timings.emplace_back(name, s); }
  void add_metric(const std::string& name, double v, const std::string&) { metrics.emplace_back(name, v); }
  double metric(const std::string& name) const {
    for (const auto& m : metrics)
      if (m.first == name) return m.second;
    return -1.0;
  }
};
struct CommonOpts {
  std::string method = "nfft-lanczos";
  int k = 3;
  std::uint64_t seed = 1;
  double tol = 1e-10;
};
struct PointCloud {
  MatrixXd coordinates;
};
double lanczos_tol(const CommonOpts& opts) { return opts.tol; }

EigenPairs solve_pairs(const PointCloud& cloud, const KernelSpec& kernel, const FastsumParams& params,
                       const CommonOpts& opts, Report* report) {
  LanczosOptions lopts;
  lopts.tol = lanczos_tol(opts);
  lopts.seed = opts.seed;
  EigenPairs pairs;
  if (opts.method == "nfft-lanczos" || opts.method == "direct") {
    // ---- begin commands.cpp:171-188 (verbatim) ----
    const AdjacencyBackend backend = opts.method == "direct"
                                         ? AdjacencyBackend::Direct
                                         : AdjacencyBackend::Fastsum;
    Timer setup;
    AdjacencyOperator op(cloud.coordinates, kernel, params, backend);
    report->add_timing("setup", setup.seconds());
    Timer solve;
    LanczosInfo info;
    pairs = lanczos_largest(adjacency_handle(op), opts.k, lopts, &info);
    report->add_timing("solve", solve.seconds());
    report->add_metric("lanczos_iterations", info.iterations,
                       "Lanczos steps executed");
    report->add_metric("lanczos_converged", info.converged ? 1.0 : 0.0,
                       "1 if every wanted Ritz pair met the tolerance");
    report->add_metric(
        "max_residual_operator", max_residual(adjacency_handle(op), pairs),
        "max_i ||A v_i - lambda_i v_i||_2 with the operator used for the "
        "solve (approximate for nfft-lanczos)");
    // ---- end commands.cpp:171-188 ----
  }
  return pairs;
}
}  // namespace refcli

// dense symmetric test operator with the given spectrum (test_spectral.cpp
// with_spectrum): Q diag(s) Q^T, Q from Gram-Schmidt on seeded columns
static MatrixXd with_spectrum(const std::vector<double>& s, std::uint64_t seed) {
  const Index n = static_cast<Index>(s.size());
  std::mt19937_64 rng(seed);
  std::normal_distribution<double> g;
  MatrixXd q(n, n);
  for (Index j = 0; j < n; ++j) {
    for (Index i = 0; i < n; ++i) q(i, j) = g(rng);
    for (int pass = 0; pass < 2; ++pass)
      for (Index c = 0; c < j; ++c) {
        double d = 0.0;
        for (Index i = 0; i < n; ++i) d += q(i, c) * q(i, j);
        for (Index i = 0; i < n; ++i) q(i, j) -= d * q(i, c);
      }
    double nr = 0.0;
    for (Index i = 0; i < n; ++i) nr += q(i, j) * q(i, j);
    nr = std::sqrt(nr);
    for (Index i = 0; i < n; ++i) q(i, j) /= nr;
  }
  MatrixXd a(n, n);
  for (Index i = 0; i < n; ++i)
    for (Index j = 0; j < n; ++j) {
      double v = 0.0;
      for (Index c = 0; c < n; ++c) v += q(i, c) * s[static_cast<size_t>(c)] * q(j, c);
      a(i, j) = v;
    }
  return a;
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
  // the reference's own call site: lanczos_largest(adjacency_handle(op), ...)
  // + max_residual(adjacency_handle(op), pairs) (commands.cpp:171-188)
  {
    refcli::PointCloud cloud;
    cloud.coordinates = random_nodes(3000, 3, 77, -0.2, 0.2);
    refcli::CommonOpts opts;
    refcli::Report report;
    EigenPairs pairs = refcli::solve_pairs(cloud, KernelSpec::gaussian(0.35), FastsumParams{32, 4, 4, 0.0, 2.0}, opts,
                                           &report);
    CHECK(pairs.count() == 3 && std::abs(pairs.values(0) - 1.0) <= 1e-8);
    CHECK(report.metric("lanczos_converged") == 1.0 && report.metric("lanczos_iterations") > 3);
    CHECK(report.metric("max_residual_operator") >= 0.0 && report.metric("max_residual_operator") <= 1e-8);
    CHECK(report.timings.size() == 2);
    // the same through the AdjacencyOperator overload: identical
    AdjacencyOperator op(cloud.coordinates, KernelSpec::gaussian(0.35), FastsumParams{32, 4, 4, 0.0, 2.0});
    LanczosOptions lo;
    lo.tol = 1e-10;
    EigenPairs direct = lanczos_largest(op, 3, lo);
    for (int i = 0; i < 3; ++i) CHECK(direct.values(i) == pairs.values(i));
    // laplacian_handle: lambda_L = 1 - lambda_A (spectral.cpp:98-103)
    EigenPairs lp = lanczos_largest(laplacian_handle(op), 2, lo);
    CHECK(lp.count() == 2 && lp.values(0) > 1.0);
    refcli::CommonOpts dopts;
    dopts.method = "direct";
    refcli::Report dreport;
    EigenPairs dp = refcli::solve_pairs(cloud, KernelSpec::gaussian(0.35), FastsumParams{32, 4, 4, 0.0, 2.0}, dopts,
                                        &dreport);
    CHECK(std::abs(dp.values(1) - pairs.values(1)) <= 1e-4);
  }
  // generic operators through dense_handle (test_spectral.cpp:84-140)
  {
    MatrixXd d5(5, 5);
    for (int i = 0; i < 5; ++i) d5(i, i) = 5.0 - i;
    LanczosInfo info;
    EigenPairs p = lanczos_largest(dense_handle(d5), 2, {}, &info);
    CHECK(info.converged);
    CHECK(std::abs(p.values(0) - 5.0) <= 1e-10 * 5.0 && std::abs(p.values(1) - 4.0) <= 1e-10 * 4.0);
    CHECK(std::abs(std::abs(p.vectors(0, 0)) - 1.0) <= 1e-10 && std::abs(std::abs(p.vectors(1, 1)) - 1.0) <= 1e-10);
    CHECK(p.vectors(0, 0) > 0.0 && p.vectors(1, 1) > 0.0);

    MatrixXd swap(2, 2);
    swap(0, 1) = swap(1, 0) = 1.0;
    SymmetricOperatorHandle sw = dense_handle(swap);
    EigenPairs ps = lanczos_largest(sw, 2, {}, &info);
    CHECK(info.converged && info.iterations == 2);
    CHECK(std::abs(ps.values(0) - 1.0) <= 1e-12 && std::abs(ps.values(1) + 1.0) <= 1e-12);
    CHECK(max_residual(sw, ps) <= 1e-12);

    std::vector<double> spec(30);
    for (int i = 0; i < 30; ++i) spec[static_cast<size_t>(i)] = 10.0 / (1.0 + i);
    SymmetricOperatorHandle syn = dense_handle(with_spectrum(spec, 5));
    EigenPairs pz = lanczos_largest(syn, 6);
    double gram = 0.0;
    for (int a = 0; a < 6; ++a)
      for (int b = 0; b < 6; ++b) {
        double d = 0.0;
        for (int i = 0; i < 30; ++i) d += pz.vectors(i, a) * pz.vectors(i, b);
        gram = std::max(gram, std::abs(d - (a == b ? 1.0 : 0.0)));
      }
    CHECK(gram <= 1e-8);
    CHECK(max_residual(syn, pz) <= 1e-9);
    for (int i = 0; i < 6; ++i) CHECK(std::abs(pz.values(i) - spec[static_cast<size_t>(i)]) <= 1e-10 * spec[static_cast<size_t>(i)]);

    // shift invariance (test_spectral.cpp:125-140)
    std::vector<double> s25(25);
    for (int i = 0; i < 25; ++i) s25[static_cast<size_t>(i)] = 5.0 * std::pow(0.8, i);
    MatrixXd a = with_spectrum(s25, 9), shifted = a;
    for (int i = 0; i < 25; ++i) shifted(i, i) += 2.75;
    LanczosOptions o31;
    o31.seed = 31;
    EigenPairs base = lanczos_largest(dense_handle(a), 4, o31);
    EigenPairs moved = lanczos_largest(dense_handle(shifted), 4, o31);
    for (int i = 0; i < 4; ++i) {
      CHECK(std::abs((moved.values(i) - base.values(i)) - 2.75) <= 1e-10 * 2.75);
      double dn = 0.0;
      for (int r = 0; r < 25; ++r) dn += std::pow(moved.vectors(r, i) - base.vectors(r, i), 2);
      CHECK(std::sqrt(dn) <= 1e-6);
    }
  }
  std::printf("dropin_test: %d failure(s)\n", failures);
  return failures;
}
