// workload.cpp -- seeded synthetic stand-ins for the five BASELINE.json
// configurations (the paper's spiral / crescent / photo datasets are not in
// this container).  Compiled into the product library AND
// into oracle/liboracle.so, so bench.py's reference arm generates the same
// arrays without loading the product.  std::mt19937_64 + libstdc++ distributions,
// as the reference's own generators use (dataset.cpp, spectral.cpp:152-156).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <random>
#include <string>
#include <vector>

#include "fgs_b200.h"

namespace {

thread_local std::string g_werr;

struct Info {
  int64_t n;
  int d;
  double sigma;
  int N, m, p, k;
};

bool info_of(int config, Info* out) {
  switch (config) {
    case 1: *out = {20000, 3, 0.35, 32, 4, 4, 10}; return true;
    case 2: *out = {100000, 2, 0.05, 64, 6, 6, 10}; return true;
    case 3: *out = {480000, 3, 90.0, 32, 4, 4, 4}; return true;
    case 4: *out = {2000000, 3, 0.4, 64, 6, 6, 20}; return true;
    case 5: *out = {10000000, 3, 0.3, 64, 8, 8, 16}; return true;
    default: return false;
  }
}

// direction ~ normalised N(0, I), radius = R U^(1/d): uniform in the d-ball
void ball(std::mt19937_64& rng, int d, double R, double* v) {
  std::normal_distribution<double> g;
  std::uniform_real_distribution<double> u(0.0, 1.0);
  double s = 0.0;
  for (int t = 0; t < d; ++t) {
    v[t] = g(rng);
    s += v[t] * v[t];
  }
  const double len = std::sqrt(s);
  const double r = R * std::pow(u(rng), 1.0 / d);
  for (int t = 0; t < d; ++t) v[t] = len > 0.0 ? v[t] * (r / len) : 0.0;
}

}  // namespace

extern "C" {

fgs_status fgs_workload_info(int config, int64_t* n, int* d, double* sigma, int* N, int* m, int* p, int* k) {
  Info i;
  if (!info_of(config, &i)) {
    g_werr = "config must be 1..5";
    return FGS_EPARAM;
  }
  if (n) *n = i.n;
  if (d) *d = i.d;
  if (sigma) *sigma = i.sigma;
  if (N) *N = i.N;
  if (m) *m = i.m;
  if (p) *p = i.p;
  if (k) *k = i.k;
  return FGS_OK;
}

fgs_status fgs_workload_generate(int config, uint64_t seed, double* X) {
  return fgs_workload_generate_n(config, seed, 0, X);
}

fgs_status fgs_workload_generate_n(int config, uint64_t seed, int64_t n_points, double* X) {
  Info in;
  if (!info_of(config, &in) || !X || n_points < 0) return FGS_EPARAM;
  if (config == 3 && n_points != 0 && n_points != in.n) return FGS_EPARAM;  // the image has fixed size
  const int64_t n = n_points > 0 ? n_points : in.n;
  const int d = in.d;
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> U(0.0, 1.0);
  std::normal_distribution<double> G(0.0, 1.0);
  double v[3];
  switch (config) {
    case 1:  // uniform in the ball of radius 0.2
      for (int64_t j = 0; j < n; ++j) {
        ball(rng, 3, 0.2, v);
        for (int t = 0; t < 3; ++t) X[t * n + j] = v[t];
      }
      break;
    case 2: {  // disk r<=1 + annulus sector r in [1.5,2.5], theta in [0,pi]; N(0,0.05^2) jitter; x0.1
      const double pi = 3.141592653589793;
      for (int64_t j = 0; j < n; ++j) {
        double r, th;
        if (j < n / 2) {
          r = std::sqrt(U(rng));
          th = 2.0 * pi * U(rng);
        } else {
          r = std::sqrt(1.5 * 1.5 + U(rng) * (2.5 * 2.5 - 1.5 * 1.5));
          th = pi * U(rng);
        }
        double x = r * std::cos(th) + 0.05 * G(rng);
        double y = r * std::sin(th) + 0.05 * G(rng);
        X[j] = 0.1 * x;
        X[n + j] = 0.1 * y;
      }
      break;
    }
    case 3: {  // 800x600 Voronoi image, 8 sites, colours U[0,255]^3, N(0,5^2) noise, clip, uint8
      const int W = 800, H = 600, S = 8;
      double sx[S], sy[S], col[S][3];
      for (int s = 0; s < S; ++s) {
        sx[s] = U(rng) * W;
        sy[s] = U(rng) * H;
        for (int c = 0; c < 3; ++c) col[s][c] = 255.0 * U(rng);
      }
      for (int64_t j = 0; j < n; ++j) {
        const int px = static_cast<int>(j % W), py = static_cast<int>(j / W);
        int best = 0;
        double bd = 1e300;
        for (int s = 0; s < S; ++s) {
          const double dx = px + 0.5 - sx[s], dy = py + 0.5 - sy[s];
          const double dd = dx * dx + dy * dy;
          if (dd < bd) {
            bd = dd;
            best = s;
          }
        }
        for (int c = 0; c < 3; ++c) {
          double val = col[best][c] + 5.0 * G(rng);
          val = std::min(255.0, std::max(0.0, val));
          X[c * n + j] = std::nearbyint(val);  // image_to_nodes reads uint8 (dataset.cpp:368-382)
        }
      }
      break;
    }
    case 4: {  // 5-component isotropic GMM, means U[-1,1]^3, std 0.15; rescaled to max norm 0.25
      double mu[5][3];
      for (int c = 0; c < 5; ++c)
        for (int t = 0; t < 3; ++t) mu[c][t] = -1.0 + 2.0 * U(rng);
      std::uniform_int_distribution<int> comp(0, 4);
      double maxn = 0.0;
      for (int64_t j = 0; j < n; ++j) {
        const int c = comp(rng);
        double s = 0.0;
        for (int t = 0; t < 3; ++t) {
          const double x = mu[c][t] + 0.15 * G(rng);
          X[t * n + j] = x;
          s += x * x;
        }
        maxn = std::max(maxn, std::sqrt(s));
      }
      const double f = 0.25 / maxn;
      for (int64_t i = 0; i < 3 * n; ++i) X[i] *= f;
      break;
    }
    case 5:  // uniform in the ball of radius 0.25
      for (int64_t j = 0; j < n; ++j) {
        ball(rng, 3, 0.25, v);
        for (int t = 0; t < 3; ++t) X[t * n + j] = v[t];
      }
      break;
  }
  (void)d;
  return FGS_OK;
}

fgs_status fgs_workload_vectors(int64_t n, int nvec, uint64_t seed, double* out) {
  if (!out || n < 0 || nvec < 0) return FGS_EPARAM;
  std::mt19937_64 rng(seed);
  std::normal_distribution<double> G(0.0, 1.0);
  for (int64_t i = 0; i < n * nvec; ++i) out[i] = G(rng);
  return FGS_OK;
}

}  // extern "C"
