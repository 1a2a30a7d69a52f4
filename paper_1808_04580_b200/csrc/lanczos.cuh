// lanczos.cuh -- device Lanczos (spectral.cpp:141-256) over a Core.
#pragma once

#include <cstdint>
#include <vector>

namespace fgsb {

class Core;

struct LanczosResult {
  std::vector<double> values;         // descending Ritz values (count = min(k, m))
  std::vector<double> local_vectors;  // n_local x count, internal order, column-major
  int iterations = 0;
  bool converged = false;
  double apply_ms = 0.0, reorth_ms = 0.0, loop_ms = 0.0;  // device apply / reorth, host wall of the loop
};

LanczosResult lanczos_device(Core& c, int which, int k, int max_iter, double tol, uint64_t seed, bool want_vectors);
void tridiagonal_eigen(int m, std::vector<double>& diag, const std::vector<double>& offd, std::vector<double>& z);

}  // namespace fgsb
