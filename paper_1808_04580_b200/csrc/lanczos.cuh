// lanczos.cuh -- device Lanczos (spectral.cpp:141-256) over a Core.
#pragma once

#include <cstdint>
#include <vector>

#include "core.cuh"

namespace fgsb {

struct LanczosResult {
  std::vector<double> values;         // descending Ritz values (count = min(k, m))
  DBuf<double> vectors_dev;  // n_local x count Ritz vectors on the device, internal order
  int iterations = 0;
  bool converged = false;
  double apply_ms = 0.0, reorth_ms = 0.0, loop_ms = 0.0;  // device apply / reorth, host wall of the loop
};

LanczosResult lanczos_device(Core& c, int which, int k, int max_iter, double tol, uint64_t seed, bool want_vectors);
// caller-order, sign-normalised (make_eigenpairs) Ritz vectors, columns in
// `order`, copied to host_out (n x order.size(), column-major)
void lanczos_finish_vectors(Core& c, LanczosResult& r, const std::vector<int>& order, double* host_out);
void tridiagonal_eigen(int m, std::vector<double>& diag, const std::vector<double>& offd, std::vector<double>& z);
// lanczos_largest over a host-callback operator (SymmetricOperatorHandle)
using OperatorApply = int (*)(void* ctx, const double* x, double* y, int64_t n);
void lanczos_operator(int64_t n, OperatorApply apply, void* ctx, int device, int k, int max_iter, double tol,
                      uint64_t seed, double* values, double* vectors, int* count, int* iterations, int* converged);

}  // namespace fgsb
