// nystrom.hpp -- sketch-based Nystrom eigenpairs over a Core (nystrom.cu).
#pragma once

#include <cstdint>
#include <vector>

#include "core.cuh"

namespace fgsb {

// spectral.cpp:384-444 on the device: descending values (returned) and the
// sign-normalised caller-order vectors (n x k column-major) to vectors_host
std::vector<double> nystrom_gaussian(Core& c, int k, int L, int M, uint64_t seed, double* vectors_host);
// symmetric eigenproblem (ascending, Eigen's convention), host Jacobi
void symmetric_eigen(int s, std::vector<double> a, std::vector<double>& vals, std::vector<double>& vecs);

}  // namespace fgsb
