// cg.hpp -- device conjugate gradients over a Core (cg.cu).
#pragma once

#include "core.cuh"

namespace fgsb {

enum CgSystem { CG_SSL = 0, CG_KRR = 1 };  // (I + beta L_s) x = f  /  (W~ + beta I) x = f
enum CgStatusCode { CG_CONVERGED = 0, CG_MAX_ITERATIONS = 1, CG_INDEFINITE = 2 };  // spectral.hpp:120-124

struct CgOutcome {
  int iterations = 0;
  CgStatusCode status = CG_MAX_ITERATIONS;
};

// spectral.cpp:446-495 on the device; f and x in caller order on the host
CgOutcome cg_solve(Core& c, CgSystem system, double beta, const double* f_host, double tol, int max_iter,
                   double* x_host);

}  // namespace fgsb
