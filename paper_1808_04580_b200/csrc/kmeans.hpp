// kmeans.hpp -- device k-means / spectral clustering driver (kmeans.cu).
#pragma once

#include <cstdint>

namespace fgsb {

// learn.cpp:140-167.  points column-major n x dim (host, or device when
// on_device); normalize_rows = spectral_cluster's unit-row step.  Outputs on
// the host: labels[n], centroids k x dim column-major (nullable), wcss
// (nullable).
void kmeans_run(const double* points, bool on_device, int64_t n, int dim, int k, int restarts, int max_iter,
                uint64_t seed, int device, bool normalize_rows, int* labels_out, double* centroids_out,
                double* wcss_out);

}  // namespace fgsb
