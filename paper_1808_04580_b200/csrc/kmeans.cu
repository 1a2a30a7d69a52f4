// kmeans.cu -- k-means++ / Lloyd k-means and spectral clustering on the GPU
// (learn.cpp:17-167: nearest_centroid, plus_plus_init, lloyd_run, kmeans,
// spectral_cluster).
//
// Split: every O(n k dim) pass runs on the device; the random stream stays
// on the host so it is consumed exactly as the reference consumes it
// (std::mt19937_64(seed) shared across restarts, uniform_int_distribution
// <Eigen::Index> for the first centre, uniform_real_distribution(0,1) per
// further centre, the all-zero-distance fallback draw).  Arithmetic mirrors
// the reference's scalar order: squared distances are left-to-right sums of
// squares without FMA contraction; centroid sums run per cluster over points
// in increasing index order within fixed chunks, and the chunk partials are
// then added in chunk order (so a centroid can differ from the serial sum by
// rounding only); ties go to the lowest cluster / first point exactly as the
// reference's strict comparisons.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <limits>
#include <random>
#include <vector>

#include "common.cuh"
#include "core.cuh"
#include "kmeans.hpp"

namespace fgsb {
namespace {

constexpr int kChunk = 256;  // points per serial chunk (sums / scans)

inline int cdiv(int64_t a, int64_t b) { return static_cast<int>((a + b - 1) / b); }

__device__ __forceinline__ double sqdist(const double* pts, int64_t n, int64_t i, int dim, const double* cen, int k,
                                         int c) {
  double s = 0.0;
  for (int t = 0; t < dim; ++t) {
    const double df = __dsub_rn(pts[t * n + i], cen[t * k + c]);
    s = __dadd_rn(s, __dmul_rn(df, df));
  }
  return s;
}

// d2[i] = |p_i - c|^2 (mode 0) or min(d2[i], |p_i - c|^2) (mode 1)
__global__ void km_dist_kernel(const double* pts, int64_t n, int dim, const double* cen, int k, int c, double* d2,
                               int mode) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  const double v = sqdist(pts, n, i, dim, cen, k, c);
  d2[i] = mode == 0 ? v : fmin(d2[i], v);
}

// d2[i] = |p_i - c_{label_i}|^2
__global__ void km_own_dist_kernel(const double* pts, int64_t n, int dim, const double* cen, int k, const int* labels,
                                   double* d2) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  d2[i] = sqdist(pts, n, i, dim, cen, k, labels[i]);
}

// serial sum of each chunk
__global__ void km_chunk_sum_kernel(const double* v, int64_t n, double* out, int nchunks) {
  const int ch = blockIdx.x * blockDim.x + threadIdx.x;
  if (ch >= nchunks) return;
  const int64_t lo = static_cast<int64_t>(ch) * kChunk, hi = min(n, lo + kChunk);
  double s = 0.0;
  for (int64_t i = lo; i < hi; ++i) s += v[i];
  out[ch] = s;
}

// total = serial sum of the chunk sums (one thread)
__global__ void km_total_kernel(const double* chunk, int nchunks, double* total) {
  double s = 0.0;
  for (int c = 0; c < nchunks; ++c) s += chunk[c];
  *total = s;
}

// first i with running sum >= target (learn.cpp:47-55); n - 1 if none
__global__ void km_pick_kernel(const double* v, int64_t n, const double* chunk, int nchunks, double target,
                               long long* pick) {
  double running = 0.0;
  int c = 0;
  for (; c < nchunks; ++c) {
    if (running + chunk[c] >= target) break;
    running += chunk[c];
  }
  long long out = n - 1;
  if (c < nchunks) {
    const int64_t lo = static_cast<int64_t>(c) * kChunk, hi = min(n, lo + kChunk);
    for (int64_t i = lo; i < hi; ++i) {
      running += v[i];
      if (running >= target) {
        out = i;
        break;
      }
    }
  }
  *pick = out;
}

// copy point row i into centroid slot c
__global__ void km_take_kernel(const double* pts, int64_t n, int dim, const long long* idx, double* cen, int k, int c) {
  const int t = threadIdx.x;
  if (t < dim) cen[t * k + c] = pts[t * n + *idx];
}

// nearest centroid (strict <, lowest index wins: learn.cpp:17-28)
__global__ void km_assign_kernel(const double* pts, int64_t n, int dim, const double* cen, int k, int* labels,
                                 int* changed) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  int best = 0;
  double bd = sqdist(pts, n, i, dim, cen, k, 0);
  for (int c = 1; c < k; ++c) {
    const double dc = sqdist(pts, n, i, dim, cen, k, c);
    if (dc < bd) {
      bd = dc;
      best = c;
    }
  }
  if (labels[i] != best) {
    labels[i] = best;
    *changed = 1;
  }
}

// per chunk, per (cluster, component): serial sum over the chunk's points in
// index order; slot dim holds the count
__global__ void km_partial_kernel(const double* pts, int64_t n, int dim, const int* labels, int k, double* part) {
  const int ch = blockIdx.x;
  const int64_t lo = static_cast<int64_t>(ch) * kChunk, hi = min(n, lo + kChunk);
  const int w = dim + 1;
  for (int pair = threadIdx.x; pair < k * w; pair += blockDim.x) {
    const int c = pair / w, t = pair - c * w;
    double s = 0.0;
    for (int64_t i = lo; i < hi; ++i)
      if (labels[i] == c) s += (t < dim) ? pts[t * n + i] : 1.0;
    part[static_cast<int64_t>(ch) * k * w + pair] = s;
  }
}

__global__ void km_reduce_partial_kernel(const double* part, int nchunks, int kw, double* out) {
  const int pair = blockIdx.x * blockDim.x + threadIdx.x;
  if (pair >= kw) return;
  double s = 0.0;
  for (int ch = 0; ch < nchunks; ++ch) s += part[static_cast<int64_t>(ch) * kw + pair];
  out[pair] = s;
}

// per chunk: first index of the maximum (strict >, learn.cpp:111-119)
__global__ void km_chunk_argmax_kernel(const double* v, int64_t n, double* cmax, long long* carg, int nchunks) {
  const int ch = blockIdx.x * blockDim.x + threadIdx.x;
  if (ch >= nchunks) return;
  const int64_t lo = static_cast<int64_t>(ch) * kChunk, hi = min(n, lo + kChunk);
  double best = -1.0;
  long long arg = lo;
  for (int64_t i = lo; i < hi; ++i)
    if (v[i] > best) {
      best = v[i];
      arg = i;
    }
  cmax[ch] = best;
  carg[ch] = arg;
}

__global__ void km_argmax_kernel(const double* cmax, const long long* carg, int nchunks, long long* out) {
  double best = -1.0;
  long long arg = 0;
  for (int c = 0; c < nchunks; ++c)
    if (cmax[c] > best) {
      best = cmax[c];
      arg = carg[c];
    }
  *out = arg;
}

// unit-normalised rows (learn.cpp:160-164): norm = sqrt(serial sum of squares)
__global__ void km_normalize_rows_kernel(double* v, int64_t n, int dim) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  double s = 0.0;
  for (int t = 0; t < dim; ++t) s = __dadd_rn(s, __dmul_rn(v[t * n + i], v[t * n + i]));
  const double nrm = sqrt(s);
  if (nrm > 0.0)
    for (int t = 0; t < dim; ++t) v[t * n + i] = v[t * n + i] / nrm;
}

struct KMeansState {
  int64_t n;
  int dim, k, nchunks;
  cudaStream_t s;
  DBuf<double> pts, d2, cen, chunk, part, red, cmax;
  DBuf<int> labels, changed;
  DBuf<long long> pick, carg;
  DBuf<double> total;

  int blocks() const { return cdiv(n, 256); }

  double sum_of(const double* v) {  // chunked serial sum -> host
    km_chunk_sum_kernel<<<cdiv(nchunks, 128), 128, 0, s>>>(v, n, chunk.p, nchunks);
    km_total_kernel<<<1, 1, 0, s>>>(chunk.p, nchunks, total.p);
    double h = 0.0;
    FGS_CUDA(cudaMemcpyAsync(&h, total.p, sizeof(double), cudaMemcpyDeviceToHost, s));
    FGS_CUDA(cudaStreamSynchronize(s));
    return h;
  }
  int64_t download_pick() {
    long long h = 0;
    FGS_CUDA(cudaMemcpyAsync(&h, pick.p, sizeof(h), cudaMemcpyDeviceToHost, s));
    FGS_CUDA(cudaStreamSynchronize(s));
    return static_cast<int64_t>(h);
  }
  void take(int c, int64_t i) {
    const long long hi = static_cast<long long>(i);
    FGS_CUDA(cudaMemcpyAsync(pick.p, &hi, sizeof(hi), cudaMemcpyHostToDevice, s));
    km_take_kernel<<<1, 32 * cdiv(dim, 32), 0, s>>>(pts.p, n, dim, pick.p, cen.p, k, c);
  }

  // learn.cpp:30-75
  void plus_plus(std::mt19937_64& rng) {
    std::uniform_int_distribution<int64_t> any(0, n - 1);
    std::uniform_real_distribution<double> unif(0.0, 1.0);
    std::vector<char> chosen(static_cast<size_t>(n), 0);
    const int64_t first = any(rng);
    take(0, first);
    chosen[static_cast<size_t>(first)] = 1;
    km_dist_kernel<<<blocks(), 256, 0, s>>>(pts.p, n, dim, cen.p, k, 0, d2.p, 0);
    for (int c = 1; c < k; ++c) {
      const double tot = sum_of(d2.p);
      int64_t p = -1;
      if (tot > 0.0) {
        const double target = unif(rng) * tot;
        km_pick_kernel<<<1, 1, 0, s>>>(d2.p, n, chunk.p, nchunks, target, pick.p);
        p = download_pick();
      } else {
        std::vector<int64_t> open;
        for (int64_t i = 0; i < n; ++i)
          if (!chosen[static_cast<size_t>(i)]) open.push_back(i);
        if (open.empty())
          p = any(rng);
        else
          p = open[std::uniform_int_distribution<size_t>(0, open.size() - 1)(rng)];
      }
      take(c, p);
      chosen[static_cast<size_t>(p)] = 1;
      km_dist_kernel<<<blocks(), 256, 0, s>>>(pts.p, n, dim, cen.p, k, c, d2.p, 1);
    }
  }

  // learn.cpp:77-136; returns wcss, leaves labels / centroids on the device
  double lloyd(int max_iter, std::mt19937_64& rng) {
    plus_plus(rng);
    FGS_CUDA(cudaMemsetAsync(labels.p, 0xff, sizeof(int) * n, s));  // -1
    const int w = dim + 1;
    std::vector<double> red_h(static_cast<size_t>(k * w)), cen_h(static_cast<size_t>(k * dim));
    for (int iter = 0; iter < max_iter; ++iter) {
      FGS_CUDA(cudaMemsetAsync(changed.p, 0, sizeof(int), s));
      km_assign_kernel<<<blocks(), 256, 0, s>>>(pts.p, n, dim, cen.p, k, labels.p, changed.p);
      km_partial_kernel<<<nchunks, 128, 0, s>>>(pts.p, n, dim, labels.p, k, part.p);
      km_reduce_partial_kernel<<<cdiv(k * w, 128), 128, 0, s>>>(part.p, nchunks, k * w, red.p);
      int changed_h = 0;
      FGS_CUDA(cudaMemcpyAsync(red_h.data(), red.p, sizeof(double) * k * w, cudaMemcpyDeviceToHost, s));
      FGS_CUDA(cudaMemcpyAsync(cen_h.data(), cen.p, sizeof(double) * k * dim, cudaMemcpyDeviceToHost, s));
      FGS_CUDA(cudaMemcpyAsync(&changed_h, changed.p, sizeof(int), cudaMemcpyDeviceToHost, s));
      FGS_CUDA(cudaStreamSynchronize(s));
      bool ch = changed_h != 0;
      for (int c = 0; c < k; ++c) {
        const double cnt = red_h[static_cast<size_t>(c * w + dim)];
        if (cnt > 0.0) {
          for (int t = 0; t < dim; ++t)
            cen_h[static_cast<size_t>(t * k + c)] = red_h[static_cast<size_t>(c * w + t)] / cnt;
        } else {  // empty: re-seed at the point farthest from its (current) centroid
          FGS_CUDA(cudaMemcpyAsync(cen.p, cen_h.data(), sizeof(double) * k * dim, cudaMemcpyHostToDevice, s));
          km_own_dist_kernel<<<blocks(), 256, 0, s>>>(pts.p, n, dim, cen.p, k, labels.p, d2.p);
          km_chunk_argmax_kernel<<<cdiv(nchunks, 128), 128, 0, s>>>(d2.p, n, cmax.p, carg.p, nchunks);
          km_argmax_kernel<<<1, 1, 0, s>>>(cmax.p, carg.p, nchunks, pick.p);
          const int64_t far = download_pick();
          for (int t = 0; t < dim; ++t) {
            double v = 0.0;
            FGS_CUDA(cudaMemcpy(&v, pts.p + t * n + far, sizeof(double), cudaMemcpyDeviceToHost));
            cen_h[static_cast<size_t>(t * k + c)] = v;
          }
          FGS_CUDA(cudaMemcpyAsync(labels.p + far, &c, sizeof(int), cudaMemcpyHostToDevice, s));
          FGS_CUDA(cudaStreamSynchronize(s));
          ch = true;
        }
      }
      FGS_CUDA(cudaMemcpyAsync(cen.p, cen_h.data(), sizeof(double) * k * dim, cudaMemcpyHostToDevice, s));
      if (!ch) break;
    }
    km_own_dist_kernel<<<blocks(), 256, 0, s>>>(pts.p, n, dim, cen.p, k, labels.p, d2.p);
    return sum_of(d2.p);
  }
};

}  // namespace

void kmeans_run(const double* points, bool on_device, int64_t n, int dim, int k, int restarts, int max_iter,
                uint64_t seed, int device, bool normalize_rows, int* labels_out, double* centroids_out,
                double* wcss_out) {
  if (n < 1) fail(FGS_ESHAPE, "k-means needs at least one point");
  if (dim < 1) fail(FGS_ESHAPE, "points need at least one component");
  if (k < 1 || k > n) fail(FGS_EPARAM, "cluster count must lie in [1, point count]");
  if (restarts < 1 || max_iter < 1) fail(FGS_EPARAM, "restarts and max_iter must be positive");
  FGS_CUDA(cudaSetDevice(device));
  KMeansState st;
  st.n = n;
  st.dim = dim;
  st.k = k;
  st.nchunks = cdiv(n, kChunk);
  FGS_CUDA(cudaStreamCreateWithFlags(&st.s, cudaStreamNonBlocking));
  struct StreamGuard {
    cudaStream_t s;
    ~StreamGuard() {
      cudaStreamSynchronize(s);
      cudaStreamDestroy(s);
    }
  } guard{st.s};
  st.pts.alloc(static_cast<size_t>(n) * dim);
  FGS_CUDA(cudaMemcpyAsync(st.pts.p, points, sizeof(double) * n * dim,
                           on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st.s));
  if (normalize_rows) km_normalize_rows_kernel<<<st.blocks(), 256, 0, st.s>>>(st.pts.p, n, dim);
  st.d2.alloc(static_cast<size_t>(n));
  st.cen.alloc(static_cast<size_t>(k) * dim);
  st.chunk.alloc(static_cast<size_t>(st.nchunks));
  st.part.alloc(static_cast<size_t>(st.nchunks) * k * (dim + 1));
  st.red.alloc(static_cast<size_t>(k) * (dim + 1));
  st.cmax.alloc(static_cast<size_t>(st.nchunks));
  st.carg.alloc(static_cast<size_t>(st.nchunks));
  st.labels.alloc(static_cast<size_t>(n));
  st.changed.alloc(1);
  st.pick.alloc(1);
  st.total.alloc(1);

  std::mt19937_64 rng(seed);
  double best = std::numeric_limits<double>::infinity();
  std::vector<int> best_labels(static_cast<size_t>(n));
  std::vector<double> best_cen(static_cast<size_t>(k) * dim);
  for (int a = 0; a < restarts; ++a) {
    const double w = st.lloyd(max_iter, rng);
    if (w < best) {  // learn.cpp:151-153: strict, the first of equal runs is kept
      best = w;
      FGS_CUDA(cudaMemcpyAsync(best_labels.data(), st.labels.p, sizeof(int) * n, cudaMemcpyDeviceToHost, st.s));
      FGS_CUDA(cudaMemcpyAsync(best_cen.data(), st.cen.p, sizeof(double) * k * dim, cudaMemcpyDeviceToHost, st.s));
      FGS_CUDA(cudaStreamSynchronize(st.s));
    }
  }
  FGS_CUDA(cudaGetLastError());
  std::copy(best_labels.begin(), best_labels.end(), labels_out);
  if (centroids_out) std::copy(best_cen.begin(), best_cen.end(), centroids_out);
  if (wcss_out) *wcss_out = best;
}

}  // namespace fgsb
