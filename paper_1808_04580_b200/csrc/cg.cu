// cg.cu -- conjugate gradients on the device (spectral.cpp:446-495
// cg_solve) for the two matvec consumers the reference builds on it:
//   kernel_ssl_solve (learn.cpp:364-381):  (I + beta L_s) x = f
//   krr_fit          (learn.cpp:403-430):  (W~ + beta I) alpha = f
// Same recurrences, the same "confirm on the true residual" restart and the
// same status rules as the reference; vectors stay in HBM in the handle's
// internal order, every operator application is the handle's graph-cached
// apply, and the dot products are fixed-order block sums (bitwise
// reproducible).  Two scalars come back to the host per iteration
// (curvature, residual norm) to drive the control flow.
#include <cuda_runtime.h>

#include <cmath>
#include <vector>

#include "cg.hpp"
#include "common.cuh"
#include "core.cuh"

namespace fgsb {
namespace {

constexpr int kThreads = 256;
constexpr int kRows = 8;  // rows per thread per block
constexpr int kBlockRows = kThreads * kRows;

inline int cdiv(int64_t a, int64_t b) { return static_cast<int>((a + b - 1) / b); }

// block-fixed-order sum of v[r]; written to partial[blockIdx.x]
__device__ __forceinline__ void block_sum(double v, double* partial) {
  __shared__ double red[kThreads];
  red[threadIdx.x] = v;
  __syncthreads();
  for (int s = kThreads / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) partial[blockIdx.x] = red[0];
}

__global__ void dot_kernel(const double* __restrict__ a, const double* __restrict__ b, int64_t n,
                           double* __restrict__ partial) {
  double s = 0.0;
  const int64_t r0 = static_cast<int64_t>(blockIdx.x) * kBlockRows + threadIdx.x;
#pragma unroll
  for (int i = 0; i < kRows; ++i) {
    const int64_t r = r0 + static_cast<int64_t>(i) * kThreads;
    if (r < n) s += a[r] * b[r];
  }
  block_sum(s, partial);
}

// x += step p;  r -= step ap;  partial = sum r^2
__global__ void step_kernel(double* __restrict__ x, double* __restrict__ r, const double* __restrict__ p,
                            const double* __restrict__ ap, double step, int64_t n, double* __restrict__ partial) {
  double s = 0.0;
  const int64_t r0 = static_cast<int64_t>(blockIdx.x) * kBlockRows + threadIdx.x;
#pragma unroll
  for (int i = 0; i < kRows; ++i) {
    const int64_t k = r0 + static_cast<int64_t>(i) * kThreads;
    if (k < n) {
      x[k] += step * p[k];
      const double rk = r[k] - step * ap[k];
      r[k] = rk;
      s += rk * rk;
    }
  }
  block_sum(s, partial);
}

// r = b - ax;  partial = sum r^2
__global__ void residual_kernel(const double* __restrict__ b, const double* __restrict__ ax, double* __restrict__ r,
                                int64_t n, double* __restrict__ partial) {
  double s = 0.0;
  const int64_t r0 = static_cast<int64_t>(blockIdx.x) * kBlockRows + threadIdx.x;
#pragma unroll
  for (int i = 0; i < kRows; ++i) {
    const int64_t k = r0 + static_cast<int64_t>(i) * kThreads;
    if (k < n) {
      const double rk = b[k] - ax[k];
      r[k] = rk;
      s += rk * rk;
    }
  }
  block_sum(s, partial);
}

// out = sum of partial[0..nb) in a fixed order (one warp)
__global__ void finish_kernel(const double* __restrict__ partial, int nb, double* __restrict__ out) {
  double s = 0.0;
  for (int b = threadIdx.x; b < nb; b += 32) s += partial[b];
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) s += __shfl_down_sync(0xffffffffu, s, off);
  if (threadIdx.x == 0) *out = s;
}

// p = r + beta p
__global__ void direction_kernel(double* __restrict__ p, const double* __restrict__ r, double beta, int64_t n) {
  const int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (k < n) p[k] = r[k] + beta * p[k];
}

// y = cx x + cy y, no contraction: (x + beta * (L x)) / ((W x) + beta * x)
__global__ void combine_kernel(const double* __restrict__ x, double* __restrict__ y, double cx, double cy, int64_t n) {
  const int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (k < n) y[k] = __dadd_rn(__dmul_rn(cx, x[k]), __dmul_rn(cy, y[k]));
}

}  // namespace

CgOutcome cg_solve(Core& c, CgSystem system, double beta, const double* f_host, double tol, int max_iter,
                   double* x_host) {
  if (c.world > 1) fail(FGS_EPARAM, "cg_solve needs an unsharded handle");
  if (!(tol > 0.0)) fail(FGS_EPARAM, "tolerance must be positive");
  if (max_iter < 1) fail(FGS_EPARAM, "max_iter must be positive");
  if (system == CG_SSL && !(beta >= 0.0)) fail(FGS_EPARAM, "beta must be nonnegative");
  if (system == CG_KRR && !(beta > 0.0)) fail(FGS_EPARAM, "beta must be positive");
  const int64_t n = c.n;
  cudaStream_t st = c.stream;
  CgOutcome out;
  if (system == CG_SSL && beta == 0.0) {  // learn.cpp:368-373: the identity system
    for (int64_t i = 0; i < n; ++i) x_host[i] = f_host[i];
    out.status = CG_CONVERGED;
    return out;
  }
  // operator of the system, in the internal order
  const int epi = system == CG_SSL ? EPI_LAPLACIAN : EPI_KERNEL;
  const bool scale = system == CG_SSL;
  const double cx = system == CG_SSL ? 1.0 : beta, cy = system == CG_SSL ? beta : 1.0;

  DBuf<double> bc, b, x, r, p, ap, partial, scal;
  bc.upload(f_host, static_cast<size_t>(n), st);
  b.alloc(static_cast<size_t>(n));
  x.alloc(static_cast<size_t>(n));
  r.alloc(static_cast<size_t>(n));
  p.alloc(static_cast<size_t>(n));
  ap.alloc(static_cast<size_t>(n));
  const int nb = std::max(1, cdiv(n, kBlockRows));
  partial.alloc(static_cast<size_t>(nb));
  scal.alloc(1);
  c.permute(bc.p, n, b.p, n, 1, 0);  // caller -> internal
  FGS_CUDA(cudaMemsetAsync(x.p, 0, sizeof(double) * n, st));
  const int g = cdiv(n, 256);

  auto fetch = [&]() {
    finish_kernel<<<1, 32, 0, st>>>(partial.p, nb, scal.p);
    double h = 0.0;
    FGS_CUDA(cudaMemcpyAsync(&h, scal.p, sizeof(double), cudaMemcpyDeviceToHost, st));
    FGS_CUDA(cudaStreamSynchronize(st));
    c.launches += 1;
    return h;
  };
  auto sys_apply = [&](const double* in, double* o) {
    c.apply(epi, in, n, o, n, 1, false, scale);
    combine_kernel<<<g, 256, 0, st>>>(in, o, cx, cy, n);
    c.launches += 1;
  };
  auto finish_x = [&]() {
    c.permute(x.p, n, bc.p, n, 1, 1);  // internal -> caller
    FGS_CUDA(cudaMemcpyAsync(x_host, bc.p, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
    FGS_CUDA(cudaStreamSynchronize(st));
    FGS_CUDA(cudaGetLastError());
  };

  dot_kernel<<<nb, kThreads, 0, st>>>(b.p, b.p, n, partial.p);
  const double bnorm = std::sqrt(fetch());
  if (bnorm == 0.0) {
    out.status = CG_CONVERGED;
    finish_x();
    return out;
  }
  FGS_CUDA(cudaMemcpyAsync(r.p, b.p, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
  FGS_CUDA(cudaMemcpyAsync(p.p, b.p, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
  dot_kernel<<<nb, kThreads, 0, st>>>(r.p, r.p, n, partial.p);
  double rs = fetch();
  out.status = CG_MAX_ITERATIONS;
  for (int it = 1; it <= max_iter; ++it) {
    sys_apply(p.p, ap.p);
    dot_kernel<<<nb, kThreads, 0, st>>>(p.p, ap.p, n, partial.p);
    const double curvature = fetch();
    out.iterations = it;
    if (!(curvature > 0.0)) {
      out.status = CG_INDEFINITE;
      finish_x();
      return out;
    }
    const double step = rs / curvature;
    step_kernel<<<nb, kThreads, 0, st>>>(x.p, r.p, p.p, ap.p, step, n, partial.p);
    double rs_next = fetch();
    if (std::sqrt(rs_next) <= tol * bnorm) {
      // confirm on the true residual (the recurrence can drift)
      sys_apply(x.p, ap.p);
      residual_kernel<<<nb, kThreads, 0, st>>>(b.p, ap.p, r.p, n, partial.p);
      rs_next = fetch();
      if (std::sqrt(rs_next) <= tol * bnorm) {
        out.status = CG_CONVERGED;
        finish_x();
        return out;
      }
      FGS_CUDA(cudaMemcpyAsync(p.p, r.p, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
      rs = rs_next;
      continue;
    }
    direction_kernel<<<g, 256, 0, st>>>(p.p, r.p, rs_next / rs, n);
    c.launches += 3;
    rs = rs_next;
  }
  finish_x();
  return out;
}

}  // namespace fgsb
