// direct.cuh -- the exact O(n^2) operator behind AdjacencyBackend::Direct
// (graphop.cpp:29-34 -> fastsum.cpp:126-139 direct_apply) and the
// recompute-mode dense reference (spectral.cpp:497-554):
//   (W~ x)_j = sum_i K(||v_j - v_i||) x_i     (i = j included; the graph
//   epilogues subtract K(0) x exactly as for the fast summation).
//
// Pass 1 (direct_partial_kernel): CTA (target tile, source segment); the
// segment's sources are staged through shared memory in tiles and every
// thread accumulates its target over them in increasing source order.
// Pass 2 (direct_finish_kernel): the segment partials summed in segment
// order + the graph-operator epilogue.  Fixed order, no atomics: bitwise
// reproducible.  Kernel formulas as kernels.cpp:79-93 (r = sqrt of the
// squared distance, then the family's expression).
#pragma once

#include "common.cuh"

namespace fgsb {

constexpr int kDirectThreads = 128;  // targets per CTA
constexpr int kDirectTile = 256;     // sources per shared-memory tile
constexpr int kDirectVec = 4;        // vectors per pass

struct DirectArgs {
  const double* nodes;  // [d][n] column-major, caller order
  int64_t n;
  int d;
  int family;
  double shape;
  const double* x;
  int64_t ldx;
  const double* s;  // D^-1/2 (nullable)
  int scale_input;
  int vec0, nv;     // vectors [vec0, vec0 + nv) of this pass, nv <= kDirectVec
  int64_t seg_len;  // sources per segment
  int nseg;
  double* partial;  // [nseg][nvec][n]
  int nvec;
};

__device__ __forceinline__ double direct_kernel_value(int family, double shape, double r) {
  switch (family) {
    case FGS_GAUSSIAN: return exp(-(r * r) / (shape * shape));
    case FGS_LAPLACIAN_RBF: return exp(-r / shape);
    case FGS_MULTIQUADRIC: return sqrt(r * r + shape * shape);
    default: return 1.0 / sqrt(r * r + shape * shape);
  }
}

__global__ void __launch_bounds__(kDirectThreads) direct_partial_kernel(DirectArgs a) {
  pdl_wait();
  __shared__ double sc[3][kDirectTile];
  __shared__ double sx[kDirectVec][kDirectTile];
  const int64_t j = blockIdx.x * static_cast<int64_t>(kDirectThreads) + threadIdx.x;
  const int seg = blockIdx.y;
  const int64_t lo = seg * a.seg_len, hi = min(a.n, lo + a.seg_len);
  double vj[3] = {0.0, 0.0, 0.0};
  if (j < a.n)
    for (int t = 0; t < a.d; ++t) vj[t] = a.nodes[t * a.n + j];
  double acc[kDirectVec] = {0.0, 0.0, 0.0, 0.0};
  for (int64_t t0 = lo; t0 < hi; t0 += kDirectTile) {
    const int cnt = static_cast<int>(hi - t0 < kDirectTile ? hi - t0 : kDirectTile);
    __syncthreads();
    for (int k = threadIdx.x; k < cnt; k += kDirectThreads) {
      const int64_t i = t0 + k;
      for (int t = 0; t < a.d; ++t) sc[t][k] = a.nodes[t * a.n + i];
      const double si = (a.scale_input && a.s) ? a.s[i] : 1.0;
#pragma unroll
      for (int v = 0; v < kDirectVec; ++v) {
        double xv = 0.0;
        if (v < a.nv) {
          xv = a.x[(a.vec0 + v) * a.ldx + i];
          if (a.scale_input && a.s) xv = __dmul_rn(si, xv);
        }
        sx[v][k] = xv;
      }
    }
    __syncthreads();
    if (j < a.n) {
      for (int k = 0; k < cnt; ++k) {
        double r2 = 0.0;
        for (int t = 0; t < a.d; ++t) {
          const double df = vj[t] - sc[t][k];
          r2 += df * df;
        }
        const double kv = direct_kernel_value(a.family, a.shape, sqrt(r2));
#pragma unroll
        for (int v = 0; v < kDirectVec; ++v)
          if (v < a.nv) acc[v] += kv * sx[v][k];
      }
    }
  }
  if (j < a.n) {
#pragma unroll
    for (int v = 0; v < kDirectVec; ++v)
      if (v < a.nv) a.partial[(static_cast<int64_t>(seg) * a.nvec + a.vec0 + v) * a.n + j] = acc[v];
  }
}

struct DirectFinishArgs {
  const double* partial;  // [nseg][nvec][n]
  int nseg, nvec;
  int64_t n;
  PassArgs pa;  // epilogue, x/ldx, s, y/ldy, k0, degrees, inv_sqrt, bad_flag, caller
};

__global__ void direct_finish_kernel(DirectFinishArgs f) {
  pdl_wait();
  const int64_t j = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (j >= f.n) return;
  const PassArgs& a = f.pa;
  for (int v = 0; v < f.nvec; ++v) {
    double val = 0.0;
    for (int s = 0; s < f.nseg; ++s) val += f.partial[(static_cast<int64_t>(s) * f.nvec + v) * f.n + j];
    if (a.epilogue == EPI_DEGREE) {
      const double dg = val - a.k0;  // graphop.cpp:55-56
      a.degrees[j] = dg;
      a.inv_sqrt[j] = 1.0 / sqrt(dg);
      if (!(dg > 0.0)) atomicMin(a.bad_flag, static_cast<unsigned long long>(j));
    } else {
      const double* xv = a.x + v * a.ldx;
      a.y[v * a.ldy + j] = epilogue(a, val, j, j, xv);
    }
  }
}

}  // namespace fgsb
