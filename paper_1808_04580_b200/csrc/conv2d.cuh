// conv2d.cuh -- pruned spectral convolution for d = 2 grids (replaces cuFFT
// D2Z + multiply + Z2D; fastsum.cpp:115-117 / nfft.cpp:402-427 semantics).
//
// The multiplier is zero outside l in [-N/2, N/2] x [0, N/2] of the half
// spectrum, so only (N+1)(N/2+1) modes are ever formed:
//   row     A[u0][k1]  = sum_u1 g[u0][u1] e^{-2 pi i k1 u1 / M},  k1 in [0, N/2]
//   column  W[l0][k1]  = m~[l0][k1] sum_u0 A[u0][k1] e^{-2 pi i l0 u0 / M}
//           A'[u0][k1] = sum_l0 W[l0][k1] e^{+2 pi i l0 u0 / M}
//   row     g'[u0][u1] = sum_k1 c(k1) Re(A'[u0][k1] e^{+2 pi i k1 u1 / M}),
//           c = 1 for k1 = 0 or 2 k1 = M, else 2  (the C2R Hermitian fold)
// -- the same linear map as C2R(m~ . R2C(g)) up to rounding.  Three small
// launches of direct DFTs against an exact twiddle table (angles reduced
// mod M), each sum in a fixed order.  For C2 (M = 128, N = 64) this is
// 2.2 MFLOP per vector.
#pragma once

#include "common.cuh"

namespace fgsb {

struct Conv2Args {
  const double* grid_in;  // [M][M] per vector (stride grid_stride)
  double* grid_out;       // may alias grid_in
  cufftDoubleComplex* A;  // [M][H] per vector (stride a_stride)
  const cufftDoubleComplex* mult;  // compact window multiplier [N+1][H]
  const double2* tw;      // tw[j] = e^{-2 pi i j / M}
  int M, N, nvec;
  int64_t grid_stride, a_stride;
};

constexpr int kConvThreads = 256;

__device__ __forceinline__ void load_twiddles(double2* tws, const double2* tw, int M) {
  for (int j = threadIdx.x; j < M; j += blockDim.x) tws[j] = tw[j];
}

// A[u0][k1]: 4 lanes per output mode, each summing a quarter of the row, then
// a fixed shuffle tree.  smem: tw[M] | row[M]
__global__ void __launch_bounds__(kConvThreads) conv2_rows_fwd(Conv2Args a) {
  extern __shared__ double2 sm2[];
  const int u0 = blockIdx.x, v = blockIdx.y, M = a.M, H = a.N / 2 + 1;
  double2* tws = sm2;
  double* row = reinterpret_cast<double*>(sm2 + M);
  load_twiddles(tws, a.tw, M);
  const double* g = a.grid_in + v * a.grid_stride + static_cast<int64_t>(u0) * M;
  for (int u = threadIdx.x; u < M; u += blockDim.x) row[u] = g[u];
  __syncthreads();
  for (int t = threadIdx.x; t < 32 * ((H + 7) / 8); t += blockDim.x) {
    const int k = t >> 2, part = t & 3;
    double re = 0.0, im = 0.0;
    if (k < H) {
      const int per = (M + 3) / 4, lo = part * per, hi = min(M, lo + per);
      int idx = static_cast<int>((static_cast<int64_t>(k) * lo) % M);
      for (int u = lo; u < hi; ++u) {
        const double2 w = tws[idx];
        re = fma(row[u], w.x, re);
        im = fma(row[u], w.y, im);
        idx += k;
        if (idx >= M) idx -= M;
      }
    }
    re += __shfl_down_sync(0xffffffffu, re, 1, 4);
    im += __shfl_down_sync(0xffffffffu, im, 1, 4);
    re += __shfl_down_sync(0xffffffffu, re, 2, 4);
    im += __shfl_down_sync(0xffffffffu, im, 2, 4);
    if (part == 0 && k < H) a.A[v * a.a_stride + static_cast<int64_t>(u0) * H + k] = make_cuDoubleComplex(re, im);
  }
}

// column k1: forward to the window, multiply, back to all M rows (in place).
// smem: tw[M] | col[M] | W[N+1]
__global__ void __launch_bounds__(kConvThreads) conv2_cols(Conv2Args a) {
  extern __shared__ double2 sm2[];
  const int k1 = blockIdx.x, v = blockIdx.y, M = a.M, N = a.N, H = N / 2 + 1, hN = N / 2;
  double2* tws = sm2;
  double2* col = sm2 + M;
  double2* W = col + M;
  load_twiddles(tws, a.tw, M);
  cufftDoubleComplex* A = a.A + v * a.a_stride;
  for (int u = threadIdx.x; u < M; u += blockDim.x) {
    const cufftDoubleComplex z = A[static_cast<int64_t>(u) * H + k1];
    col[u] = make_double2(z.x, z.y);
  }
  __syncthreads();
  const int nw = (M == N) ? N : N + 1;  // M == N: l0 = +N/2 aliases -N/2
  // forward: 4 lanes per window mode
  for (int t = threadIdx.x; t < 32 * ((N + 1 + 7) / 8); t += blockDim.x) {
    const int i = t >> 2, part = t & 3;
    double re = 0.0, im = 0.0;
    if (i < nw) {
      const int step = (((i - hN) % M) + M) % M;
      const int per = (M + 3) / 4, lo = part * per, hi = min(M, lo + per);
      int idx = static_cast<int>((static_cast<int64_t>(step) * lo) % M);
      for (int u = lo; u < hi; ++u) {  // col[u] e^{-2 pi i l0 u / M}
        const double2 w = tws[idx];
        const double2 c = col[u];
        re = fma(c.x, w.x, re);
        re = fma(-c.y, w.y, re);
        im = fma(c.x, w.y, im);
        im = fma(c.y, w.x, im);
        idx += step;
        if (idx >= M) idx -= M;
      }
    }
    re += __shfl_down_sync(0xffffffffu, re, 1, 4);
    im += __shfl_down_sync(0xffffffffu, im, 1, 4);
    re += __shfl_down_sync(0xffffffffu, re, 2, 4);
    im += __shfl_down_sync(0xffffffffu, im, 2, 4);
    if (part == 0 && i < N + 1) {
      if (i < nw) {
        const cufftDoubleComplex m = a.mult[static_cast<int64_t>(i) * H + k1];
        W[i] = make_double2(re * m.x - im * m.y, re * m.y + im * m.x);
      } else {
        W[i] = make_double2(0.0, 0.0);
      }
    }
  }
  __syncthreads();
  // inverse: 2 lanes per output row, sum_l0 W[l0] e^{+2 pi i l0 u / M}
  for (int t = threadIdx.x; t < 2 * ((M + 15) / 16) * 16; t += blockDim.x) {
    const int u = t >> 1, part = t & 1;
    double re = 0.0, im = 0.0;
    if (u < M) {
      const int per = (nw + 1) / 2, lo = part * per, hi = min(nw, lo + per);
      int idx = static_cast<int>((static_cast<int64_t>((((lo - hN) % M) + M) % M) * u) % M);
      for (int i = lo; i < hi; ++i) {
        const double2 w = tws[idx];  // conj(w) = e^{+...}
        const double2 c = W[i];
        re = fma(c.x, w.x, re);
        re = fma(c.y, w.y, re);
        im = fma(c.y, w.x, im);
        im = fma(-c.x, w.y, im);
        idx += u;
        if (idx >= M) idx -= M;
      }
    }
    re += __shfl_down_sync(0xffffffffu, re, 1, 2);
    im += __shfl_down_sync(0xffffffffu, im, 1, 2);
    if (part == 0 && u < M) A[static_cast<int64_t>(u) * H + k1] = make_cuDoubleComplex(re, im);
  }
}

// g'[u0][u1] = sum_k1 c(k1) Re(A'[u0][k1] e^{+2 pi i k1 u1 / M}).  smem: tw[M] | ar[H]
__global__ void __launch_bounds__(kConvThreads) conv2_rows_inv(Conv2Args a) {
  extern __shared__ double2 sm2[];
  const int u0 = blockIdx.x, v = blockIdx.y, M = a.M, H = a.N / 2 + 1;
  double2* tws = sm2;
  double2* ar = sm2 + M;
  load_twiddles(tws, a.tw, M);
  const cufftDoubleComplex* A = a.A + v * a.a_stride + static_cast<int64_t>(u0) * H;
  for (int k = threadIdx.x; k < H; k += blockDim.x) {
    const double c = (k == 0 || 2 * k == M) ? 1.0 : 2.0;
    ar[k] = make_double2(c * A[k].x, c * A[k].y);
  }
  __syncthreads();
  double* g = a.grid_out + v * a.grid_stride + static_cast<int64_t>(u0) * M;
  for (int u = threadIdx.x; u < M; u += blockDim.x) {
    double acc0 = 0.0, acc1 = 0.0;  // two chains
    int idx = 0;
    int k = 0;
    for (; k + 1 < H; k += 2) {  // Re((x + iy)(wr - i wi)) with w = e^{-...}
      const double2 w0 = tws[idx];
      idx += u;
      if (idx >= M) idx -= M;
      const double2 w1 = tws[idx];
      idx += u;
      if (idx >= M) idx -= M;
      acc0 = fma(ar[k].x, w0.x, acc0);
      acc0 = fma(ar[k].y, w0.y, acc0);
      acc1 = fma(ar[k + 1].x, w1.x, acc1);
      acc1 = fma(ar[k + 1].y, w1.y, acc1);
    }
    if (k < H) {
      const double2 w0 = tws[idx];
      acc0 = fma(ar[k].x, w0.x, acc0);
      acc0 = fma(ar[k].y, w0.y, acc0);
    }
    g[u] = acc0 + acc1;
  }
}

}  // namespace fgsb
