// conv3d.cuh -- pruned spectral convolution for d = 3 grids: replaces cuFFT
// D2Z + multiply + Z2D (fastsum.cpp:115-117 / nfft.cpp:402-427 semantics)
// with three hand-written kernels built on conv2d.cuh's batched register FFT.
//
// The Hermitian-symmetrised multiplier m~ is zero outside the window
// l in [-N/2, N/2]^2 x [0, N/2] of the R2C half spectrum, so only the window
// is ever formed (u = grid index, k = frequency, M = 2N grid points):
//   planes_fwd (one CTA per plane u0):
//       rows     X[u1][k2]    = sum_u2 g[u0][u1][u2] e^{-2 pi i k2 u2 / M}, k2 <= N/2
//                (two real rows per complex sequence)
//       columns  Y[u0][l1][k2] = sum_u1 X[u1][k2] e^{-2 pi i l1 u1 / M},   |l1| <= N/2
//   lines (a batch of (l1, k2) lines per CTA):
//       Z[l0]    = m~[l0][l1][k2] sum_u0 Y[u0][l1][k2] e^{-2 pi i l0 u0 / M}
//       Y'[u0]   = sum_l0 Z[l0] e^{+2 pi i l0 u0 / M}
//   planes_inv (one CTA per plane u0):
//       columns  X'[u1][k2]   = sum_l1 Y'[u0][l1][k2] e^{+2 pi i l1 u1 / M}
//       rows     g'[u1][u2]   = sum_k2 c(k2) Re(X'[u1][k2] e^{+2 pi i k2 u2 / M}),
//                c = 1 for k2 = 0, else 2 (the C2R Hermitian fold; k2 <= N/2 < M/2)
// -- the same linear map as C2R(m~ . R2C(g)).  The two plane passes work on
// (N+1)(N/2+1) / M^2 ~ 1/8 of the half spectrum between them; the line pass
// touches only the window.  Every sum runs in a fixed order: bitwise
// reproducible.  Sharded handles run the planes of their slab only and sum
// the window spectra of the ranks (Core::apply_launches).
#pragma once

#include <cstdlib>
#include <string>

#include "conv2d.cuh"

namespace fgsb {

struct Conv3Args {
  const double* grid_in;          // [M][M][M] per vector (stride grid_stride)
  double* grid_out;
  double2* win;                   // [vec][M][NW][H] after planes_fwd; Y' after lines
  double2* spec;                  // [vec][NW][NW][H] window spectrum (sharded exchange), or null
  const cufftDoubleComplex* mult; // compact window multiplier [N+1][N+1][H]
  const double2* tw;              // tw[j] = e^{-2 pi i j / M}
  int M, N, nvec;
  int plane0, planes;             // planes plane0 .. plane0 + planes - 1 (mod M) of this launch
  int64_t grid_stride;
};

constexpr int kConv3Threads = 256;
// sequences per batched FFT call of the plane passes: a 64-point plane's 32
// packed row pairs in one call; 128-point planes in two (shared memory)
template <int M>
constexpr int conv3_seq() {
  return M <= 64 ? 32 : 16;
}
constexpr int kConv3Lines = 16;  // (l1, k2) lines per CTA of the line pass

__host__ __device__ inline int conv3_nw(int M, int N) { return M == N ? N : N + 1; }  // M == N: +N/2 aliases -N/2

// shared memory of the plane passes: tw[M] | X[M][H] | buf[S][M] | scratch[S][M + 16]
inline size_t conv3_plane_smem(int M, int N, int S = 0) {
  const size_t H = static_cast<size_t>(N / 2 + 1);
  if (S == 0) S = M <= 64 ? 32 : 16;
  return sizeof(double2) * (static_cast<size_t>(M) + static_cast<size_t>(M) * H + S * (2 * M + 16));
}
// line pass: tw[M] | buf[L][M] | scratch[L][M + 16]
inline size_t conv3_line_smem(int M) {
  return sizeof(double2) * (static_cast<size_t>(M) + static_cast<size_t>(kConv3Lines) * (2 * M + 16));
}

template <int M, int S = conv3_seq<M>(), int NT = kConv3Threads>
__global__ void __launch_bounds__(NT) conv3_planes_fwd_kernel(Conv3Args a) {
  extern __shared__ double2 sm3[];
  const int N = a.N, H = N / 2 + 1, hN = N / 2, NW = conv3_nw(M, N);
  const int u0 = (a.plane0 + static_cast<int>(blockIdx.x) % a.planes) & (M - 1);  // cyclic slab
  const int v = static_cast<int>(blockIdx.x) / a.planes;
  double2* tws = sm3;
  double2* X = tws + M;
  double2* buf = X + M * H;
  double2* scr = buf + S * M;
  pdl_wait();
  for (int j = threadIdx.x; j < M; j += blockDim.x) tws[j] = a.tw[j];
  __syncthreads();
  const double* g = a.grid_in + v * a.grid_stride + static_cast<int64_t>(u0) * M * M;
  // rows: 2p and 2p+1 packed as z_p = g[2p] + i g[2p+1], S pairs per round
  for (int p0 = 0; p0 < M / 2; p0 += S) {
    const int np = min(S, M / 2 - p0);
    fft_batch<M, false>(
        scr, np, tws,
        [&](int p, int u) {
          const int r = 2 * (p0 + p);
          return make_double2(__ldg(g + r * M + u), __ldg(g + (r + 1) * M + u));
        },
        [&](int p, int k, double2 z) { buf[p * M + k] = z; });
    __syncthreads();
    for (int t = threadIdx.x; t < np * H; t += blockDim.x) {
      const int p = t / H, k = t - p * H;
      const double2 z = buf[p * M + k];
      const double2 zc = buf[p * M + ((M - k) & (M - 1))];
      const int r = 2 * (p0 + p);
      X[r * H + k] = make_double2(0.5 * (z.x + zc.x), 0.5 * (z.y - zc.y));        // row 2p
      X[(r + 1) * H + k] = make_double2(0.5 * (z.y + zc.y), -0.5 * (z.x - zc.x));  // row 2p + 1
    }
    __syncthreads();
  }
  // columns k2: keep |l1| <= N/2, window index i = l1 + N/2
  double2* out = a.win + (static_cast<int64_t>(v) * M + u0) * NW * H;
  for (int c0 = 0; c0 < H; c0 += S) {
    const int nc = min(S, H - c0);
    fft_batch<M, false>(
        scr, nc, tws, [&](int j, int u) { return X[u * H + c0 + j]; },
        [&](int j, int q, double2 f) {
          const int i = (q + hN) & (M - 1);
          if (i < NW) out[i * H + c0 + j] = f;
        });
    __syncthreads();
  }
}

template <int M>
__global__ void __launch_bounds__(kConv3Threads) conv3_lines_kernel(Conv3Args a, int apply_mult, int inverse_only) {
  extern __shared__ double2 sm3[];
  const int N = a.N, H = N / 2 + 1, hN = N / 2, NW = conv3_nw(M, N);
  const int L = NW * H;
  const int nblk = (L + kConv3Lines - 1) / kConv3Lines;
  const int v = static_cast<int>(blockIdx.x) / nblk;
  const int l0 = (static_cast<int>(blockIdx.x) % nblk) * kConv3Lines;
  const int nl = min(kConv3Lines, L - l0);
  double2* tws = sm3;
  double2* buf = tws + M;
  double2* scr = buf + kConv3Lines * M;
  pdl_wait();
  for (int j = threadIdx.x; j < M; j += blockDim.x) tws[j] = a.tw[j];
  __syncthreads();
  double2* w = a.win + static_cast<int64_t>(v) * M * L;
  double2* sp = a.spec ? a.spec + static_cast<int64_t>(v) * NW * L : nullptr;
  if (!inverse_only) {
    // forward along u0 over this launch's planes; the window spectrum goes
    // to `spec` (sharded: the ranks' partial sums are added afterwards) or
    // straight into the multiply
    fft_batch<M, false>(
        scr, nl, tws,
        [&](int s, int u) {
          return (((u - a.plane0) & (M - 1)) < a.planes) ? w[static_cast<int64_t>(u) * L + l0 + s]
                                                            : make_double2(0.0, 0.0);
        },
        [&](int s, int q, double2 f) {
          const int i = (q + hN) & (M - 1);
          if (sp) {
            if (i < NW) sp[static_cast<int64_t>(i) * L + l0 + s] = f;
          } else {
            buf[s * M + q] = (i < NW && apply_mult)
                                 ? cmul(f, a.mult[static_cast<int64_t>(i) * L + l0 + s])
                                 : ((i < NW) ? f : make_double2(0.0, 0.0));
          }
        });
    __syncthreads();
    if (sp) return;
  } else {
    // sharded second half: the summed window spectrum times the multiplier
    for (int t = threadIdx.x; t < nl * M; t += blockDim.x) {
      const int s = t / M, q = t - s * M;
      const int i = (q + hN) & (M - 1);
      buf[s * M + q] = (i < NW) ? cmul(sp[static_cast<int64_t>(i) * L + l0 + s], a.mult[static_cast<int64_t>(i) * L + l0 + s])
                                : make_double2(0.0, 0.0);
    }
    __syncthreads();
  }
  // inverse along u0, only the planes this launch's owner interpolates from
  fft_batch<M, true>(
      scr, nl, tws, [&](int s, int q) { return buf[s * M + q]; },
      [&](int s, int u, double2 y) {
        if (((u - a.plane0) & (M - 1)) < a.planes) w[static_cast<int64_t>(u) * L + l0 + s] = y;
      });
}

template <int M, int S = conv3_seq<M>(), int NT = kConv3Threads>
__global__ void __launch_bounds__(NT) conv3_planes_inv_kernel(Conv3Args a) {
  extern __shared__ double2 sm3[];
  const int N = a.N, H = N / 2 + 1, hN = N / 2, NW = conv3_nw(M, N);
  const int u0 = (a.plane0 + static_cast<int>(blockIdx.x) % a.planes) & (M - 1);  // cyclic slab
  const int v = static_cast<int>(blockIdx.x) / a.planes;
  double2* tws = sm3;
  double2* X = tws + M;
  double2* buf = X + M * H;
  double2* scr = buf + S * M;
  pdl_wait();
  for (int j = threadIdx.x; j < M; j += blockDim.x) tws[j] = a.tw[j];
  __syncthreads();
  const double2* in = a.win + (static_cast<int64_t>(v) * M + u0) * NW * H;
  // columns k2: inverse along u1 from the kept l1
  for (int c0 = 0; c0 < H; c0 += S) {
    const int nc = min(S, H - c0);
    fft_batch<M, true>(
        scr, nc, tws,
        [&](int j, int q) {
          const int i = (q + hN) & (M - 1);
          return i < NW ? in[i * H + c0 + j] : make_double2(0.0, 0.0);
        },
        [&](int j, int u, double2 y) { X[u * H + c0 + j] = y; });
    __syncthreads();
  }
  // rows: Z = S_even + i S_odd, S the Hermitian extension of X' (C2R)
  double* g = a.grid_out + v * a.grid_stride + static_cast<int64_t>(u0) * M * M;
  for (int p0 = 0; p0 < M / 2; p0 += S) {
    const int np = min(S, M / 2 - p0);
    fft_batch<M, true>(
        scr, np, tws,
        [&](int p, int q) {
          const double2* ae = X + (2 * (p0 + p)) * H;
          const double2* ao = ae + H;
          double2 z = make_double2(0.0, 0.0);
          if (q == 0 || 2 * q == M) {
            if (q < H) z = make_double2(ae[q].x, ao[q].x);  // real parts only
          } else if (q < H) {
            z = make_double2(ae[q].x - ao[q].y, ae[q].y + ao[q].x);
          } else if (M - q < H) {
            const int k = M - q;
            z = make_double2(ae[k].x + ao[k].y, ao[k].x - ae[k].y);
          }
          return z;
        },
        [&](int p, int u, double2 y) {
          const int r = 2 * (p0 + p);
          g[r * M + u] = y.x;
          g[(r + 1) * M + u] = y.y;
        });
    __syncthreads();
  }
}

inline bool conv3_supported(int M) { return M == 32 || M == 64 || M == 128; }

// wide plane passes for 128-point planes: 512 threads, 32 sequences per
// round (rows in 2 rounds instead of 4, columns in 2 instead of 3; 204 KB of
// shared memory, one CTA per SM) -- the plane passes are latency-bound
// rounds of FFTs, and a sharded rank or a single vector has few planes
inline bool conv3_wide() {
  static const bool on = [] {
    const char* e = std::getenv("FGS_CONV3_WIDE");
    return !(e && std::string(e) == "0");
  }();
  return on;
}

template <int M>
void conv3_launch_t(const Conv3Args& a, int stage, int apply_mult, int inverse_only, cudaStream_t s) {
  const int H = a.N / 2 + 1, L = conv3_nw(M, a.N) * H;
  constexpr bool kWide = M == 128;
  constexpr int SW = kWide ? 32 : conv3_seq<M>(), NW_ = kWide ? 512 : kConv3Threads;
  static const bool init = [] {
    const int ps = 227 * 1024;
    FGS_CUDA(cudaFuncSetAttribute(reinterpret_cast<const void*>(conv3_planes_fwd_kernel<M>),
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, ps));
    FGS_CUDA(cudaFuncSetAttribute(reinterpret_cast<const void*>(conv3_planes_inv_kernel<M>),
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, ps));
    FGS_CUDA(cudaFuncSetAttribute(reinterpret_cast<const void*>(conv3_planes_fwd_kernel<M, SW, NW_>),
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, ps));
    FGS_CUDA(cudaFuncSetAttribute(reinterpret_cast<const void*>(conv3_planes_inv_kernel<M, SW, NW_>),
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, ps));
    FGS_CUDA(cudaFuncSetAttribute(reinterpret_cast<const void*>(conv3_lines_kernel<M>),
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, ps));
    return true;
  }();
  (void)init;
  const dim3 block(kConv3Threads);
  const bool wide = kWide && conv3_wide();
  if (stage == 1) {
    launch_ex(conv3_lines_kernel<M>, dim3(((L + kConv3Lines - 1) / kConv3Lines) * a.nvec), block, conv3_line_smem(M), s,
              a, apply_mult, inverse_only);
  } else if (wide) {
    const size_t sm = conv3_plane_smem(M, a.N, SW);
    if (stage == 0)
      launch_ex(conv3_planes_fwd_kernel<M, SW, NW_>, dim3(a.planes * a.nvec), dim3(NW_), sm, s, a);
    else
      launch_ex(conv3_planes_inv_kernel<M, SW, NW_>, dim3(a.planes * a.nvec), dim3(NW_), sm, s, a);
  } else if (stage == 0) {
    launch_ex(conv3_planes_fwd_kernel<M>, dim3(a.planes * a.nvec), block, conv3_plane_smem(M, a.N), s, a);
  } else {
    launch_ex(conv3_planes_inv_kernel<M>, dim3(a.planes * a.nvec), block, conv3_plane_smem(M, a.N), s, a);
  }
}

// stage 0: planes_fwd, 1: lines, 2: planes_inv
inline void conv3_launch(const Conv3Args& a, int stage, int apply_mult, int inverse_only, cudaStream_t s) {
  switch (a.M) {
    case 32: return conv3_launch_t<32>(a, stage, apply_mult, inverse_only, s);
    case 64: return conv3_launch_t<64>(a, stage, apply_mult, inverse_only, s);
    default: return conv3_launch_t<128>(a, stage, apply_mult, inverse_only, s);
  }
}

}  // namespace fgsb
