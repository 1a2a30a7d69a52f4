// conv2d.cuh -- one-launch spectral convolution for d = 2 grids: replaces
// cuFFT D2Z + multiply + Z2D (fastsum.cpp:115-117 / nfft.cpp:402-427
// semantics) with a single thread-block-cluster kernel.
//
// The multiplier is zero outside l in [-N/2, N/2] x [0, N/2] of the half
// spectrum, so only those modes are carried between the passes:
//   rows     A[u0][k1]  = sum_u1 g[u0][u1] e^{-2 pi i k1 u1 / M},  k1 in [0, N/2]
//   columns  W[l0][k1]  = m~[l0][k1] sum_u0 A[u0][k1] e^{-2 pi i l0 u0 / M}
//            A'[u0][k1] = sum_l0 W[l0][k1] e^{+2 pi i l0 u0 / M}
//   rows     g'[u0][u1] = sum_k1 c(k1) Re(A'[u0][k1] e^{+2 pi i k1 u1 / M}),
//            c = 1 for k1 = 0 or 2 k1 = M, else 2  (the C2R Hermitian fold)
// -- the same linear map as C2R(m~ . R2C(g)).
//
// One cluster of kClusterCtas CTAs per vector.  CTA c owns grid rows
// [c R, (c+1) R), R = M / kClusterCtas, and the kept column modes
// k1 = c, c + 8, ...:
//   1. its rows, two real rows packed per complex sequence, through a
//      two-pass register FFT; the kept modes unpacked and pushed into the
//      column owners' shared memory (distributed shared memory stores);
//   2. cluster barrier; its columns: FFT, window multiply, inverse FFT,
//      results pushed back into the row owners' A2 through DSMEM;
//   3. cluster barrier; its rows' Hermitian spectra (two rows per complex
//      sequence again) inverse-transformed and stored.
// Every sum is in a fixed order (no atomics): bitwise reproducible.
// Requires M a power of two, 16 <= M, smem within the opt-in limit.
#pragma once

#include <cooperative_groups.h>

#include "common.cuh"

namespace fgsb {

#ifdef FGS_CONV2_TRACE  // phase timestamps (tools/conv2_bench.cu only)
__device__ unsigned long long g_conv2_trace[16];
#define CONV2_MARK(i)                                                                  \
  do {                                                                                 \
    if (blockIdx.x == 0 && threadIdx.x == 0) {                                         \
      unsigned long long t_;                                                           \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                           \
      g_conv2_trace[i] = t_;                                                           \
    }                                                                                  \
  } while (0)
#else
#define CONV2_MARK(i) \
  do {                \
  } while (0)
#endif

constexpr int kClusterCtas = 16;  // non-portable cluster size (B200 allows 16)
constexpr int kConvThreads = 256;

struct Conv2Args {
  const double* grid_in;  // [M][M] per vector (stride grid_stride)
  double* grid_out;       // may alias grid_in
  const cufftDoubleComplex* mult;  // compact window multiplier [N+1][H]
  const double2* tw;      // tw[j] = e^{-2 pi i j / M}
  int M, logM, N, nvec;
  int64_t grid_stride;
};

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}

// In-register radix-2 DIT FFT of P points (P a power of two, compile-time),
// twiddles W_P^j = tws[j M / P] (conjugated for the inverse).
template <int P, int M, bool INV>
__device__ __forceinline__ void reg_fft(double2 (&v)[P], const double2* tws) {
#pragma unroll
  for (int i = 0; i < P; ++i) {  // bit-reversal permutation
    int r = 0;
#pragma unroll
    for (int b = 1, x = i; b < P; b <<= 1, x >>= 1) r = (r << 1) | (x & 1);
    if (r > i) {
      const double2 t = v[i];
      v[i] = v[r];
      v[r] = t;
    }
  }
#pragma unroll
  for (int h = 1; h < P; h <<= 1) {
#pragma unroll
    for (int j = 0; j < h; ++j) {
      double2 w = tws[j * (M / (2 * h))];
      if (INV) w.y = -w.y;
#pragma unroll
      for (int i = j; i < P; i += 2 * h) {
        const double2 a = v[i];
        const double2 b = (j == 0) ? v[i + h] : cmul(v[i + h], w);
        v[i] = make_double2(a.x + b.x, a.y + b.y);
        v[i + h] = make_double2(a.x - b.x, a.y - b.y);
      }
    }
  }
}

__host__ __device__ constexpr int ilog2c(int x) { return x <= 1 ? 0 : 1 + ilog2c(x / 2); }

// Split M = P * Q used by the two-pass FFT.
template <int M> struct FftSplit;
template <> struct FftSplit<16> { static constexpr int P = 4, Q = 4; };
template <> struct FftSplit<32> { static constexpr int P = 4, Q = 8; };
template <> struct FftSplit<64> { static constexpr int P = 8, Q = 8; };
template <> struct FftSplit<128> { static constexpr int P = 8, Q = 16; };
template <> struct FftSplit<256> { static constexpr int P = 16, Q = 16; };

// Padded transpose scratch per sequence: P rows of Q + 1.
template <int M> __host__ __device__ constexpr int fft_scratch() { return FftSplit<M>::P * (FftSplit<M>::Q + 1); }

// Batched length-M FFT ("four-step"): element idx of sequence s comes from
// ld(s, idx); pass 1 does P-point DFTs over n2 of x[n1 + Q n2] and the twiddle
// W_M^{n1 k2} into the padded scratch t[s][k2][n1]; pass 2 does Q-point DFTs
// over n1 and hands X[k2 + P k1] to st(s, k2 + P k1, value).  One barrier
// (between the passes); the caller orders scratch reuse and st's effects.
template <int M, bool INV, class Ld, class St>
__device__ __forceinline__ void fft_batch(double2* t, int nseq, const double2* tws, Ld ld, St st) {
  constexpr int P = FftSplit<M>::P, Q = FftSplit<M>::Q, TS = fft_scratch<M>();
  for (int w = threadIdx.x; w < nseq * Q; w += blockDim.x) {
    const int s = w / Q, n1 = w - s * Q;
    double2 v[P];
#pragma unroll
    for (int n2 = 0; n2 < P; ++n2) v[n2] = ld(s, n1 + Q * n2);
    reg_fft<P, M, INV>(v, tws);
#pragma unroll
    for (int k2 = 0; k2 < P; ++k2) {
      double2 tw = tws[(n1 * k2) & (M - 1)];
      if (INV) tw.y = -tw.y;
      t[s * TS + k2 * (Q + 1) + n1] = (k2 == 0) ? v[k2] : cmul(v[k2], tw);
    }
  }
  __syncthreads();
  for (int w = threadIdx.x; w < nseq * P; w += blockDim.x) {
    const int s = w / P, k2 = w - s * P;
    double2 v[Q];
#pragma unroll
    for (int n1 = 0; n1 < Q; ++n1) v[n1] = t[s * TS + k2 * (Q + 1) + n1];
    reg_fft<Q, M, INV>(v, tws);
#pragma unroll
    for (int k1 = 0; k1 < Q; ++k1) st(s, k2 + P * k1, v[k1]);
  }
}

__device__ __forceinline__ void conv_cp_async16(void* smem, const void* gmem) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem));
}

// smem: tw[M] | buf[S][M] | scratch[S][P(Q+1)] | colbuf[C][M] | A2[R][H] |
//       mw[C][N+1]  (S = max(R / 2, C), C = ceil(H / kClusterCtas))
__host__ __device__ inline int conv2_cols(int N) { return (N / 2 + 1 + kClusterCtas - 1) / kClusterCtas; }
__host__ __device__ inline int conv2_seqs(int M, int N) {
  const int R = M / kClusterCtas, nc = conv2_cols(N);
  return R / 2 > nc ? R / 2 : nc;
}
inline size_t conv2_smem(int M, int N) {
  const int R = M / kClusterCtas, H = N / 2 + 1, S = conv2_seqs(M, N);
  // scratch P (Q + 1) <= M + 16 for every split
  const size_t C = static_cast<size_t>(conv2_cols(N));
  return sizeof(double2) * (static_cast<size_t>(M) + static_cast<size_t>(S) * (2 * M + 16) + C * M +
                            static_cast<size_t>(R) * H + C * (N + 1));
}

template <int M>
__global__ void __cluster_dims__(kClusterCtas, 1, 1) __launch_bounds__(kConvThreads)
    conv2_cluster_kernel(Conv2Args a) {
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  extern __shared__ double2 sm2[];
  const int N = a.N, H = N / 2 + 1, hN = N / 2;
  const int R = M / kClusterCtas, S = conv2_seqs(M, N), C = conv2_cols(N);
  const int c = static_cast<int>(cluster.block_rank());
  const int v = blockIdx.x / kClusterCtas;
  const int nc = (H - c + kClusterCtas - 1) / kClusterCtas;  // my columns k1 = c + j kClusterCtas
  const int nw = (M == N) ? N : N + 1;                      // M == N: l0 = +N/2 aliases -N/2
  double2* tws = sm2;
  double2* buf0 = sm2 + M;
  double2* scr = buf0 + S * M;
  double2* colbuf = scr + S * (M + 16);
  double2* A2 = colbuf + C * M;
  double2* mw = A2 + R * H;
  const double* gin = a.grid_in + v * a.grid_stride + static_cast<int64_t>(c) * R * M;
  double* gout = a.grid_out + v * a.grid_stride + static_cast<int64_t>(c) * R * M;
  CONV2_MARK(0);
  pdl_wait();
  asm volatile("barrier.cluster.arrive.relaxed.aligned;\n" ::: "memory");
  // my columns' window multipliers, asynchronously (first used after the
  // first cluster barrier)
  for (int t = threadIdx.x; t < nc * nw; t += blockDim.x) {
    const int j = t / nw, i = t - j * nw;
    conv_cp_async16(mw + j * (N + 1) + i, a.mult + static_cast<int64_t>(i) * H + c + j * kClusterCtas);
  }
  asm volatile("cp.async.commit_group;\n" ::);
  for (int j = threadIdx.x; j < M; j += blockDim.x) tws[j] = a.tw[j];
  __syncthreads();
  CONV2_MARK(1);
  // 1) my rows, 2p and 2p+1 packed as z_p = g[2p] + i g[2p+1]
  const int np = R / 2;
  fft_batch<M, false>(
      scr, np, tws,
      [&](int p, int u) { return make_double2(__ldg(gin + (2 * p) * M + u), __ldg(gin + (2 * p + 1) * M + u)); },
      [&](int p, int k, double2 z) { buf0[p * M + k] = z; });
  __syncthreads();
  CONV2_MARK(2);
  // every CTA of the cluster has started (arrived) before peers' smem is written
  asm volatile("barrier.cluster.wait.aligned;\n" ::: "memory");
  for (int t = threadIdx.x; t < np * H; t += blockDim.x) {
    const int p = t / H, k = t - p * H;
    const double2 z = buf0[p * M + k];
    const double2 zc = buf0[p * M + ((M - k) & (M - 1))];
    // A_even = (Z_k + conj Z_{M-k}) / 2, A_odd = (Z_k - conj Z_{M-k}) / 2i,
    // pushed into column k's owner: colbuf[k / 8][row]
    double2* col = cluster.map_shared_rank(colbuf, k % kClusterCtas) + (k / kClusterCtas) * M + c * R + 2 * p;
    col[0] = make_double2(0.5 * (z.x + zc.x), 0.5 * (z.y - zc.y));
    col[1] = make_double2(0.5 * (z.y + zc.y), -0.5 * (z.x - zc.x));
  }
  asm volatile("cp.async.wait_all;\n" ::: "memory");
  CONV2_MARK(3);
  cluster.sync();
  CONV2_MARK(4);
  // 2) my columns: gathered through DSMEM, FFT, window multiply, inverse FFT,
  //    scattered back into the owners' A2 through DSMEM
  if (nc > 0) {
    fft_batch<M, false>(
        scr, nc, tws,
        [&](int j, int u) { return colbuf[j * M + u]; },
        [&](int j, int q, double2 f) {
          const int i = (q + hN) & (M - 1);  // window index of frequency q (mod M)
          buf0[j * M + q] = (i < nw) ? cmul(f, mw[j * (N + 1) + i]) : make_double2(0.0, 0.0);
        });
    __syncthreads();
    CONV2_MARK(5);
    fft_batch<M, true>(
        scr, nc, tws, [&](int j, int q) { return buf0[j * M + q]; },
        [&](int j, int u, double2 y) {
          double2* A2r = cluster.map_shared_rank(A2, u / R);
          A2r[(u % R) * H + c + j * kClusterCtas] = y;
        });
  }
  CONV2_MARK(6);
  cluster.sync();
  CONV2_MARK(7);
  // 3) my rows: Z = S_even + i S_odd, S the Hermitian extension of A2 (C2R)
  fft_batch<M, true>(
      scr, np, tws,
      [&](int p, int q) {
        const double2* ae = A2 + (2 * p) * H;
        const double2* ao = A2 + (2 * p + 1) * H;
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
        gout[(2 * p) * M + u] = y.x;
        gout[(2 * p + 1) * M + u] = y.y;
      });
  CONV2_MARK(8);
}

// Host dispatch over the supported grid sizes (M = 32 ... 256).
inline bool conv2_supported(int M) { return M == 32 || M == 64 || M == 128 || M == 256; }  // M / 16 rows, paired
inline const void* conv2_kernel_ptr(int M) {
  switch (M) {
    case 32: return reinterpret_cast<const void*>(conv2_cluster_kernel<32>);
    case 64: return reinterpret_cast<const void*>(conv2_cluster_kernel<64>);
    case 128: return reinterpret_cast<const void*>(conv2_cluster_kernel<128>);
    default: return reinterpret_cast<const void*>(conv2_cluster_kernel<256>);
  }
}
inline void conv2_allow_cluster(const void* k) {
  FGS_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
}
inline void conv2_launch(const Conv2Args& a, size_t smem, cudaStream_t stream) {
  static const bool allowed = [] {
    conv2_allow_cluster(reinterpret_cast<const void*>(conv2_cluster_kernel<32>));
    conv2_allow_cluster(reinterpret_cast<const void*>(conv2_cluster_kernel<64>));
    conv2_allow_cluster(reinterpret_cast<const void*>(conv2_cluster_kernel<128>));
    conv2_allow_cluster(reinterpret_cast<const void*>(conv2_cluster_kernel<256>));
    return true;
  }();
  (void)allowed;
  const dim3 grid(kClusterCtas * a.nvec), block(kConvThreads);
  switch (a.M) {
    case 32: launch_ex(conv2_cluster_kernel<32>, grid, block, smem, stream, a); break;
    case 64: launch_ex(conv2_cluster_kernel<64>, grid, block, smem, stream, a); break;
    case 128: launch_ex(conv2_cluster_kernel<128>, grid, block, smem, stream, a); break;
    default: launch_ex(conv2_cluster_kernel<256>, grid, block, smem, stream, a); break;
  }
}

}  // namespace fgsb
