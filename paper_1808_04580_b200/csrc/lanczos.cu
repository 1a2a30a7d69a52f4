// lanczos.cu -- device-resident Lanczos with full two-pass classical
// Gram-Schmidt reorthogonalisation over the fast graph operator
// (reference: spectral.cpp:141-256, lanczos_largest).
//
// The Krylov basis lives in HBM in the operator's internal point order (rows
// = this shard's slice), column-major with leading dimension n_local, and
// grows geometrically like the reference's conservativeResize
// (spectral.cpp:159,222-224).  Every reduction is a fixed-order two-stage
// tree (block partials -> ordered final sum), so a run is bitwise
// reproducible.  Sharded runs add one NCCL allreduce per reduction.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <limits>
#include <numeric>
#include <random>

#include "core.cuh"
#include "lanczos.cuh"
#include "nccl_shim.hpp"
#include "tma.cuh"

namespace fgsb {

namespace {

#ifndef FGS_LZ_RPT
#define FGS_LZ_RPT 8
#endif
#ifndef FGS_LZ_THREADS
#define FGS_LZ_THREADS 256
#endif
constexpr int kRedThreads = FGS_LZ_THREADS;
constexpr int kRowsPerThread = FGS_LZ_RPT;  // tuning builds: FGS_NVCC_DEFINES="FGS_LZ_RPT=4" 
constexpr int kRowsPerBlock = kRedThreads * kRowsPerThread;

inline int ceil_div(int64_t a, int64_t b) { return static_cast<int>((a + b - 1) / b); }

// partial[b][j] = sum over block b's rows of Q[r, j] * z[r], j < m
// (32 columns at a time per warp, transposed through a warp butterfly).
// zr: this thread's rows r = row0 + tid + i * kRedThreads, i < kRowsPerThread.
__device__ __forceinline__ void multidot_block(const double* __restrict__ Q, int64_t ldq, int m,
                                               const double (&zr)[kRowsPerThread], int64_t row0, int64_t n,
                                               double* __restrict__ partial) {
  __shared__ double red[kRedThreads / 32][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int j0 = 0; j0 < m; j0 += 32) {
    double p[32];
#pragma unroll
    for (int c = 0; c < 32; ++c) {
      double acc = 0.0;
      if (j0 + c < m) {
        // the column's loads first, read-only path: inlined into the fused
        // kernels (which also store) nvcc otherwise issued load, fma, load,
        // ... one latency per row (3.5 vs 0.9 us per column at C2)
        const double* col = Q + static_cast<int64_t>(j0 + c) * ldq;
        double qv[kRowsPerThread];
#pragma unroll
        for (int i = 0; i < kRowsPerThread; ++i) {
          const int64_t r = row0 + threadIdx.x + static_cast<int64_t>(i) * kRedThreads;
          qv[i] = r < n ? __ldg(col + r) : 0.0;
        }
#pragma unroll
        for (int i = 0; i < kRowsPerThread; ++i) {
          const int64_t r = row0 + threadIdx.x + static_cast<int64_t>(i) * kRedThreads;
          if (r < n) acc = fma(qv[i], zr[i], acc);
        }
      }
      p[c] = acc;
    }
#pragma unroll
    for (int sft = 16; sft >= 1; sft >>= 1) {
      const bool upper = (lane & sft) != 0;
#pragma unroll
      for (int k = 0; k < sft; ++k) {
        const double send = upper ? p[k] : p[k + sft];
        const double keep = upper ? p[k + sft] : p[k];
        p[k] = keep + __shfl_xor_sync(0xffffffffu, send, sft);
      }
    }
    red[warp][lane] = p[0];
    __syncthreads();
    if (warp == 0) {
      double s = 0.0;
#pragma unroll
      for (int w = 0; w < kRedThreads / 32; ++w) s += red[w][lane];
      if (j0 + lane < m) partial[static_cast<int64_t>(blockIdx.x) * m + j0 + lane] = s;
    }
    __syncthreads();
  }
}

__device__ __forceinline__ void load_rows(const double* __restrict__ z, int64_t row0, int64_t n,
                                          double (&zr)[kRowsPerThread]) {
#pragma unroll
  for (int i = 0; i < kRowsPerThread; ++i) {
    const int64_t r = row0 + threadIdx.x + static_cast<int64_t>(i) * kRedThreads;
    zr[i] = r < n ? z[r] : 0.0;
  }
}

__global__ void __launch_bounds__(kRedThreads) multidot_kernel(const double* __restrict__ Q, int64_t ldq, int m,
                                                               const double* __restrict__ z, int64_t n,
                                                               double* __restrict__ partial) {
  pdl_wait();  // PDL launches in the fused step: predecessor complete
  const int64_t row0 = static_cast<int64_t>(blockIdx.x) * kRowsPerBlock;
  double zr[kRowsPerThread];
  load_rows(z, row0, n, zr);
  multidot_block(Q, ldq, m, zr, row0, n, partial);
}

// ---- fused single-device step kernels ------------------------------------
// The block partials are summed by the last block to finish (an atomic
// ticket), in exactly reduce_partials_kernel's order, so the fused step is
// bitwise identical to the unfused one while launching half the kernels
// (C2: ~13 launches of a few microseconds each per step were most of the
// reorthogonalisation time).
__device__ __forceinline__ bool last_block_done(unsigned* ticket) {
  __shared__ bool last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  __syncthreads();
  if (last) __threadfence();
  return last;
}

__device__ __forceinline__ void reduce_cols_block(const double* partial, int nblocks, int m, double* __restrict__ out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int j = warp; j < m; j += kRedThreads / 32) {
    double s = 0.0;
    for (int b = lane; b < nblocks; b += 32) s += __ldcg(partial + static_cast<int64_t>(b) * m + j);
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) s += __shfl_down_sync(0xffffffffu, s, off);
    if (lane == 0) out[j] = s;
  }
}

// out[0..m) = Q^T z (one launch)
__global__ void __launch_bounds__(kRedThreads) multidot_reduce_kernel(const double* __restrict__ Q, int64_t ldq, int m,
                                                                      const double* __restrict__ z, int64_t n,
                                                                      double* partial, unsigned* ticket,
                                                                      double* __restrict__ out) {
  pdl_wait();  // PDL launches in the fused step: predecessor complete
  const int64_t row0 = static_cast<int64_t>(blockIdx.x) * kRowsPerBlock;
  double zr[kRowsPerThread];
  load_rows(z, row0, n, zr);
  multidot_block(Q, ldq, m, zr, row0, n, partial);
  if (ticket && last_block_done(ticket)) {  // else the caller launches reduce_partials_kernel
    reduce_cols_block(partial, gridDim.x, m, out);
    if (threadIdx.x == 0) *ticket = 0u;
  }
}

// z -= alpha q_cur + beta q_prev (three_term_kernel), then out = Q^T z
__global__ void __launch_bounds__(kRedThreads) three_term_multidot_kernel(
    double* __restrict__ z, const double* __restrict__ qcur, const double* __restrict__ qprev,
    const double* __restrict__ alpha, const double* __restrict__ beta, const double* __restrict__ Q, int64_t ldq,
    int m, int64_t n, double* partial, unsigned* ticket, double* __restrict__ out) {
  pdl_wait();  // PDL launches in the fused step: predecessor complete
  const int64_t row0 = static_cast<int64_t>(blockIdx.x) * kRowsPerBlock;
  const double a = alpha[0], b = qprev ? beta[0] : 0.0;
  double zr[kRowsPerThread];
#pragma unroll
  for (int i = 0; i < kRowsPerThread; ++i) {
    const int64_t r = row0 + threadIdx.x + static_cast<int64_t>(i) * kRedThreads;
    double v = 0.0;
    if (r < n) {
      v = z[r] - a * qcur[r];
      if (qprev) v -= b * qprev[r];
      z[r] = v;
    }
    zr[i] = v;
  }
  multidot_block(Q, ldq, m, zr, row0, n, partial);
  if (ticket && last_block_done(ticket)) {  // else the caller launches reduce_partials_kernel
    reduce_cols_block(partial, gridDim.x, m, out);
    if (threadIdx.x == 0) *ticket = 0u;
  }
}

// |z|^2 (multidot_kernel of z with itself), then step m's scalars
// (lanczos_scalars_kernel) in the last block
__global__ void __launch_bounds__(kRedThreads) norm_scalars_kernel(
    const double* __restrict__ z, int64_t n, double* partial, unsigned* ticket, const double* __restrict__ alpha,
    double* __restrict__ nrm2, double* __restrict__ beta, double* __restrict__ st, int step) {
  pdl_wait();  // PDL launches in the fused step: predecessor complete
  const int64_t row0 = static_cast<int64_t>(blockIdx.x) * kRowsPerBlock;
  double zr[kRowsPerThread];
  load_rows(z, row0, n, zr);
  multidot_block(z, n, 1, zr, row0, n, partial);
  if (last_block_done(ticket)) {
    reduce_cols_block(partial, gridDim.x, 1, nrm2 + (step - 1));
    __syncthreads();
    if (threadIdx.x == 0) {
      const double a = alpha[step - 1];
      const double b = sqrt(nrm2[step - 1]);
      const double bp = step >= 2 ? beta[step - 2] : 0.0;
      const double scale = fmax(st[0], fabs(a) + b + bp);
      st[0] = scale;
      beta[step - 1] = b;
      if (b > 1e-14 * fmax(scale, 1.0) && st[2] == 0.0) {
        st[1] = 1.0 / b;
      } else {
        st[1] = 0.0;
        if (st[2] == 0.0) st[2] = static_cast<double>(step);
      }
      *ticket = 0u;
    }
  }
}

// q_{m+1} = z / beta into the basis and the apply input
__global__ void scale2_kernel(const double* __restrict__ z, const double* __restrict__ inv, double* __restrict__ out,
                              double* __restrict__ out2, int64_t n) {
  pdl_wait();  // PDL launches in the fused step: predecessor complete
  const int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (r < n) {
    const double v = z[r] * inv[0];
    out[r] = v;
    out2[r] = v;
  }
}

// out[j] = sum_b partial[b][j]: one warp per column, lanes take block
// residues mod 32 in increasing order, then a fixed shuffle tree
// (deterministic; the serial per-column loop cost ~0.5 ms at n = 2M)
__global__ void reduce_partials_kernel(const double* __restrict__ partial, int nblocks, int m,
                                       double* __restrict__ out, int take_sqrt) {
  pdl_wait();  // PDL launches in the fused step: predecessor complete
  const int j = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (j >= m) return;
  double s = 0.0;
  for (int b = lane; b < nblocks; b += 32) s += partial[static_cast<int64_t>(b) * m + j];
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) s += __shfl_down_sync(0xffffffffu, s, off);
  if (lane == 0) out[j] = take_sqrt ? sqrt(s) : s;
}

// column-wise first index of the largest |v| (make_eigenpairs' convention,
// spectral.cpp:120-124): per block (max, first index), then ordered fold
__global__ void colmax_partial_kernel(const double* __restrict__ V, int64_t ldv, int64_t n, int chunk,
                                      double* __restrict__ pval, int64_t* __restrict__ pidx,
                                      double* __restrict__ psigned) {
  __shared__ double sv[256];
  __shared__ int64_t si[256];
  const int col = blockIdx.y;
  const int64_t r0 = static_cast<int64_t>(blockIdx.x) * chunk;
  const int64_t r1 = r0 + chunk < n ? r0 + chunk : n;
  double best = -1.0;
  int64_t bi = -1;
  for (int64_t r = r0 + threadIdx.x; r < r1; r += blockDim.x) {
    const double v = fabs(V[col * ldv + r]);
    if (v > best) {
      best = v;
      bi = r;
    }
  }
  sv[threadIdx.x] = best;
  si[threadIdx.x] = bi;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      const double v2 = sv[threadIdx.x + s];
      const int64_t i2 = si[threadIdx.x + s];
      if (v2 > sv[threadIdx.x] || (v2 == sv[threadIdx.x] && i2 >= 0 && (si[threadIdx.x] < 0 || i2 < si[threadIdx.x]))) {
        sv[threadIdx.x] = v2;
        si[threadIdx.x] = i2;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const int64_t slot = static_cast<int64_t>(col) * gridDim.x + blockIdx.x;
    pval[slot] = sv[0];
    pidx[slot] = si[0];
    psigned[slot] = si[0] >= 0 ? V[col * ldv + si[0]] : 0.0;  // the entry itself, before any scaling
  }
}

// sign[col] = -1 if V[first argmax |.|] < 0; then V[:, col] *= sign.  The
// signed entry comes from colmax_partial_kernel: every block of a column
// scales V in place, so no block may read V to decide the sign.
__global__ void colsign_kernel(double* __restrict__ V, int64_t ldv, int64_t n, const double* __restrict__ pval,
                               const double* __restrict__ psigned, int nparts) {
  const int col = blockIdx.y;
  __shared__ double sgn;
  if (threadIdx.x == 0) {
    double best = -1.0, at = 0.0;
    for (int p = 0; p < nparts; ++p) {  // parts in row order: first index wins ties
      const double v = pval[static_cast<int64_t>(col) * nparts + p];
      if (v > best) {
        best = v;
        at = psigned[static_cast<int64_t>(col) * nparts + p];
      }
    }
    sgn = (n > 0 && at < 0.0) ? -1.0 : 1.0;
  }
  __syncthreads();
  for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; r < n;
       r += static_cast<int64_t>(gridDim.x) * blockDim.x)
    V[col * ldv + r] *= sgn;
}

__global__ void unpermute_cols_kernel(const double* __restrict__ Vi, int64_t ldi, double* __restrict__ Vc,
                                      int64_t ldc, const int* __restrict__ perm, const int* __restrict__ order,
                                      int64_t n) {
  const int col = blockIdx.y;
  const int src = order[col];
  for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; r < n;
       r += static_cast<int64_t>(gridDim.x) * blockDim.x)
    Vc[col * ldc + perm[r]] = Vi[src * ldi + r];
}

// z[r] -= sum_j Q[r, j] * h[j]   (the GEMV of one CGS pass, spectral.cpp:195)
__global__ void update_kernel(const double* __restrict__ Q, int64_t ldq, int m, const double* __restrict__ h,
                              double* __restrict__ z, int64_t n) {
  pdl_wait();  // PDL launches in the fused step: predecessor complete
  extern __shared__ double hs[];
  for (int j = threadIdx.x; j < m; j += blockDim.x) hs[j] = h[j];
  __syncthreads();
  const int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (r >= n) return;
  double acc = 0.0;
  int j = 0;
  for (; j + 4 <= m; j += 4) {
    const double q0 = Q[static_cast<int64_t>(j) * ldq + r];
    const double q1 = Q[static_cast<int64_t>(j + 1) * ldq + r];
    const double q2 = Q[static_cast<int64_t>(j + 2) * ldq + r];
    const double q3 = Q[static_cast<int64_t>(j + 3) * ldq + r];
    acc = fma(q0, hs[j], acc);
    acc = fma(q1, hs[j + 1], acc);
    acc = fma(q2, hs[j + 2], acc);
    acc = fma(q3, hs[j + 3], acc);
  }
  for (; j < m; ++j) acc = fma(Q[static_cast<int64_t>(j) * ldq + r], hs[j], acc);
  z[r] -= acc;
}

// The first CGS pass's update and the second pass's projection in ONE read
// of the basis (3 basis sweeps per step instead of 4): each block stages its
// kTile3 rows of all m columns in shared memory (m bulk copies on one
// mbarrier), forms z' = z - Q h1 for its rows in update_kernel's exact
// operation order, stores z', and writes its partials of Q^T z' column-major
// (partial[j][block]) for reduce_colmajor_kernel.  m <= kTile3Cols.
// (A persistent, double-buffered variant -- one or two blocks per SM walking
// the tiles -- measured 18-21 ms per C4 solve against 10.8 ms for this one:
// four warps per SM cannot hide the tile's compute.)
constexpr int kTile3 = 128;       // rows per block (= threads)
constexpr int kTile3Cols = 128;   // basis columns the tile holds (128 KB of shared memory)

__global__ void __launch_bounds__(kTile3) update_multidot_kernel(const double* __restrict__ Q, int64_t ldq, int m,
                                                                 const double* __restrict__ h, double* __restrict__ z,
                                                                 int64_t n, double* __restrict__ partial) {
  pdl_wait();  // PDL launches in the fused step: predecessor complete
  extern __shared__ __align__(16) double tile[];  // [m][kTile3] | z'[kTile3] | h[m] | mbarrier
  double* zs = tile + static_cast<size_t>(m) * kTile3;
  double* hs = zs + kTile3;
  unsigned long long* mb = reinterpret_cast<unsigned long long*>(hs + ((m + 1) & ~1));
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int64_t r0 = static_cast<int64_t>(blockIdx.x) * kTile3;
  const int rows = static_cast<int>(n - r0 < kTile3 ? n - r0 : kTile3);
  const bool bulk = rows == kTile3 && (ldq & 1) == 0;  // 16-byte aligned full columns
  if (bulk) {
    if (t == 0) {
      mbar_init(mb, 1);
      mbar_init_fence();
      mbar_expect_tx(mb, static_cast<unsigned>(m) * kTile3 * 8u);
    }
    __syncthreads();
    for (int j = t; j < m; j += kTile3)  // one 1 KB copy per column
      bulk_g2s(tile + static_cast<size_t>(j) * kTile3, Q + static_cast<int64_t>(j) * ldq + r0, kTile3 * 8u, mb);
  } else {
    for (int j = 0; j < m; ++j)
      tile[static_cast<size_t>(j) * kTile3 + t] = t < rows ? Q[static_cast<int64_t>(j) * ldq + r0 + t] : 0.0;
  }
  for (int j = t; j < m; j += kTile3) hs[j] = h[j];
  if (bulk) mbar_wait(mb, 0);
  __syncthreads();
  // z' = z - Q h (update_kernel's order: 4-column groups, fma chain over j)
  double acc = 0.0;
  int j = 0;
  for (; j + 4 <= m; j += 4) {
    acc = fma(tile[static_cast<size_t>(j) * kTile3 + t], hs[j], acc);
    acc = fma(tile[static_cast<size_t>(j + 1) * kTile3 + t], hs[j + 1], acc);
    acc = fma(tile[static_cast<size_t>(j + 2) * kTile3 + t], hs[j + 2], acc);
    acc = fma(tile[static_cast<size_t>(j + 3) * kTile3 + t], hs[j + 3], acc);
  }
  for (; j < m; ++j) acc = fma(tile[static_cast<size_t>(j) * kTile3 + t], hs[j], acc);
  double zv = 0.0;
  if (t < rows) {
    zv = z[r0 + t] - acc;
    z[r0 + t] = zv;
  }
  zs[t] = zv;
  __syncthreads();
  // block partials of Q^T z': warp w takes columns j = w (mod 4), each lane
  // rows lane + 32 i in increasing i, then a fixed shuffle tree
  for (int c = warp; c < m; c += kTile3 / 32) {
    const double* col = tile + static_cast<size_t>(c) * kTile3;
    double sacc = 0.0;
#pragma unroll
    for (int i = 0; i < kTile3 / 32; ++i) sacc = fma(col[lane + 32 * i], zs[lane + 32 * i], sacc);
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) sacc += __shfl_down_sync(0xffffffffu, sacc, off);
    if (lane == 0) partial[static_cast<int64_t>(c) * gridDim.x + blockIdx.x] = sacc;
  }
}

inline size_t update_multidot_smem(int m) {
  return sizeof(double) * (static_cast<size_t>(m) * kTile3 + kTile3 + ((m + 1) & ~1) + 2);
}

// out[j] = sum_b partial[j][b] (column-major partials, one block per
// column): thread t sums b = t, t + 256, ... in order, then a fixed tree
__global__ void __launch_bounds__(256) reduce_colmajor_kernel(const double* __restrict__ partial, int nblocks,
                                                               double* __restrict__ out) {
  pdl_wait();  // PDL launches in the fused step: predecessor complete
  __shared__ double red[256];
  const double* col = partial + static_cast<int64_t>(blockIdx.x) * nblocks;
  double s = 0.0;
  for (int b = threadIdx.x; b < nblocks; b += 256) s += col[b];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = 128; w >= 1; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[blockIdx.x] = red[0];
}

// z -= alpha q_{m-1} + beta q_{m-2}  (spectral.cpp:186-191); alpha and the
// previous beta are read from device memory (the host runs ahead)
__global__ void three_term_kernel(double* __restrict__ z, const double* __restrict__ qcur,
                                  const double* __restrict__ qprev, const double* __restrict__ alpha,
                                  const double* __restrict__ beta, int64_t n) {
  const int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (r >= n) return;
  double v = z[r] - alpha[0] * qcur[r];
  if (qprev) v -= beta[0] * qprev[r];
  z[r] = v;
}

// step m's scalars on the device: beta = sqrt(|z|^2), the running scale
// max(|alpha| + beta + beta_prev) and the breakdown test
// beta > 1e-14 max(scale, 1) (spectral.cpp:197-199, 225); inv = 1 / beta.
// st[0] = scale, st[1] = 1 / beta (0 on breakdown), st[2] = first
// breakdown step (+1) or 0.
__global__ void lanczos_scalars_kernel(const double* __restrict__ alpha, const double* __restrict__ nrm2,
                                       double* __restrict__ beta, double* __restrict__ st, int m) {
  const double a = alpha[m - 1];
  const double b = sqrt(nrm2[m - 1]);
  const double bp = m >= 2 ? beta[m - 2] : 0.0;
  const double scale = fmax(st[0], fabs(a) + b + bp);
  st[0] = scale;
  if (b > 1e-14 * fmax(scale, 1.0) && st[2] == 0.0) {
    beta[m - 1] = b;
    st[1] = 1.0 / b;
  } else {
    beta[m - 1] = b;  // the raw value, for the convergence estimate
    st[1] = 0.0;
    if (st[2] == 0.0) st[2] = static_cast<double>(m);
  }
}

__global__ void scale_dev_kernel(const double* __restrict__ z, const double* __restrict__ inv,
                                 double* __restrict__ out, int64_t n) {
  const int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (r < n) out[r] = z[r] * inv[0];
}

__global__ void scale_kernel(const double* __restrict__ z, double inv, double* __restrict__ out, int64_t n) {
  const int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (r < n) out[r] = z[r] * inv;
}

// V[:, i] = Q_m S[:, i]   (Ritz vectors, spectral.cpp:250); S row-major m x k
template <int KC>
__global__ void ritz_kernel(const double* __restrict__ Q, int64_t ldq, int m, const double* __restrict__ S, int k,
                            int c0, double* __restrict__ V, int64_t ldv, int64_t n) {
  const int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (r >= n) return;
  double acc[KC];
#pragma unroll
  for (int i = 0; i < KC; ++i) acc[i] = 0.0;
  for (int j = 0; j < m; ++j) {
    const double q = Q[static_cast<int64_t>(j) * ldq + r];
#pragma unroll
    for (int i = 0; i < KC; ++i)
      if (c0 + i < k) acc[i] = fma(q, __ldg(S + static_cast<int64_t>(j) * k + c0 + i), acc[i]);
  }
#pragma unroll
  for (int i = 0; i < KC; ++i)
    if (c0 + i < k) V[static_cast<int64_t>(c0 + i) * ldv + r] = acc[i];
}

// ---- start vector on the device (spectral.cpp:152-156) ---------------------
// std::mt19937_64 as a sequence: w[0..312) is the seeded state, and every
// later word is w[k + 312] = w[k + 156] ^ twist(w[k], w[k + 1]); output j is
// temper(w[312 + j]).  The 156 words of one round depend only on earlier
// rounds, so one CTA produces them in parallel per round from a ring of 1024
// words (a round reads [k, k + 312) and writes [k + 312, k + 468)).
constexpr int kMtN = 312, kMtM = 156;

__device__ __forceinline__ unsigned long long mt_next(unsigned long long a, unsigned long long b,
                                                      unsigned long long c) {
  const unsigned long long y = (a & 0xFFFFFFFF80000000ull) | (b & 0x7FFFFFFFull);
  return c ^ (y >> 1) ^ ((y & 1ull) ? 0xB5026F5AA96619E9ull : 0ull);
}

__device__ __forceinline__ unsigned long long mt_temper(unsigned long long y) {
  y ^= (y >> 29) & 0x5555555555555555ull;
  y ^= (y << 17) & 0x71D67FFFEDA60000ull;
  y ^= (y << 37) & 0xFFF7EEE000000000ull;
  return y ^ (y >> 43);
}

// uniform_real_distribution<double>(-1, 1) over libstdc++'s
// generate_canonical<double, 53>: one 64-bit draw, (double) r / 2^64 clamped
// below 1, then u * (b - a) + a
__device__ __forceinline__ double mt_uniform(unsigned long long r) {
  double u = __dmul_rn(__ull2double_rn(r), 0x1p-64);
  if (u >= 1.0) u = 0x1.fffffffffffffp-1;
  return __dadd_rn(__dmul_rn(u, 2.0), -1.0);
}

__global__ void __launch_bounds__(kMtM) mt_uniform_kernel(const unsigned long long* __restrict__ seeded, int64_t n,
                                                          double* __restrict__ out) {
  __shared__ unsigned long long ring[1024];
  for (int i = threadIdx.x; i < kMtN; i += blockDim.x) ring[i] = seeded[i];
  __syncthreads();
  for (int64_t base = 0; base < n; base += kMtM) {
    const int64_t k = base + threadIdx.x;
    const unsigned long long w = mt_next(ring[k & 1023], ring[(k + 1) & 1023], ring[(k + kMtM) & 1023]);
    ring[(k + kMtN) & 1023] = w;
    if (k < n) out[k] = mt_uniform(mt_temper(w));
    __syncthreads();
  }
}

constexpr int kSqBlocks = 256, kSqThreads = 256;

// fixed-order sum of squares: block b's rows, then a block tree
__global__ void __launch_bounds__(kSqThreads) sumsq_partial_kernel(const double* __restrict__ v, int64_t n,
                                                                   double* __restrict__ partial) {
  __shared__ double red[kSqThreads];
  const int64_t per = (n + gridDim.x - 1) / gridDim.x;
  const int64_t lo = blockIdx.x * per, hi = lo + per < n ? lo + per : n;
  double acc = 0.0;
  for (int64_t r = lo + threadIdx.x; r < hi; r += blockDim.x) acc = fma(v[r], v[r], acc);
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int s = kSqThreads / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) partial[blockIdx.x] = red[0];
}

// basis[:, 0][p] = start[perm[offset + p]] / |start| (every block sums the
// partials in the same order)
__global__ void __launch_bounds__(kSqThreads) start_scatter_kernel(const double* __restrict__ start,
                                                                   const double* __restrict__ partial,
                                                                   const int* __restrict__ perm, int64_t offset,
                                                                   int64_t nl, double* __restrict__ q) {
  __shared__ double red[kSqBlocks];
  for (int i = threadIdx.x; i < kSqBlocks; i += blockDim.x) red[i] = partial[i];
  __syncthreads();
  for (int s = kSqBlocks / 2; s > 0; s >>= 1) {
    for (int i = threadIdx.x; i < s; i += blockDim.x) red[i] += red[i + s];
    __syncthreads();
  }
  const double sn = sqrt(red[0]);
  for (int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; p < nl;
       p += static_cast<int64_t>(gridDim.x) * blockDim.x)
    q[p] = start[perm[offset + p]] / sn;
}

}  // namespace

// ---------------------------------------------------------------------------
// Symmetric tridiagonal eigensolver (the role of Eigen's
// SelfAdjointEigenSolver::computeFromTridiagonal, spectral.cpp:174-179):
// implicit QL with Wilkinson shifts; eigenvalues ascending, eigenvectors
// as columns of z (column-major m x m).
// ---------------------------------------------------------------------------
void tridiagonal_eigen(int m, std::vector<double>& dg, const std::vector<double>& offd, std::vector<double>& z) {
  const double eps = std::numeric_limits<double>::epsilon();
  z.assign(static_cast<size_t>(m) * m, 0.0);
  for (int i = 0; i < m; ++i) z[static_cast<size_t>(i) * m + i] = 1.0;
  std::vector<double> e(static_cast<size_t>(m), 0.0);
  for (int i = 0; i + 1 < m; ++i) e[static_cast<size_t>(i)] = offd[static_cast<size_t>(i)];
  for (int l = 0; l < m; ++l) {
    for (int iter = 0;; ++iter) {
      int mm = l;
      while (mm < m - 1 && std::abs(e[mm]) > eps * (std::abs(dg[mm]) + std::abs(dg[mm + 1]))) ++mm;
      if (mm == l) break;
      if (iter > 64) fail(FGS_ENUMERIC, "tridiagonal eigensolver did not converge");
      double g = (dg[l + 1] - dg[l]) / (2.0 * e[l]);
      double r = std::hypot(g, 1.0);
      g = dg[mm] - dg[l] + e[l] / (g + std::copysign(r, g));
      double s = 1.0, c = 1.0, p = 0.0;
      bool deflated = false;
      for (int i = mm - 1; i >= l; --i) {
        double f = s * e[i], bb = c * e[i];
        r = std::hypot(f, g);
        e[i + 1] = r;
        if (r == 0.0) {
          dg[i + 1] -= p;
          e[mm] = 0.0;
          deflated = true;
          break;
        }
        s = f / r;
        c = g / r;
        g = dg[i + 1] - p;
        r = (dg[i] - g) * s + 2.0 * c * bb;
        p = s * r;
        dg[i + 1] = g + p;
        g = c * r - bb;
        double* zi = &z[static_cast<size_t>(i) * m];
        double* zi1 = &z[static_cast<size_t>(i + 1) * m];
        for (int k = 0; k < m; ++k) {
          const double t = zi1[k];
          zi1[k] = s * zi[k] + c * t;
          zi[k] = c * zi[k] - s * t;
        }
      }
      if (deflated) continue;
      dg[l] -= p;
      e[l] = g;
      e[mm] = 0.0;
    }
  }
  std::vector<int> order(static_cast<size_t>(m));
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return dg[a] < dg[b]; });
  std::vector<double> d2(static_cast<size_t>(m)), z2(z.size());
  for (int i = 0; i < m; ++i) {
    d2[static_cast<size_t>(i)] = dg[static_cast<size_t>(order[i])];
    std::copy(&z[static_cast<size_t>(order[i]) * m], &z[static_cast<size_t>(order[i]) * m] + m,
              &z2[static_cast<size_t>(i) * m]);
  }
  dg.swap(d2);
  z.swap(z2);
}

// ---------------------------------------------------------------------------
LanczosResult lanczos_device(Core& c, int which, int k, int max_iter, double tol, uint64_t seed, bool want_vectors) {
  const int64_t n = c.n, nl = c.n_local;
  if (k < 1) fail(FGS_EPARAM, "at least one eigenpair must be requested");
  if (k > n) fail(FGS_EPARAM, "requested pairs must not exceed the operator dimension");
  if (max_iter < 1) fail(FGS_EPARAM, "max_iter must be positive");
  if (!(tol > 0.0)) fail(FGS_EPARAM, "tolerance must be positive");
  const double kEps = std::numeric_limits<double>::epsilon();
  cudaStream_t st = c.stream;
  const int epi = which == 0 ? EPI_NORMALIZED : EPI_LAPLACIAN;
  const auto entry = std::chrono::steady_clock::now();

  // start vector: mt19937_64(seed) uniform(-1, 1) over the caller order,
  // normalised (spectral.cpp:152-156), drawn on the device (the host draw +
  // permutation cost 27 ms of a 137 ms C4 solve); the host generator is
  // advanced past those n draws only if a breakdown restart needs it
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> unif(-1.0, 1.0);
  bool rng_at_restart = false;
  std::vector<double> local;
  {
    unsigned long long seeded[kMtN];
    seeded[0] = seed;
    for (int i = 1; i < kMtN; ++i)  // the standard's seeding (mersenne_twister_engine::seed)
      seeded[i] = 6364136223846793005ull * (seeded[i - 1] ^ (seeded[i - 1] >> 62)) + static_cast<unsigned long long>(i);
    c.lz_mt.upload(seeded, kMtN, st);
    c.lz_start.alloc(static_cast<size_t>(n));
    c.lz_sq.alloc(kSqBlocks);
    mt_uniform_kernel<<<1, kMtM, 0, st>>>(c.lz_mt.p, n, c.lz_start.p);
    sumsq_partial_kernel<<<kSqBlocks, kSqThreads, 0, st>>>(c.lz_start.p, n, c.lz_sq.p);
    c.launches += 2;
  }

  // initial basis width: the reference grows from 64 columns geometrically
  // (conservativeResize); k-dependent pre-sizing (4k + 8, C4's k = 20
  // converges in 76 steps) avoids the first solve's 2x reallocation and
  // basis copy (1 GB at C4)
  int64_t cap = std::min<int64_t>(std::min<int64_t>(n, std::max<int64_t>(max_iter, 1)),
                                  std::max<int64_t>(64, 4 * static_cast<int64_t>(k) + 8));
  // workspace kept on the handle between solves: no re-allocation, and the
  // apply's input/output addresses stay fixed, so its cached CUDA graph is
  // replayed instead of re-captured on every call
  DBuf<double>& basis = c.lz_basis;
  DBuf<double>& z = c.lz_z;
  DBuf<double>& partial = c.lz_partial;
  DBuf<double>& hbuf = c.lz_hbuf;
  DBuf<double>& scal = c.lz_scal;
  DBuf<double>& qin = c.lz_qin;
  basis.alloc(static_cast<size_t>(std::max<int64_t>(nl, 1)) * cap);
  cap = std::max<int64_t>(cap, std::min<int64_t>(n, static_cast<int64_t>(basis.n) / std::max<int64_t>(nl, 1)));
  z.alloc(static_cast<size_t>(std::max<int64_t>(nl, 1)));
  qin.alloc(static_cast<size_t>(std::max<int64_t>(nl, 1)));  // fixed apply input -> graph-cached apply
  const int nblk = std::max(1, ceil_div(nl, kRowsPerBlock));
  hbuf.alloc(static_cast<size_t>(std::min<int64_t>(n, max_iter) + 2));
  partial.alloc(static_cast<size_t>(nblk) * (std::min<int64_t>(n, max_iter) + 2));
  // partials of the staged-tile update + projection (steps with <= kTile3Cols columns)
  const int nblk3 = std::max(1, ceil_div(nl, kTile3));
  DBuf<double>& partial3 = c.lz_partial3;
  partial3.alloc(static_cast<size_t>(nblk3) * kTile3Cols);
  {
    static bool attr = false;
    if (!attr) {
      FGS_CUDA(cudaFuncSetAttribute(reinterpret_cast<const void*>(update_multidot_kernel),
                                    cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(update_multidot_smem(kTile3Cols))));
      attr = true;
    }
  }
  scal.alloc(4);
  start_scatter_kernel<<<std::max(1, std::min(ceil_div(std::max<int64_t>(nl, 1), kSqThreads), 1184)), kSqThreads, 0,
                         st>>>(c.lz_start.p, c.lz_sq.p, c.perm.p, c.offset, nl, basis.p);
  ++c.launches;

  auto allreduce = [&](double* v, int count) {
    if (c.sharded)
      nccl_check(nccl().all_reduce(v, v, static_cast<size_t>(count), ncclDouble, ncclSum, c.comm, st),
                 "ncclAllReduce in Lanczos");
  };
  // out[0..m) = Q[:, 0..m)^T v  (global, fixed order)
  auto multidot = [&](const double* Q, int m, const double* v, double* out) {
    multidot_kernel<<<nblk, kRedThreads, 0, st>>>(Q, nl, m, v, nl, partial.p);
    reduce_partials_kernel<<<ceil_div(m, 8), 256, 0, st>>>(partial.p, nblk, m, out, 0);
    c.launches += 2;
    allreduce(out, m);
  };
  auto update = [&](const double* Q, int m, const double* h, double* v) {
    update_kernel<<<ceil_div(std::max<int64_t>(nl, 1), 256), 256, sizeof(double) * m, st>>>(Q, nl, m, h, v, nl);
    ++c.launches;
  };
  auto cgs_pass = [&](int m, double* v) {  // v -= Q(Q^T v)
    multidot(basis.p, m, v, hbuf.p);
    update(basis.p, m, hbuf.p, v);
  };
  // two CGS passes (spectral.cpp:193-195) in three basis sweeps: h1 = Q^T v;
  // v -= Q h1 with h2 = Q^T v from the same staged tile; v -= Q h2
  auto cgs2 = [&](int m, double* v) {
    if (m > kTile3Cols) {
      cgs_pass(m, v);
      cgs_pass(m, v);
      return;
    }
    multidot(basis.p, m, v, hbuf.p);
    update_multidot_kernel<<<nblk3, kTile3, update_multidot_smem(m), st>>>(basis.p, nl, m, hbuf.p, v, nl,
                                                                          partial3.p);
    reduce_colmajor_kernel<<<m, 256, 0, st>>>(partial3.p, nblk3, hbuf.p);
    c.launches += 2;
    allreduce(hbuf.p, m);
    update(basis.p, m, hbuf.p, v);
  };
  auto norm_of = [&](const double* v) -> double {
    multidot(v, 1, v, scal.p + 1);
    double h = 0.0;
    FGS_CUDA(cudaMemcpyAsync(&h, scal.p + 1, sizeof(double), cudaMemcpyDeviceToHost, st));
    FGS_CUDA(cudaStreamSynchronize(st));
    return std::sqrt(h);
  };

  std::vector<double> alphas, betas, tvals, tvecs;
  int tri_size = 0, iterations = 0, next_check = k;
  double scale = 0.0;
  bool converged = false;
  auto solve_tri = [&](int m) {
    tvals.assign(alphas.begin(), alphas.begin() + m);
    std::vector<double> sub(betas.begin(), betas.begin() + (m - 1));
    tridiagonal_eigen(m, tvals, sub, tvecs);
    tri_size = m;
  };

  // Run-ahead recurrence: alpha_m, |z|^2 and beta_m live in device arrays
  // and step m's 1/beta is formed on the device (lanczos_scalars_kernel), so
  // the host enqueues steps without waiting and synchronises only where the
  // reference needs host values: its geometric convergence checks
  // (spectral.cpp:200-215), the iteration cap, basis growth, or a
  // breakdown -- which rolls the run back to that step and takes the
  // reference's random restart (spectral.cpp:225-238) on the host.
  const int64_t amax = std::min<int64_t>(n, max_iter) + 2;
  DBuf<double>& dalpha = c.lz_alpha;
  DBuf<double>& dnrm = c.lz_nrm;
  DBuf<double>& dbeta = c.lz_beta;
  DBuf<double>& dst = c.lz_st;
  dalpha.alloc(static_cast<size_t>(amax));
  dnrm.alloc(static_cast<size_t>(amax));
  dbeta.alloc(static_cast<size_t>(amax));
  dst.alloc(4);
  FGS_CUDA(cudaMemsetAsync(dst.p, 0, 4 * sizeof(double), st));
  const int gsz = ceil_div(std::max<int64_t>(nl, 1), 256);

  // per-phase device timing (operator applies vs reorthogonalisation)
  std::vector<cudaEvent_t>& evpool = c.lz_events;  // kept on the handle: no create/destroy per solve
  auto ev_at = [&](size_t i) {
    while (evpool.size() <= i) {
      cudaEvent_t e;
      FGS_CUDA(cudaEventCreate(&e));
      evpool.push_back(e);
    }
    return evpool[i];
  };
  double apply_ms = 0.0, reorth_ms = 0.0;
  const auto wall0 = std::chrono::steady_clock::now();
  static const bool trace = std::getenv("FGS_LANCZOS_TRACE") != nullptr;
  auto now_ms = [] {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
  };
  double t_launch = 0.0, t_sync = 0.0, t_tri = 0.0;
  int syncs = 0;

  // enqueue step mm (1-based): z = A q_mm, alpha, three-term, CGS2, |z|^2,
  // scalars, q_{mm+1} = z / beta (when the basis has room)
  // single device: fused step kernels (last-block reductions, the three-term
  // folded into the first Gram-Schmidt product, the second update into the
  // norm and the scalars), bitwise identical to the unfused sequence below,
  // which sharded runs keep for their allreduces; FGS_LANCZOS_FUSED=0 forces it
  static const bool fused_env = [] {
    const char* e = std::getenv("FGS_LANCZOS_FUSED");
    return !(e && std::atoi(e) == 0);
  }();
  const bool fused = fused_env && !c.sharded;
  DBuf<unsigned>& ticket = c.lz_ticket;
  if (!ticket.p) {
    ticket.alloc(4);
    FGS_CUDA(cudaMemsetAsync(ticket.p, 0, 4 * sizeof(unsigned), st));
  }
  int qin_holds = 0;  // basis column (1-based) currently in qin, 0 = none
  auto enqueue_fused = [&](int mm, size_t evbase) {
    const double* qcur = basis.p + static_cast<int64_t>(mm - 1) * nl;
    FGS_CUDA(cudaEventRecord(ev_at(evbase), st));
    if (qin_holds != mm) FGS_CUDA(cudaMemcpyAsync(qin.p, qcur, sizeof(double) * nl, cudaMemcpyDeviceToDevice, st));
    c.apply(epi, qin.p, nl, z.p, nl, 1, false, true);
    FGS_CUDA(cudaEventRecord(ev_at(evbase + 1), st));
    // one block sums the partials when they are few (C2: 49 blocks); many
    // blocks x columns (C4: 977 x 76) would serialise on it, so those
    // products keep the separate column-parallel reduction
    const bool tail = static_cast<int64_t>(nblk) * mm <= 8192;
    const dim3 gb(nblk), tb(kRedThreads), gu(gsz), tu(256), gr(ceil_div(mm, 8));
    const double* qprev = mm >= 2 ? basis.p + static_cast<int64_t>(mm - 2) * nl : nullptr;
    unsigned* tk = tail ? ticket.p : nullptr;
    launch_ex(multidot_reduce_kernel, gb, tb, 0, st, qcur, nl, 1, z.p, nl, partial.p, ticket.p, dalpha.p + (mm - 1));
    launch_ex(three_term_multidot_kernel, gb, tb, 0, st, z.p, qcur, qprev, dalpha.p + (mm - 1),
              mm >= 2 ? dbeta.p + (mm - 2) : dbeta.p, basis.p, nl, mm, nl, partial.p, tk, hbuf.p);
    if (!tail) {
      launch_ex(reduce_partials_kernel, gr, tu, 0, st, partial.p, nblk, mm, hbuf.p, 0);
      ++c.launches;
    }
    if (mm <= kTile3Cols) {  // first update + second projection from one staged tile (cgs2)
      launch_ex(update_multidot_kernel, dim3(nblk3), dim3(kTile3), update_multidot_smem(mm), st, basis.p, nl, mm,
                hbuf.p, z.p, nl, partial3.p);
      launch_ex(reduce_colmajor_kernel, dim3(mm), dim3(256), 0, st, partial3.p, nblk3, hbuf.p);
      ++c.launches;
    } else {
      launch_ex(update_kernel, gu, tu, sizeof(double) * mm, st, basis.p, nl, mm, hbuf.p, z.p, nl);
      launch_ex(multidot_reduce_kernel, gb, tb, 0, st, basis.p, nl, mm, z.p, nl, partial.p, tk, hbuf.p);
      if (!tail) {
        launch_ex(reduce_partials_kernel, gr, tu, 0, st, partial.p, nblk, mm, hbuf.p, 0);
        ++c.launches;
      }
    }
    launch_ex(update_kernel, gu, tu, sizeof(double) * mm, st, basis.p, nl, mm, hbuf.p, z.p, nl);
    launch_ex(norm_scalars_kernel, gb, tb, 0, st, z.p, nl, partial.p, ticket.p, dalpha.p, dnrm.p, dbeta.p, dst.p, mm);
    c.launches += 6;
    if (mm < cap) {
      launch_ex(scale2_kernel, gu, tu, 0, st, z.p, dst.p + 1, basis.p + static_cast<int64_t>(mm) * nl, qin.p, nl);
      ++c.launches;
      qin_holds = mm + 1;
    } else {
      qin_holds = 0;
    }
    FGS_CUDA(cudaEventRecord(ev_at(evbase + 2), st));
  };
  auto enqueue_step = [&](int mm, size_t evbase) {
    if (fused) return enqueue_fused(mm, evbase);
    const double* qcur = basis.p + static_cast<int64_t>(mm - 1) * nl;
    FGS_CUDA(cudaEventRecord(ev_at(evbase), st));
    FGS_CUDA(cudaMemcpyAsync(qin.p, qcur, sizeof(double) * nl, cudaMemcpyDeviceToDevice, st));
    c.apply(epi, qin.p, nl, z.p, nl, 1, false, true);
    FGS_CUDA(cudaEventRecord(ev_at(evbase + 1), st));
    multidot(qcur, 1, z.p, dalpha.p + (mm - 1));
    three_term_kernel<<<gsz, 256, 0, st>>>(z.p, qcur, mm >= 2 ? basis.p + static_cast<int64_t>(mm - 2) * nl : nullptr,
                                           dalpha.p + (mm - 1), mm >= 2 ? dbeta.p + (mm - 2) : dbeta.p, nl);
    cgs2(mm, z.p);
    multidot(z.p, 1, z.p, dnrm.p + (mm - 1));
    lanczos_scalars_kernel<<<1, 1, 0, st>>>(dalpha.p, dnrm.p, dbeta.p, dst.p, mm);
    if (mm < cap) scale_dev_kernel<<<gsz, 256, 0, st>>>(z.p, dst.p + 1, basis.p + static_cast<int64_t>(mm) * nl, nl);
    c.launches += 3;
    FGS_CUDA(cudaEventRecord(ev_at(evbase + 2), st));
  };

  while (true) {
    const int m0 = static_cast<int>(alphas.size()) + 1;  // first step of this batch
    // last step before the host must look: check point, cap, basis room, n
    int mt = m0;
    while (true) {
      const bool check = mt >= k && mt >= next_check;
      const bool stop = iterations + (mt - m0 + 1) >= max_iter || mt == static_cast<int>(n) || mt == cap;
      if (check || stop) break;
      ++mt;
    }
    const double h0 = now_ms();
    for (int mm = m0; mm <= mt; ++mm) enqueue_step(mm, 3 * static_cast<size_t>(mm - m0));
    const double h1 = now_ms();
    const int cnt = mt - m0 + 1;
    std::vector<double> ha(static_cast<size_t>(cnt)), hb(static_cast<size_t>(cnt)), hs(3);
    FGS_CUDA(cudaMemcpyAsync(ha.data(), dalpha.p + (m0 - 1), sizeof(double) * cnt, cudaMemcpyDeviceToHost, st));
    FGS_CUDA(cudaMemcpyAsync(hb.data(), dbeta.p + (m0 - 1), sizeof(double) * cnt, cudaMemcpyDeviceToHost, st));
    FGS_CUDA(cudaMemcpyAsync(hs.data(), dst.p, sizeof(double) * 3, cudaMemcpyDeviceToHost, st));
    FGS_CUDA(cudaStreamSynchronize(st));
    ++syncs;
    const double h2 = now_ms();
    t_launch += h1 - h0;
    t_sync += h2 - h1;
    const int mb = static_cast<int>(hs[2]);  // first breakdown step of the batch, or 0
    const int last_valid = mb > 0 ? mb : mt;  // steps after a breakdown ran on garbage
    for (int mm = m0; mm <= last_valid; ++mm) {
      float t01 = 0.f, t12 = 0.f;
      const size_t e = 3 * static_cast<size_t>(mm - m0);
      FGS_CUDA(cudaEventElapsedTime(&t01, ev_at(e), ev_at(e + 1)));
      FGS_CUDA(cudaEventElapsedTime(&t12, ev_at(e + 1), ev_at(e + 2)));
      apply_ms += t01;
      reorth_ms += t12;
    }
    iterations += last_valid - m0 + 1;
    // steps m0 .. last_valid - 1 continue normally: alpha and beta accepted
    for (int mm = m0; mm < last_valid; ++mm) {
      const double beta_prev = mm >= 2 ? betas[static_cast<size_t>(mm - 2)] : 0.0;
      alphas.push_back(ha[static_cast<size_t>(mm - m0)]);
      scale = std::max(scale, std::abs(alphas.back()) + hb[static_cast<size_t>(mm - m0)] + beta_prev);
      betas.push_back(hb[static_cast<size_t>(mm - m0)]);
    }
    // the batch's last valid step: the reference's per-step decisions
    const int m = last_valid;
    const double alpha = ha[static_cast<size_t>(m - m0)], beta = hb[static_cast<size_t>(m - m0)];
    const double beta_prev = m >= 2 ? betas[static_cast<size_t>(m - 2)] : 0.0;
    alphas.push_back(alpha);
    scale = std::max(scale, std::abs(alpha) + beta + beta_prev);
    const bool last = iterations >= max_iter || m == static_cast<int>(n);
    const double h3 = now_ms();
    if (m >= k && (m >= next_check || last)) {  // spectral.cpp:200-215
      solve_tri(m);
      bool all_small = true;
      for (int i = 0; i < k && all_small; ++i) {
        const double theta = tvals[static_cast<size_t>(m - 1 - i)];
        const double est = beta * std::abs(tvecs[static_cast<size_t>(m - 1 - i) * m + (m - 1)]);
        if (est > tol * std::max(std::abs(theta), kEps * std::max(scale, 1.0))) all_small = false;
      }
      if (all_small) {
        converged = true;
        break;
      }
      next_check = m + std::max(8, m / 8);
    }
    if (iterations >= max_iter) break;
    if (m == static_cast<int>(n)) {
      converged = true;
      break;
    }
    const bool grew = m == cap;
    if (grew) {  // geometric growth (conservativeResize)
      const int64_t ncap = std::min<int64_t>(n, cap * 2);
      DBuf<double> nb;
      nb.alloc(static_cast<size_t>(std::max<int64_t>(nl, 1)) * ncap);
      FGS_CUDA(cudaMemcpyAsync(nb.p, basis.p, sizeof(double) * nl * cap, cudaMemcpyDeviceToDevice, st));
      FGS_CUDA(cudaStreamSynchronize(st));
      std::swap(basis.p, nb.p);
      std::swap(basis.n, nb.n);
      cap = ncap;
    }
    const double h4 = now_ms();
    t_tri += h4 - h3;
    double* qnext = basis.p + static_cast<int64_t>(m) * nl;
    if (mb == 0 && beta > 1e-14 * std::max(scale, 1.0)) {
      betas.push_back(beta);
      if (grew) {  // q_{m+1} was not formed before the basis had room
        scale_dev_kernel<<<gsz, 256, 0, st>>>(z.p, dst.p + 1, qnext, nl);
        ++c.launches;
      }
      // the reference divides z / beta; multiplying by the reciprocal
      // differs by one rounding (<= 1 ulp per entry)
    } else {
      // breakdown: fresh random direction orthogonal to the basis
      // (spectral.cpp:59-75, 225-238), same RNG stream as the start vector
      qin_holds = 0;  // the host forms q_{m+1}
      if (!rng_at_restart) {  // the start vector's n draws happened on the device
        rng.discard(static_cast<unsigned long long>(n));
        local.resize(static_cast<size_t>(std::max<int64_t>(nl, 1)));
        rng_at_restart = true;
      }
      bool found = false;
      for (int attempt = 0; attempt < 8 && !found; ++attempt) {
        std::vector<double> v(static_cast<size_t>(n));
        for (int64_t i = 0; i < n; ++i) v[static_cast<size_t>(i)] = unif(rng);
        for (int64_t p = 0; p < nl; ++p) local[static_cast<size_t>(p)] = v[static_cast<size_t>(c.host_perm[static_cast<size_t>(c.offset + p)])];
        FGS_CUDA(cudaMemcpyAsync(z.p, local.data(), sizeof(double) * nl, cudaMemcpyHostToDevice, st));
        cgs_pass(m, z.p);
        cgs_pass(m, z.p);
        const double nv = norm_of(z.p);
        if (nv > 1e-8) {
          scale_kernel<<<gsz, 256, 0, st>>>(z.p, 1.0 / nv, qnext, nl);
          ++c.launches;
          found = true;
        }
      }
      if (!found) {
        converged = true;
        break;
      }
      betas.push_back(0.0);
      // device state for the next step: beta_m = 0 (the three-term's
      // beta_prev), breakdown flag cleared, scale as on the host
      const double zero = 0.0, reset[3] = {scale, 0.0, 0.0};
      FGS_CUDA(cudaMemcpyAsync(dbeta.p + (m - 1), &zero, sizeof(double), cudaMemcpyHostToDevice, st));
      FGS_CUDA(cudaMemcpyAsync(dst.p, reset, 3 * sizeof(double), cudaMemcpyHostToDevice, st));
      FGS_CUDA(cudaStreamSynchronize(st));
    }
  }

  if (trace)
    std::fprintf(stderr, "[lanczos] host syncs %d\n", syncs);
  if (trace)
    std::fprintf(stderr,
                 "[lanczos] iters %d  device apply %.2f ms  reorth %.2f ms | host launch %.2f ms  sync-wait %.2f ms  "
                 "tridiag %.2f ms  loop wall %.2f ms\n",
                 iterations, apply_ms, reorth_ms, t_launch, t_sync, t_tri,
                 std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - wall0).count());
  const int m = static_cast<int>(alphas.size());
  if (tri_size != m) solve_tri(m);
  const int wanted = std::min(k, m);
  LanczosResult res;
  res.iterations = iterations;
  res.converged = converged;
  res.apply_ms = apply_ms;
  res.reorth_ms = reorth_ms;
  res.loop_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - wall0).count();
  res.values.resize(static_cast<size_t>(wanted));
  std::vector<double> S(static_cast<size_t>(m) * wanted);  // row-major m x wanted
  for (int i = 0; i < wanted; ++i) {
    res.values[static_cast<size_t>(i)] = tvals[static_cast<size_t>(m - 1 - i)];
    for (int j = 0; j < m; ++j)
      S[static_cast<size_t>(j) * wanted + i] = tvecs[static_cast<size_t>(m - 1 - i) * m + j];
  }
  if (want_vectors) {
    DBuf<double>& dS = c.lz_S;
    dS.upload(S.data(), S.size(), st);
    res.vectors_dev = std::move(c.lz_vecs);  // handed back by lanczos_finish_vectors
    res.vectors_dev.alloc(static_cast<size_t>(std::max<int64_t>(nl, 1)) * wanted);
    for (int c0 = 0; c0 < wanted; c0 += 8) {
      ritz_kernel<8><<<ceil_div(std::max<int64_t>(nl, 1), 128), 128, 0, st>>>(basis.p, nl, m, dS.p, wanted, c0,
                                                                             res.vectors_dev.p, nl, nl);
      ++c.launches;
    }
  }
  FGS_CUDA(cudaStreamSynchronize(st));
  FGS_CUDA(cudaGetLastError());
  if (trace) {
    const auto end = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[lanczos] prologue %.2f ms  loop %.2f ms  ritz %.2f ms\n",
                 std::chrono::duration<double, std::milli>(wall0 - entry).count(), res.loop_ms,
                 std::chrono::duration<double, std::milli>(end - wall0).count() - res.loop_ms);
  }
  return res;
}

namespace {
__global__ void div_scalar_kernel(const double* __restrict__ z, double beta, double* __restrict__ out, int64_t n) {
  const int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (r < n) out[r] = z[r] / beta;  // basis.col(m) = z / beta (spectral.cpp:227)
}
}  // namespace

// lanczos_largest over a generic symmetric operator given as a host callback
// (the reference's SymmetricOperatorHandle, spectral.hpp:18-30: dense_handle,
// user operators).  The recurrence runs on the device -- basis in HBM,
// alpha, the three-term update, both classical Gram-Schmidt passes and beta
// by the same fixed-order kernels as lanczos_device -- and each step moves
// q_m to the host for the caller's apply and z back.  Control flow, start
// vector, convergence schedule, breakdown restart and Ritz conventions are
// spectral.cpp:141-256's; q_{m+1} = z / beta by division as the reference.
void lanczos_operator(int64_t n, OperatorApply apply, void* ctx, int device, int k, int max_iter, double tol,
                      uint64_t seed, double* values, double* vectors, int* count, int* iterations, int* converged) {
  if (n < 1 || apply == nullptr) fail(FGS_EPARAM, "operator handle is empty");
  if (k < 1) fail(FGS_EPARAM, "at least one eigenpair must be requested");
  if (k > n) fail(FGS_EPARAM, "requested pairs must not exceed the operator dimension");
  if (max_iter < 1) fail(FGS_EPARAM, "max_iter must be positive");
  if (!(tol > 0.0)) fail(FGS_EPARAM, "tolerance must be positive");
  const double kEps = std::numeric_limits<double>::epsilon();
  FGS_CUDA(cudaSetDevice(device));
  cudaStream_t st;
  FGS_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  struct StreamGuard {
    cudaStream_t s;
    ~StreamGuard() {
      cudaStreamSynchronize(s);
      cudaStreamDestroy(s);
    }
  } guard{st};

  std::mt19937_64 rng(seed);  // spectral.cpp:152-156
  std::uniform_real_distribution<double> unif(-1.0, 1.0);
  std::vector<double> hx(static_cast<size_t>(n)), hy(static_cast<size_t>(n));
  for (int64_t i = 0; i < n; ++i) hx[static_cast<size_t>(i)] = unif(rng);
  double sn = 0.0;
  for (double v : hx) sn += v * v;
  sn = std::sqrt(sn);
  for (double& v : hx) v /= sn;  // start.normalize()

  int64_t cap = std::min<int64_t>(n, 64);
  const int64_t amax = std::min<int64_t>(n, max_iter) + 2;
  const int nblk = std::max(1, ceil_div(n, kRowsPerBlock));
  const int gsz = ceil_div(n, 256);
  DBuf<double> basis, z, hbuf, partial, dalpha, dbeta, dnrm;
  basis.alloc(static_cast<size_t>(n) * cap);
  z.alloc(static_cast<size_t>(n));
  hbuf.alloc(static_cast<size_t>(amax));
  partial.alloc(static_cast<size_t>(nblk) * amax);
  dalpha.alloc(static_cast<size_t>(amax));
  dbeta.alloc(static_cast<size_t>(amax));
  dnrm.alloc(static_cast<size_t>(amax));
  FGS_CUDA(cudaMemcpyAsync(basis.p, hx.data(), sizeof(double) * n, cudaMemcpyHostToDevice, st));

  auto multidot = [&](const double* Q, int m, const double* v, double* out) {
    multidot_kernel<<<nblk, kRedThreads, 0, st>>>(Q, n, m, v, n, partial.p);
    reduce_partials_kernel<<<ceil_div(m, 8), 256, 0, st>>>(partial.p, nblk, m, out, 0);
  };
  auto cgs_pass = [&](int m, double* v) {  // v -= Q (Q^T v)
    multidot(basis.p, m, v, hbuf.p);
    update_kernel<<<gsz, 256, sizeof(double) * m, st>>>(basis.p, n, m, hbuf.p, v, n);
  };
  auto host_scalar = [&](const double* d) {
    double h = 0.0;
    FGS_CUDA(cudaMemcpyAsync(&h, d, sizeof(double), cudaMemcpyDeviceToHost, st));
    FGS_CUDA(cudaStreamSynchronize(st));
    return h;
  };

  std::vector<double> alphas, betas, tvals, tvecs;
  int tri_size = 0, iters = 0, next_check = k;
  double scale = 0.0;
  bool conv = false;
  auto solve_tri = [&](int m) {
    tvals.assign(alphas.begin(), alphas.begin() + m);
    std::vector<double> sub(betas.begin(), betas.begin() + (m - 1));
    tridiagonal_eigen(m, tvals, sub, tvecs);
    tri_size = m;
  };
  while (true) {
    const int m = static_cast<int>(alphas.size()) + 1;
    const double* qcur = basis.p + static_cast<int64_t>(m - 1) * n;
    FGS_CUDA(cudaMemcpyAsync(hx.data(), qcur, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
    FGS_CUDA(cudaStreamSynchronize(st));
    if (apply(ctx, hx.data(), hy.data(), n) != 0) fail(FGS_ENUMERIC, "operator apply callback failed");
    FGS_CUDA(cudaMemcpyAsync(z.p, hy.data(), sizeof(double) * n, cudaMemcpyHostToDevice, st));
    ++iters;
    multidot(qcur, 1, z.p, dalpha.p + (m - 1));  // alpha = q_m . z
    three_term_kernel<<<gsz, 256, 0, st>>>(z.p, qcur, m >= 2 ? qcur - n : nullptr, dalpha.p + (m - 1),
                                           m >= 2 ? dbeta.p + (m - 2) : dbeta.p, n);
    cgs_pass(m, z.p);  // full reorthogonalisation, twice (spectral.cpp:193-195)
    cgs_pass(m, z.p);
    multidot(z.p, 1, z.p, dnrm.p + (m - 1));
    const double alpha = host_scalar(dalpha.p + (m - 1));
    const double beta = std::sqrt(host_scalar(dnrm.p + (m - 1)));
    const double beta_prev = m >= 2 ? betas[static_cast<size_t>(m - 2)] : 0.0;
    alphas.push_back(alpha);
    scale = std::max(scale, std::abs(alpha) + beta + beta_prev);
    const bool last = iters >= max_iter || m == static_cast<int>(n);
    if (m >= k && (m >= next_check || last)) {  // spectral.cpp:200-215
      solve_tri(m);
      bool all_small = true;
      for (int i = 0; i < k && all_small; ++i) {
        const double theta = tvals[static_cast<size_t>(m - 1 - i)];
        const double est = beta * std::abs(tvecs[static_cast<size_t>(m - 1 - i) * m + (m - 1)]);
        if (est > tol * std::max(std::abs(theta), kEps * std::max(scale, 1.0))) all_small = false;
      }
      if (all_small) {
        conv = true;
        break;
      }
      next_check = m + std::max(8, m / 8);
    }
    if (iters >= max_iter) break;
    if (m == static_cast<int>(n)) {
      conv = true;
      break;
    }
    if (m == cap) {  // basis.conservativeResize(NoChange, min(n, 2 cap))
      const int64_t ncap = std::min<int64_t>(n, cap * 2);
      DBuf<double> nb;
      nb.alloc(static_cast<size_t>(n) * ncap);
      FGS_CUDA(cudaMemcpyAsync(nb.p, basis.p, sizeof(double) * n * cap, cudaMemcpyDeviceToDevice, st));
      FGS_CUDA(cudaStreamSynchronize(st));
      std::swap(basis.p, nb.p);
      std::swap(basis.n, nb.n);
      cap = ncap;
    }
    double* qnext = basis.p + static_cast<int64_t>(m) * n;
    if (beta > 1e-14 * std::max(scale, 1.0)) {
      betas.push_back(beta);
      FGS_CUDA(cudaMemcpyAsync(dbeta.p + (m - 1), &betas.back(), sizeof(double), cudaMemcpyHostToDevice, st));
      div_scalar_kernel<<<gsz, 256, 0, st>>>(z.p, beta, qnext, n);
    } else {  // breakdown (spectral.cpp:59-75, 225-238)
      bool found = false;
      for (int attempt = 0; attempt < 8 && !found; ++attempt) {
        for (int64_t i = 0; i < n; ++i) hx[static_cast<size_t>(i)] = unif(rng);
        FGS_CUDA(cudaMemcpyAsync(z.p, hx.data(), sizeof(double) * n, cudaMemcpyHostToDevice, st));
        cgs_pass(m, z.p);
        cgs_pass(m, z.p);
        multidot(z.p, 1, z.p, hbuf.p);
        const double nv = std::sqrt(host_scalar(hbuf.p));
        if (nv > 1e-8) {
          div_scalar_kernel<<<gsz, 256, 0, st>>>(z.p, nv, qnext, n);
          found = true;
        }
      }
      if (!found) {
        conv = true;
        break;
      }
      betas.push_back(0.0);
      FGS_CUDA(cudaMemcpyAsync(dbeta.p + (m - 1), &betas.back(), sizeof(double), cudaMemcpyHostToDevice, st));
    }
    FGS_CUDA(cudaGetLastError());
  }
  const int m = static_cast<int>(alphas.size());
  if (tri_size != m) solve_tri(m);
  const int wanted = std::min(k, m);
  std::vector<double> vals(static_cast<size_t>(wanted)), S(static_cast<size_t>(m) * wanted);
  for (int i = 0; i < wanted; ++i) {
    vals[static_cast<size_t>(i)] = tvals[static_cast<size_t>(m - 1 - i)];
    for (int j = 0; j < m; ++j) S[static_cast<size_t>(j) * wanted + i] = tvecs[static_cast<size_t>(m - 1 - i) * m + j];
  }
  std::vector<double> V;
  if (vectors) {  // V = Q_m S on the device (spectral.cpp:250)
    DBuf<double> dS, dV;
    dS.upload(S.data(), S.size(), st);
    dV.alloc(static_cast<size_t>(n) * wanted);
    for (int c0 = 0; c0 < wanted; c0 += 8)
      ritz_kernel<8><<<ceil_div(n, 128), 128, 0, st>>>(basis.p, n, m, dS.p, wanted, c0, dV.p, n, n);
    V.resize(static_cast<size_t>(n) * wanted);
    FGS_CUDA(cudaMemcpyAsync(V.data(), dV.p, sizeof(double) * V.size(), cudaMemcpyDeviceToHost, st));
    FGS_CUDA(cudaStreamSynchronize(st));
  }
  FGS_CUDA(cudaGetLastError());
  // make_eigenpairs (spectral.cpp:105-127)
  std::vector<int> order(static_cast<size_t>(wanted));
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return vals[static_cast<size_t>(a)] > vals[static_cast<size_t>(b)]; });
  for (int i = 0; i < wanted; ++i) {
    const int src = order[static_cast<size_t>(i)];
    values[i] = vals[static_cast<size_t>(src)];
    if (vectors) {
      const double* col = V.data() + static_cast<size_t>(src) * n;
      int64_t at = 0;
      for (int64_t r = 1; r < n; ++r)
        if (std::abs(col[r]) > std::abs(col[at])) at = r;
      const double sg = col[at] < 0.0 ? -1.0 : 1.0;
      for (int64_t r = 0; r < n; ++r) vectors[static_cast<size_t>(i) * n + r] = sg * col[r];
    }
  }
  if (count) *count = wanted;
  if (iterations) *iterations = iters;
  if (converged) *converged = conv ? 1 : 0;
}

void lanczos_finish_vectors(Core& c, LanczosResult& r, const std::vector<int>& order, double* host_out) {
  const int64_t n = c.n;
  const int cnt = static_cast<int>(order.size());
  if (cnt == 0) return;
  cudaStream_t st = c.stream;
  DBuf<int>& dorder = c.lz_order;
  dorder.upload(order.data(), order.size(), st);
  DBuf<double>& Vc = c.lz_vc;
  Vc.alloc(static_cast<size_t>(n) * cnt);
  const int gx = std::max(1, std::min(ceil_div(n, 256), 4096));
  unpermute_cols_kernel<<<dim3(gx, cnt), 256, 0, st>>>(r.vectors_dev.p, n, Vc.p, n, c.perm.p, dorder.p, n);
  const int chunk = 1 << 16;
  const int parts = std::max(1, ceil_div(n, chunk));
  DBuf<double>& pval = c.lz_pval;
  DBuf<double>& psigned = c.lz_psigned;
  DBuf<int64_t>& pidx = c.lz_pidx;
  pval.alloc(static_cast<size_t>(parts) * cnt);
  psigned.alloc(static_cast<size_t>(parts) * cnt);
  pidx.alloc(static_cast<size_t>(parts) * cnt);
  colmax_partial_kernel<<<dim3(parts, cnt), 256, 0, st>>>(Vc.p, n, n, chunk, pval.p, pidx.p, psigned.p);
  colsign_kernel<<<dim3(gx, cnt), 256, 0, st>>>(Vc.p, n, n, pval.p, psigned.p, parts);
  c.launches += 3;
  const auto t0 = std::chrono::steady_clock::now();
  c.host_copy(false, host_out, Vc.p, sizeof(double) * n * cnt);
  FGS_CUDA(cudaGetLastError());
  if (std::getenv("FGS_LANCZOS_TRACE"))
    std::fprintf(stderr, "[lanczos] vectors copy-out %.2f ms\n",
                 std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
  c.lz_vecs = std::move(r.vectors_dev);  // keep the device Ritz block for the next solve
}

}  // namespace fgsb
