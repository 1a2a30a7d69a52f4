// kernels.cuh -- hand-written sm_100a kernels of the NFFT fast-summation
// matvec (reference path: fastsum.cpp:111-118 -> nfft.cpp:402-438).
//
// Design: points are kept permanently in an internal order
// sorted by (tile, cell), where a cell is the first window tap
// u0 = ceil(v M - m) per dimension.  All points of one cell share the same
// (2m)^d footprint, so the spread and the interpolation are, per cell, a
// small dense contraction over the cell's points:
//     spread : G[a,c,e] += sum_j (x_j wa_j[a]) wc_j[c] we_j[e]
//     interp : y_j       = sum_{a,c} wa_j[a] wc_j[c] sum_e we_j[e] G[a,c,e]
// One CTA owns one work item (a run list inside one tile).  Each thread owns
// fixed (a, c, e-segment) "units" of the footprint: in the spread it keeps the
// E accumulators of its unit in registers across a staged chunk of <= 32
// points (no atomics, no shared-memory fp64 CAS), in the interpolation it
// keeps E grid values in registers and produces per-point partials that a
// warp butterfly + cross-warp shared-memory sum reduce.  Window taps of a
// chunk are one contiguous [q][d][2m] block in HBM (internal order), staged to
// shared memory with 16-byte coalesced loads and read back as broadcasts.
// The spread never touches the global grid: each CTA writes its tile box to
// a private slot and `assemble_kernel` sums the slots per grid cell in a
// fixed order, which makes every apply bitwise deterministic (the contract
// of fastsum.hpp:55-56) without fp64 atomics.
#pragma once

#include "common.cuh"

namespace fgsb {

constexpr double kPiD = 3.141592653589793238462643383279502884;

// ---------------------------------------------------------------------------
// Kaiser-Bessel window, operation-for-operation as nfft.cpp:161-169 (explicit
// _rn intrinsics keep nvcc from contracting into FMAs, so the tap values match
// the serial reference to libm accuracy).
// ---------------------------------------------------------------------------
__device__ __forceinline__ double kb_window(double diff, int m, int M, double b) {
  const double md = static_cast<double>(m);
  const double t1 = __dmul_rn(static_cast<double>(M), diff);
  const double arg = __dsub_rn(__dmul_rn(md, md), __dmul_rn(t1, t1));
  if (arg <= 0.0) return __ddiv_rn(b, kPiD);
  const double t = __dsqrt_rn(arg);
  if (t < 1e-8) {
    double num = __dmul_rn(__dmul_rn(__dmul_rn(__dmul_rn(b, b), b), t), t);
    return __ddiv_rn(__dadd_rn(b, __ddiv_rn(num, 6.0)), kPiD);
  }
  return __ddiv_rn(sinh(__dmul_rn(b, t)), __dmul_rn(kPiD, t));
}

// u0 = ceil(v M - m) exactly as nfft.cpp:358 (no FMA contraction)
__device__ __forceinline__ int first_tap(double v, int M, int m) {
  return static_cast<int>(ceil(__dsub_rn(__dmul_rn(v, static_cast<double>(M)), static_cast<double>(m))));
}

// ---------------------------------------------------------------------------
// Plan-time kernels
// ---------------------------------------------------------------------------
struct PointArgs {
  const double* nodes;  // caller order, column-major n x d (unscaled)
  int64_t n;
  int d, M, m, B, nt;
  double rho;
  int apply_rho;        // FastsumPlan scales by rho (fastsum.cpp:88); NfftPlan does not
  unsigned long long* keys;
  int* idx;
  unsigned long long* bad_range;  // min caller index with a scaled node outside [-1/2, 1/2)
  int rot0;                        // dim-0 tile rotation: key tile t0' = (t0 - rot0) mod nt
};

// dim-0 tiles holding at least one point (sharded plans rotate the dim-0
// tile order so the cloud is contiguous and every rank's slice is one slab)
__global__ void tile0_occupancy_kernel(PointArgs a, int* occ) {
  const int64_t j = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (j >= a.n) return;
  double v = a.nodes[j];
  if (a.apply_rho) v = __dmul_rn(a.rho, v);
  if (!(v >= -0.5 && v < 0.5)) v = 0.0;
  const int u0 = first_tap(v, a.M, a.m);
  const int w = ((u0 % a.M) + a.M) % a.M;
  occ[w / a.B] = 1;
}

// Scaled node, cell key = (tile, cell-in-tile).  rho * v is the exact IEEE
// product MatrixXd(rho * nodes) forms (fastsum.cpp:91).
__global__ void point_keys_kernel(PointArgs a) {
  const int64_t j = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (j >= a.n) return;
  unsigned long long tile = 0, cell = 0;
  for (int t = 0; t < a.d; ++t) {
    double v = a.nodes[t * a.n + j];
    if (a.apply_rho) v = __dmul_rn(a.rho, v);
    if (!(v >= -0.5 && v < 0.5)) {
      atomicMin(a.bad_range, static_cast<unsigned long long>(j));
      v = 0.0;
    }
    int u0 = first_tap(v, a.M, a.m);
    int w = ((u0 % a.M) + a.M) % a.M;
    int tt = w / a.B;
    if (t == 0) tt = (tt - a.rot0 + a.nt) % a.nt;
    tile = tile * a.nt + tt;
    cell = cell * a.B + w % a.B;
  }
  unsigned long long bd = 1;
  for (int t = 0; t < a.d; ++t) bd *= a.B;
  a.keys[j] = tile * bd + cell;
  a.idx[j] = static_cast<int>(j);
}

struct TapArgs {
  const double* nodes;
  int64_t n;       // caller count (column stride of nodes)
  int64_t count;   // internal points to fill
  const int* perm; // internal -> caller
  int d, M, m;
  double rho, b;
  int apply_rho;
  double* taps;    // [count][d][2m]
  const int* rows; // slot layout: row -> caller index (-1: pad row, zero taps); nullable
  int stride;      // doubles per row (0: d 2m)
};

// Window taps of every point in internal order (nfft.cpp:355-365).
__global__ void taps_kernel(TapArgs a) {
  const int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (p >= a.count) return;
  const int T = 2 * a.m;
  const int stride = a.stride ? a.stride : a.d * T;
  double* out = a.taps + p * stride;
  const int j = a.rows ? a.rows[p] : a.perm[p];
  if (j < 0) {  // pad slot of the run-aligned layout: zero taps
    for (int k = 0; k < stride; ++k) out[k] = 0.0;
    return;
  }
  for (int t = 0; t < a.d; ++t) {
    double v = a.nodes[t * a.n + j];
    if (a.apply_rho) v = __dmul_rn(a.rho, v);
    if (!(v >= -0.5 && v < 0.5)) v = 0.0;
    const int u0 = first_tap(v, a.M, a.m);
    for (int k = 0; k < T; ++k) {
      const int u = u0 + k;
      const double diff = __dsub_rn(v, __ddiv_rn(static_cast<double>(u), static_cast<double>(a.M)));
      out[t * T + k] = kb_window(diff, a.m, a.M, a.b);
    }
  }
  for (int k = a.d * T; k < stride; ++k) out[k] = 0.0;
}

// ---------------------------------------------------------------------------
// Unit geometry of the cell contraction: rows (a, c) x e-segments of E.
// ---------------------------------------------------------------------------
template <int D>
struct Canon;  // canonical 3-D view of the footprint / box
template <>
struct Canon<3> {
  __device__ static int rows(int T) { return T * T; }
};
template <>
struct Canon<2> {
  __device__ static int rows(int T) { return T; }
};
template <>
struct Canon<1> {
  __device__ static int rows(int) { return 1; }
};

constexpr int kQ = 32;  // points staged per chunk (one butterfly width)

// Stage q points' taps (q*taps doubles, 16-byte aligned since 2m is even).
__device__ __forceinline__ void stage_taps(double* __restrict__ stg, const double* __restrict__ src, int count,
                                           int tid, int nt) {
  const double2* s2 = reinterpret_cast<const double2*>(src);
  double2* d2 = reinterpret_cast<double2*>(stg);
  const int n2 = count >> 1;
  for (int k = tid; k < n2; k += nt) d2[k] = __ldg(s2 + k);
}

// ---------------------------------------------------------------------------
// Spread: per item, accumulate the tile box in shared memory through
// register-blocked cell contractions, then write the box to the item's
// private slot.  T = 2m (0: runtime T), E = e-values per unit.
// Shared memory: box (box_stride doubles) | stage (kQ*D*T) | xs (kQ).
// ---------------------------------------------------------------------------
template <int D, int T_, int E, int NT>
__global__ void __launch_bounds__(NT) spread_kernel(PassArgs a, int Trt, int box_stride_smem) {
  extern __shared__ __align__(16) double smem[];
  const int T = T_ > 0 ? T_ : Trt;
  const int TAPS = D * T;
  const int tid = threadIdx.x;
  const DItem it = a.items[blockIdx.x];
  const int bx1 = it.e1, bx2 = it.e2;
  const int V = it.e0 * it.e1 * it.e2;
  double* S = smem;
  double* stg = smem + box_stride_smem;
  double* xs = stg + kQ * TAPS;
  const int SP = T / E;
  const int U = Canon<D>::rows(T) * SP;
  const int nitems = gridDim.x;

  for (int vec = 0; vec < a.nvec; ++vec) {
    for (int v = tid; v < V; v += NT) S[v] = 0.0;
    const double* xv = a.x + vec * a.ldx;
    for (int r = it.run_begin; r < it.run_end; ++r) {
      const DRun run = a.runs[r];
      const int o0 = run.off & 1023, o1 = (run.off >> 10) & 1023, o2 = (run.off >> 20) & 1023;
      for (int base = 0; base < run.pcount; base += kQ) {
        const int q = min(kQ, run.pcount - base);
        const int64_t p0 = static_cast<int64_t>(run.pstart) + base;
        __syncthreads();  // previous chunk fully consumed
        stage_taps(stg, a.taps + p0 * TAPS, q * TAPS, tid, NT);
        if (tid < q) {
          const int64_t ip = p0 + tid;
          const int64_t ix = a.perm ? static_cast<int64_t>(a.perm[ip]) : ip;
          double xval = xv[ix];
          if (a.scale_input) xval = __dmul_rn(a.s[ip], xval);  // scaled = s .* x (graphop.cpp:96)
          xs[tid] = xval;
        }
        __syncthreads();
        for (int u = tid; u < U; u += NT) {
          const int row = u / SP;
          const int e0 = (u - row * SP) * E;
          const int ra = D == 3 ? row / T : 0;
          const int rc = D == 3 ? row - ra * T : (D == 2 ? row : 0);
          const int sidx = ((o0 + ra) * bx1 + (o1 + rc)) * bx2 + o2 + e0;
          double acc[E];
#pragma unroll
          for (int e = 0; e < E; ++e) acc[e] = S[sidx + e];
          for (int i = 0; i < q; ++i) {
            const double* w = stg + i * TAPS;
            double uu;
            const double* we;
            if (D == 3) {
              uu = (xs[i] * w[ra]) * w[T + rc];  // (x wa) wc, nfft.cpp:308-311
              we = w + 2 * T;
            } else if (D == 2) {
              uu = xs[i] * w[rc];
              we = w + T;
            } else {
              uu = xs[i];
              we = w;
            }
#pragma unroll
            for (int e = 0; e < E; ++e) acc[e] = fma(uu, we[e0 + e], acc[e]);
          }
#pragma unroll
          for (int e = 0; e < E; ++e) S[sidx + e] = acc[e];
        }
      }
    }
    __syncthreads();
    double* out = a.priv + (static_cast<int64_t>(vec) * nitems + blockIdx.x) * a.box_stride;
    for (int v = tid; v < V; v += NT) out[v] = S[v];
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// Deterministic grid assembly: grid cell g = sum, in increasing item order,
// of the private-box entries that map onto g (CSR built at plan time).  A
// pure gather: no atomics, fixed summation order -> bitwise reproducible.
// ---------------------------------------------------------------------------
struct AssembleArgs {
  const int* ptr;       // grid_elems + 1
  const int* idx;       // private-box entry offsets
  const double* priv;
  int64_t priv_stride;  // per vector
  double* grid;
  int64_t grid_stride;
  int nvec;
};

// One launch for all list-length classes (cells sorted by class at plan
// time; classes are warp-aligned, heaviest first so the long lists start in
// the first wave): warps [0, w2) take one long list each (> 64 entries, 32
// lanes), [w2, w2 + w1) four medium lists (9-64, 8 lanes each), the rest 32
// short lists (one lane each).  Per cell the arithmetic is
// assemble_kernel<L>'s for its class.  C2's lists average 17 entries but
// 88 % of the entries sit in lists of 65-291, which 8 lanes per cell walked
// as ~20 serial L2 round trips: the straggler set the kernel's length.
// L lanes per cell each sum a contiguous slice of the cell's entry list in
// order, then the slices are combined by a fixed shuffle tree -> bitwise
// reproducible (no atomics, fixed summation order).
struct AssembleMixedArgs {
  AssembleArgs a;    // ptr, idx, priv, grid, nvec
  const int* cells;  // class 2 cells | class 1 cells | class 0 cells
  int64_t n0, n1, n2, w1, w2;
};

template <int L, bool MULTI>
__device__ __forceinline__ void assemble_cell(const AssembleArgs& a, int64_t g, bool valid, int sub) {
  int b = 0, e = 0;
  if (valid) {
    const int b0 = a.ptr[g], e0 = a.ptr[g + 1];
    const int per = (e0 - b0 + L - 1) / L;
    b = min(e0, b0 + sub * per);
    e = min(e0, b + per);
  }
  const int cnt = e - b;
  constexpr int H = 16;  // slices up to H entries: indices loaded once, all values in flight per vector
  // multi-vector blocks only (a separate instantiation: the extra registers
  // cost the single-vector kernel its occupancy -- C4 assemble 47 -> 72 us)
  if (MULTI && __all_sync(0xffffffffu, cnt <= H)) {
    int ii[H];
#pragma unroll
    for (int u = 0; u < H; ++u) ii[u] = u < cnt ? __ldg(a.idx + b + u) : 0;
    for (int v = 0; v < a.nvec; ++v) {
      const double* pv = a.priv + v * a.priv_stride;
      double vv[H];
#pragma unroll
      for (int u = 0; u < H; ++u) vv[u] = u < cnt ? pv[ii[u]] : 0.0;
      double acc = 0.0;
#pragma unroll
      for (int u = 0; u < H; ++u)
        if (u < cnt) acc += vv[u];  // entry order, as the batched loop below
#pragma unroll
      for (int off = 1; off < L; off <<= 1) acc += __shfl_down_sync(0xffffffffu, acc, off, L);
      if (valid && sub == 0) a.grid[v * a.grid_stride + g] = acc;
    }
    return;
  }
  for (int v = 0; v < a.nvec; ++v) {
    const double* pv = a.priv + v * a.priv_stride;
    double acc = 0.0;
    int l = b;
    for (; l + 4 <= e; l += 4) {
      const int i0 = __ldg(a.idx + l), i1 = __ldg(a.idx + l + 1), i2 = __ldg(a.idx + l + 2), i3 = __ldg(a.idx + l + 3);
      const double v0 = pv[i0], v1 = pv[i1], v2 = pv[i2], v3 = pv[i3];
      acc += v0;
      acc += v1;
      acc += v2;
      acc += v3;
    }
    for (; l < e; ++l) acc += pv[__ldg(a.idx + l)];
#pragma unroll
    for (int off = 1; off < L; off <<= 1) acc += __shfl_down_sync(0xffffffffu, acc, off, L);
    if (valid && sub == 0) a.grid[v * a.grid_stride + g] = acc;
  }
}

template <bool MULTI>
__global__ void assemble_mixed_kernel(AssembleMixedArgs m) {
  pdl_wait();
  const int64_t gw = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (gw < m.w2) {
    const int64_t ci = gw;
    const bool valid = ci < m.n2;
    assemble_cell<32, MULTI>(m.a, valid ? m.cells[ci] : 0, valid, lane);
  } else if (gw < m.w2 + m.w1) {
    const int64_t ci = (gw - m.w2) * 4 + (lane >> 3);
    const bool valid = ci < m.n1;
    assemble_cell<8, MULTI>(m.a, valid ? m.cells[m.n2 + ci] : 0, valid, lane & 7);
  } else {
    const int64_t ci = (gw - m.w2 - m.w1) * 32 + lane;
    const bool valid = ci < m.n0;
    assemble_cell<1, MULTI>(m.a, valid ? m.cells[m.n2 + m.n1 + ci] : 0, valid, 0);
  }
}

// ---------------------------------------------------------------------------
// Spectral multiply on the R2C half spectrum by the Hermitian-symmetrised
// multiplier  m~_k = (m_k + conj(m_-k)) / 2,  m_k = out_factor * bhat_l *
// prod_t deconv(l_t)^2 on wrap(I_N), 0 elsewhere.  This reproduces
// out_factor * Re(forward(bhat .* adjoint(x))) (fastsum.cpp:115-117,
// nfft.cpp:429-438) including the unpaired -N/2 planes; the multiplier is
// stored compactly over l in [-N/2, N/2]^(d-1) x [0, N/2].
// ---------------------------------------------------------------------------
struct MultiplyArgs {
  cufftDoubleComplex* spec;
  const cufftDoubleComplex* mult;
  int64_t spec_stride;
  int64_t total;  // per vector
  int nvec;
  int D, M, N;
};

__global__ void multiply_kernel(MultiplyArgs a) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= a.total) return;
  const int H = a.M / 2 + 1;
  const int hN = a.N / 2;
  const int W = a.N + 1;
  int k2 = static_cast<int>(i % H);
  int64_t rest = i / H;
  int l[3] = {0, 0, k2};
  int D = a.D;
  if (D >= 2) {
    int k1 = static_cast<int>(rest % a.M);
    rest /= a.M;
    l[1] = k1 < (a.M + 1) / 2 ? k1 : k1 - a.M;
  }
  if (D == 3) {
    int k0 = static_cast<int>(rest);
    l[0] = k0 < (a.M + 1) / 2 ? k0 : k0 - a.M;
  }
  // M == N: representative of k = M/2 is -N/2 (still inside the window)
  bool inside = l[2] <= hN;
  if (D >= 2) inside = inside && l[1] >= -hN && l[1] <= hN;
  if (D == 3) inside = inside && l[0] >= -hN && l[0] <= hN;
  int64_t midx = l[2];
  if (D >= 2) midx += static_cast<int64_t>(l[1] + hN) * (hN + 1);
  if (D == 3) midx += static_cast<int64_t>(l[0] + hN) * W * (hN + 1);
  cufftDoubleComplex m = inside ? a.mult[midx] : make_cuDoubleComplex(0.0, 0.0);
  for (int v = 0; v < a.nvec; ++v) {
    cufftDoubleComplex z = a.spec[v * a.spec_stride + i];
    a.spec[v * a.spec_stride + i] =
        make_cuDoubleComplex(z.x * m.x - z.y * m.y, z.x * m.y + z.y * m.x);
  }
}

// ---------------------------------------------------------------------------
// Interpolation: per item, load the tile box of the real grid into shared
// memory; per staged chunk of <= 32 points each thread contracts its units
// (E grid values in registers) against the points' taps, a warp butterfly
// transposes the 32 per-point partials onto the lanes, warps are summed in
// shared memory, and the graph-operator epilogue is applied in place.
// Shared memory: box | stage | xs(unused) | red (NT/32 * 32).
// ---------------------------------------------------------------------------
__device__ __forceinline__ double epilogue(const PassArgs& a, double val, int64_t ip, int64_t ix,
                                           const double* xv) {
  switch (a.epilogue) {
    case EPI_KERNEL: return val;
    case EPI_WEIGHT: return val - a.k0 * xv[ix];
    case EPI_NORMALIZED: {
      const double s = a.s[ip];
      const double scaled = __dmul_rn(s, xv[ix]);
      return s * (val - a.k0 * scaled);
    }
    case EPI_LAPLACIAN: {
      const double s = a.s[ip];
      const double x = xv[ix];
      const double scaled = __dmul_rn(s, x);
      return x - s * (val - a.k0 * scaled);
    }
    default: return val;
  }
}

template <int D, int T_, int E, int NT>
__global__ void __launch_bounds__(NT) interp_kernel(PassArgs a, int Trt, int box_stride_smem) {
  extern __shared__ __align__(16) double smem[];
  const int T = T_ > 0 ? T_ : Trt;
  const int TAPS = D * T;
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  constexpr int NW = NT / 32;
  const DItem it = a.items[blockIdx.x];
  const int bx1 = it.e1, bx2 = it.e2;
  const int V = it.e0 * it.e1 * it.e2;
  const int Md0 = D == 3 ? a.M : 1, Md1 = D >= 2 ? a.M : 1, Md2 = a.M;
  double* S = smem;
  double* stg = smem + box_stride_smem;
  double* red = stg + kQ * TAPS + kQ;
  const int SP = T / E;
  const int U = Canon<D>::rows(T) * SP;

  for (int vec = 0; vec < a.nvec; ++vec) {
    const double* g = a.grid + vec * a.grid_stride;
    for (int v = tid; v < V; v += NT) {
      const int x2 = v % bx2, x1 = (v / bx2) % bx1, x0 = v / (bx2 * bx1);
      int g0 = it.a0 + x0, g1 = it.a1 + x1, g2 = it.a2 + x2;
      g0 %= Md0;
      g1 %= Md1;
      g2 %= Md2;
      S[v] = g[(static_cast<int64_t>(g0) * Md1 + g1) * Md2 + g2];
    }
    const double* xv = a.x + vec * a.ldx;
    double* yv = a.y ? a.y + vec * a.ldy : nullptr;
    for (int r = it.run_begin; r < it.run_end; ++r) {
      const DRun run = a.runs[r];
      const int o0 = run.off & 1023, o1 = (run.off >> 10) & 1023, o2 = (run.off >> 20) & 1023;
      for (int base = 0; base < run.pcount; base += kQ) {
        const int q = min(kQ, run.pcount - base);
        const int64_t p0 = static_cast<int64_t>(run.pstart) + base;
        __syncthreads();  // box loaded / previous chunk consumed
        stage_taps(stg, a.taps + p0 * TAPS, q * TAPS, tid, NT);
        __syncthreads();
        double p[kQ];
#pragma unroll
        for (int i = 0; i < kQ; ++i) p[i] = 0.0;
        for (int u = tid; u < U; u += NT) {
          const int row = u / SP;
          const int e0 = (u - row * SP) * E;
          const int ra = D == 3 ? row / T : 0;
          const int rc = D == 3 ? row - ra * T : (D == 2 ? row : 0);
          const int sidx = ((o0 + ra) * bx1 + (o1 + rc)) * bx2 + o2 + e0;
          double gv[E];
#pragma unroll
          for (int e = 0; e < E; ++e) gv[e] = S[sidx + e];
#pragma unroll
          for (int i = 0; i < kQ; ++i) {
            if (i < q) {
              const double* w = stg + i * TAPS;
              double uu;
              const double* we;
              if (D == 3) {
                uu = w[ra] * w[T + rc];
                we = w + 2 * T;
              } else if (D == 2) {
                uu = w[rc];
                we = w + T;
              } else {
                uu = 1.0;
                we = w;
              }
              double rs = 0.0;
#pragma unroll
              for (int e = 0; e < E; ++e) rs = fma(we[e0 + e], gv[e], rs);
              p[i] = fma(uu, rs, p[i]);
            }
          }
        }
        // warp transpose-reduce: lane l ends with the warp sum of point l
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
        red[warp * 32 + lane] = p[0];
        __syncthreads();
        if (tid < q) {
          double val = 0.0;
#pragma unroll
          for (int w = 0; w < NW; ++w) val += red[w * 32 + tid];
          const int64_t ip = p0 + tid;
          const int64_t ix = a.perm ? static_cast<int64_t>(a.perm[ip]) : ip;
          if (a.epilogue == EPI_DEGREE) {
            const double dg = val - a.k0;  // graphop.cpp:55-56
            a.degrees[ip] = dg;
            a.inv_sqrt[ip] = 1.0 / sqrt(dg);  // rsqrt (graphop.cpp:65)
            if (!(dg > 0.0)) atomicMin(a.bad_flag, static_cast<unsigned long long>(a.caller[ip]));
          } else {
            yv[ix] = epilogue(a, val, ip, ix, xv);
          }
        }
      }
    }
    __syncthreads();
  }
}

}  // namespace fgsb
