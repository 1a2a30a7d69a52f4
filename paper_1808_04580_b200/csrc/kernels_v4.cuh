// kernels_v4.cuh -- fp64 tensor-core (DMMA, mma.sync.m8n8k4.f64) spread for
// d = 3, 2m in {8, 12} (dense cells; 2m = 16 takes kernels_v6.cuh) and the
// d = 2 spread / interpolation.  The d = 3 interpolation moved to
// kernels_v5.cuh / kernels_v6.cuh; the pair algebra below is shared.
//
// Per run (points sharing one footprint) both passes are small GEMMs over the
// footprint's (a, c) "pairs":
//   interp: Z[j][(a,c)] = sum_e  we_j[e] g[(a,c)][e]          M = 8 points, K = e, N = pairs
//           y_j        = sum_a wa_j[a] sum_c wc_j[c] Z[j][(a,c)]   (scalar, 1/(2m) of the flops)
//   spread: G[(a,c)][e] += sum_j (wa_j[a] wc_j[c]) (x_j we_j[e])   M = pairs, K = 4 points, N = e
// One DMMA = 256 fp64 FMAs from register operands, so the fp64 pipe is fed
// with ~8x fewer issued instructions and no shared-memory operand per FMA
// (the limiter of the scalar kernels: ncu short-scoreboard / wait stalls).
// Measured on this B200: DMMA 36.7 TFLOP/s = DFMA 36.6 TFLOP/s peak.
//
// Pair tiling: an 8-wide MMA tile covers 2 a-values x 4 c-values,
//   n (or m) in 0..7  <->  (a = 2 ta + n / 4, c = 4 tc + n % 4),
// so for the C-fragment element (lane, i) the a-offset is (lane&3)/2 and the
// c-offset 2 (lane&1) + i: every lane touches only 2m/2 a-taps and 2m/2
// c-taps of its point, held in registers with compile-time indices.
// Fragment layouts (checked on the B200 by tools/dmma_layout_check.cu):
//   A 8x4 row: lane holds A[lane/4][lane%4];  B 4x8 col: B[lane%4][lane/4];
//   C 8x8: lane holds C[lane/4][2 (lane%4) + i], i = 0, 1.
// Groups of G warps share one footprint (G > 1 splits the a range: 2m = 12
// G = 2; 2m = 16 G = 4 spread / 2 interpolation); P groups per CTA walk different K-steps / batches of each staged
// chunk.  Results are bitwise deterministic (fixed MMA and reduction order).
#pragma once

#include <type_traits>

#include "kernels_v2.cuh"

namespace fgsb {

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

template <int T, bool INTERP, int PS = 0, int QSZ = 0>
struct Blk4 {
  // QSZ = 0: default chunk (64 for 2m in {8, 16}, 32 for 2m = 12 interpolation)
  // warps per footprint group: more warps per footprint = fewer registers
  // per lane (ncu: 236-255 regs capped occupancy at 8 warps/SM with G = 1)
#ifndef FGS_G12_INTERP
#define FGS_G12_INTERP 2
#endif
  // 2m = 16 spread: one group of 8 warps (each warp one a-tile pair, all c
  // and e): no turn-based flush barriers (C5 spread 64.5 -> 57.9 ms per
  // 16-vector block; G = 4 x 2 streams before)
  static constexpr int G = T == 16 ? (INTERP ? 2 : 8) : (T == 12 ? (INTERP ? FGS_G12_INTERP : 2) : 1);
  static constexpr int TA = T / 2;           // a-tiles (2 a each)
  static constexpr int TC = T / 4;           // c-tiles (4 c each)
  static constexpr int TAW = TA / G;         // a-tiles per warp
  static constexpr int TW = TAW * TC;        // pair tiles per warp
  static constexpr int KS = T / 4;           // interp K-steps over e
  static constexpr int NE = (T + 7) / 8;     // spread N-tiles over e (2m = 12 pads 12 -> 16)
  // groups (point streams) per CTA; PS > 0 overrides the default
  // (2m = 16 spread: 2 streams, C5 64.9 -> 62.2 ms per 16-vector block)
  static constexpr int P = PS > 0 ? PS : (T == 8 ? 4 : ((T == 16 && !INTERP) ? 1 : 2));
  static constexpr int NT = 32 * G * P;
  // points per staged chunk (2m = 12: spread 64 -- C4 spread 412 -> 391 us
  // with the private group boxes -- interp 32)
  static constexpr int QS = QSZ > 0 ? QSZ : ((T == 12 && INTERP) ? 32 : 64);
  static constexpr int TAPS = 3 * T;
  // staged row stride: = 4 or 12 (mod 16 doubles) so the 4 (spread) or 8
  // (interp) points a warp reads per LDS fall on distinct bank pairs; 2m = 16
  // rows of 48 doubles all started on the same bank (ncu: 9e9 conflicts, C5)
  static constexpr int STRIDE = (TAPS % 16 == 4 || TAPS % 16 == 12) ? TAPS
                              : (TAPS % 16 == 0 ? TAPS + 4 : TAPS + ((12 - TAPS % 16 + 16) % 16));
};

// cp.async a chunk of q points' taps into rows of STRIDE doubles
template <class I>
__device__ __forceinline__ I pmin(I x, I y) { return x < y ? x : y; }

template <int TAPS, int STRIDE>
__device__ __forceinline__ void v4_issue_chunk(double* buf, const double* taps, int64_t p, int q, int tid, int nt) {
  constexpr int H = TAPS / 2;  // 16-byte pieces per point
  const double* src = taps + p * TAPS;
  const int n16 = q * H;
  for (int k = tid; k < n16; k += nt) {
    const int pt = k / H, r = k - pt * H;
    cp_async16(buf + pt * STRIDE + 2 * r, src + 2 * k);
  }
}

// ---------------------------------------------------------------------------
// spread.  smem: box | stage[2][QS*TAPS] | xs[2][QS]
// ---------------------------------------------------------------------------
template <int T, int PS, int QSZ>
__global__ void __launch_bounds__(Blk4<T, false, PS, QSZ>::NT) spread_v4_kernel(PassArgs a, int box_stride_smem) {
  pdl_wait();
  using B = Blk4<T, false, PS, QSZ>;
  constexpr int NT = B::NT, QS = B::QS, TAPS = B::TAPS, P = B::P, SR = B::STRIDE;
  constexpr int TAW = B::TAW, TC = B::TC, TW = B::TW, NE = B::NE;
  extern __shared__ __align__(16) double smem[];
  // P >= 4 groups: one private box per group (flushes need no barrier; the
  // boxes are summed in group order at the end of the item).  Fewer groups:
  // one shared box, groups flush in turn (the extra box costs occupancy).
  constexpr bool PRIV = P >= 4;
  constexpr int NB = PRIV ? P : 1;
  double* S = smem;
  double* stg = smem + NB * box_stride_smem;
  double* xs = stg + 2 * QS * SR;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int grp = warp / B::G, wg = warp % B::G;
  const int q = lane & 3, r8 = lane >> 2;
  const int ta0 = wg * TAW;
  const DItem it = a.items[blockIdx.x];
  const int bx1 = it.e1, bx2 = it.e2;
  const int V = it.e0 * it.e1 * it.e2;
  const int64_t p_begin = it.p_begin, p_end = it.p_end;
  const int nch = static_cast<int>((p_end - p_begin + QS - 1) / QS);

  for (int vec = 0; vec < a.nvec; ++vec) {
    // slot layout (2m = 12 dense plans): x pre-gathered into slot order
    const double* xv = a.xs ? a.xs + vec * a.ldxs : a.x + vec * a.ldx;
    for (int g = 0; g < NB; ++g)
      for (int v = tid; v < V; v += NT) S[g * box_stride_smem + v] = 0.0;
    v4_issue_chunk<TAPS, SR>(stg, a.taps, p_begin, static_cast<int>(lmin(QS, p_end - p_begin)), tid, NT);
    cp_async_commit();
    if (tid < QS && p_begin + tid < p_end) xs[tid] = a.xs ? xv[p_begin + tid] : v2_x(a, xv, p_begin + tid);
    int r = it.run_begin;
    DRun run = a.runs[r];
    double C[TW][NE][2];
#pragma unroll
    for (int t = 0; t < TW; ++t)
#pragma unroll
      for (int ne = 0; ne < NE; ++ne) C[t][ne][0] = C[t][ne][1] = 0.0;

    // flush this group's accumulators of `run`: into its own box (PRIV: the
    // G warps of a group own disjoint a-rows, lanes disjoint (c, e), so no
    // barrier), else into the shared box with the groups in turn
    auto flush_into = [&](double* Sg) {
      const int o0 = run.off & 1023, o1 = (run.off >> 10) & 1023, o2 = (run.off >> 20) & 1023;
#pragma unroll
      for (int t = 0; t < TW; ++t) {
        const int ta = ta0 + t / TC, tc = t % TC;
        const int aa = 2 * ta + (r8 >> 2), cc = 4 * tc + (r8 & 3);
        double* row = Sg + ((o0 + aa) * bx1 + (o1 + cc)) * bx2 + o2;
#pragma unroll
        for (int ne = 0; ne < NE; ++ne)
#pragma unroll
          for (int i = 0; i < 2; ++i) {
            const int e = 8 * ne + 2 * q + i;
            if (e < T) row[e] += C[t][ne][i];
            C[t][ne][i] = 0.0;
          }
      }
    };
    auto flush = [&]() {
      if constexpr (PRIV) {
        flush_into(S + grp * box_stride_smem);
      } else if constexpr (P == 1) {
        // one group: its warps own disjoint a-rows of THIS run's footprint,
        // but consecutive runs' footprints overlap at other offsets, so
        // every warp finishes this flush before any flushes the next run
        flush_into(S);
        __syncthreads();
      } else {
        for (int g = 0; g < P; ++g) {
          if (g == grp) flush_into(S);
          __syncthreads();
        }
      }
    };

    for (int k = 0; k < nch; ++k) {
      const int64_t c0 = p_begin + static_cast<int64_t>(k) * QS;
      const int64_t c1 = lmin(c0 + QS, p_end);
      const int buf = k & 1;
      cp_async_wait_0();
      __syncthreads();
      const bool more = k + 1 < nch;
      double xnext = 0.0;
      int qn = 0;
      if (more) {
        qn = static_cast<int>(lmin(QS, p_end - c1));
        v4_issue_chunk<TAPS, SR>(stg + (buf ^ 1) * QS * SR, a.taps, c1, qn, tid, NT);
        cp_async_commit();
        if (tid < qn) xnext = a.xs ? xv[c1 + tid] : v2_x(a, xv, c1 + tid);
      }
      const double* sb = stg + buf * QS * SR;
      const double* xb = xs + buf * QS;
      while (true) {
        const int64_t rs = run.pstart, re_ = static_cast<int64_t>(run.pstart) + run.pcount;
        const int64_t s0 = rs > c0 ? rs : c0, s1 = lmin(re_, c1);
        // K-steps of 4 points aligned to the chunk; group grp takes every P-th
        for (int64_t k0 = c0 + 4 * grp; k0 < s1; k0 += 4 * P) {
          if (k0 + 4 <= s0) continue;
          const int64_t jp = k0 + q;  // this lane's point of the K-step
          const bool ok = jp >= s0 && jp < s1;
          const double* w = sb + (ok ? (jp - c0) : 0) * SR;
          const double xj = ok ? xb[jp - c0] : 0.0;
          double wa[TAW], wc[TC];
#pragma unroll
          for (int t = 0; t < TAW; ++t) wa[t] = w[2 * (ta0 + t) + (r8 >> 2)];
#pragma unroll
          for (int t = 0; t < TC; ++t) wc[t] = w[T + 4 * t + (r8 & 3)];
          double bF[NE];  // x_j we_j[e], e = 8 ne + lane/4
#pragma unroll
          for (int ne = 0; ne < NE; ++ne) {
            const int e = 8 * ne + r8;
            bF[ne] = e < T ? xj * w[2 * T + e] : 0.0;
          }
          double af[TW];  // wa wc of pair (lane/4 row), all tiles first
#pragma unroll
          for (int t = 0; t < TW; ++t) af[t] = wa[t / TC] * wc[t % TC];
#pragma unroll
          for (int ne = 0; ne < NE; ++ne)
#pragma unroll
            for (int t = 0; t < TW; ++t) dmma(C[t][ne][0], C[t][ne][1], af[t], bF[ne]);
        }
        if (re_ <= c1) {  // run ends inside this chunk
          flush();
          if (++r >= it.run_end) break;
          run = a.runs[r];
          continue;
        }
        break;
      }
      if (more && tid < qn) xs[(buf ^ 1) * QS + tid] = xnext;
    }
    __syncthreads();
    double* out = a.priv + (static_cast<int64_t>(vec) * gridDim.x + blockIdx.x) * a.box_stride;
    for (int v = tid; v < V; v += NT) {
      double sum = S[v];
#pragma unroll
      for (int g = 1; g < NB; ++g) sum += S[g * box_stride_smem + v];
      out[v] = sum;
    }
    __syncthreads();
  }
}


// ===========================================================================
// d = 2 tensor-core variants (2m in {8, 12, 16}).  The footprint is a
// (2m) x (2m) block g[c][e]:
//   interp: Z[j][c] = sum_e we_j[e] g[c][e]   M = 8 points, K = e, N = c (padded to 8k)
//           y_j = sum_c wc_j[c] Z[j][c]
//   spread: G[c][e] += sum_j (x_j wc_j[c]) we_j[e]   M = c, K = 4 points, N = e
// One warp per point stream, P streams per CTA, the same chunk / run / flush
// protocol as the d = 3 kernels above.
// ===========================================================================
template <int T, int PS = 4>
struct Blk4d2 {
  static constexpr int NC = (T + 7) / 8;  // c tiles (M or N dimension, padded)
  static constexpr int NE = (T + 7) / 8;  // e tiles (spread N dimension, padded)
  static constexpr int KS = T / 4;        // interp K-steps over e
  static constexpr int P = PS;  // point streams (warps) per CTA
  static constexpr int NT = 32 * P;
  static constexpr int QS = 32;
  static constexpr int TAPS = 2 * T;
  static constexpr int STRIDE = (TAPS % 16 == 4 || TAPS % 16 == 12) ? TAPS
                              : (TAPS % 16 == 0 ? TAPS + 4 : TAPS + ((12 - TAPS % 16 + 16) % 16));
  // points whose caller-order inputs are staged at once (a multiple of QS)
  static constexpr int XW = NT > 64 ? NT : 64;
};

// Per-point inputs of a window of internal points [w0, min(w0 + XW, p_end))
// staged in shared memory with every load of the window in flight at once:
// the caller-order gather x[perm[j]] is a two-load dependent chain, and
// fetched one chunk at a time it stalled the 2-D kernels for ~30 % (spread)
// and ~11 % (interp) of their samples (ncu source page, r01_c2_full).
//   xs[o]  spread: x (times s when the pass scales its input), as v2_x
//   xs[o], ixs[o]  interp: epilogue input x and the caller index of the store
template <int NT, int XW>
__device__ __forceinline__ void v4_stage_spread_x(const PassArgs& a, const double* xv, int64_t w0, int64_t p_end,
                                                  double* xs, int tid) {
  constexpr int U = XW / NT;
  int64_t ix[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int64_t j = w0 + u * NT + tid;
    ix[u] = j < p_end ? (a.perm ? static_cast<int64_t>(a.perm[j]) : j) : -1;
  }
  double xr[U], sr[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    xr[u] = ix[u] >= 0 ? xv[ix[u]] : 0.0;
    sr[u] = ix[u] >= 0 && a.scale_input ? a.s[w0 + u * NT + tid] : 1.0;
  }
#pragma unroll
  for (int u = 0; u < U; ++u)
    if (ix[u] >= 0) xs[u * NT + tid] = a.scale_input ? __dmul_rn(sr[u], xr[u]) : xr[u];
}

template <int NT, int XW>
__device__ __forceinline__ void v4_stage_interp_x(const PassArgs& a, const double* xv, int64_t w0, int64_t p_end,
                                                  double* xs, int64_t* ixs, int tid) {
  constexpr int U = XW / NT;
  const bool need_x = xv && a.epilogue != EPI_KERNEL && a.epilogue != EPI_DEGREE;
  int64_t ix[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int64_t j = w0 + u * NT + tid;
    ix[u] = j < p_end ? (a.perm ? static_cast<int64_t>(a.perm[j]) : j) : -1;
  }
  double xr[U];
#pragma unroll
  for (int u = 0; u < U; ++u) xr[u] = need_x && ix[u] >= 0 ? xv[ix[u]] : 0.0;
#pragma unroll
  for (int u = 0; u < U; ++u)
    if (ix[u] >= 0) {
      xs[u * NT + tid] = xr[u];
      ixs[u * NT + tid] = ix[u];
    }
}

template <int T, int PS = 4>
__global__ void __launch_bounds__(Blk4d2<T, PS>::NT) interp_v4_2d_kernel(PassArgs a, int box_stride_smem) {
  pdl_wait();
  using B = Blk4d2<T, PS>;
  constexpr int NT = B::NT, QS = B::QS, TAPS = B::TAPS, P = B::P, SR = B::STRIDE, NC = B::NC, KS = B::KS;
  constexpr int XW = B::XW;
  extern __shared__ __align__(16) double smem[];
  double* S = smem;
  double* stg = smem + box_stride_smem;
  double* xs = stg + 2 * QS * SR;
  int64_t* ixs = reinterpret_cast<int64_t*>(xs + XW);
  const int tid = threadIdx.x, lane = tid & 31, grp = tid >> 5;
  const int q = lane & 3, r8 = lane >> 2;
  const DItem it = a.items[blockIdx.x];
  const int bx2 = it.e2;
  const int V = it.e1 * it.e2;
  const int M = a.M;
  const int64_t p_begin = it.p_begin, p_end = it.p_end;
  const int nch = static_cast<int>((p_end - p_begin + QS - 1) / QS);

  for (int vec = 0; vec < a.nvec; ++vec) {
    const double* gv = a.grid + vec * a.grid_stride;
    const double* xv = a.x ? a.x + vec * a.ldx : nullptr;
    double* yv = a.y ? a.y + vec * a.ldy : nullptr;
    v4_issue_chunk<TAPS, SR>(stg, a.taps, p_begin, static_cast<int>(lmin(QS, p_end - p_begin)), tid, NT);
    cp_async_commit();
    v4_stage_interp_x<NT, XW>(a, xv, p_begin, p_end, xs, ixs, tid);
    {  // floor(v / bx2) by multiply-shift (exact while v bx2 < 2^20), wraps by compare-and-subtract
      const unsigned mdiv = (1u << 20) / static_cast<unsigned>(bx2) + 1u;
      for (int v = tid; v < V; v += NT) {
        const int x1 = static_cast<int>((static_cast<unsigned>(v) * mdiv) >> 20), x2 = v - x1 * bx2;
        int g1 = it.a1 + x1, g2 = it.a2 + x2;
        if (g1 >= M) g1 = g1 - M < M ? g1 - M : g1 % M;
        if (g2 >= M) g2 = g2 - M < M ? g2 - M : g2 % M;
        S[v] = gv[static_cast<int64_t>(g1) * M + g2];
      }
    }
    int r = it.run_begin;
    DRun run = a.runs[r];
    int loaded = -1;
    double gB[NC][KS];  // B[k = e][n = c]: g[c = 8 nc + lane/4][e = 4 ks + lane%4]
    for (int k = 0; k < nch; ++k) {
      const int64_t c0 = p_begin + static_cast<int64_t>(k) * QS;
      const int64_t c1 = lmin(c0 + QS, p_end);
      const int buf = k & 1;
      const int xo = (k * QS) % XW;  // chunk offset in the staged window
      if (k > 0 && xo == 0) {        // next window (items longer than XW points)
        __syncthreads();
        v4_stage_interp_x<NT, XW>(a, xv, c0, p_end, xs, ixs, tid);
      }
      cp_async_wait_0();
      __syncthreads();
      if (k + 1 < nch) {
        v4_issue_chunk<TAPS, SR>(stg + (buf ^ 1) * QS * SR, a.taps, c1, static_cast<int>(lmin(QS, p_end - c1)), tid, NT);
        cp_async_commit();
      }
      const double* sb = stg + buf * QS * SR;
      for (int64_t b0 = c0 + 8 * grp; b0 < c1; b0 += 8 * P) {
        const int64_t ipt = b0 + r8;
        const bool in_chunk = ipt < c1;
        const double* w = sb + (in_chunk ? (ipt - c0) : 0) * SR;
        double xin = 0.0, sin_ = 1.0;
        int64_t ix = 0;
        if (q == 0 && in_chunk) {
          const int o = xo + static_cast<int>(ipt - c0);
          ix = ixs[o];
          xin = xs[o];
          if (a.epilogue == EPI_NORMALIZED || a.epilogue == EPI_LAPLACIAN) sin_ = a.s[ipt];
        }
        double wc[NC][2];  // c = 8 nc + 2 q + i
#pragma unroll
        for (int nc = 0; nc < NC; ++nc)
#pragma unroll
          for (int i = 0; i < 2; ++i) {
            const int cc = 8 * nc + 2 * q + i;
            wc[nc][i] = cc < T ? w[cc] : 0.0;
          }
        double yacc = 0.0;
        while (true) {
          while (static_cast<int64_t>(run.pstart) + run.pcount <= b0 && r + 1 < it.run_end) run = a.runs[++r];
          if (loaded != r) {
            const int o1 = (run.off >> 10) & 1023, o2 = (run.off >> 20) & 1023;
#pragma unroll
            for (int nc = 0; nc < NC; ++nc) {
              const int cc = 8 * nc + r8;
              const double* row = S + (o1 + (cc < T ? cc : 0)) * bx2 + o2 + q;
#pragma unroll
              for (int ks = 0; ks < KS; ++ks) gB[nc][ks] = cc < T ? row[4 * ks] : 0.0;
            }
            loaded = r;
          }
          const int64_t rs = run.pstart, re_ = static_cast<int64_t>(run.pstart) + run.pcount;
          const bool mine = in_chunk && ipt >= rs && ipt < re_;
          double aF[KS];
#pragma unroll
          for (int ks = 0; ks < KS; ++ks) aF[ks] = mine ? w[T + 4 * ks + q] : 0.0;
#pragma unroll
          for (int nc = 0; nc < NC; ++nc) {
            double z0 = 0.0, z1 = 0.0;
#pragma unroll
            for (int ks = 0; ks < KS; ++ks) dmma(z0, z1, aF[ks], gB[nc][ks]);
            yacc = fma(wc[nc][0], z0, yacc);
            yacc = fma(wc[nc][1], z1, yacc);
          }
          if (re_ < lmin(b0 + 8, c1) && r + 1 < it.run_end) {
            run = a.runs[++r];
            continue;
          }
          break;
        }
        yacc += __shfl_xor_sync(0xffffffffu, yacc, 1);
        yacc += __shfl_xor_sync(0xffffffffu, yacc, 2);
        if (q == 0 && in_chunk) {
          const double val = yacc;
          if (a.epilogue == EPI_DEGREE) {
            const double dg = val - a.k0;  // graphop.cpp:55-56
            a.degrees[ipt] = dg;
            a.inv_sqrt[ipt] = 1.0 / sqrt(dg);
            if (!(dg > 0.0)) atomicMin(a.bad_flag, static_cast<unsigned long long>(a.caller[ipt]));
          } else {
            double out;
            switch (a.epilogue) {
              case EPI_KERNEL: out = val; break;
              case EPI_WEIGHT: out = val - a.k0 * xin; break;
              case EPI_NORMALIZED: out = sin_ * (val - a.k0 * __dmul_rn(sin_, xin)); break;
              default: out = xin - sin_ * (val - a.k0 * __dmul_rn(sin_, xin)); break;
            }
            yv[ix] = out;
          }
        }
      }
    }
    cp_async_wait_0();
    __syncthreads();
  }
}

template <int T, int PS>
__global__ void __launch_bounds__(Blk4d2<T, PS>::NT) spread_v4_2d_kernel(PassArgs a, int box_stride_smem) {
  pdl_wait();
  using B = Blk4d2<T, PS>;
  constexpr int NT = B::NT, QS = B::QS, TAPS = B::TAPS, P = B::P, SR = B::STRIDE, NC = B::NC, NE = B::NE;
  constexpr int XW = B::XW;
  extern __shared__ __align__(16) double smem[];
  // one private box per point stream (a d = 2 box is a few KB): flushes need
  // no barrier, the boxes are summed in stream order at the end of the item
  constexpr int NB = P;
  double* S = smem;
  double* stg = smem + NB * box_stride_smem;
  double* xs = stg + 2 * QS * SR;
  const int tid = threadIdx.x, lane = tid & 31, grp = tid >> 5;
  const int q = lane & 3, r8 = lane >> 2;
  const DItem it = a.items[blockIdx.x];
  const int bx2 = it.e2;
  const int V = it.e1 * it.e2;
  const int64_t p_begin = it.p_begin, p_end = it.p_end;
  const int nch = static_cast<int>((p_end - p_begin + QS - 1) / QS);

  for (int vec = 0; vec < a.nvec; ++vec) {
    // slot layout (2m = 12 dense plans): x pre-gathered into slot order
    const double* xv = a.xs ? a.xs + vec * a.ldxs : a.x + vec * a.ldx;
    for (int g = 0; g < NB; ++g)
      for (int v = tid; v < V; v += NT) S[g * box_stride_smem + v] = 0.0;
    v4_issue_chunk<TAPS, SR>(stg, a.taps, p_begin, static_cast<int>(lmin(QS, p_end - p_begin)), tid, NT);
    cp_async_commit();
    v4_stage_spread_x<NT, XW>(a, xv, p_begin, p_end, xs, tid);
    int r = it.run_begin;
    DRun run = a.runs[r];
    double C[NC][NE][2];  // C[m = c][n = e]: lane holds c = 8 mc + lane/4, e = 8 ne + 2 (lane%4) + i
#pragma unroll
    for (int mc = 0; mc < NC; ++mc)
#pragma unroll
      for (int ne = 0; ne < NE; ++ne) C[mc][ne][0] = C[mc][ne][1] = 0.0;
    auto flush = [&]() {
      const int o1 = (run.off >> 10) & 1023, o2 = (run.off >> 20) & 1023;
      double* Sg = S + grp * box_stride_smem;
#pragma unroll
      for (int mc = 0; mc < NC; ++mc) {
        const int cc = 8 * mc + r8;
        double* row = Sg + (o1 + (cc < T ? cc : 0)) * bx2 + o2;
#pragma unroll
        for (int ne = 0; ne < NE; ++ne)
#pragma unroll
          for (int i = 0; i < 2; ++i) {
            const int e = 8 * ne + 2 * q + i;
            if (cc < T && e < T) row[e] += C[mc][ne][i];
            C[mc][ne][i] = 0.0;
          }
      }
      __syncwarp();
    };
    for (int k = 0; k < nch; ++k) {
      const int64_t c0 = p_begin + static_cast<int64_t>(k) * QS;
      const int64_t c1 = lmin(c0 + QS, p_end);
      const int buf = k & 1;
      const int xo = (k * QS) % XW;  // chunk offset in the staged window
      if (k > 0 && xo == 0) {        // next window (items longer than XW points)
        __syncthreads();
        v4_stage_spread_x<NT, XW>(a, xv, c0, p_end, xs, tid);
      }
      cp_async_wait_0();
      __syncthreads();
      if (k + 1 < nch) {
        v4_issue_chunk<TAPS, SR>(stg + (buf ^ 1) * QS * SR, a.taps, c1, static_cast<int>(lmin(QS, p_end - c1)), tid, NT);
        cp_async_commit();
      }
      const double* sb = stg + buf * QS * SR;
      const double* xb = xs + xo;
      while (true) {
        const int64_t rs = run.pstart, re_ = static_cast<int64_t>(run.pstart) + run.pcount;
        const int64_t s0 = rs > c0 ? rs : c0, s1 = lmin(re_, c1);
        // first K-step of this group that reaches the run (k0 + 4 > s0);
        // d = 2 only (C2 spread 16.2 -> 14.8 us; the d = 3 kernel's schedule
        // got worse with it, C4 412 -> 452 us)
        int64_t kfirst = c0 + 4 * grp;
        if (s0 > kfirst + 3) kfirst += (s0 - kfirst - 3 + 4 * P - 1) / (4 * P) * (4 * P);
        for (int64_t k0 = kfirst; k0 < s1; k0 += 4 * P) {
          const int64_t jp = k0 + q;
          const bool ok = jp >= s0 && jp < s1;
          const double* w = sb + (ok ? (jp - c0) : 0) * SR;
          const double xj = ok ? xb[jp - c0] : 0.0;
          double af[NC], bF[NE];
#pragma unroll
          for (int mc = 0; mc < NC; ++mc) {
            const int cc = 8 * mc + r8;
            af[mc] = cc < T ? xj * w[cc] : 0.0;  // x wc
          }
#pragma unroll
          for (int ne = 0; ne < NE; ++ne) {
            const int e = 8 * ne + r8;
            bF[ne] = e < T ? w[T + e] : 0.0;  // we
          }
#pragma unroll
          for (int mc = 0; mc < NC; ++mc)
#pragma unroll
            for (int ne = 0; ne < NE; ++ne) dmma(C[mc][ne][0], C[mc][ne][1], af[mc], bF[ne]);
        }
        if (re_ <= c1) {
          flush();
          if (++r >= it.run_end) break;
          run = a.runs[r];
          continue;
        }
        break;
      }
    }
    __syncthreads();
    double* out = a.priv + (static_cast<int64_t>(vec) * gridDim.x + blockIdx.x) * a.box_stride;
    for (int v = tid; v < V; v += NT) {
      double sum = S[v];
#pragma unroll
      for (int g = 1; g < NB; ++g) sum += S[g * box_stride_smem + v];
      out[v] = sum;
    }
    __syncthreads();
  }
}

}  // namespace fgsb
