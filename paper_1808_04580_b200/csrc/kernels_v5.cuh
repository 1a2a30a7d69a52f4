// kernels_v5.cuh -- d = 3 interpolation on the fp64 tensor cores with the
// grid block streamed from shared memory (2m in {8, 12, 16}).
//
// Per run (points sharing one footprint) the interpolation is the small GEMM
//   Z[j][(a,c)] = sum_e we_j[e] g[(a,c)][e]      M = 8 points, K = e, N = pairs
//   y_j         = sum_a wa_j[a] sum_c wc_j[c] Z[j][(a,c)]
// (kernels_v4.cuh explains the 2a x 4c pair tiling and the DMMA fragment
// layouts).  The v4 kernel kept the run's whole grid block in registers as B
// fragments (64 doubles per lane at 2m = 16, 255 registers, 8 warps per SM,
// G warps sharing one point batch through shared-memory partials and CTA
// barriers).  Here every warp owns whole 8-point batches over ALL pairs and
// reads each B fragment from the item's box in shared memory right before its
// DMMA: ~100 registers, 16 warps per SM, no cross-warp reduction and no CTA
// barrier after the box load.  The box rows are padded to a stride = 4
// (mod 8) doubles so a B-fragment load (4 c-rows x 4 e per half-warp) hits 16
// distinct bank pairs.  Each warp stages its next batch's taps (8 points x 3
// x 2m doubles) into its own shared-memory slot with cp.async while it
// computes the current one (per-warp double buffer, no CTA-wide staging).
// Per lane and batch: 2m^3 / 8 DMMAs (2m = 16: 128) against as many LDS.64.
#pragma once

#include "kernels_v4.cuh"

namespace fgsb {

// padded x2-stride of an item box in shared memory: the smallest s >= e2
// with s = 4 (mod 8)
__host__ __device__ __forceinline__ int v5_pad(int e2) { return e2 + ((12 - e2 % 8) % 8); }

template <int T>
struct Blk5 {
  static constexpr int TA = T / 2;  // a-tiles (2 a each)
  static constexpr int TC = T / 4;  // c-tiles (4 c each)
  static constexpr int KS = T / 4;  // K-steps over e
  static constexpr int W = 8;       // warps per CTA (independent point streams)
  static constexpr int NT = 32 * W;
  static constexpr int TAPS = 3 * T;
  // staged tap row stride: = 4 (mod 16) doubles -> the 8 points of a batch
  // sit on distinct bank groups when a lane reads its taps
  static constexpr int STRIDE = TAPS % 16 == 4 ? TAPS : TAPS + ((20 - TAPS % 16) % 16);
  static constexpr int SLOT = 8 * STRIDE;  // one batch of taps
};

// doubles of dynamic shared memory beyond the padded box
template <int T>
constexpr size_t v5_extra_doubles() {
  return 2 * static_cast<size_t>(Blk5<T>::W) * Blk5<T>::SLOT;
}

// stage the taps of points [b0, b0 + cnt) into a warp's slot (cp.async,
// 16-byte pieces, all lanes of the warp)
template <int T>
__device__ __forceinline__ void v5_stage_batch(double* slot, const double* taps, int64_t b0, int cnt, int lane) {
  using B = Blk5<T>;
  constexpr int H = B::TAPS / 2;  // 16-byte pieces per point
  const double* src = taps + b0 * B::TAPS;
  for (int k = lane; k < cnt * H; k += 32) {
    const int pt = k / H, r = k - pt * H;
    cp_async16(slot + pt * B::STRIDE + 2 * r, src + 2 * k);
  }
  cp_async_commit();
}

// The item's grid block -> the (padded) box: flat element loop, nine loads
// in flight per thread, indices by multiply-shift division and
// compare-and-subtract wrap.  (The flat loop it
// replaces did two integer divisions and three modulos per element -- ~100
// instructions each, 12-17 % of the interpolation's instruction stream at
// configs 5 / 4, in kernels whose limit is the issue slot.)
__device__ __forceinline__ int v5_wrap(int g, int M) {  // g in [0, M + ext): g mod M
  if (g >= M) {
    g -= M;
    if (g >= M) g %= M;
  }
  return g;
}

template <int NT>
__device__ __forceinline__ void v5_load_box(double* S, const double* gv, const DItem& it, int M, int bx1, int sp2,
                                            int tid) {
  constexpr int U = 9;  // loads in flight per thread (a 13^3 box is one round trip, 19^3 three)
  const int e1 = it.e1, e2 = it.e2, total = it.e0 * e1 * e2;
  // floor(v / e) = (v m) >> 20, m = floor(2^20 / e) + 1, exact while v e < 2^20:
  // a box that fits shared memory has extents <= 30, 30^4 < 2^20
  const unsigned m1 = (1u << 20) / static_cast<unsigned>(e1) + 1u, m2 = (1u << 20) / static_cast<unsigned>(e2) + 1u;
  for (int v0 = tid; v0 < total; v0 += NT * U) {
    double val[U];
    int so[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int v = v0 + u * NT;
      const bool ok = v < total;
      const int row = static_cast<int>((static_cast<unsigned>(v) * m2) >> 20);
      const int x0 = static_cast<int>((static_cast<unsigned>(row) * m1) >> 20);
      const int x2 = v - row * e2, x1 = row - x0 * e1;
      const int g0 = v5_wrap(it.a0 + x0, M), g1 = v5_wrap(it.a1 + x1, M), g2 = v5_wrap(it.a2 + x2, M);
      so[u] = ok ? (x0 * bx1 + x1) * sp2 + x2 : -1;
      val[u] = ok ? gv[(static_cast<int64_t>(g0) * M + g1) * M + g2] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (so[u] >= 0) S[so[u]] = val[u];
  }
}

template <int T>
__global__ void __launch_bounds__(Blk5<T>::NT, 2) interp_v5_kernel(PassArgs a, int box_doubles) {
  pdl_wait();
  using B = Blk5<T>;
  constexpr int TA = B::TA, TC = B::TC, KS = B::KS, W = B::W, NT = B::NT, SR = B::STRIDE;
  extern __shared__ __align__(16) double smem[];
  double* S = smem;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int q = lane & 3, r8 = lane >> 2;
  double* slots = smem + box_doubles + static_cast<size_t>(warp) * 2 * B::SLOT;
  const DItem it = a.items[blockIdx.x];
  const int bx1 = it.e1, e2 = it.e2, sp2 = v5_pad(e2);
  const int rows = it.e0 * it.e1;
  const int M = a.M;
  const int64_t p_begin = it.p_begin, p_end = it.p_end;
  const int nb = static_cast<int>((p_end - p_begin + 7) / 8);  // 8-point batches of the item
  // B-fragment walk of a pair tile: a-tile stride, c-tile stride
  const int ra = 2 * bx1 * sp2, rc = 4 * sp2;

  for (int vec = 0; vec < a.nvec; ++vec) {
    const double* gv = a.grid + vec * a.grid_stride;
    const double* xv = a.x ? a.x + vec * a.ldx : nullptr;
    double* yv = a.y ? a.y + vec * a.ldy : nullptr;
    // this warp's first batch: taps in flight while the box loads
    if (warp < nb)
      v5_stage_batch<T>(slots, a.taps, p_begin + 8 * warp, static_cast<int>(lmin(8, p_end - p_begin - 8 * warp)), lane);
    if (vec > 0) __syncthreads();  // every warp is done with the previous vector's box
    v5_load_box<NT>(S, gv, it, M, bx1, sp2, tid);
    __syncthreads();

    int r = it.run_begin;
    int cur = 0;  // slot of the batch being computed
    for (int b = warp; b < nb; b += W) {
      const int64_t b0 = p_begin + 8 * static_cast<int64_t>(b);
      const int cnt = static_cast<int>(lmin(8, p_end - b0));
      const int bn = b + W;
      if (bn < nb)  // next batch of this warp into the other slot
        v5_stage_batch<T>(slots + (cur ^ 1) * B::SLOT, a.taps, p_begin + 8 * static_cast<int64_t>(bn),
                          static_cast<int>(lmin(8, p_end - p_begin - 8 * static_cast<int64_t>(bn))), lane);
      if (bn < nb)
        cp_async_wait_1();
      else
        cp_async_wait_0();
      __syncwarp();
      const int64_t ipt = b0 + r8;  // this lane's point (A rows / C rows)
      const bool in = r8 < cnt;
      const double* w = slots + cur * B::SLOT + (in ? r8 : 0) * SR;
      // epilogue operands (lane q == 0 of each point)
      double xin = 0.0, sin_ = 1.0;
      int64_t ix = 0;
      if (q == 0 && in) {
        ix = a.perm ? static_cast<int64_t>(a.perm[ipt]) : ipt;
        if (xv && a.epilogue != EPI_KERNEL && a.epilogue != EPI_DEGREE) xin = xv[ix];
        if (a.epilogue == EPI_NORMALIZED || a.epilogue == EPI_LAPLACIAN) sin_ = a.s[ipt];
      }
      double wa[TA], wc[TC][2], we[KS];
#pragma unroll
      for (int t = 0; t < TA; ++t) wa[t] = w[2 * t + (q >> 1)];
#pragma unroll
      for (int t = 0; t < TC; ++t) {
        wc[t][0] = w[T + 4 * t + 2 * (q & 1)];
        wc[t][1] = w[T + 4 * t + 2 * (q & 1) + 1];
      }
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) we[ks] = w[2 * T + 4 * ks + q];
      // runs meeting this batch (runs are in point order; the cursor only
      // moves forward with the warp's batches)
      while (static_cast<int64_t>(a.runs[r].pstart) + a.runs[r].pcount <= b0 && r + 1 < it.run_end) ++r;
      double yacc = 0.0;
      int rr = r;
      while (true) {
        const DRun run = a.runs[rr];
        const int64_t rs = run.pstart, re_ = static_cast<int64_t>(run.pstart) + run.pcount;
        const bool mine = in && ipt >= rs && ipt < re_;
        double aF[KS];
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) aF[ks] = mine ? we[ks] : 0.0;
        const int o0 = run.off & 1023, o1 = (run.off >> 10) & 1023, o2 = (run.off >> 20) & 1023;
        // this lane's B-fragment element: pair (a = r8 / 4, c = r8 % 4) of a
        // tile, e = 4 ks + q
        const double* gb = S + ((o0 + (r8 >> 2)) * bx1 + (o1 + (r8 & 3))) * sp2 + o2 + q;
#pragma unroll
        for (int ta = 0; ta < TA; ++ta) {
          double z[TC][2];
#pragma unroll
          for (int tc = 0; tc < TC; ++tc) z[tc][0] = z[tc][1] = 0.0;
#pragma unroll
          for (int ks = 0; ks < KS; ++ks)
#pragma unroll
            for (int tc = 0; tc < TC; ++tc) dmma(z[tc][0], z[tc][1], aF[ks], gb[ta * ra + tc * rc + 4 * ks]);
          double K = 0.0;
#pragma unroll
          for (int tc = 0; tc < TC; ++tc) {
            K = fma(wc[tc][0], z[tc][0], K);
            K = fma(wc[tc][1], z[tc][1], K);
          }
          yacc = fma(wa[ta], K, yacc);
        }
        if (re_ < b0 + cnt && rr + 1 < it.run_end) {  // the batch continues in the next run
          ++rr;
          continue;
        }
        break;
      }
      r = rr;
      // the 4 lanes of each point hold disjoint pair columns
      yacc += __shfl_xor_sync(0xffffffffu, yacc, 1);
      yacc += __shfl_xor_sync(0xffffffffu, yacc, 2);
      if (q == 0 && in) {
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
      __syncwarp();  // the slot is restaged two batches later
      cur ^= 1;
    }
    cp_async_wait_0();
  }
}

}  // namespace fgsb

namespace fgsb {

// ---------------------------------------------------------------------------
// d = 3 spread, 2m in {12, 16}: W warps share every K-step of a run and each
// warp owns the item-box rows x0 = w (mod W).  In a run with footprint
// origin o0 the warp's a-values are a = (w - o0 mod W) + W i, i < 2m / W, so
// its accumulators (2m/W a-rows x 2m c x 2m e of the footprint) flush into
// box rows no other warp ever writes: no barrier per run (the v4 kernel's
// warps owned footprint-relative a-rows, which overlap between consecutive
// runs, and needed a CTA barrier around every flush).
//   G[(a,c)][e] += sum_j (wa_j[a] wc_j[c]) (x_j we_j[e])   M = 8 pairs, K = 4 points, N = 8 e
// The chunk staging (cp.async, double buffer) is the v4 kernel's.
// ---------------------------------------------------------------------------
template <int T, int W>
struct Blk5s {
  static constexpr int NT = 32 * W;
  static constexpr int RW = T / W;      // a-rows per warp
  static constexpr int TAW = RW / 2;    // a-tiles (2 rows) per warp
  static constexpr int TC = T / 4;      // c-tiles (4 c)
  static constexpr int NE = (T + 7) / 8;  // e-tiles (2m = 12 pads 12 -> 16)
  static constexpr int TW = TAW * TC;
  static constexpr int QS = 64;
  static constexpr int TAPS = 3 * T;
  static constexpr int STRIDE = Blk4<T, false>::STRIDE;
  static_assert(T % W == 0 && RW % 2 == 0, "each warp owns whole a-tiles");
};

template <int T, int W>
constexpr size_t v5s_extra_doubles() {
  using B = Blk5s<T, W>;
  return 2 * static_cast<size_t>(B::QS) * B::STRIDE + 2 * B::QS;
}

template <int T, int W>
__global__ void __launch_bounds__(Blk5s<T, W>::NT, 2) spread_v5_kernel(PassArgs a, int box_stride_smem) {
  pdl_wait();
  using B = Blk5s<T, W>;
  constexpr int NT = B::NT, QS = B::QS, TAPS = B::TAPS, SR = B::STRIDE;
  constexpr int TAW = B::TAW, TC = B::TC, TW = B::TW, NE = B::NE;
  extern __shared__ __align__(16) double smem[];
  double* S = smem;
  double* stg = smem + box_stride_smem;
  double* xs = stg + 2 * QS * SR;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int q = lane & 3, r8 = lane >> 2;
  const DItem it = a.items[blockIdx.x];
  const int bx1 = it.e1, bx2 = it.e2;
  const int V = it.e0 * it.e1 * it.e2;
  const int64_t p_begin = it.p_begin, p_end = it.p_end;
  const int nch = static_cast<int>((p_end - p_begin + QS - 1) / QS);

  for (int vec = 0; vec < a.nvec; ++vec) {
    const double* xv = a.x + vec * a.ldx;
    for (int v = tid; v < V; v += NT) S[v] = 0.0;
    v4_issue_chunk<TAPS, SR>(stg, a.taps, p_begin, static_cast<int>(lmin(QS, p_end - p_begin)), tid, NT);
    cp_async_commit();
    if (tid < QS && p_begin + tid < p_end) xs[tid] = v2_x(a, xv, p_begin + tid);
    int r = it.run_begin;
    DRun run = a.runs[r];
    double C[TW][NE][2];
#pragma unroll
    for (int t = 0; t < TW; ++t)
#pragma unroll
      for (int ne = 0; ne < NE; ++ne) C[t][ne][0] = C[t][ne][1] = 0.0;
    // this warp's first a-row of the run's footprint (box row = warp mod W)
    auto first_a = [&](const DRun& rn) { return ((warp - (rn.off & 1023)) % W + W) % W; };
    int a0 = first_a(run);

    auto flush = [&]() {
      const int o0 = run.off & 1023, o1 = (run.off >> 10) & 1023, o2 = (run.off >> 20) & 1023;
#pragma unroll
      for (int t = 0; t < TW; ++t) {
        const int ta = t / TC, tc = t % TC;
        const int aa = a0 + W * (2 * ta + (r8 >> 2)), cc = 4 * tc + (r8 & 3);
        double* row = S + ((o0 + aa) * bx1 + (o1 + cc)) * bx2 + o2;
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
        if (tid < qn) xnext = v2_x(a, xv, c1 + tid);
      }
      const double* sb = stg + buf * QS * SR;
      const double* xb = xs + buf * QS;
      while (true) {
        const int64_t rs = run.pstart, re_ = static_cast<int64_t>(run.pstart) + run.pcount;
        const int64_t s0 = rs > c0 ? rs : c0, s1 = lmin(re_, c1);
        // K-steps of 4 points aligned to the chunk, from the one holding s0
        for (int64_t k0 = c0 + ((s0 - c0) & ~int64_t{3}); k0 < s1; k0 += 4) {
          const int64_t jp = k0 + q;  // this lane's point of the K-step
          const bool ok = jp >= s0 && jp < s1;
          const double* w = sb + (ok ? (jp - c0) : 0) * SR;
          const double xj = ok ? xb[jp - c0] : 0.0;
          double wa[TAW], wc[TC];
#pragma unroll
          for (int t = 0; t < TAW; ++t) wa[t] = w[a0 + W * (2 * t + (r8 >> 2))];
#pragma unroll
          for (int t = 0; t < TC; ++t) wc[t] = w[T + 4 * t + (r8 & 3)];
          double bF[NE];  // x_j we_j[e], e = 8 ne + lane/4
#pragma unroll
          for (int ne = 0; ne < NE; ++ne) {
            const int e = 8 * ne + r8;
            bF[ne] = e < T ? xj * w[2 * T + e] : 0.0;
          }
          double af[TW];  // wa wc of pair (lane/4 row)
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
          a0 = first_a(run);
          continue;
        }
        break;
      }
      if (more && tid < qn) xs[(buf ^ 1) * QS + tid] = xnext;
    }
    __syncthreads();
    double* out = a.priv + (static_cast<int64_t>(vec) * gridDim.x + blockIdx.x) * a.box_stride;
    for (int v = tid; v < V; v += NT) out[v] = S[v];
    __syncthreads();
  }
}

}  // namespace fgsb
