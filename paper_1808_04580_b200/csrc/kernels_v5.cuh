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
    for (int v = tid; v < rows * e2; v += NT) {
      const int row = v / e2, x2 = v - row * e2;
      const int x0 = row / bx1, x1 = row - x0 * bx1;
      S[row * sp2 + x2] = gv[(static_cast<int64_t>((it.a0 + x0) % M) * M + (it.a1 + x1) % M) * M + (it.a2 + x2) % M];
    }
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
