// kernels_v3.cuh -- warp-resident-footprint interpolation for dense runs
// (d = 3, 2m in {8, 12, 16}).
//
// v2 splits a footprint over the whole CTA and must reduce every 16-point
// batch across warps behind a CTA barrier; ncu on config 4 showed that
// barrier plus the serial e-chains ("wait" + "barrier" stalls) capping the
// fp64 pipe at ~16 % realtime.  Here a group of G warps (G = 1 for 2m <= 12,
// 2 for 2m = 16) holds the run's entire (2m)^3 grid block in registers
// (Ra x Rc x Re values per lane) and the CTA's P groups walk different
// 16-point batches of each staged chunk:
//   * the contraction per point is Ra*Rc independent e-chains, then Ra
//     c-chains, then one a-chain -- 16 points in flight per lane;
//   * the 16 per-point partials of a warp are transposed by a 16-wide
//     butterfly; groups of two warps add their halves through shared memory
//     behind a 64-thread named barrier (2m = 16 only);
//   * the only CTA barrier is the one per staged chunk (cp.async pipeline).
#pragma once

#include "kernels_v2.cuh"

namespace fgsb {

template <int T>
struct Blk3 {
  static constexpr int G = T == 16 ? 2 : 1;   // warps per footprint group
  static constexpr int Ra = T == 16 ? 2 : (T == 12 ? 3 : 2);
  static constexpr int Rc = T == 16 ? 4 : (T == 12 ? 3 : 2);
  static constexpr int Re = T == 16 ? 8 : (T == 12 ? 6 : 4);
  static constexpr int AG = T / Ra, CG = T / Rc, EG = T / Re;
  static constexpr int LANES = AG * CG * EG;  // == 32 * G
  static constexpr int P = T == 16 ? 2 : (T == 12 ? 2 : 4);  // point streams per CTA
  static constexpr int NT = 32 * G * P;
  static constexpr int QB = 16;
  static constexpr int QS = P * QB;
  static constexpr int TAPS = 3 * T;
  static_assert(LANES == 32 * G, "footprint must map onto whole warps");
};

template <int T>
__global__ void __launch_bounds__(Blk3<T>::NT) interp_v3_kernel(PassArgs a, int box_stride_smem) {
  using B = Blk3<T>;
  constexpr int NT = B::NT, QS = B::QS, QB = B::QB, TAPS = B::TAPS, G = B::G;
  constexpr int Ra = B::Ra, Rc = B::Rc, Re = B::Re;
  extern __shared__ __align__(16) double smem[];
  double* S = smem;
  double* stg = smem + box_stride_smem;
  double* red = stg + 2 * QS * TAPS;  // [P][G][QB]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int grp = warp / G, wg = warp % G;  // group, warp within group
  const int l = wg * 32 + lane;             // lane within group
  const int ua = (l / (B::EG * B::CG)) * Ra;
  const int uc = ((l / B::EG) % B::CG) * Rc;
  const int ue = (l % B::EG) * Re;
  const DItem it = a.items[blockIdx.x];
  const int bx1 = it.e1, bx2 = it.e2;
  const int V = it.e0 * it.e1 * it.e2;
  const int M = a.M;
  const int64_t p_begin = it.p_begin, p_end = it.p_end;
  const int nch = static_cast<int>((p_end - p_begin + QS - 1) / QS);

  for (int vec = 0; vec < a.nvec; ++vec) {
    const double* gv = a.grid + vec * a.grid_stride;
    const double* xv = a.x ? a.x + vec * a.ldx : nullptr;
    double* yv = a.y ? a.y + vec * a.ldy : nullptr;
    v2_issue_chunk<TAPS>(stg, a.taps, p_begin, static_cast<int>(lmin(QS, p_end - p_begin)), tid, NT);
    cp_async_commit();
    for (int v = tid; v < V; v += NT) {
      const int x2 = v % bx2, x1 = (v / bx2) % bx1, x0 = v / (bx2 * bx1);
      S[v] = gv[(static_cast<int64_t>((it.a0 + x0) % M) * M + (it.a1 + x1) % M) * M + (it.a2 + x2) % M];
    }
    int r = it.run_begin;
    DRun run = a.runs[r];
    int loaded = -1;  // run whose block sits in g
    double g[Ra][Rc][Re];

    for (int k = 0; k < nch; ++k) {
      const int64_t c0 = p_begin + static_cast<int64_t>(k) * QS;
      const int64_t c1 = lmin(c0 + QS, p_end);
      const int buf = k & 1;
      cp_async_wait_0();
      __syncthreads();  // chunk k (and at k = 0 the box) visible; chunk k-1 consumed
      if (k + 1 < nch) {
        v2_issue_chunk<TAPS>(stg + (buf ^ 1) * QS * TAPS, a.taps, c1, static_cast<int>(lmin(QS, p_end - c1)), tid, NT);
        cp_async_commit();
      }
      const int64_t b0 = c0 + static_cast<int64_t>(grp) * QB;
      if (b0 >= c1) continue;
      const int qb = static_cast<int>(lmin(QB, c1 - b0));
      // prefetch the epilogue operands of this lane's point
      double xin = 0.0, sin_ = 1.0;
      int64_t ix = 0;
      if (wg == 0 && lane < qb) {
        const int64_t ip = b0 + lane;
        ix = a.perm ? static_cast<int64_t>(a.perm[ip]) : ip;
        if (xv && a.epilogue != EPI_KERNEL && a.epilogue != EPI_DEGREE) xin = xv[ix];
        if (a.epilogue == EPI_NORMALIZED || a.epilogue == EPI_LAPLACIAN) sin_ = a.s[ip];
      }
      const double* sb = stg + buf * QS * TAPS;
      double p[QB];
#pragma unroll
      for (int i = 0; i < QB; ++i) p[i] = 0.0;
      while (true) {
        // advance to the run containing the next unprocessed point of the batch
        while (static_cast<int64_t>(run.pstart) + run.pcount <= b0 && r + 1 < it.run_end) run = a.runs[++r];
        if (loaded != r) {
          const int o0 = run.off & 1023, o1 = (run.off >> 10) & 1023, o2 = (run.off >> 20) & 1023;
#pragma unroll
          for (int aa = 0; aa < Ra; ++aa)
#pragma unroll
            for (int cc = 0; cc < Rc; ++cc) {
              const double* row = S + ((o0 + ua + aa) * bx1 + (o1 + uc + cc)) * bx2 + o2 + ue;
#pragma unroll
              for (int e = 0; e < Re; ++e) g[aa][cc][e] = row[e];
            }
          loaded = r;
        }
        const int64_t rs = run.pstart, re_ = static_cast<int64_t>(run.pstart) + run.pcount;
        const int64_t s0 = rs > b0 ? rs : b0, s1 = lmin(re_, b0 + qb);
        const bool whole = s0 == b0 && s1 == b0 + QB;
        auto point = [&](int64_t ip) -> double {
          const double* w = sb + (ip - c0) * TAPS;
          double wa[Ra], wc[Rc], we[Re];
#pragma unroll
          for (int aa = 0; aa < Ra; ++aa) wa[aa] = w[ua + aa];
#pragma unroll
          for (int cc = 0; cc < Rc; ++cc) wc[cc] = w[T + uc + cc];
          if constexpr (Re % 2 == 0) {
            const double2* w2 = reinterpret_cast<const double2*>(w + 2 * T + ue);  // ue even: 16-byte aligned
#pragma unroll
            for (int e = 0; e < Re / 2; ++e) {
              const double2 t = w2[e];
              we[2 * e] = t.x;
              we[2 * e + 1] = t.y;
            }
          } else {
#pragma unroll
            for (int e = 0; e < Re; ++e) we[e] = w[2 * T + ue + e];
          }
          double pa = 0.0;
#pragma unroll
          for (int aa = 0; aa < Ra; ++aa) {
            double pc = 0.0;
#pragma unroll
            for (int cc = 0; cc < Rc; ++cc) {
              double r0 = 0.0, r1 = 0.0;  // two half-chains per row
#pragma unroll
              for (int e = 0; e < Re; e += 2) {
                r0 = fma(we[e], g[aa][cc][e], r0);
                if (e + 1 < Re) r1 = fma(we[e + 1], g[aa][cc][e + 1], r1);
              }
              pc = fma(wc[cc], r0 + r1, pc);
            }
            pa = fma(wa[aa], pc, pa);
          }
          return pa;
        };
        if (whole) {  // branch-free: 16 independent points for the scheduler
#pragma unroll
          for (int i = 0; i < QB; ++i) p[i] += point(b0 + i);
        } else {
#pragma unroll
          for (int i = 0; i < QB; ++i) {
            const int64_t ip = b0 + i;
            if (ip >= s0 && ip < s1) p[i] += point(ip);
          }
        }
        if (re_ < b0 + qb && r + 1 < it.run_end) {  // batch continues in the next run
          run = a.runs[++r];
          continue;
        }
        break;
      }
      // 16-wide warp butterfly: lane l (and l ^ 16) holds the warp sum of point l & 15
#pragma unroll
      for (int sft = 8; sft >= 1; sft >>= 1) {
        const bool upper = (lane & sft) != 0;
#pragma unroll
        for (int kk = 0; kk < sft; ++kk) {
          const double send = upper ? p[kk] : p[kk + sft];
          const double keep = upper ? p[kk + sft] : p[kk];
          p[kk] = keep + __shfl_xor_sync(0xffffffffu, send, sft);
        }
      }
      p[0] += __shfl_xor_sync(0xffffffffu, p[0], 16);
      double val = p[0];
      if (G > 1) {
        double* rg = red + grp * G * QB;
        if (wg > 0 && lane < QB) rg[wg * QB + lane] = val;
        asm volatile("bar.sync %0, %1;\n" ::"r"(1 + grp), "r"(32 * G) : "memory");
        if (wg == 0 && lane < QB)
#pragma unroll
          for (int w2 = 1; w2 < G; ++w2) val += rg[w2 * QB + lane];
        asm volatile("bar.sync %0, %1;\n" ::"r"(1 + grp), "r"(32 * G) : "memory");
      }
      if (wg == 0 && lane < qb) {
        const int64_t ip = b0 + lane;
        if (a.epilogue == EPI_DEGREE) {
          const double dg = val - a.k0;  // graphop.cpp:55-56
          a.degrees[ip] = dg;
          a.inv_sqrt[ip] = 1.0 / sqrt(dg);
          if (!(dg > 0.0)) atomicMin(a.bad_flag, static_cast<unsigned long long>(a.caller[ip]));
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
    cp_async_wait_0();
    __syncthreads();
  }
}

}  // namespace fgsb
