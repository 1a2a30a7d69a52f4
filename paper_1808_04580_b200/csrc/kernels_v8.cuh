// kernels_v8.cuh -- d = 3, 2m = 12 spread over the run-aligned slot layout
// (config 4: n = 2M Gaussian mixture, N = 64, m = 6).
//
// A DMMA tile is 8 wide, 2m = 12 is not: the v4 spread (M = (a, c) pairs,
// N = e padded 12 -> 16) spent a quarter of its tensor instructions on zero
// columns.  Here the e range is split 8 + 4:
//   e in [0, 8)   one DMMA per pair tile and K-step of 4 slots,
//   e in [8, 12)  plain DFMAs on the SAME A operand: lane (r8, q) already
//                 holds the pair product of row r8 for point q, so it
//                 accumulates its own point's 4 tail columns
//                 D[t][e'] += af[t] * we_q[8 + e'] and the 4 q-lanes are summed
//                 once per run (a 4 x 4 transpose-reduce: 3 shuffles).
// On this B200 a DFMA costs the fp64 pipe ~2.25 cycles for 32 FMAs, a DMMA 16
// for 256 -- nearly the same rate, and mixing them is free
// (tools/dmma_dfma_probe.cu: 3 DMMA + 12 DFMA = 81 cycles, ideal 72) -- so the
// tail costs about half a padded DMMA's pipe time.
//
// W = 6 / H warps; warp w owns the box c-rows = w (mod W) -- in a run with
// origin o1 its 2 H c values are cw + W j, cw = (w - o1) mod W -- and all 12
// a: 3 H pair tiles of 4 a x 2 c,
//   tile (t, h), row r8:  a = 4 t + r8 / 2,  c = cw + W (r8 % 2) + 2 W h.
// Flushes of consecutive runs never touch another warp's rows, so there is
// no barrier per run (the v4 kernel's two point streams flushed in turn
// through two CTA barriers per run).  x is folded into wc once per K-step.
// Measured (config 4): 0.356 ms with 2, 4 or 6 c-rows per warp (H = 1, 2, 3)
// and 12-24 warps per SM alike -- neither shared-memory bandwidth (73 % of the
// LSU wavefront peak at H = 1, 40 % at H = 2) nor occupancy binds; what does
// is issue slots: a DMMA holds its scheduler's issue port for 16 cycles and
// every other instruction adds its own.  H = 2 issues the
// fewest instructions per FMA that still fit 4 CTAs per SM.
// Staging is the v6 spread's ring of bulk-copied chunks on full/empty
// mbarriers.  The slot rows are 36 doubles (wa | wc | we), = 4 (mod 16), so
// the 4 slots of a K-step sit on distinct bank groups.
#pragma once

#include "kernels_v6.cuh"

namespace fgsb {

#ifndef FGS_V8S_QS
#define FGS_V8S_QS 64
#endif
#ifndef FGS_V8S_NS
#define FGS_V8S_NS 2
#endif
#ifndef FGS_V8S_H
#define FGS_V8S_H 2
#endif
#ifndef FGS_V8S_MINB
#define FGS_V8S_MINB 4
#endif
// H = c-pairs per warp: W = 6 / H warps, warp w owns the box c-rows = w (mod W)
template <int H_>
struct Blk8s {
  static constexpr int T = 12;
  static constexpr int H = H_;
  static constexpr int W = 6 / H;
  static_assert(W * H == 6, "H in {1, 2, 3}");
  static constexpr int NT = 32 * W;
  static constexpr int QS = FGS_V8S_QS;      // slots per staged chunk (multiple of kSlotAlign)
  static constexpr int NS = FGS_V8S_NS;      // ring stages
  static constexpr int MINB = FGS_V8S_MINB;  // CTAs per SM the registers are budgeted for
  static constexpr int SR = slot_row<12>();  // 36
};
using Blk8 = Blk8s<FGS_V8S_H>;

// staging doubles beyond the box: taps [NS][QS][SR] | x [NS][QS] | full[NS] | empty[NS]
constexpr size_t v8s_extra_doubles() {
  return static_cast<size_t>(Blk8::NS) * Blk8::QS * (Blk8::SR + 1) + 2 * Blk8::NS;
}

template <int H>
__global__ void __launch_bounds__(Blk8s<H>::NT, Blk8s<H>::MINB) spread_v8_kernel(PassArgs a_, int box_stride_smem) {
  pdl_wait();
  PassArgs a = a_;
  const ItemOfBlock ib = vsplit_narrow(a);
  using B = Blk8s<H>;
  constexpr int T = B::T, NT = B::NT, QS = B::QS, SR = B::SR, NS = B::NS, W = B::W;
  extern __shared__ __align__(16) double smem[];
  double* S = smem;
  double* stg = smem + box_stride_smem;
  double* xst = stg + NS * QS * SR;
  unsigned long long* full = reinterpret_cast<unsigned long long*>(xst + NS * QS);
  unsigned long long* empty = full + NS;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int q = lane & 3, r8 = lane >> 2;
  // this lane's pair row of tile (t, h): a = 4 t + ah, c = cw + ch + 2 W h
  const int ah = r8 >> 1, ch = W * (r8 & 1);
  const DItem it = a.items[ib.item];
  const int bx1 = it.e1, bx2 = it.e2;
  const int V = it.e0 * bx1 * bx2;
  const int s_begin = it.p_begin, s_end = it.p_end;  // slots, multiples of kSlotAlign
  const int nch = (s_end - s_begin + QS - 1) / QS;
  const int total = nch * a.nvec;  // chunks of the whole kernel (vector-major)

  if (tid == 0) {
    for (int i = 0; i < NS; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], W);
    }
    mbar_init_fence();
  }
  __syncthreads();
  // producer (thread 0): chunk g = (vector g / nch, chunk g % nch) -> stage g % NS
  auto issue = [&](int g) {
    const int st = g % NS, vec = g / nch, c0 = s_begin + (g - vec * nch) * QS;
    const int cnt = min(QS, s_end - c0);
    fence_proxy_async();
    mbar_expect_tx(&full[st], static_cast<unsigned>(cnt) * (SR + 1) * 8u);
    bulk_g2s(stg + st * QS * SR, a.taps + static_cast<int64_t>(c0) * SR, static_cast<unsigned>(cnt) * SR * 8u,
             &full[st]);
    bulk_g2s(xst + st * QS, a.xs + vec * a.ldxs + c0, static_cast<unsigned>(cnt) * 8u, &full[st]);
  };
  if (tid == 0)
    for (int g = 0; g < NS - 1 && g < total; ++g) issue(g);

  int g = 0;  // chunk being consumed
  for (int vec = 0; vec < a.nvec; ++vec) {
    if (vec > 0) __syncthreads();  // the previous vector's box has been written out
    for (int v = tid; v < V; v += NT) S[v] = 0.0;
    __syncthreads();
    int r = it.run_begin;
    DRun run = a.runs[r];
    DRun nxt = a.runs[min(r + 1, it.run_end - 1)];    // one run ahead
    int cur = run.pstart;                             // K-step cursor (slots)
    int kend = run.pstart + ((run.pcount + 3) & ~3);  // the run's last K-step end
    // this warp's first c in the run (1026 = 0 mod W)
    int cw = (warp + 1026 - ((run.off >> 10) & 1023)) % W;
    double C[H][3][2];  // DMMA accumulators: e = 2 q + i
    double D[H][3][4];  // this lane's point q, e = 8 + e'
#pragma unroll
    for (int h = 0; h < H; ++h)
#pragma unroll
      for (int t = 0; t < 3; ++t) {
        C[h][t][0] = C[h][t][1] = 0.0;
#pragma unroll
        for (int e = 0; e < 4; ++e) D[h][t][e] = 0.0;
      }

    auto flush = [&]() {
      const int o0 = run.off & 1023, o1 = (run.off >> 10) & 1023, o2 = (run.off >> 20) & 1023;
      const bool odd = q & 1, hi = q & 2;
      const int et = 8 + ((q & 1) << 1) + (q >> 1);  // the tail column this lane ends up with
#pragma unroll
      for (int h = 0; h < H; ++h)
#pragma unroll
        for (int t = 0; t < 3; ++t) {
          // 4 x 4 transpose-reduce of the tail partials over the 4 q-lanes
          const double k0 = odd ? D[h][t][2] : D[h][t][0], k1 = odd ? D[h][t][3] : D[h][t][1];
          const double s0 = odd ? D[h][t][0] : D[h][t][2], s1 = odd ? D[h][t][1] : D[h][t][3];
          const double u0 = k0 + __shfl_xor_sync(0xffffffffu, s0, 1);
          const double u1 = k1 + __shfl_xor_sync(0xffffffffu, s1, 1);
          const double keep = hi ? u1 : u0, send = hi ? u0 : u1;
          const double tail = keep + __shfl_xor_sync(0xffffffffu, send, 2);
          double* row = S + ((o0 + 4 * t + ah) * bx1 + (o1 + cw + ch + 2 * W * h)) * bx2 + o2;
          row[2 * q] += C[h][t][0];
          row[2 * q + 1] += C[h][t][1];
          row[et] += tail;
          C[h][t][0] = C[h][t][1] = 0.0;
#pragma unroll
          for (int e = 0; e < 4; ++e) D[h][t][e] = 0.0;
        }
    };

    bool done = false;
    for (int k = 0; k < nch; ++k, ++g) {
      // keep NS - 1 chunks in flight: chunk g + NS - 1 reuses the stage of
      // chunk g - 1, free once every warp has released it
      if (tid == 0 && g + NS - 1 < total) {
        if (g >= 1) mbar_wait(&empty[(g - 1) % NS], ((g - 1) / NS) & 1);
        issue(g + NS - 1);
      }
      const int c0 = s_begin + k * QS;
      const int cend = min(c0 + QS, s_end);
      const int st = g % NS;
      const double* buf = stg + st * QS * SR;
      const double* xb = xst + st * QS;
      mbar_wait(&full[st], (g / NS) & 1);
      if (!done) {
        while (true) {
          const int stop = min(kend, cend);
          const double* row = buf + (cur - c0 + q) * SR;
          const double* xr = xb + (cur - c0 + q);
          for (; cur < stop; cur += 4, row += 4 * SR, xr += 4) {
            const double xv = *xr;
            const double w0 = row[ah], w1 = row[4 + ah], w2 = row[8 + ah];
            const double b = row[2 * T + r8];
            const double2 t01 = *reinterpret_cast<const double2*>(row + 2 * T + 8);
            const double2 t23 = *reinterpret_cast<const double2*>(row + 2 * T + 10);
#pragma unroll
            for (int h = 0; h < H; ++h) {
              const double xw = row[T + cw + ch + 2 * W * h] * xv;  // x wc[c]
              const double af[3] = {w0 * xw, w1 * xw, w2 * xw};
#pragma unroll
              for (int t = 0; t < 3; ++t) dmma(C[h][t][0], C[h][t][1], af[t], b);
#pragma unroll
              for (int t = 0; t < 3; ++t) {
                D[h][t][0] = fma(af[t], t01.x, D[h][t][0]);
                D[h][t][1] = fma(af[t], t01.y, D[h][t][1]);
                D[h][t][2] = fma(af[t], t23.x, D[h][t][2]);
                D[h][t][3] = fma(af[t], t23.y, D[h][t][3]);
              }
            }
          }
          if (cur < kend) break;  // the run continues in the next chunk
          flush();
          if (++r >= it.run_end) {
            done = true;
            break;
          }
          run = nxt;
          nxt = a.runs[min(r + 1, it.run_end - 1)];
          cur = run.pstart;
          kend = run.pstart + ((run.pcount + 3) & ~3);
          cw = (warp + 1026 - ((run.off >> 10) & 1023)) % W;
          if (cur >= cend) break;
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
    }
    __syncthreads();  // every warp's flushes are in the box
    double* out = a.priv + (static_cast<int64_t>(vec) * ib.nitems + ib.item) * a.box_stride;
    for (int v = tid; v < V; v += NT) out[v] = S[v];
  }
}

}  // namespace fgsb
