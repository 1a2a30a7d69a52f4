// kernels_v6.cuh -- d = 3, 2m = 16 spread and interpolation over the
// run-aligned slot layout (config 5: ~73 points per footprint).
//
// The plan lays every item's runs (points sharing one footprint) out in a
// slot space where each run starts on a multiple of 8 slots; the pad slots
// map to no point (slots[s] = -1: zero taps, x = 0, no output).  K-steps of
// 4 slots (spread) and batches of 8 slots (interpolation) then never
// straddle two runs, so the inner loops carry no per-lane run masks, no run
// cursor compares and no partial-batch re-runs (v5: a batch crossing a run
// boundary ran the whole footprint twice; ~10 % of the interpolation's
// DMMAs at config 5).
//
// Spread, per run and K-step of 4 slots (points k):
//   G[a][(c, e)] += sum_k wa_k[a] * ((x_k wc_k[c]) we_k[e])
//   A = wa (8 a x 4 points, straight from the staged taps, no product),
//   B = (x wc) we (4 points x 8 e of one c): one DMUL per fragment.
// x multiplies the staged wc per K-step (x0 = x wc[c0], x1 = x wc[c0 + 8]),
// so a warp's K-step is 7 LDS + 6 DMUL +
// 8 DMMA (v5: 8 LDS + 6 DMUL, plus the lane masks).  (Folding x into wc
// once per slot cooperatively -- each warp a share of a chunk, one chunk
// ahead, a `folded` mbarrier -- saves 2 DMUL per K-step but re-couples the
// warps like a per-chunk barrier: C5 spread 48.9 -> 51.7 ms.)  Warp w owns the box
// c-rows = w (mod 8): in a run with origin o1 its two c values are
// c0 = (w - o1) mod 8 and c0 + 8, both a-tiles and both e-halves (16
// accumulators per lane); flushes of consecutive runs never touch another
// warp's rows, so no barrier per run.
//
// Interpolation: the v5 kernel (per-warp 8-point batches, B fragments from
// the bank-padded box) with one run per batch.
//
// Staging is TMA bulk copies (cp.async.bulk, completion on mbarriers): the
// plan stores the taps in slot order with rows padded to the staged row
// stride (52 doubles), so a spread chunk (64 slots, 26.6 KB) and an
// interpolation batch (8 slots, 3.3 KB) are one contiguous copy each, issued
// by one thread, with no per-thread address math and no dependent index
// loads in the staging path.  The spread's x comes pre-gathered in slot order
// (slot_gather_kernel: one pass over the block, pads 0, s applied).
#pragma once

#include "kernels_v5.cuh"
#include "tma.cuh"

namespace fgsb {

constexpr int kSlotAlign = 8;  // run starts in the slot space
// doubles per slot-ordered taps row: wa | wc | we | pad, = 4 (mod 16) -- the
// interpolation's staged row (Blk5<T>::STRIDE): 52 for 2m = 16, 36 for 2m = 12
// (= 3 2m, the v4 spread's staging stride, so it reads the slot rows as is)
template <int T>
constexpr int slot_row() {
  return Blk5<T>::STRIDE;
}
constexpr int kSlotRow = slot_row<16>();
inline int slot_row_of(int T) { return T == 16 ? slot_row<16>() : slot_row<12>(); }
static_assert(slot_row<12>() == 36, "2m = 12 slot rows are unpadded");

#ifndef FGS_V6S_QS
#define FGS_V6S_QS 64
#endif
#ifndef FGS_V6S_NS
#define FGS_V6S_NS 2
#endif
#ifndef FGS_V6S_MINB
#define FGS_V6S_MINB 2
#endif
struct Blk6s {
  static constexpr int T = 16;
  static constexpr int W = 8;       // warps; warp w owns box c-rows = w (mod 8)
  static constexpr int NT = 32 * W;
  // slots per staged chunk (multiple of kSlotAlign): 64 x 2 stages (C5 spread
  // 48.5 -> 47.25 ms against 32 x 4 once the taps come from L2: half the
  // per-chunk barrier waits and index math)
  static constexpr int QS = FGS_V6S_QS;
  static constexpr int NS = FGS_V6S_NS;  // ring stages
  static constexpr int MINB = FGS_V6S_MINB;  // CTAs per SM the registers are budgeted for
  // staged slot row = the global slot-ordered taps row: wa[16] | wc[16] |
  // we[16] | pad; 52 = 4 (mod 16) doubles -> the 4 slots of a K-step sit on
  // distinct bank groups
  static constexpr int SR = kSlotRow;
};

// staging doubles beyond the box: taps [NS][QS][SR] | x [NS][QS] | full[NS] | empty[NS]
constexpr size_t v6s_extra_doubles() {
  return static_cast<size_t>(Blk6s::NS) * Blk6s::QS * (Blk6s::SR + 1) + 2 * Blk6s::NS;
}

// the vectors gathered into slot order for the spread: xs[v][s] = s[src] x[src]
// (scale_input) or x[src], 0 on pad slots (v2_x over the slot map)
__global__ void slot_gather_kernel(PassArgs a, int64_t nslots, double* out) {
  pdl_wait();
  if (a.perm != nullptr) {
    // caller order: x[perm[src]] is a random gather, so one vector at a time
    // (an 80 MB vector stays in L2; all vectors of a slot at once measured
    // 98.7 -> 99.9 ms on the caller-order config-5 block)
    const int64_t total = nslots * a.nvec;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
      const int64_t v = i / nslots, sl = i - v * nslots;
      const int src = a.slots[sl];
      double val = 0.0;
      if (src >= 0) {
        val = a.x[v * a.ldx + a.perm[src]];
        if (a.scale_input) val = __dmul_rn(a.s[src], val);
      }
      out[v * nslots + sl] = val;
    }
    return;
  }
  // internal order: one thread per slot, all vectors of the block -- the slot
  // map and s are read once per slot instead of once per (slot, vector)
  // (config 5, 16 vectors: 1.13 -> 0.5 ms)
  for (int64_t sl = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; sl < nslots;
       sl += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int src = a.slots[sl];
    if (src < 0) {
      for (int v = 0; v < a.nvec; ++v) out[v * nslots + sl] = 0.0;
      continue;
    }
    const double sc = a.scale_input ? a.s[src] : 1.0;
    const double* xp = a.x + src;
    double* op = out + sl;
    int v = 0;
    for (; v + 4 <= a.nvec; v += 4) {
      double val[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) val[u] = xp[(v + u) * a.ldx];
#pragma unroll
      for (int u = 0; u < 4; ++u) op[(v + u) * nslots] = a.scale_input ? __dmul_rn(sc, val[u]) : val[u];
    }
    for (; v < a.nvec; ++v) {
      const double val = xp[v * a.ldx];
      op[v * nslots] = a.scale_input ? __dmul_rn(sc, val) : val;
    }
  }
}

__global__ void __launch_bounds__(Blk6s::NT, Blk6s::MINB) spread_v6_kernel(PassArgs a_, int box_stride_smem) {
  pdl_wait();
  PassArgs a = a_;
  const ItemOfBlock ib = vsplit_narrow(a);
  using B = Blk6s;
  constexpr int T = B::T, NT = B::NT, QS = B::QS, SR = B::SR, NS = B::NS, W = B::W;
  extern __shared__ __align__(16) double smem[];
  double* S = smem;
  double* stg = smem + box_stride_smem;
  double* xst = stg + NS * QS * SR;
  unsigned long long* full = reinterpret_cast<unsigned long long*>(xst + NS * QS);
  unsigned long long* empty = full + NS;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int q = lane & 3, r8 = lane >> 2;
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
    __syncthreads();  // flushes of this vector may start as soon as a warp finishes its first run
    int r = it.run_begin;
    DRun run = a.runs[r];
    DRun nxt = a.runs[min(r + 1, it.run_end - 1)];    // one run ahead: the load is off the flush path
    int cur = run.pstart;                             // K-step cursor (slots)
    int kend = run.pstart + ((run.pcount + 3) & ~3);  // the run's last K-step end
    int cw = (warp - ((run.off >> 10) & 1023)) & 7;   // this warp's first c in the run
    double C[2][2][2][2];  // [a-tile][c][e-half][pair]
#pragma unroll
    for (int t = 0; t < 2; ++t)
#pragma unroll
      for (int c = 0; c < 2; ++c)
#pragma unroll
        for (int h = 0; h < 2; ++h) C[t][c][h][0] = C[t][c][h][1] = 0.0;

    auto flush = [&]() {
      const int o0 = run.off & 1023, o1 = (run.off >> 10) & 1023, o2 = (run.off >> 20) & 1023;
#pragma unroll
      for (int t = 0; t < 2; ++t)
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          double* row = S + ((o0 + 8 * t + r8) * bx1 + (o1 + cw + 8 * c)) * bx2 + o2 + 2 * q;
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            row[8 * h] += C[t][c][h][0];
            row[8 * h + 1] += C[t][c][h][1];
            C[t][c][h][0] = C[t][c][h][1] = 0.0;
          }
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
            const double a0 = row[r8], a1 = row[8 + r8];
            const double x0 = row[T + cw] * xv, x1 = row[T + cw + 8] * xv;
            const double e0 = row[2 * T + r8], e1 = row[2 * T + 8 + r8];
            const double b00 = x0 * e0, b01 = x0 * e1, b10 = x1 * e0, b11 = x1 * e1;
            dmma(C[0][0][0][0], C[0][0][0][1], a0, b00);
            dmma(C[1][0][0][0], C[1][0][0][1], a1, b00);
            dmma(C[0][0][1][0], C[0][0][1][1], a0, b01);
            dmma(C[1][0][1][0], C[1][0][1][1], a1, b01);
            dmma(C[0][1][0][0], C[0][1][0][1], a0, b10);
            dmma(C[1][1][0][0], C[1][1][0][1], a1, b10);
            dmma(C[0][1][1][0], C[0][1][1][1], a0, b11);
            dmma(C[1][1][1][0], C[1][1][1][1], a1, b11);
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
          cw = (warp - ((run.off >> 10) & 1023)) & 7;
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

// ---------------------------------------------------------------------------
// interpolation over run-aligned 8-slot batches (see kernels_v5.cuh for the
// fragment layout); each warp stages its next batch's 8 taps rows with one
// bulk copy on its own mbarrier pair (double buffer)
// ---------------------------------------------------------------------------
template <int T>
constexpr size_t v6i_extra_doubles() {
  return v5_extra_doubles<T>() + 2 * static_cast<size_t>(Blk5<T>::W);
}

// EXT > 0: the box is laid out with the plan's maximal extent (tile B + 2m - 1)
// in every item, so the B-fragment offsets ta ra + tc rc + 4 ks are immediates
// (runtime strides cost ~2 IMADs per DMMA at 2m = 12, and a DMMA's issue slot
// is the kernel's limit); EXT = 0: per-item strides.
template <int T, int EXT>
__global__ void __launch_bounds__(Blk5<T>::NT, 2) interp_v6_kernel(PassArgs a_, int box_doubles) {
  pdl_wait();
  PassArgs a = a_;
  const ItemOfBlock ib = vsplit_narrow(a);
  using B = Blk5<T>;
  constexpr int TA = B::TA, TC = B::TC, KS = B::KS, W = B::W, NT = B::NT, SR = B::STRIDE;
  static_assert(SR == slot_row<T>(), "staged row = global slot-ordered row");
  extern __shared__ __align__(16) double smem[];
  double* S = smem;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int q = lane & 3, r8 = lane >> 2;
  double* slots = smem + box_doubles + static_cast<size_t>(warp) * 2 * B::SLOT;
  unsigned long long* mb =
      reinterpret_cast<unsigned long long*>(smem + box_doubles + static_cast<size_t>(W) * 2 * B::SLOT) + 2 * warp;
  const DItem it = a.items[ib.item];
  const int e1 = it.e1, e2 = it.e2;
  const int bx1 = EXT > 0 ? EXT : e1, sp2 = EXT > 0 ? v5_pad(EXT) : v5_pad(e2);  // box strides
  const int rows = it.e0 * e1;
  const int M = a.M;
  const int s_begin = it.p_begin;
  const int nb = (it.p_end - s_begin) / 8;  // 8-slot batches of the item
  const int ra = 2 * bx1 * sp2, rc = 4 * sp2;
  if (lane == 0) {
    mbar_init(&mb[0], 1);
    mbar_init(&mb[1], 1);
    mbar_init_fence();
  }
  __syncwarp();
  auto issue = [&](unsigned g, int batch) {  // lane 0
    const int b = static_cast<int>(g & 1u);
    fence_proxy_async();
    mbar_expect_tx(&mb[b], 8u * SR * 8u);
    bulk_g2s(slots + b * B::SLOT, a.taps + static_cast<int64_t>(s_begin + 8 * batch) * SR, 8u * SR * 8u, &mb[b]);
  };

  unsigned g = 0;  // batches this warp consumed (all vectors): buffer g & 1, phase (g >> 1) & 1
  for (int vec = 0; vec < a.nvec; ++vec) {
    const double* gv = a.grid + vec * a.grid_stride;
    const double* xv = a.x ? a.x + vec * a.ldx : nullptr;
    double* yv = a.y ? a.y + vec * a.ldy : nullptr;
    if (warp < nb && lane == 0) issue(g, warp);
    if (vec > 0) __syncthreads();  // every warp is done with the previous vector's box
    v5_load_box<NT>(S, gv, it, M, bx1, sp2, tid);
    __syncthreads();

    // per batch: its run's footprint offset (plan array, one per 8 slots) and
    // this lane's point, loaded one batch ahead with the epilogue operands
    const bool need_x = xv && a.epilogue != EPI_KERNEL && a.epilogue != EPI_DEGREE;
    const bool need_s = a.epilogue == EPI_NORMALIZED || a.epilogue == EPI_LAPLACIAN;
    int src_n = -1, off_n = 0;
    if (warp < nb) {
      src_n = a.slots[s_begin + 8 * warp + r8];
      off_n = a.boff[(s_begin >> 3) + warp];
    }
    for (int bt = warp; bt < nb; bt += W, ++g) {
      const int src = src_n, off = off_n;
      if (bt + W < nb) {
        if (lane == 0) issue(g + 1, bt + W);
        src_n = a.slots[s_begin + 8 * (bt + W) + r8];
        off_n = a.boff[(s_begin >> 3) + bt + W];
      }
      // epilogue operands (lane q == 0 of each real point; others read index 0)
      const bool mine = q == 0 && src >= 0;
      const int64_t ix = mine ? (a.perm ? static_cast<int64_t>(a.perm[src]) : src) : 0;
      const double xin = need_x && mine ? xv[ix] : 0.0;
      const double sin_ = need_s && mine ? a.s[src] : 1.0;
      mbar_wait(&mb[g & 1u], (g >> 1) & 1u);
      const double* w = slots + (g & 1u) * B::SLOT + r8 * SR;
      double wa[TA], wc[TC][2], aF[KS];
#pragma unroll
      for (int t = 0; t < TA; ++t) wa[t] = w[2 * t + (q >> 1)];
#pragma unroll
      for (int t = 0; t < TC; ++t) {
        wc[t][0] = w[T + 4 * t + 2 * (q & 1)];
        wc[t][1] = w[T + 4 * t + 2 * (q & 1) + 1];
      }
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) aF[ks] = w[2 * T + 4 * ks + q];  // zero on pad slots
      const int o0 = off & 1023, o1 = (off >> 10) & 1023, o2 = (off >> 20) & 1023;
      const double* gb = S + ((o0 + (r8 >> 2)) * bx1 + (o1 + (r8 & 3))) * sp2 + o2 + q;
      double yacc = 0.0;
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
      yacc += __shfl_xor_sync(0xffffffffu, yacc, 1);
      yacc += __shfl_xor_sync(0xffffffffu, yacc, 2);
      if (mine) {
        const double val = yacc;
        if (a.epilogue == EPI_DEGREE) {
          const double dg = val - a.k0;  // graphop.cpp:55-56
          a.degrees[src] = dg;
          a.inv_sqrt[src] = 1.0 / sqrt(dg);
          if (!(dg > 0.0)) atomicMin(a.bad_flag, static_cast<unsigned long long>(a.caller[src]));
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
      __syncwarp();  // the buffer is restaged by the next-but-one batch
    }
  }
}

// ---------------------------------------------------------------------------
// interpolation, two batches per B-fragment load (interp_v7_kernel<T>).
// A warp takes units of two consecutive 8-slot batches (16 slots, one bulk
// copy).  When both batches belong to the same run they share every B
// fragment: each grid value read from the box feeds two DMMAs (the A
// fragments of the two batches), halving the shared-memory loads per DMMA.
// The unit's taps move to registers right after they land, so one staging
// buffer per warp suffices (the next unit is copied into it while this one
// computes).  A unit whose batches straddle two runs runs them one by one.
// ---------------------------------------------------------------------------
template <int T>
struct V7Frag {
  double aF[Blk5<T>::KS];
  double wa[Blk5<T>::TA];
  double wc[Blk5<T>::TC][2];
};

template <int T>
__device__ __forceinline__ void v7_load(V7Frag<T>& f, const double* w, int q) {
#pragma unroll
  for (int t = 0; t < Blk5<T>::TA; ++t) f.wa[t] = w[2 * t + (q >> 1)];
#pragma unroll
  for (int t = 0; t < Blk5<T>::TC; ++t) {
    f.wc[t][0] = w[T + 4 * t + 2 * (q & 1)];
    f.wc[t][1] = w[T + 4 * t + 2 * (q & 1) + 1];
  }
#pragma unroll
  for (int ks = 0; ks < Blk5<T>::KS; ++ks) f.aF[ks] = w[2 * T + 4 * ks + q];  // zero on pad slots
}

// y partial of NB (1 or 2) batches sharing the footprint block gb
template <int T, int NB>
__device__ __forceinline__ void v7_compute(const V7Frag<T>* f, const double* gb, int ra, int rc, double* yacc) {
  constexpr int TA = Blk5<T>::TA, TC = Blk5<T>::TC, KS = Blk5<T>::KS;
#pragma unroll
  for (int h = 0; h < NB; ++h) yacc[h] = 0.0;
#pragma unroll
  for (int ta = 0; ta < TA; ++ta) {
    double z[NB][TC][2];
#pragma unroll
    for (int h = 0; h < NB; ++h)
#pragma unroll
      for (int tc = 0; tc < TC; ++tc) z[h][tc][0] = z[h][tc][1] = 0.0;
#pragma unroll
    for (int ks = 0; ks < KS; ++ks)
#pragma unroll
      for (int tc = 0; tc < TC; ++tc) {
        const double bv = gb[ta * ra + tc * rc + 4 * ks];
#pragma unroll
        for (int h = 0; h < NB; ++h) dmma(z[h][tc][0], z[h][tc][1], f[h].aF[ks], bv);
      }
#pragma unroll
    for (int h = 0; h < NB; ++h) {
      double K = 0.0;
#pragma unroll
      for (int tc = 0; tc < TC; ++tc) {
        K = fma(f[h].wc[tc][0], z[h][tc][0], K);
        K = fma(f[h].wc[tc][1], z[h][tc][1], K);
      }
      yacc[h] = fma(f[h].wa[ta], K, yacc[h]);
    }
  }
}

template <int T, int EXT>
__global__ void __launch_bounds__(Blk5<T>::NT, 2) interp_v7_kernel(PassArgs a_, int box_doubles) {
  pdl_wait();
  PassArgs a = a_;
  const ItemOfBlock ib = vsplit_narrow(a);
  using B = Blk5<T>;
  constexpr int W = B::W, NT = B::NT, SR = B::STRIDE;
  static_assert(SR == slot_row<T>(), "staged row = global slot-ordered row");
  extern __shared__ __align__(16) double smem[];
  double* S = smem;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int q = lane & 3, r8 = lane >> 2;
  double* buf = smem + box_doubles + static_cast<size_t>(warp) * 2 * B::SLOT;  // 16 slot rows
  unsigned long long* mb =
      reinterpret_cast<unsigned long long*>(smem + box_doubles + static_cast<size_t>(W) * 2 * B::SLOT) + warp;
  const DItem it = a.items[ib.item];
  const int e1 = it.e1, e2 = it.e2;
  const int bx1 = EXT > 0 ? EXT : e1, sp2 = EXT > 0 ? v5_pad(EXT) : v5_pad(e2);  // box strides
  const int rows = it.e0 * e1;
  const int M = a.M;
  const int s_begin = it.p_begin;
  const int nb = (it.p_end - s_begin) / 8;  // 8-slot batches of the item
  const int nu = (nb + 1) / 2;             // units of two batches
  const int ra = 2 * bx1 * sp2, rc = 4 * sp2;
  const int bbase = s_begin >> 3;          // global index of the item's first batch
  if (lane == 0) {
    mbar_init(mb, 1);
    mbar_init_fence();
  }
  __syncwarp();
  auto issue = [&](int u) {  // lane 0: the unit's 8 or 16 taps rows, one bulk copy
    const int cnt = min(2, nb - 2 * u) * 8;
    fence_proxy_async();
    mbar_expect_tx(mb, static_cast<unsigned>(cnt) * SR * 8u);
    bulk_g2s(buf, a.taps + static_cast<int64_t>(s_begin + 16 * u) * SR, static_cast<unsigned>(cnt) * SR * 8u, mb);
  };
  const bool need_s = a.epilogue == EPI_NORMALIZED || a.epilogue == EPI_LAPLACIAN;
  unsigned phase = 0;

  for (int vec = 0; vec < a.nvec; ++vec) {
    const double* gv = a.grid + vec * a.grid_stride;
    const double* xv = a.x ? a.x + vec * a.ldx : nullptr;
    double* yv = a.y ? a.y + vec * a.ldy : nullptr;
    const bool need_x = xv && a.epilogue != EPI_KERNEL && a.epilogue != EPI_DEGREE;
    if (warp < nu && lane == 0) issue(warp);
    if (vec > 0) __syncthreads();  // every warp is done with the previous vector's box
    v5_load_box<NT>(S, gv, it, M, bx1, sp2, tid);
    __syncthreads();

    // a unit's slot map entries and run offsets are loaded one unit ahead
    // (at the top of the unit they were a dependent global load in front of
    // the epilogue operands and the footprint address: 4.6 % of the stall
    // samples)
    int src_n[2] = {-1, -1}, off_n[2] = {0, 0};
    auto prefetch = [&](int u) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int b = min(2 * u + h, nb - 1);
        src_n[h] = 2 * u + h < nb ? a.slots[s_begin + 8 * b + r8] : -1;
        off_n[h] = a.boff[bbase + b];
      }
    };
    if (warp < nu) prefetch(warp);
    for (int u = warp; u < nu; u += W) {
      const int nbat = min(2, nb - 2 * u);
      const int src[2] = {src_n[0], src_n[1]}, off[2] = {off_n[0], off_n[1]};
      if (u + W < nu) prefetch(u + W);
      double xin[2], sin_[2];
      int64_t ix[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const bool mine = q == 0 && src[h] >= 0;
        ix[h] = mine ? (a.perm ? static_cast<int64_t>(a.perm[src[h]]) : src[h]) : 0;
        xin[h] = need_x && mine ? xv[ix[h]] : 0.0;
        sin_[h] = need_s && mine ? a.s[src[h]] : 1.0;
      }
      mbar_wait(mb, phase);
      phase ^= 1u;
      V7Frag<T> f[2];
      v7_load<T>(f[0], buf + r8 * SR, q);
      if (nbat == 2) v7_load<T>(f[1], buf + (8 + r8) * SR, q);
      __syncwarp();  // every lane has its taps: the buffer takes the next unit
      if (u + W < nu && lane == 0) issue(u + W);
      double yacc[2] = {0.0, 0.0};
      auto footprint = [&](int o) {
        const int o0 = o & 1023, o1 = (o >> 10) & 1023, o2 = (o >> 20) & 1023;
        return S + ((o0 + (r8 >> 2)) * bx1 + (o1 + (r8 & 3))) * sp2 + o2 + q;
      };
      if (nbat == 2 && off[0] == off[1]) {
        v7_compute<T, 2>(f, footprint(off[0]), ra, rc, yacc);
      } else {
        v7_compute<T, 1>(&f[0], footprint(off[0]), ra, rc, &yacc[0]);
        if (nbat == 2) v7_compute<T, 1>(&f[1], footprint(off[1]), ra, rc, &yacc[1]);
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        double yv_ = yacc[h];
        yv_ += __shfl_xor_sync(0xffffffffu, yv_, 1);
        yv_ += __shfl_xor_sync(0xffffffffu, yv_, 2);
        if (q == 0 && src[h] >= 0) {
          const int sr = src[h];
          if (a.epilogue == EPI_DEGREE) {
            const double dg = yv_ - a.k0;  // graphop.cpp:55-56
            a.degrees[sr] = dg;
            a.inv_sqrt[sr] = 1.0 / sqrt(dg);
            if (!(dg > 0.0)) atomicMin(a.bad_flag, static_cast<unsigned long long>(a.caller[sr]));
          } else {
            double out;
            switch (a.epilogue) {
              case EPI_KERNEL: out = yv_; break;
              case EPI_WEIGHT: out = yv_ - a.k0 * xin[h]; break;
              case EPI_NORMALIZED: out = sin_[h] * (yv_ - a.k0 * __dmul_rn(sin_[h], xin[h])); break;
              default: out = xin[h] - sin_[h] * (yv_ - a.k0 * __dmul_rn(sin_[h], xin[h])); break;
            }
            yv[ix[h]] = out;
          }
        }
      }
    }
  }
}

}  // namespace fgsb
