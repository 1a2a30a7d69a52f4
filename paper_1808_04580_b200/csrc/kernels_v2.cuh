// kernels_v2.cuh -- register-blocked, cp.async-pipelined spread and
// interpolation kernels (the fast path for 2m <= 16).
//
// Work item = one CTA = a contiguous range of the internal point order inside
// one spatial tile, split into runs of equal first tap u0 (same footprint).
// Points stream through shared memory in chunks of QS points with a
// two-stage cp.async pipeline (chunk k+1 in flight while chunk k is
// contracted); chunks ignore run boundaries.
//
// Each thread owns a block of the (2m)^d footprint: one a (d = 3), Rc
// consecutive c rows and Re consecutive e values.  Per staged point it reads
// 1 + Rc/2 + Re/2 broadcast 16-byte words from shared memory for Rc*Re fp64
// FMAs (e.g. 7 loads : 32 FMAs at 2m = 16), which keeps the fp64 pipe, not
// the shared-memory crossbar, the limiter.
//   spread : acc[c][e] += ((x wa[a]) wc[c]) we[e] over the run's points in
//            registers; flushed to the item box in shared memory when the run
//            ends (one barrier between runs orders the box updates).
//   interp : g[c][e] of the run stay in registers across chunks; per batch of
//            16 points each thread forms wa[a] sum_c wc[c] sum_e we[e] g[c][e],
//            a 16-wide warp butterfly + shared-memory sum over warps reduces,
//            and the graph-operator epilogue runs in place.
#pragma once

#include "kernels.cuh"

namespace fgsb {

__device__ __forceinline__ int64_t lmin(int64_t x, int64_t y) { return x < y ? x : y; }

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_1() { asm volatile("cp.async.wait_group 1;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_0() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

// Footprint blocking per (d, 2m): rows of Rc c-values x Re e-values per thread.
template <int D, int T>
struct Blk {
  static constexpr int Rc = D == 1 ? 1
                            : D == 2 ? 1
                            : (T == 16 ? 4 : T == 12 ? 3 : T == 14 ? 2 : T == 10 ? 2 : T == 8 ? 2 : T == 6 ? 2 : 1);
  static constexpr int Re = D == 1 ? (T >= 2 ? 2 : 1)
                            : D == 2 ? (T >= 2 ? 2 : 1)
                            : (T == 16 ? 8 : T == 12 ? 6 : T == 14 ? 14 : T == 10 ? 5 : T == 8 ? 4 : T == 6 ? 3
                               : T == 4 ? 2 : 1);
  static constexpr int CG = D >= 2 ? T / Rc : 1;  // c groups
  static constexpr int EG = T / Re;               // e groups
  static constexpr int U = (D == 3 ? T : 1) * CG * EG;
  static constexpr int NT = ((U + 31) / 32) * 32;
  static constexpr int QS = 32;  // points per staged chunk
  static constexpr int QB = 16;  // points per interpolation reduction batch
  static constexpr int TAPS = D * T;
  static_assert(T % Rc == 0 && T % Re == 0, "blocking must tile the footprint");
};

struct V2Geom {  // unit of this thread
  int a, c0, e0;
  bool active;
};

template <int D, int T>
__device__ __forceinline__ V2Geom v2_unit(int tid) {
  using B = Blk<D, T>;
  V2Geom g;
  g.active = tid < B::U;
  const int u = g.active ? tid : 0;
  g.e0 = (u % B::EG) * B::Re;
  g.c0 = ((u / B::EG) % B::CG) * B::Rc;
  g.a = D == 3 ? u / (B::EG * B::CG) : 0;
  return g;
}

// issue the cp.async copies of chunk [p, p+q) (taps) into stage buffer `buf`
template <int TAPS>
__device__ __forceinline__ void v2_issue_chunk(double* buf, const double* taps, int64_t p, int q, int tid, int nt) {
  const double* src = taps + p * TAPS;
  const int n16 = q * TAPS / 2;
  for (int k = tid; k < n16; k += nt) cp_async16(buf + 2 * k, src + 2 * k);
}

// x value (optionally scaled by s) of internal point ip
__device__ __forceinline__ double v2_x(const PassArgs& a, const double* xv, int64_t ip) {
  const int64_t ix = a.perm ? static_cast<int64_t>(a.perm[ip]) : ip;
  double v = xv[ix];
  if (a.scale_input) v = __dmul_rn(a.s[ip], v);
  return v;
}

// ---------------------------------------------------------------------------
// spread (v2).  Shared memory: box | stage[2][QS*TAPS] | xs[2][QS]
// ---------------------------------------------------------------------------
template <int D, int T>
__global__ void __launch_bounds__(Blk<D, T>::NT) spread_v2_kernel(PassArgs a, int box_stride_smem) {
  using B = Blk<D, T>;
  constexpr int NT = B::NT, QS = B::QS, TAPS = B::TAPS, Rc = B::Rc, Re = B::Re;
  extern __shared__ __align__(16) double smem[];
  double* S = smem;
  double* stg = smem + box_stride_smem;
  double* xs = stg + 2 * QS * TAPS;
  const int tid = threadIdx.x;
  const DItem it = a.items[blockIdx.x];
  const int bx1 = it.e1, bx2 = it.e2;
  const int V = it.e0 * it.e1 * it.e2;
  const V2Geom ug = v2_unit<D, T>(tid);
  const int64_t p_begin = it.p_begin, p_end = it.p_end;
  const int nch = static_cast<int>((p_end - p_begin + QS - 1) / QS);

  for (int vec = 0; vec < a.nvec; ++vec) {
    const double* xv = a.x + vec * a.ldx;
    for (int v = tid; v < V; v += NT) S[v] = 0.0;
    // prologue: chunk 0 in flight, its x values staged directly
    v2_issue_chunk<TAPS>(stg, a.taps, p_begin, static_cast<int>(lmin(QS, p_end - p_begin)), tid, NT);
    cp_async_commit();
    if (tid < QS && p_begin + tid < p_end) xs[tid] = v2_x(a, xv, p_begin + tid);

    int r = it.run_begin;
    DRun run = a.runs[r];
    double acc[Rc][Re];
#pragma unroll
    for (int c = 0; c < Rc; ++c)
#pragma unroll
      for (int e = 0; e < Re; ++e) acc[c][e] = 0.0;

    for (int k = 0; k < nch; ++k) {
      const int64_t c0 = p_begin + static_cast<int64_t>(k) * QS;
      const int64_t c1 = lmin(c0 + QS, p_end);
      const int buf = k & 1;
      cp_async_wait_0();
      __syncthreads();  // chunk k (taps + xs) visible; chunk k-1 fully consumed
      const bool more = k + 1 < nch;
      double xnext = 0.0;
      int qn = 0;
      if (more) {  // prefetch chunk k+1 into the buffer chunk k-1 used
        qn = static_cast<int>(lmin(QS, p_end - c1));
        v2_issue_chunk<TAPS>(stg + (buf ^ 1) * QS * TAPS, a.taps, c1, qn, tid, NT);
        cp_async_commit();
        if (tid < qn) xnext = v2_x(a, xv, c1 + tid);
      }
      const double* sb = stg + buf * QS * TAPS;
      const double* xb = xs + buf * QS;
      while (true) {
        const int64_t rs = run.pstart, re_ = static_cast<int64_t>(run.pstart) + run.pcount;
        const int s0 = static_cast<int>(max(rs, c0) - c0), s1 = static_cast<int>(min(re_, c1) - c0);
        if (ug.active && s0 < s1) {
          // operands of one point: u = x wa (d = 3) or x, the Rc wc and Re we taps
          auto fetch = [&](int i, double& u, double* uc, double* ue) {
            const double* w = sb + i * TAPS;
            u = xb[i];
            if (D == 3) u = u * w[ug.a];  // x wa (nfft.cpp:308)
            const double* wc = D == 3 ? w + T : w;
            const double* we = w + (D - 1) * T;
#pragma unroll
            for (int c = 0; c < Rc; ++c) uc[c] = D >= 2 ? wc[ug.c0 + c] : 1.0;
#pragma unroll
            for (int e = 0; e < Re; ++e) ue[e] = we[ug.e0 + e];
          };
          double u, uc[Rc], ue[Re];
          fetch(s0, u, uc, ue);
          for (int i = s0; i < s1; ++i) {
            double nu, nuc[Rc], nue[Re];
            if (i + 1 < s1) fetch(i + 1, nu, nuc, nue);  // next point's loads in flight
#pragma unroll
            for (int c = 0; c < Rc; ++c) {
              const double v = D >= 2 ? u * uc[c] : u;  // (x wa) wc
#pragma unroll
              for (int e = 0; e < Re; ++e) acc[c][e] = fma(v, ue[e], acc[c][e]);
            }
            if (i + 1 < s1) {
              u = nu;
#pragma unroll
              for (int c = 0; c < Rc; ++c) uc[c] = nuc[c];
#pragma unroll
              for (int e = 0; e < Re; ++e) ue[e] = nue[e];
            }
          }
        }
        if (re_ <= c1) {  // run ends inside this chunk: flush its block into the box
          if (ug.active) {
            const int o0 = run.off & 1023, o1 = (run.off >> 10) & 1023, o2 = (run.off >> 20) & 1023;
#pragma unroll
            for (int c = 0; c < Rc; ++c) {
              double* row = S + ((o0 + ug.a) * bx1 + (o1 + ug.c0 + c)) * bx2 + o2 + ug.e0;
#pragma unroll
              for (int e = 0; e < Re; ++e) {
                row[e] += acc[c][e];
                acc[c][e] = 0.0;
              }
            }
          }
          if (++r >= it.run_end) break;
          run = a.runs[r];
          __syncthreads();  // order this run's box update before the next run's
          continue;
        }
        break;
      }
      if (more && tid < qn) xs[(buf ^ 1) * QS + tid] = xnext;  // xs[buf^1] last read in chunk k-1
    }
    __syncthreads();
    double* out = a.priv + (static_cast<int64_t>(vec) * gridDim.x + blockIdx.x) * a.box_stride;
    for (int v = tid; v < V; v += NT) out[v] = S[v];
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// interpolation (v2).  Shared memory: box | stage[2][QS*TAPS] | xs[2][QS] |
// red[2][NW][16]
// ---------------------------------------------------------------------------
template <int D, int T>
__global__ void __launch_bounds__(Blk<D, T>::NT) interp_v2_kernel(PassArgs a, int box_stride_smem) {
  using B = Blk<D, T>;
  constexpr int NT = B::NT, QS = B::QS, QB = B::QB, TAPS = B::TAPS, Rc = B::Rc, Re = B::Re;
  constexpr int NW = NT / 32;
  extern __shared__ __align__(16) double smem[];
  double* S = smem;
  double* stg = smem + box_stride_smem;
  double* red = stg + 2 * QS * TAPS + 2 * QS;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const DItem it = a.items[blockIdx.x];
  const int bx1 = it.e1, bx2 = it.e2;
  const int V = it.e0 * it.e1 * it.e2;
  const int Md0 = D == 3 ? a.M : 1, Md1 = D >= 2 ? a.M : 1, Md2 = a.M;
  const V2Geom ug = v2_unit<D, T>(tid);
  const int64_t p_begin = it.p_begin, p_end = it.p_end;
  const int nch = static_cast<int>((p_end - p_begin + QS - 1) / QS);
  int rb = 0;  // red double buffer

  for (int vec = 0; vec < a.nvec; ++vec) {
    const double* gv = a.grid + vec * a.grid_stride;
    const double* xv = a.x ? a.x + vec * a.ldx : nullptr;
    double* yv = a.y ? a.y + vec * a.ldy : nullptr;
    v2_issue_chunk<TAPS>(stg, a.taps, p_begin, static_cast<int>(lmin(QS, p_end - p_begin)), tid, NT);
    cp_async_commit();
    for (int v = tid; v < V; v += NT) {
      const int x2 = v % bx2, x1 = (v / bx2) % bx1, x0 = v / (bx2 * bx1);
      const int g0 = (it.a0 + x0) % Md0, g1 = (it.a1 + x1) % Md1, g2 = (it.a2 + x2) % Md2;
      S[v] = gv[(static_cast<int64_t>(g0) * Md1 + g1) * Md2 + g2];
    }
    __syncthreads();  // box complete

    int r = it.run_begin;
    DRun run = a.runs[r];
    double g[Rc][Re];
    auto load_g = [&]() {
      if (!ug.active) return;
      const int o0 = run.off & 1023, o1 = (run.off >> 10) & 1023, o2 = (run.off >> 20) & 1023;
#pragma unroll
      for (int c = 0; c < Rc; ++c) {
        const double* row = S + ((o0 + ug.a) * bx1 + (o1 + ug.c0 + c)) * bx2 + o2 + ug.e0;
#pragma unroll
        for (int e = 0; e < Re; ++e) g[c][e] = row[e];
      }
    };
    load_g();

    for (int k = 0; k < nch; ++k) {
      const int64_t c0 = p_begin + static_cast<int64_t>(k) * QS;
      const int64_t c1 = lmin(c0 + QS, p_end);
      const int buf = k & 1;
      if (k + 1 < nch) {
        const int qn = static_cast<int>(lmin(QS, p_end - c1));
        v2_issue_chunk<TAPS>(stg + (buf ^ 1) * QS * TAPS, a.taps, c1, qn, tid, NT);
        cp_async_commit();
        cp_async_wait_1();
      } else {
        cp_async_wait_0();
      }
      __syncthreads();
      const double* sb = stg + buf * QS * TAPS;
      for (int64_t b0 = c0; b0 < c1; b0 += QB) {
        const int qb = static_cast<int>(lmin(QB, c1 - b0));
        // prefetch this thread's epilogue operands (their latency hides under the batch)
        int64_t eix = 0;
        double exin = 0.0, esin = 1.0;
        if (tid < qb) {
          const int64_t ip = b0 + tid;
          eix = a.perm ? static_cast<int64_t>(a.perm[ip]) : ip;
          if (xv && a.epilogue != EPI_KERNEL && a.epilogue != EPI_DEGREE) exin = xv[eix];
          if (a.epilogue == EPI_NORMALIZED || a.epilogue == EPI_LAPLACIAN) esin = a.s[ip];
        }
        double p[QB];
#pragma unroll
        for (int i = 0; i < QB; ++i) p[i] = 0.0;
        while (true) {
          const int64_t rs = run.pstart, re_ = static_cast<int64_t>(run.pstart) + run.pcount;
          const int64_t s0 = max(rs, b0), s1 = min(re_, b0 + qb);
          if (ug.active && s0 < s1) {
#pragma unroll
            for (int i = 0; i < QB; ++i) {
              const int64_t ip = b0 + i;
              if (ip >= s0 && ip < s1) {
                const double* w = sb + (ip - c0) * TAPS;
                const double* wc = D == 3 ? w + T : w;
                const double* we = w + (D - 1) * T;
                double acc = 0.0;
#pragma unroll
                for (int c = 0; c < Rc; ++c) {
                  double rsum = 0.0;
#pragma unroll
                  for (int e = 0; e < Re; ++e) rsum = fma(we[ug.e0 + e], g[c][e], rsum);
                  acc = D >= 2 ? fma(wc[ug.c0 + c], rsum, acc) : acc + rsum;
                }
                p[i] = D == 3 ? fma(w[ug.a], acc, p[i]) : p[i] + acc;
              }
            }
          }
          if (re_ <= b0 + qb && r + 1 < it.run_end) {
            ++r;
            run = a.runs[r];
            load_g();
            continue;
          }
          break;
        }
        // 16-wide butterfly: lane l (and l ^ 16) ends with the warp sum of point l & 15
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
        double* rbuf = red + rb * NW * QB;
        if (lane < QB) rbuf[warp * QB + lane] = p[0];
        __syncthreads();
        if (tid < qb) {
          double val = 0.0;
#pragma unroll
          for (int w = 0; w < NW; ++w) val += rbuf[w * QB + tid];
          const int64_t ip = b0 + tid;
          if (a.epilogue == EPI_DEGREE) {
            const double dg = val - a.k0;  // graphop.cpp:55-56
            a.degrees[ip] = dg;
            a.inv_sqrt[ip] = 1.0 / sqrt(dg);
            if (!(dg > 0.0)) atomicMin(a.bad_flag, static_cast<unsigned long long>(a.caller[ip]));
          } else {
            double out;
            switch (a.epilogue) {
              case EPI_KERNEL: out = val; break;
              case EPI_WEIGHT: out = val - a.k0 * exin; break;
              case EPI_NORMALIZED: out = esin * (val - a.k0 * __dmul_rn(esin, exin)); break;
              default: out = exin - esin * (val - a.k0 * __dmul_rn(esin, exin)); break;
            }
            yv[eix] = out;
          }
        }
        rb ^= 1;  // the next batch writes the other red buffer: no second barrier
      }
      __syncthreads();  // buffer `buf` fully consumed before chunk k+2 overwrites it
    }
    __syncthreads();
  }
}

}  // namespace fgsb
