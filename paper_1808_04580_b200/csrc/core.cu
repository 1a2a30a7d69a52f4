// core.cu -- plan construction and apply orchestration of the B200 fast
// summation (reference: nfft.cpp:328-438, kernels.cpp:266-335,
// fastsum.cpp:69-118, graphop.cpp:36-103).
#include <cub/cub.cuh>

#include <algorithm>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>
#include <cstring>
#include <numeric>
#include <thread>

#include "core.cuh"
#include "kernels.cuh"
#include "kernels_v2.cuh"
#include "kernels_v4.cuh"
#include "kernels_v6.cuh"
#include "kernels_v8.cuh"
#include "conv2d.cuh"
#include "conv3d.cuh"
#include "direct.cuh"
#include "nccl_shim.hpp"

namespace fgsb {

void validate_params(const Params& p) {  // fastsum.cpp:25-36
  if (p.N < 2 || p.N % 2 != 0) fail(FGS_EPARAM, "bandwidth must be even and >= 2");
  if (p.m < 1 || p.m > 32) fail(FGS_EPARAM, "cutoff must lie in [1, 32]");
  if (p.p < 1 || p.p > 8) fail(FGS_EPARAM, "smoothness order must lie in [1, 8]");
  if (!(p.eps_b >= 0.0) || !(p.eps_b < 0.5)) fail(FGS_EPARAM, "blend width must lie in [0, 1/2)");
  if (!(p.oversampling >= 1.0)) fail(FGS_EPARAM, "oversampling factor must be >= 1");
}

namespace {

inline int ceil_div(int64_t a, int64_t b) { return static_cast<int>((a + b - 1) / b); }

// ---- small device kernels of the complex NfftPlan path -------------------
__global__ void merge_complex_kernel(const double* re, const double* im, cufftDoubleComplex* out, int64_t n) {
  int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i < n) out[i] = make_cuDoubleComplex(re[i], im[i]);
}
__global__ void split_complex_kernel(const cufftDoubleComplex* in, double* re, double* im, int64_t n) {
  int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i < n) {
    re[i] = in[i].x;
    im[i] = in[i].y;
  }
}

// grid offset of frequency multi-index f in FrequencyIndexSet order
__device__ __forceinline__ int64_t freq_to_grid(int64_t f, int D, int N, int M, double* dec,
                                                const double* deconv) {
  int64_t g = 0, stride = 1;
  double prod = 1.0;
  double fac[3];
  int64_t rest = f;
  for (int t = D - 1; t >= 0; --t) {
    int a = static_cast<int>(rest % N);
    rest /= N;
    int l = a - N / 2;
    int k = (l + M) % M;
    g += k * stride;
    stride *= M;
    fac[t] = deconv[a];
  }
  // (deconv[a] * deconv[c]) * deconv[e] as nfft.cpp:200-201
  prod = fac[0];
  for (int t = 1; t < D; ++t) prod = prod * fac[t];
  *dec = prod;
  return g;
}

// place_coefficients (nfft.cpp:174-213) into a zeroed complex grid
__global__ void place_kernel(const cufftDoubleComplex* fhat, cufftDoubleComplex* grid, int64_t F, int D, int N,
                             int M, const double* deconv) {
  int64_t f = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (f >= F) return;
  double dec;
  int64_t g = freq_to_grid(f, D, N, M, &dec, deconv);
  cufftDoubleComplex v = fhat[f];
  grid[g] = make_cuDoubleComplex(v.x * dec, v.y * dec);
}

// extract_coefficients (nfft.cpp:216-250)
__global__ void extract_kernel(const cufftDoubleComplex* grid, cufftDoubleComplex* fhat, int64_t F, int D, int N,
                               int M, const double* deconv) {
  int64_t f = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (f >= F) return;
  double dec;
  int64_t g = freq_to_grid(f, D, N, M, &dec, deconv);
  cufftDoubleComplex v = grid[g];
  fhat[f] = make_cuDoubleComplex(v.x * dec, v.y * dec);
}

// ---- sharded spectrum exchange: window <-> half spectrum ------------------
struct WindowArgs {
  cufftDoubleComplex* spec;
  cufftDoubleComplex* window;
  const cufftDoubleComplex* mult;
  int64_t spec_stride, window_stride, total;
  int nvec, D, M, N;
};

__device__ __forceinline__ bool window_to_spec(int64_t w, int D, int M, int N, int64_t* sidx) {
  const int hN = N / 2, W = N + 1, H = M / 2 + 1;
  int l2 = static_cast<int>(w % (hN + 1));
  int64_t rest = w / (hN + 1);
  int l1 = 0, l0 = 0;
  if (D >= 2) {
    l1 = static_cast<int>(rest % W) - hN;
    rest /= W;
  }
  if (D == 3) l0 = static_cast<int>(rest) - hN;
  if (l2 > M / 2) return false;
  if (M == N && ((D >= 2 && l1 == hN) || (D == 3 && l0 == hN))) return false;  // aliases -N/2
  int64_t s = l2;
  if (D >= 2) s += static_cast<int64_t>((l1 + M) % M) * H;
  if (D == 3) s += static_cast<int64_t>((l0 + M) % M) * H * M;
  *sidx = s;
  return true;
}

__global__ void pack_window_kernel(WindowArgs a) {
  int64_t w = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (w >= a.total) return;
  int64_t s;
  bool ok = window_to_spec(w, a.D, a.M, a.N, &s);
  for (int v = 0; v < a.nvec; ++v)
    a.window[v * a.window_stride + w] = ok ? a.spec[v * a.spec_stride + s] : make_cuDoubleComplex(0.0, 0.0);
}

__global__ void unpack_multiply_kernel(WindowArgs a) {
  int64_t w = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (w >= a.total) return;
  int64_t s;
  if (!window_to_spec(w, a.D, a.M, a.N, &s)) return;
  cufftDoubleComplex m = a.mult[w];
  for (int v = 0; v < a.nvec; ++v) {
    cufftDoubleComplex z = a.window[v * a.window_stride + w];
    a.spec[v * a.spec_stride + s] = make_cuDoubleComplex(z.x * m.x - z.y * m.y, z.x * m.y + z.y * m.x);
  }
}

__global__ void fill_kernel(double* x, int64_t n, double v) {
  int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i < n) x[i] = v;
}

__global__ void permute_kernel(const double* x, int64_t ldx, double* y, int64_t ldy, const int* perm, int64_t n,
                               int nvec, int direction) {
  int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  const int64_t c = perm[i];
  for (int v = 0; v < nvec; ++v) {
    if (direction == 0)
      y[v * ldy + i] = x[v * ldx + c];  // caller -> internal
    else
      y[v * ldy + c] = x[v * ldx + i];  // internal -> caller
  }
}

// ---- launch policy ----------------------------------------------------------
// d = 3, 2m in {8, 12, 16}: fp64 tensor-core (DMMA) kernels (kernels_v4.cuh);
// the spread needs dense runs (>= kDenseRun points per cell), sparser plans
// use the register-blocked cp.async kernel (kernels_v2.cuh).  d = 2, 2m in
// {8, 12, 16}: the d = 2 DMMA kernels, same rule.  Other 2m <= 16: v2
// kernels; 2m > 16: runtime-2m single-value kernels (kernels.cuh).
// cudaFuncSetAttribute is a driver call; raise each kernel's dynamic shared
// memory limit once, not on every launch (ncu/launch-overhead hygiene)
void set_smem(const void* func, size_t smem) {
  static std::mutex mu;
  static std::map<const void*, size_t> done;
  std::lock_guard<std::mutex> lock(mu);
  auto it = done.find(func);
  if (it != done.end() && it->second >= smem) return;
  FGS_CUDA(cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  done[func] = smem;
}

// the tensor-core spread needs runs of >= this many points (K-steps of 4,
// one block flush per run); sparser plans use the scalar register-blocked one
// d = 3, 2m = 16: 4 -- the slot-layout tensor kernels beat the scalar spread from
// ~4 points per run (config 5 at 1.25M points, ~9 per run: 471 -> 700
// matvecs/s); other 2m keep 12.  FGS_DENSE_RUN overrides (tuning).
double dense_run_threshold(int T, int d) {
  static const double forced = [] {
    const char* e = std::getenv("FGS_DENSE_RUN");
    return e ? std::atof(e) : -1.0;
  }();
  if (forced >= 0.0) return forced;
  return T == 16 && d == 3 ? 4.0 : 12.0;
}
#define kDenseRun (dense_run_threshold(T, d))

template <int D, int T>
constexpr bool has_v4_3d() {
  return D == 3 && (T == 8 || T == 12 || T == 16);
}
template <int D, int T>
constexpr bool has_v4_2d() {
  return D == 2 && (T == 8 || T == 12 || T == 16);
}

// d = 2 tensor-core kernels: point-stream warps per CTA (interpolation 2:
// C2 22.8 k vs 22.2 k with 4, 21.7 k with 1; spread 1)
constexpr int kInterp2dP = 2;
// d = 3 interpolation over the point order (plans without the slot layout):
// per-warp point batches with B fragments from the box (kernels_v5.cuh)
// d = 3 spread, 2m in {12, 16}: warps own box rows x0 = w (mod W), no
// barrier per run (kernels_v5.cuh); FGS_SPREAD_V5=0 builds the v4 kernel
#ifndef FGS_SPREAD_V5
#define FGS_SPREAD_V5 1
#endif
#ifndef FGS_V5S_W16
#define FGS_V5S_W16 8
#endif
template <int T>
constexpr bool use_spread_v5() {  // 2m = 12 (C4) measured slower: 449 vs 391 us
  return FGS_SPREAD_V5 != 0 && T == 16;
}
template <int T>
constexpr int v5s_w() {
  return T == 16 ? FGS_V5S_W16 : T / 2;
}
constexpr int kSpread2dP = 1;
constexpr int kVSplitDefault = 16;  // one vector per CTA: C5 taps traffic 68.7 -> ~8 GB per block (L2 hits), 98.8 -> 97.9 ms
// d = 3, 2m = 16 dense plans: run-aligned slot layout + kernels_v6.cuh
// (FGS_V6=0: the v5 kernels over the plain point order)
// slot-layout interpolation with two batches per B-fragment load
// (interp_v7_kernel); FGS_INTERP_V7=0 selects interp_v6_kernel
bool interp_v7_on() {
  static const bool on = [] {
    const char* e = std::getenv("FGS_INTERP_V7");
    return !(e && std::string(e) == "0");
  }();
  return on;
}
bool spread_v8_on() {
  static const bool on = [] {
    const char* e = std::getenv("FGS_SPREAD_V8");
    return !(e && std::string(e) == "0");
  }();
  return on;
}
// slot-layout kernels: CTAs per item of a vector block (vsplit_narrow,
// common.cuh); FGS_VSPLIT overrides (tuning)
int vsplit_for(int nvec) {
  static const int forced = [] {
    const char* e = std::getenv("FGS_VSPLIT");
    return e ? std::atoi(e) : 0;
  }();
  const int vs = forced > 0 ? forced : kVSplitDefault;
  return std::max(1, std::min(vs, nvec));
}
bool v6_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("FGS_V6");
    return !(e && std::string(e) == "0");
  }();
  return on;
}
// staged input window (Blk4d2::XW) of the d = 2 variant with P streams
constexpr size_t xw2d(int p) { return static_cast<size_t>(p * 32 > 64 ? p * 32 : 64); }

template <int T, bool INTERP>
constexpr size_t v4_stage_doubles() {
  using B = Blk4<T, INTERP>;
  return INTERP ? 2 * static_cast<size_t>(B::QS) * B::STRIDE + 2 * static_cast<size_t>(B::QS) * (B::G + 3)
                : 2 * static_cast<size_t>(B::QS) * B::STRIDE + 2 * B::QS;
}

// private spread boxes of the d = 3 DMMA spread (P when P >= 4, else one shared box)
int v4_spread_groups(int T) {
  if (T == 16 && FGS_SPREAD_V5) return 1;  // spread_v5: one box
  switch (T) {
    case 8: return Blk4<8, false>::P >= 4 ? Blk4<8, false>::P : 1;
    case 12: return Blk4<12, false>::P >= 4 ? Blk4<12, false>::P : 1;
    case 16: return Blk4<16, false>::P >= 4 ? Blk4<16, false>::P : 1;
    default: return 1;
  }
}

// shared-memory doubles beyond the box, and threads, of the kernel that
// dispatch() will launch for (D, T)
struct LaunchShape {
  int nt;
  size_t extra_spread, extra_interp;
};

template <int D, int T>
LaunchShape shape_t(bool dense) {
  using B = Blk<D, T>;
  const size_t base = 2 * static_cast<size_t>(B::QS) * B::TAPS + 2 * B::QS;
  size_t interp = base + 2 * static_cast<size_t>(B::NT / 32) * B::QB;
  size_t spread = base;
  if constexpr (has_v4_3d<D, T>()) {
    interp = v5_extra_doubles<T>();
    if (dense) {
      if constexpr (use_spread_v5<T>())
        spread = v5s_extra_doubles<T, v5s_w<T>()>();
      else
        spread = v4_stage_doubles<T, false>();
    }
  }
  if constexpr (has_v4_2d<D, T>()) {
    using B4 = Blk4d2<T>;
    // taps double buffer + staged inputs (interp: x and caller index)
    interp = 2 * static_cast<size_t>(B4::QS) * B4::STRIDE + 2 * xw2d(kInterp2dP);
    if (dense) spread = 2 * static_cast<size_t>(B4::QS) * B4::STRIDE + xw2d(kSpread2dP);
  }
  return {B::NT, spread, interp};
}

template <int D>
LaunchShape shape_of(int T, bool dense) {
  switch (T) {
    case 2: return shape_t<D, 2>(dense);
    case 4: return shape_t<D, 4>(dense);
    case 6: return shape_t<D, 6>(dense);
    case 8: return shape_t<D, 8>(dense);
    case 10: return shape_t<D, 10>(dense);
    case 12: return shape_t<D, 12>(dense);
    case 14: return shape_t<D, 14>(dense);
    case 16: return shape_t<D, 16>(dense);
    default: break;
  }
  const size_t base = static_cast<size_t>(kQ) * D * T + kQ;
  return {256, base, base + 256};
}

template <class K, class... Args>
void launch_smem(K k, int nitems, int nt, size_t smem, cudaStream_t s, Args... args) {
  set_smem(reinterpret_cast<const void*>(k), smem);
  launch_ex(k, nitems, nt, smem, s, args...);
}

template <int D, int T>
void launch_t(bool interp, bool dense, const PassArgs& a, int nitems, size_t smem, int box_stride, int box_pad_arg,
              cudaStream_t s) {
  if constexpr (has_v4_2d<D, T>()) {
    if (interp)
      return launch_smem(interp_v4_2d_kernel<T, kInterp2dP>, nitems, Blk4d2<T, kInterp2dP>::NT, smem, s, a, box_stride);
    if (dense)
      return launch_smem(spread_v4_2d_kernel<T, kSpread2dP>, nitems, Blk4d2<T, kSpread2dP>::NT, smem, s, a, box_stride);
  }
  if constexpr (D == 3 && (T == 16 || T == 12)) {
    if (a.slots != nullptr) {  // run-aligned slot layout: v6 interpolation; 2m = 16 v6 spread
      if (interp) {
        // two batches per B load: 2m = 16 (C5 interp 48.8 -> 47.8 ms); 2m = 12
        // does not gain (C4 314 -> 332 us with per-item strides, 313 = 313 us
        // with the fixed ones: fewer K-steps per B fragment)
        // (from 16 points per run: sparser plans rarely pair two batches of
        // one run, and v6 is 2 % faster there -- config 5 at 1.25M points)
        // fixed box strides for the plan's tile size (B = 2: 2m + 1, B = 4: 2m + 3)
        if constexpr (T == 16)
          if (interp_v7_on() && a.pair_batches) {
            if (a.box_ext == T + 1)
              return launch_smem(interp_v7_kernel<T, T + 1>, nitems, Blk5<T>::NT, smem, s, a, box_pad_arg);
            if (a.box_ext == T + 3)
              return launch_smem(interp_v7_kernel<T, T + 3>, nitems, Blk5<T>::NT, smem, s, a, box_pad_arg);
            return launch_smem(interp_v7_kernel<T, 0>, nitems, Blk5<T>::NT, smem, s, a, box_pad_arg);
          }
        if (a.box_ext == T + 1)
          return launch_smem(interp_v6_kernel<T, T + 1>, nitems, Blk5<T>::NT, smem, s, a, box_pad_arg);
        if (a.box_ext == T + 3)
          return launch_smem(interp_v6_kernel<T, T + 3>, nitems, Blk5<T>::NT, smem, s, a, box_pad_arg);
        return launch_smem(interp_v6_kernel<T, 0>, nitems, Blk5<T>::NT, smem, s, a, box_pad_arg);
      }
      if constexpr (T == 16) return launch_smem(spread_v6_kernel, nitems, Blk6s::NT, smem, s, a, box_stride);
      // 2m = 12: e split 8 (DMMA) + 4 (DFMA), warps own box c-rows (kernels_v8.cuh);
      // FGS_SPREAD_V8=0: the v4 spread below reads the slot rows (stride 3 2m) and the slot-ordered x
      if (spread_v8_on()) return launch_smem(spread_v8_kernel<Blk8::H>, nitems, Blk8::NT, smem, s, a, box_stride);
    }
  }
  if constexpr (has_v4_3d<D, T>()) {
    if (interp) return launch_smem(interp_v5_kernel<T>, nitems, Blk5<T>::NT, smem, s, a, box_pad_arg);
    if (dense) {
      if constexpr (use_spread_v5<T>()) {
        constexpr int W = v5s_w<T>();
        return launch_smem(spread_v5_kernel<T, W>, nitems, Blk5s<T, W>::NT, smem, s, a, box_stride);
      } else {
        return launch_smem(spread_v4_kernel<T, 0, 0>, nitems, Blk4<T, false>::NT, smem, s, a, box_stride);
      }
    }
  }
  constexpr int NT = Blk<D, T>::NT;
  if (interp)
    launch_smem(interp_v2_kernel<D, T>, nitems, NT, smem, s, a, box_stride);
  else
    launch_smem(spread_v2_kernel<D, T>, nitems, NT, smem, s, a, box_stride);
}

template <int D>
void dispatch(bool interp, bool dense, int T, const PassArgs& a, int nitems, size_t smem, int box_stride, int box_pad,
              cudaStream_t s) {
  switch (T) {
    case 2: return launch_t<D, 2>(interp, dense, a, nitems, smem, box_stride, box_pad, s);
    case 4: return launch_t<D, 4>(interp, dense, a, nitems, smem, box_stride, box_pad, s);
    case 6: return launch_t<D, 6>(interp, dense, a, nitems, smem, box_stride, box_pad, s);
    case 8: return launch_t<D, 8>(interp, dense, a, nitems, smem, box_stride, box_pad, s);
    case 10: return launch_t<D, 10>(interp, dense, a, nitems, smem, box_stride, box_pad, s);
    case 12: return launch_t<D, 12>(interp, dense, a, nitems, smem, box_stride, box_pad, s);
    case 14: return launch_t<D, 14>(interp, dense, a, nitems, smem, box_stride, box_pad, s);
    case 16: return launch_t<D, 16>(interp, dense, a, nitems, smem, box_stride, box_pad, s);
    default: break;
  }
  // runtime-2m kernels (m > 8): one value per unit, 256 threads
  if (interp) {
    auto k = interp_kernel<D, 0, 1, 256>;
    set_smem(reinterpret_cast<const void*>(k), smem);
    k<<<nitems, 256, smem, s>>>(a, T, box_stride);
  } else {
    auto k = spread_kernel<D, 0, 1, 256>;
    set_smem(reinterpret_cast<const void*>(k), smem);
    k<<<nitems, 256, smem, s>>>(a, T, box_stride);
  }
}

}  // namespace

// ===========================================================================
Core::Core(const double* nodes_colmajor, int64_t n_, int d_, Kind kind_, const KernelSpec& kernel_,
           const Params& params_, int device_, int rank_, int world_, const void* nccl_id)
    : kind(kind_), d(d_), n(n_), rank(rank_), world(world_), kernel(kernel_), params(params_), device(device_) {
  if (kind == FASTSUM) {
    validate_params(params);
    if (n == 0) fail(FGS_ESHAPE, "node set is empty");
    if (d < 1 || d > 3) fail(FGS_ESHAPE, "nodes must have 1, 2, or 3 columns");
    check_spec(kernel);
  } else if (kind == DIRECT) {
    if (n == 0) fail(FGS_ESHAPE, "node set is empty");
    if (d < 1 || d > 3) fail(FGS_EPARAM, "node dimension must be 1, 2, or 3");
    check_spec(kernel);
  } else {
    if (d < 1 || d > 3) fail(FGS_EPARAM, "dims must be 1, 2, or 3, got " + std::to_string(d));
    if (params.N < 2 || params.N % 2 != 0)
      fail(FGS_EPARAM, "bandwidth must be even and >= 2, got " + std::to_string(params.N));
    if (n == 0) fail(FGS_ESHAPE, "node set is empty");
    if (params.m < 1 || params.m > 32)
      fail(FGS_EPARAM, "cutoff must lie in [1, 32], got " + std::to_string(params.m));
    if (!(params.oversampling >= 1.0)) fail(FGS_EPARAM, "oversampling factor must be >= 1");
  }
  if (world < 1 || rank < 0 || rank >= world) fail(FGS_EPARAM, "invalid shard rank/world");
  if (n > INT_MAX) fail(FGS_ERESOURCE, "more than 2^31-1 nodes are not supported");
  N = params.N;
  m = params.m;
  T = 2 * m;
  FGS_CUDA(cudaSetDevice(device));
  FGS_CUDA(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
  if (kind == DIRECT) {  // exact operator: raw nodes, no rescaling (graphop.cpp:29-34, fastsum.cpp:126-139)
    if (world != 1 || nccl_id) fail(FGS_EPARAM, "the direct backend is single-device");
    k0 = kernel_value(kernel, 0.0);
    scaled = kernel;
    n_local = n;
    offset = 0;
    nodes_d.upload(nodes_colmajor, static_cast<size_t>(n) * d, stream);
    host_perm.resize(static_cast<size_t>(n));
    for (int64_t j = 0; j < n; ++j) host_perm[static_cast<size_t>(j)] = static_cast<int>(j);
    perm.upload(host_perm.data(), host_perm.size(), stream);
    FGS_CUDA(cudaStreamSynchronize(stream));
    return;
  }

  if (kind == FASTSUM) {
    // common rescaling into the ball of radius 1/4 - eps_b/2 (fastsum.cpp:79-88)
    const double radius = 0.25 - 0.5 * params.eps_b;
    if (!(radius > 0.0)) fail(FGS_EPARAM, "blend width leaves no node radius");
    double maxnorm = 0.0;
    for (int64_t j = 0; j < n; ++j) {
      double s = 0.0;
      for (int t = 0; t < d; ++t) {
        const double v = nodes_colmajor[t * n + j];
        s += v * v;
      }
      const double nr = std::sqrt(s);
      if (j == 0 || nr > maxnorm) maxnorm = nr;
    }
    rho = (maxnorm > radius) ? radius / maxnorm : 1.0;
    scaled = kernel;
    scaled.shape = kernel.shape * rho;
    out_factor = 1.0;
    if (kernel.family == FGS_MULTIQUADRIC) out_factor = 1.0 / rho;
    if (kernel.family == FGS_INV_MULTIQUADRIC) out_factor = rho;
    k0 = kernel_value(kernel, 0.0);
    reg = RegKernel(scaled, params.eps_b, params.p);
  }

  // NFFT geometry (nfft.cpp:343-354)
  M = 2 * static_cast<int>(std::ceil(params.oversampling * N / 2.0));
  b_kb = kPi * (2.0 - static_cast<double>(N) / M);
  deconv.resize(static_cast<size_t>(N));
  for (int a = 0; a < N; ++a) {
    const double l = a - N / 2;
    const double arg = b_kb * b_kb - std::pow(2.0 * kPi * l / M, 2);
    deconv[static_cast<size_t>(a)] = 1.0 / i0_series(m * std::sqrt(std::max(arg, 0.0)));
  }
  double gsz = 1.0;
  for (int t = 0; t < d; ++t) gsz *= M;
  if (gsz > 2.0e9) fail(FGS_ERESOURCE, "oversampled grid exceeds 2^31 points");
  B = d == 3 ? 4 : (d == 2 ? 8 : 32);
  if (const char* e = std::getenv("FGS_TILE_B")) B = std::max(1, std::atoi(e));  // tuning override
  if (B > M) B = M;
  nt = ceil_div(M, B);
  ntiles = 1;
  for (int t = 0; t < d; ++t) ntiles *= nt;
  grid_elems = 1;
  for (int t = 0; t < d; ++t) grid_elems *= M;
  spec_elems = grid_elems / M * (M / 2 + 1);
  window_elems = (N / 2 + 1);
  for (int t = 0; t + 1 < d; ++t) window_elems *= (N + 1);
  deconv_d.upload(deconv.data(), deconv.size(), stream);

  build_plan(nodes_colmajor);
  if (kind == FASTSUM) build_coefficients();
  if (kind == FASTSUM && (d == 2 || d == 3)) {  // twiddles e^{-2 pi i j / M} for the pruned convolutions
    std::vector<double2> tw(static_cast<size_t>(M));
    for (int j = 0; j < M; ++j) {
      const double ang = 2.0 * kPi * static_cast<double>(j) / M;
      tw[static_cast<size_t>(j)] = make_double2(std::cos(ang), -std::sin(ang));
    }
    tw2.upload(tw.data(), tw.size(), stream);
  }
  if (nccl_id != nullptr) {  // sharded handle (world may be 1: exercises the exchange path)
    sharded = true;
    ncclUniqueId id;
    std::memcpy(&id, nccl_id, sizeof(id));
    nccl_check(nccl().comm_init_rank(&comm, world, id, rank), "ncclCommInitRank");
  }
  FGS_CUDA(cudaStreamSynchronize(stream));
}

Core::~Core() {
  cudaSetDevice(device);
  if (stream) cudaStreamSynchronize(stream);
  for (auto& kv : ws_) {
    if (kv.second->has_plans) {
      cufftDestroy(kv.second->r2c);
      cufftDestroy(kv.second->c2r);
    }
    if (kv.second->has_z2z) cufftDestroy(kv.second->z2z);
  }
  ws_.clear();
  for (auto& g : graphs_) cudaGraphExecDestroy(g.exec);
  graphs_.clear();
  for (auto& evs : ev_pending_)
    for (cudaEvent_t e : evs) cudaEventDestroy(e);
  for (cudaEvent_t e : ev_pool_) cudaEventDestroy(e);
  for (cudaEvent_t e : lz_events) cudaEventDestroy(e);
  for (cudaEvent_t e : pipe_ev) cudaEventDestroy(e);
  if (cp_in) cudaStreamDestroy(cp_in);
  if (cp_out) cudaStreamDestroy(cp_out);
  if (comm) nccl().comm_destroy(comm);
  if (bounce) cudaFreeHost(bounce);
  if (own_stream && stream) cudaStreamDestroy(stream);
}

namespace {
constexpr size_t kBounceChunk = size_t(4) << 20;
constexpr size_t kBounceMin = size_t(16) << 20;  // below: one plain async copy (8 MB: 1.8 vs 2.8 ms)
}  // namespace

void Core::host_copy(bool to_device, void* dst, const void* src, size_t bytes) {
  const void* host = to_device ? src : dst;
  cudaPointerAttributes at{};
  const bool pinned = cudaPointerGetAttributes(&at, host) == cudaSuccess && at.type == cudaMemoryTypeHost;
  cudaGetLastError();
  const int hw = static_cast<int>(std::thread::hardware_concurrency());
  const int T = std::max(1, std::min(8, hw / 2));
  if (bytes < kBounceMin || pinned || T < 2) {
    FGS_CUDA(cudaMemcpyAsync(dst, src, bytes, to_device ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToHost, stream));
    if (!to_device || pinned) FGS_CUDA(cudaStreamSynchronize(stream));
    return;
  }
  if (!bounce || bounce_threads < T) {
    if (bounce) FGS_CUDA(cudaFreeHost(bounce));
    bounce = nullptr;
    FGS_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&bounce), kBounceChunk * T, cudaHostAllocPortable));
    bounce_threads = T;
  }
  cudaEvent_t ready;
  FGS_CUDA(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
  FGS_CUDA(cudaEventRecord(ready, stream));
  std::vector<std::thread> workers;
  std::vector<cudaError_t> errs(static_cast<size_t>(T), cudaSuccess);
  for (int t = 0; t < T; ++t) {
    workers.emplace_back([&, t] {
      cudaError_t e = cudaSetDevice(device);
      cudaStream_t s = nullptr;
      if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
      if (e == cudaSuccess) e = cudaStreamWaitEvent(s, ready, 0);
      char* buf = bounce + kBounceChunk * static_cast<size_t>(t);
      const size_t lo = bytes * static_cast<size_t>(t) / T, hi = bytes * static_cast<size_t>(t + 1) / T;
      for (size_t off = lo; off < hi && e == cudaSuccess; off += kBounceChunk) {
        const size_t len = std::min(kBounceChunk, hi - off);
        if (to_device) {
          std::memcpy(buf, static_cast<const char*>(src) + off, len);
          e = cudaMemcpyAsync(static_cast<char*>(dst) + off, buf, len, cudaMemcpyHostToDevice, s);
          if (e == cudaSuccess) e = cudaStreamSynchronize(s);  // before the bounce is refilled
        } else {
          e = cudaMemcpyAsync(buf, static_cast<const char*>(src) + off, len, cudaMemcpyDeviceToHost, s);
          if (e == cudaSuccess) e = cudaStreamSynchronize(s);
          if (e == cudaSuccess) std::memcpy(static_cast<char*>(dst) + off, buf, len);
        }
      }
      if (s) cudaStreamDestroy(s);
      errs[static_cast<size_t>(t)] = e;
    });
  }
  for (auto& w : workers) w.join();
  cudaEventDestroy(ready);
  for (cudaError_t e : errs) FGS_CUDA(e);
}

void Core::set_stream(cudaStream_t s) {
  FGS_CUDA(cudaStreamSynchronize(stream));
  for (auto& g : graphs_) cudaGraphExecDestroy(g.exec);
  graphs_.clear();
  if (own_stream) cudaStreamDestroy(stream);
  stream = s;
  own_stream = false;
  for (auto& kv : ws_) {
    if (kv.second->has_plans) {
      FGS_CUFFT(cufftSetStream(kv.second->r2c, stream));
      FGS_CUFFT(cufftSetStream(kv.second->c2r, stream));
    }
    if (kv.second->has_z2z) FGS_CUFFT(cufftSetStream(kv.second->z2z, stream));
  }
}

void Core::build_plan(const double* nodes_colmajor) {
  DBuf<double> dnodes;
  dnodes.upload(nodes_colmajor, static_cast<size_t>(n) * d, stream);
  DBuf<unsigned long long> keys, keys_sorted, bad;
  DBuf<int> idx;
  keys.alloc(n);
  keys_sorted.alloc(n);
  idx.alloc(n);
  perm.alloc(n);
  bad.alloc(1);
  unsigned long long init = ULLONG_MAX;
  FGS_CUDA(cudaMemcpyAsync(bad.p, &init, sizeof(init), cudaMemcpyHostToDevice, stream));

  DBuf<char> tmp, tmpb;
  DBuf<unsigned long long> uniq;
  DBuf<int> counts, nruns;
  uniq.alloc(n);
  counts.alloc(n);
  nruns.alloc(1);
  int ncells = 0;
  // keys -> stable radix sort by (tile, cell) -> run-length encode; returns
  // the number of nonempty cells (independent of the tile edge B)
  auto sort_cells = [&]() {
    PointArgs pa{dnodes.p, n, d, M, m, B, nt, rho, kind == FASTSUM ? 1 : 0, keys.p, idx.p, bad.p, 0};
    rot0 = 0;
    if (world > 1) {
      // start the dim-0 tile order after the widest empty gap of the cloud:
      // a cloud centred on 0 wraps around plane 0, and without the rotation
      // the rank whose slice spans the wrap gets two far-apart slabs
      DBuf<int> occ;
      occ.alloc(static_cast<size_t>(nt));
      FGS_CUDA(cudaMemsetAsync(occ.p, 0, sizeof(int) * nt, stream));
      tile0_occupancy_kernel<<<ceil_div(n, 256), 256, 0, stream>>>(pa, occ.p);
      ++launches;
      FGS_CUDA(cudaGetLastError());
      std::vector<int> ho(static_cast<size_t>(nt));
      FGS_CUDA(cudaMemcpyAsync(ho.data(), occ.p, sizeof(int) * nt, cudaMemcpyDeviceToHost, stream));
      FGS_CUDA(cudaStreamSynchronize(stream));
      int best = 0, run = 0;
      for (int t = 0; t < 2 * nt; ++t) {
        if (!ho[static_cast<size_t>(t % nt)]) {
          if (++run > best && run < nt) {
            best = run;
            rot0 = (t + 1) % nt;  // first tile after the gap
          }
        } else {
          run = 0;
        }
      }
      pa.rot0 = rot0;
    }
    point_keys_kernel<<<ceil_div(n, 256), 256, 0, stream>>>(pa);
    ++launches;
    FGS_CUDA(cudaGetLastError());
    unsigned long long badj = 0;
    FGS_CUDA(cudaMemcpyAsync(&badj, bad.p, sizeof(badj), cudaMemcpyDeviceToHost, stream));
    FGS_CUDA(cudaStreamSynchronize(stream));
    if (badj != ULLONG_MAX) {
      // validate_common (nfft.cpp:42-49): name the first offending node
      const int64_t j = static_cast<int64_t>(badj);
      for (int t = 0; t < d; ++t) {
        double v = nodes_colmajor[t * n + j];
        if (kind == FASTSUM) v = rho * v;
        if (!(v >= -0.5 && v < 0.5))
          fail(FGS_ERANGE, "node " + std::to_string(j) + " component " + std::to_string(t) + " = " +
                               std::to_string(v) + " outside [-1/2, 1/2)");
      }
    }
    int end_bit = 1;
    {
      double total = 1.0;
      for (int t = 0; t < d; ++t) total *= static_cast<double>(nt) * B;
      while (end_bit < 64 && std::ldexp(1.0, end_bit) < total) ++end_bit;
    }
    size_t tmp_bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, keys.p, keys_sorted.p, idx.p, perm.p, static_cast<int>(n), 0,
                                    end_bit, stream);
    tmp.alloc(tmp_bytes);
    FGS_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tmp_bytes, keys.p, keys_sorted.p, idx.p, perm.p,
                                             static_cast<int>(n), 0, end_bit, stream));
    size_t tmp2 = 0;
    cub::DeviceRunLengthEncode::Encode(nullptr, tmp2, keys_sorted.p, uniq.p, counts.p, nruns.p, static_cast<int>(n),
                                       stream);
    tmpb.alloc(tmp2);
    FGS_CUDA(cub::DeviceRunLengthEncode::Encode(tmpb.p, tmp2, keys_sorted.p, uniq.p, counts.p, nruns.p,
                                                static_cast<int>(n), stream));
    FGS_CUDA(cudaMemcpyAsync(&ncells, nruns.p, sizeof(int), cudaMemcpyDeviceToHost, stream));
    FGS_CUDA(cudaStreamSynchronize(stream));
  };
  sort_cells();
  // Very dense 3-D point sets (>= 100 points per nonempty cell: items are
  // then mostly single cells) use 2^3-cell tiles: smaller item boxes -> less
  // shared memory per CTA -> more resident warps (config 4: spread 511 ->
  // 411 us, interp 475 -> 432 us); moderate densities keep 4^3 (config 5).
  if (d == 3 && B == 4 && !std::getenv("FGS_TILE_B") && static_cast<double>(n) >= 100.0 * ncells && M >= 2) {
    B = 2;
    nt = ceil_div(M, B);
    ntiles = nt * nt * nt;
    unsigned long long init2 = ULLONG_MAX;
    FGS_CUDA(cudaMemcpyAsync(bad.p, &init2, sizeof(init2), cudaMemcpyHostToDevice, stream));
    sort_cells();
  }
  std::vector<unsigned long long> hkeys(static_cast<size_t>(ncells));
  std::vector<int> hcounts(static_cast<size_t>(ncells));
  FGS_CUDA(cudaMemcpyAsync(hkeys.data(), uniq.p, sizeof(unsigned long long) * ncells, cudaMemcpyDeviceToHost, stream));
  FGS_CUDA(cudaMemcpyAsync(hcounts.data(), counts.p, sizeof(int) * ncells, cudaMemcpyDeviceToHost, stream));
  host_perm.resize(static_cast<size_t>(n));
  FGS_CUDA(cudaMemcpyAsync(host_perm.data(), perm.p, sizeof(int) * n, cudaMemcpyDeviceToHost, stream));
  FGS_CUDA(cudaStreamSynchronize(stream));

  // shard slice of the internal order
  offset = n * rank / world;
  n_local = n * (rank + 1) / world - offset;

  // ---- work items: runs of cells inside one tile, <= chunk points ---------
  // items (CTAs) per pass: enough to fill every SM several times over; small
  // problems get short items (their cost is the serial staging chain)
  // (sharded plans: by the whole problem's size -- a C4 rank of 250k points
  // runs 592 items of ~420 points: 0.195 ms vs 0.244 ms with 2368 small ones,
  // whose box zero / write-out / assembly overhead does not shrink with n)
  int64_t target_items = n < 300000 ? 16 * 148 : 4 * 148;
  if (const char* e = std::getenv("FGS_ITEM_TARGET")) target_items = std::max<int64_t>(1, std::atoll(e));
  int chunk = static_cast<int>(std::max<int64_t>(32, std::min<int64_t>(4096, (n_local + target_items - 1) / target_items)));
  chunk = (chunk + 31) / 32 * 32;
  if (const char* e = std::getenv("FGS_CHUNK")) chunk = std::max(8, std::atoi(e));  // tuning override (cost units)
  // per-run overhead in point units (a partly filled K-step + the footprint
  // flush), FGS_RUN_COST overrides.  d = 2: 3 (C2 22.2k -> 24.1k matvecs/s:
  // sparse-region items no longer set the single wave's length); d = 3: 0
  // (C1 loses with it, C3/C4 are indifferent)
  int run_cost = d == 2 ? 3 : 0;
  if (const char* e = std::getenv("FGS_RUN_COST")) run_cost = std::max(0, std::atoi(e));
  int BD = 1;
  for (int t = 0; t < d; ++t) BD *= B;

  struct HRun {
    int pstart, pcount;
    int c[3];
  };
  struct HItem {
    int tile;
    std::vector<HRun> runs;
    int npts = 0;
    int cost = 0;  // points + run_cost per run: what a CTA's time scales with
  };
  std::vector<HItem> hitems;
  auto decode_cell = [&](unsigned long long key, int* tcoord, int* cc) {
    unsigned long long tile = key / BD, cell = key % BD;
    for (int t = 2; t >= 0; --t) {
      if (t >= 3 - d) {
        cc[t] = static_cast<int>(cell % B);
        cell /= B;
        tcoord[t] = static_cast<int>(tile % nt);
        if (t == 3 - d) tcoord[t] = (tcoord[t] + rot0) % nt;  // undo the dim-0 tile rotation
        tile /= nt;
      } else {
        cc[t] = 0;
        tcoord[t] = 0;
      }
    }
  };
  {
    int64_t start = 0;
    HItem cur;
    cur.tile = -1;
    auto flush = [&]() {
      if (!cur.runs.empty()) hitems.push_back(std::move(cur));
      cur = HItem();
      cur.tile = -1;
    };
    for (int c = 0; c < ncells; ++c) {
      const int64_t cs = start, ce = start + hcounts[static_cast<size_t>(c)];
      start = ce;
      const int64_t lo = std::max(cs, offset), hi = std::min(ce, offset + n_local);
      if (lo >= hi) continue;
      const int tile = static_cast<int>(hkeys[static_cast<size_t>(c)] / BD);
      if (tile != cur.tile) flush();
      cur.tile = tile;
      int tc[3], cc[3];
      decode_cell(hkeys[static_cast<size_t>(c)], tc, cc);
      int64_t p = lo;
      while (p < hi) {
        // item budget in cost units: a run costs run_cost plus its points
        int take = static_cast<int>(std::min<int64_t>(hi - p, chunk - cur.cost - run_cost));
        if (take <= 0) {
          if (cur.runs.empty()) {
            take = static_cast<int>(std::min<int64_t>(hi - p, chunk));  // one run alone still fits
          } else {
            flush();
            cur.tile = tile;
            continue;
          }
        }
        HRun r;
        r.pstart = static_cast<int>(p - offset);
        r.pcount = take;
        r.c[0] = cc[0];
        r.c[1] = cc[1];
        r.c[2] = cc[2];
        cur.runs.push_back(r);
        cur.npts += take;
        cur.cost += take + run_cost;
        p += take;
        if (cur.cost >= chunk) {
          flush();
          cur.tile = tile;
        }
      }
    }
    flush();
  }
  // heaviest items first (LPT order for the block scheduler)
  std::stable_sort(hitems.begin(), hitems.end(), [](const HItem& x, const HItem& y) { return x.cost > y.cost; });

  nitems = static_cast<int>(hitems.size());
  {
    size_t nr = 0;
    for (const HItem& h : hitems) nr += h.runs.size();
    mean_run = nr ? static_cast<double>(n_local) / static_cast<double>(nr) : 0.0;
  }
  std::vector<DItem> ditems;
  std::vector<DRun> druns;
  const int Md[3] = {d == 3 ? M : 1, d >= 2 ? M : 1, M};
  box_stride = 1;
  box_pad = 1;
  for (int k = 0; k < nitems; ++k) {
    const HItem& h = hitems[static_cast<size_t>(k)];
    int lo[3] = {INT_MAX, INT_MAX, INT_MAX}, hi[3] = {INT_MIN, INT_MIN, INT_MIN};
    for (const HRun& r : h.runs)
      for (int t = 0; t < 3; ++t) {
        lo[t] = std::min(lo[t], r.c[t]);
        hi[t] = std::max(hi[t], r.c[t]);
      }
    int tc[3], cc[3];
    decode_cell(static_cast<unsigned long long>(h.tile) * BD, tc, cc);
    DItem it;
    it.run_begin = static_cast<int>(druns.size());
    for (const HRun& r : h.runs) {
      DRun dr;
      dr.pstart = r.pstart;
      dr.pcount = r.pcount;
      dr.off = (r.c[0] - lo[0]) | ((r.c[1] - lo[1]) << 10) | ((r.c[2] - lo[2]) << 20);
      druns.push_back(dr);
    }
    it.run_end = static_cast<int>(druns.size());
    it.p_begin = h.runs.front().pstart;
    it.p_end = h.runs.back().pstart + h.runs.back().pcount;
    int ext[3], org[3];
    for (int t = 0; t < 3; ++t) {
      const bool used = t >= 3 - d;
      ext[t] = used ? (hi[t] - lo[t] + T) : 1;
      org[t] = used ? ((tc[t] * B + lo[t]) % M) : 0;
    }
    it.a0 = org[0];
    it.a1 = org[1];
    it.a2 = org[2];
    it.e0 = ext[0];
    it.e1 = ext[1];
    it.e2 = ext[2];
    box_stride = std::max<int64_t>(box_stride, static_cast<int64_t>(ext[0]) * ext[1] * ext[2]);
    box_pad = std::max<int64_t>(box_pad, static_cast<int64_t>(ext[0]) * ext[1] * v5_pad(ext[2]));
    ditems.push_back(it);
  }
  box_stride = (box_stride + 1) / 2 * 2;  // keep the staging area 16-byte aligned
  box_pad = (box_pad + 1) / 2 * 2;
  // dim-0 planes this rank's boxes cover: the smallest cyclic interval
  // holding them (sharded handles convolve only those planes)
  conv_plane0 = 0;
  conv_planes = M;
  if (d == 3 && world > 1 && !ditems.empty()) {
    std::vector<char> used(static_cast<size_t>(M), 0);
    for (const DItem& it : ditems)
      for (int x0 = 0; x0 < it.e0; ++x0) used[static_cast<size_t>((it.a0 + x0) % M)] = 1;
    int best_len = M, best_start = 0;  // longest cyclic run of unused planes -> its complement
    int run = 0, run_start = 0, bl = 0, bs = 0;
    for (int t = 0; t < 2 * M; ++t) {
      if (!used[static_cast<size_t>(t % M)]) {
        if (run == 0) run_start = t;
        if (++run > bl && run <= M) {
          bl = run;
          bs = run_start;
        }
      } else {
        run = 0;
      }
    }
    if (bl > 0 && bl < M) {
      best_start = (bs + bl) % M;
      best_len = M - bl;
    }
    // cyclic plane range (a point cloud centred on 0 wraps around plane 0)
    conv_plane0 = best_start;
    conv_planes = best_len;
  }
  if (std::getenv("FGS_PLAN_STATS")) {  // tuning aid: item sizes and the per-CTA shared memory
    int64_t box_sum = 0, pts_max = 0, runs_max = 0;
    for (const DItem& it : ditems) {
      box_sum += static_cast<int64_t>(it.e0) * it.e1 * it.e2;
      pts_max = std::max<int64_t>(pts_max, it.p_end - it.p_begin);
      runs_max = std::max<int64_t>(runs_max, it.run_end - it.run_begin);
    }
    std::fprintf(stderr, "[plan] n_local %lld items %d chunk %d run_cost %d mean_run %.2f | box max %lld mean %.1f | "
                 "item points max %lld runs max %lld\n", static_cast<long long>(n_local), nitems, chunk, run_cost,
                 mean_run, static_cast<long long>(box_stride),
                 nitems ? static_cast<double>(box_sum) / nitems : 0.0, static_cast<long long>(pts_max),
                 static_cast<long long>(runs_max));
  }
  if (static_cast<double>(std::max(nitems, 1)) * static_cast<double>(box_stride) > 2.0e9)
    fail(FGS_ERESOURCE, "spread workspace exceeds 2^31 entries");
  // Deterministic assembly map: for every grid cell, the private-box entries
  // (item k, local offset) that land on it, in increasing item order.
  {
    std::vector<int> cnt(static_cast<size_t>(grid_elems) + 1, 0);
    auto for_box = [&](const DItem& it, auto&& fn) {
      for (int x0 = 0; x0 < it.e0; ++x0) {
        const int64_t g0 = (it.a0 + x0) % Md[0];
        for (int x1 = 0; x1 < it.e1; ++x1) {
          const int64_t g01 = (g0 * Md[1] + (it.a1 + x1) % Md[1]) * Md[2];
          const int base = (x0 * it.e1 + x1) * it.e2;
          for (int x2 = 0; x2 < it.e2; ++x2) fn(g01 + (it.a2 + x2) % Md[2], base + x2);
        }
      }
    };
    for (int k = 0; k < nitems; ++k)
      for_box(ditems[static_cast<size_t>(k)], [&](int64_t g, int) { ++cnt[static_cast<size_t>(g) + 1]; });
    for (int64_t g = 0; g < grid_elems; ++g) cnt[static_cast<size_t>(g) + 1] += cnt[static_cast<size_t>(g)];
    std::vector<int> pos(cnt.begin(), cnt.end() - 1);
    std::vector<int> idx(static_cast<size_t>(std::max(cnt.back(), 1)));
    for (int k = 0; k < nitems; ++k) {
      const int base = static_cast<int>(static_cast<int64_t>(k) * box_stride);
      for_box(ditems[static_cast<size_t>(k)],
              [&](int64_t g, int v) { idx[static_cast<size_t>(pos[static_cast<size_t>(g)]++)] = base + v; });
    }
    asm_ptr.upload(cnt.data(), cnt.size(), stream);
    asm_idx.upload(idx.data(), idx.size(), stream);
    // lanes per cell by list length: clustered data concentrates most entries
    // in a few long lists (C3-C5: ~85 % of the entries sit in lists > 64),
    // which one lane per cell walks serially.  Cells are sorted into three
    // warp-aligned classes (<= 8 entries: one lane, 9..64: 8 lanes, > 64: a
    // warp), heaviest first, and one launch serves all three.  Cells no item
    // box touches are not listed: the spread grid is zeroed once when the
    // workspace is created and those cells are never written (the convolution
    // writes a separate output grid), so the assembly covers only the point
    // cloud's footprint (and, sharded, only this rank's slab of it).
    {
      std::vector<int> cls[3];
      for (int64_t g = 0; g < grid_elems; ++g) {
        const int len = cnt[static_cast<size_t>(g) + 1] - cnt[static_cast<size_t>(g)];
        if (len == 0) continue;
        cls[len <= 8 ? 0 : (len <= 64 ? 1 : 2)].push_back(static_cast<int>(g));
      }
      std::vector<int> all;
      for (int c = 2; c >= 0; --c) {
        asm_class_n[c] = static_cast<int64_t>(cls[c].size());
        all.insert(all.end(), cls[c].begin(), cls[c].end());  // heaviest first
      }
      if (all.empty()) all.push_back(0);
      asm_cells.upload(all.data(), all.size(), stream);
    }
  }
  if (ditems.empty()) {
    ditems.push_back(DItem{0, 0, 0, 0, 0, 1, 1, 1, 0, 0});
    nitems = 0;
  }
  // run-aligned slot layout (kernels_v6.cuh): every run starts on a
  // multiple of kSlotAlign slots, items are consecutive; same item order and
  // boxes as the point layout, so the assembly map serves both
  use_slots = false;
  if (kind == FASTSUM && d == 3 && (T == 16 || T == 12) && nitems > 0 && mean_run >= kDenseRun && v6_enabled()) {
    std::vector<DItem> sitems(ditems);
    std::vector<DRun> sruns(druns);
    std::vector<int>& smap = slot_host;
    smap.clear();
    smap.reserve(static_cast<size_t>(n_local + (n_local / 8) + 8 * druns.size()));
    int64_t sl = 0;
    for (DItem& it : sitems) {
      it.p_begin = static_cast<int>(sl);
      for (int r = it.run_begin; r < it.run_end; ++r) {
        const DRun& pr = druns[static_cast<size_t>(r)];
        sruns[static_cast<size_t>(r)].pstart = static_cast<int>(sl);
        const int padded = (pr.pcount + kSlotAlign - 1) / kSlotAlign * kSlotAlign;
        for (int j = 0; j < padded; ++j) smap.push_back(j < pr.pcount ? pr.pstart + j : -1);
        sl += padded;
      }
      it.p_end = static_cast<int>(sl);
    }
    if (sl >= (int64_t{1} << 31)) fail(FGS_ERESOURCE, "slot layout exceeds 2^31 entries");
    items6.upload(sitems.data(), sitems.size(), stream);
    runs6.upload(sruns.data(), sruns.size(), stream);
    slot_map.upload(smap.data(), smap.size(), stream);
    std::vector<int> boff(static_cast<size_t>(sl / kSlotAlign));
    for (const DItem& it : sitems)
      for (int r = it.run_begin; r < it.run_end; ++r) {
        const DRun& sr = sruns[static_cast<size_t>(r)];
        const int padded = (sr.pcount + kSlotAlign - 1) / kSlotAlign * kSlotAlign;
        for (int b = sr.pstart / kSlotAlign; b < (sr.pstart + padded) / kSlotAlign; ++b)
          boff[static_cast<size_t>(b)] = sr.off;
      }
    batch_off.upload(boff.data(), boff.size(), stream);
    use_slots = true;
    // fixed box strides for the slot-layout interpolation (tile B in {2, 4}):
    // every item's box laid out with the maximal extent B + 2m - 1
    box_ext = (B == 2 || B == 4) && !std::getenv("FGS_BOX_EXT0") ? B + T - 1 : 0;
    if (box_ext) box_pad = std::max<int64_t>(box_pad, static_cast<int64_t>(box_ext) * box_ext * v5_pad(box_ext));
  }
  items.upload(ditems.data(), ditems.size(), stream);
  if (druns.empty()) druns.push_back(DRun{0, 0, 0});
  runs.upload(druns.data(), druns.size(), stream);

  // window taps of the local slice in internal order, or (slot layout) in
  // slot order with rows padded to slot_row<2m>() doubles, pad slots zero
  if (use_slots) {
    std::vector<int> rows(slot_host.size());
    for (size_t i = 0; i < rows.size(); ++i)
      rows[i] = slot_host[i] < 0 ? -1 : host_perm[static_cast<size_t>(offset + slot_host[i])];
    DBuf<int> drows;
    drows.upload(rows.data(), rows.size(), stream);
    const int64_t ns = static_cast<int64_t>(rows.size());
    const int srow = slot_row_of(T);
    taps.alloc(static_cast<size_t>(ns) * srow);
    TapArgs ta{dnodes.p, n, ns, perm.p + offset, d, M, m, rho, b_kb, kind == FASTSUM ? 1 : 0, taps.p, drows.p, srow};
    taps_kernel<<<ceil_div(ns, 128), 128, 0, stream>>>(ta);
    ++launches;
    FGS_CUDA(cudaGetLastError());
    FGS_CUDA(cudaStreamSynchronize(stream));  // before drows is freed
    slot_host.clear();
    slot_host.shrink_to_fit();
  } else {
  taps.alloc(static_cast<size_t>(std::max<int64_t>(n_local, 1)) * d * T);
  if (n_local > 0) {
    TapArgs ta{dnodes.p, n, n_local, perm.p + offset, d, M, m, rho, b_kb, kind == FASTSUM ? 1 : 0, taps.p, nullptr, 0};
    taps_kernel<<<ceil_div(n_local, 128), 128, 0, stream>>>(ta);
    ++launches;
    FGS_CUDA(cudaGetLastError());
  }
  }
  FGS_CUDA(cudaStreamSynchronize(stream));
}

void Core::build_coefficients() {
  // bhat_l = (-1)^{sum l} N^-d FFT[K_R(j/N)] (kernels.cpp:266-335); the N^d
  // transform runs on the device (cuFFT Z2Z, FFTW_FORWARD sign)
  size_t total = 1;
  for (int t = 0; t < d; ++t) total *= static_cast<size_t>(N);
  const int half = N / 2;
  std::vector<cufftDoubleComplex> samples(total);
  int idx[3] = {0, 0, 0};
  for (size_t flat = 0; flat < total; ++flat) {
    size_t rest = flat;
    for (int t = d - 1; t >= 0; --t) {
      idx[t] = static_cast<int>(rest % N);
      rest /= N;
    }
    double s2 = 0.0;
    for (int t = 0; t < d; ++t) {
      const double y = static_cast<double>(idx[t] - half) / N;
      s2 += y * y;
    }
    samples[flat] = make_cuDoubleComplex(reg(std::sqrt(s2)), 0.0);
  }
  DBuf<cufftDoubleComplex> buf;
  buf.upload(samples.data(), total, stream);
  cufftHandle plan;
  int dims[3] = {N, N, N};
  FGS_CUFFT(cufftPlanMany(&plan, d, dims, nullptr, 1, 0, nullptr, 1, 0, CUFFT_Z2Z, 1));
  FGS_CUFFT(cufftSetStream(plan, stream));
  FGS_CUFFT(cufftExecZ2Z(plan, buf.p, buf.p, CUFFT_FORWARD));
  FGS_CUDA(cudaMemcpyAsync(samples.data(), buf.p, total * sizeof(cufftDoubleComplex), cudaMemcpyDeviceToHost, stream));
  FGS_CUDA(cudaStreamSynchronize(stream));
  cufftDestroy(plan);
  bhat.resize(total);
  const double norm = 1.0 / static_cast<double>(total);
  for (size_t flat = 0; flat < total; ++flat) {
    size_t rest = flat, bin = 0, stride = 1;
    int lsum = 0;
    for (int t = d - 1; t >= 0; --t) {
      const int a = static_cast<int>(rest % N);
      rest /= N;
      const int l = a - half;
      lsum += l;
      bin += static_cast<size_t>((l + N) % N) * stride;
      stride *= static_cast<size_t>(N);
    }
    const double sign = (lsum % 2 == 0) ? 1.0 : -1.0;
    bhat[flat] = std::complex<double>(samples[bin].x, samples[bin].y) * (sign * norm);
  }

  // compact Hermitian-symmetrised multiplier (see multiply_kernel)
  auto mval = [&](const int* k) -> std::complex<double> {  // m_k on wrap(I_N)
    size_t flat = 0;
    double dec = 1.0;
    for (int t = 0; t < d; ++t) {
      int l;
      if (k[t] < half)
        l = k[t];
      else if (k[t] >= M - half)
        l = k[t] - M;
      else
        return 0.0;
      flat = flat * N + static_cast<size_t>(l + half);
      dec = (t == 0) ? deconv[static_cast<size_t>(l + half)] : dec * deconv[static_cast<size_t>(l + half)];
    }
    return out_factor * (bhat[flat] * (dec * dec));
  };
  std::vector<cufftDoubleComplex> hm(static_cast<size_t>(window_elems));
  const int W = N + 1, hN = N / 2;
  for (int64_t w = 0; w < window_elems; ++w) {
    int l[3] = {0, 0, 0};
    l[d - 1] = static_cast<int>(w % (hN + 1));
    int64_t rest = w / (hN + 1);
    for (int t = d - 2; t >= 0; --t) {
      l[t] = static_cast<int>(rest % W) - hN;
      rest /= W;
    }
    int k[3], km[3];
    for (int t = 0; t < d; ++t) {
      k[t] = ((l[t] % M) + M) % M;
      km[t] = ((-l[t] % M) + M) % M;
    }
    std::complex<double> v = 0.5 * (mval(k) + std::conj(mval(km)));
    hm[static_cast<size_t>(w)] = make_cuDoubleComplex(v.real(), v.imag());
  }
  mult.upload(hm.data(), hm.size(), stream);
  FGS_CUDA(cudaStreamSynchronize(stream));
}

Workspace& Core::workspace(int nvec) {
  auto itw = ws_.find(nvec);
  if (itw != ws_.end()) return *itw->second;
  auto w = std::make_unique<Workspace>();
  w->nvec = nvec;
  if (kind == DIRECT) {  // segment partials [nseg][nvec][n]
    w->priv.alloc(static_cast<size_t>(direct_segments()) * nvec * n);
    auto& ref = *w;
    ws_[nvec] = std::move(w);
    return ref;
  }
  w->priv.alloc(static_cast<size_t>(std::max(nitems, 1)) * box_stride * nvec);
  w->grid.alloc(static_cast<size_t>(grid_elems) * nvec);
  FGS_CUDA(cudaMemsetAsync(w->grid.p, 0, sizeof(double) * grid_elems * nvec, stream));
  w->grid_out.alloc(static_cast<size_t>(grid_elems) * nvec);
  if (use_slots) w->xs.alloc(slot_map.n * nvec);
  if (sharded && d == 2) w->grid_sum.alloc(static_cast<size_t>(grid_elems) * nvec);
  if (use_conv3d()) {  // plane-pass window buffer (+ the sharded window spectrum)
    const int64_t nw = conv3_nw(M, N), H = N / 2 + 1;
    w->win.alloc(static_cast<size_t>(M) * nw * H * nvec);
    if (sharded) w->cspec.alloc(static_cast<size_t>(nw) * nw * H * nvec);
  }
  if (!use_conv2d() && !use_conv3d()) {  // cuFFT only where no hand-written convolution covers the grid
    w->spec.alloc(static_cast<size_t>(spec_elems) * nvec);
    if (sharded) w->window.alloc(static_cast<size_t>(window_elems) * nvec);
    int dims[3] = {M, M, M};
    FGS_CUFFT(cufftPlanMany(&w->r2c, d, dims, nullptr, 1, static_cast<int>(grid_elems), nullptr, 1,
                            static_cast<int>(spec_elems), CUFFT_D2Z, nvec));
    FGS_CUFFT(cufftPlanMany(&w->c2r, d, dims, nullptr, 1, static_cast<int>(spec_elems), nullptr, 1,
                            static_cast<int>(grid_elems), CUFFT_Z2D, nvec));
    FGS_CUFFT(cufftSetStream(w->r2c, stream));
    FGS_CUFFT(cufftSetStream(w->c2r, stream));
    w->has_plans = true;
  }
  auto& ref = *w;
  ws_[nvec] = std::move(w);
  return ref;
}

size_t Core::smem_bytes(bool interp) const {
  const bool dense = mean_run >= kDenseRun;
  const LaunchShape sh = d == 3 ? shape_of<3>(T, dense) : (d == 2 ? shape_of<2>(T, dense) : shape_of<1>(T, dense));
  size_t boxes = static_cast<size_t>(box_stride);
  if (interp && d == 3 && (T == 8 || T == 12 || T == 16)) boxes = static_cast<size_t>(box_pad);
  if (use_slots && interp)
    return (boxes + (T == 16 ? v6i_extra_doubles<16>() : v6i_extra_doubles<12>())) * sizeof(double);
  if (use_slots && !interp && T == 16) return (boxes + v6s_extra_doubles()) * sizeof(double);
  if (use_slots && !interp && T == 12 && spread_v8_on()) return (boxes + v8s_extra_doubles()) * sizeof(double);
  if (d == 3 && !interp && dense) boxes *= static_cast<size_t>(v4_spread_groups(T));  // per-group boxes
  if (d == 2 && !interp && dense && (T == 8 || T == 12 || T == 16))
    boxes *= static_cast<size_t>(kSpread2dP);  // per-stream boxes
  return (boxes + (interp ? sh.extra_interp : sh.extra_spread)) * sizeof(double);
}

bool Core::tensor_spread() const {
  return kind != DIRECT && (d == 2 || d == 3) && (T == 8 || T == 12 || T == 16) && mean_run >= kDenseRun;
}
bool Core::tensor_interp() const { return kind != DIRECT && (d == 2 || d == 3) && (T == 8 || T == 12 || T == 16); }

void Core::launch_spread(const PassArgs& a) {
  if (nitems == 0) return;
  const size_t smem = smem_bytes(false);
  if (std::getenv("FGS_PLAN_STATS") && launches == 0)
    std::fprintf(stderr, "[plan] smem per CTA: spread %zu B, interp %zu B\n", smem, smem_bytes(true));
  if (smem > 227 * 1024) fail(FGS_ERESOURCE, "tile box exceeds shared memory (cutoff too large for d = 3)");
  const bool dense = mean_run >= kDenseRun;
  const int bs = static_cast<int>(box_stride), bp = static_cast<int>(box_pad);
  if (use_slots && (T == 16 || spread_v8_on()) && a.nvec > 1) {  // spread_v6 / spread_v8: vector split
    PassArgs b = a;
    b.vsplit = vsplit_for(a.nvec);
    dispatch<3>(false, dense, T, b, nitems * b.vsplit, smem, bs, bp, stream);
    ++launches;
    FGS_CUDA(cudaGetLastError());
    return;
  }
  if (d == 3) dispatch<3>(false, dense, T, a, nitems, smem, bs, bp, stream);
  if (d == 2) dispatch<2>(false, dense, T, a, nitems, smem, bs, bp, stream);
  if (d == 1) dispatch<1>(false, dense, T, a, nitems, smem, bs, bp, stream);
  ++launches;
  FGS_CUDA(cudaGetLastError());
}

void Core::launch_interp(const PassArgs& a) {
  if (nitems == 0) return;
  const size_t smem = smem_bytes(true);
  if (smem > 227 * 1024) fail(FGS_ERESOURCE, "tile box exceeds shared memory (cutoff too large for d = 3)");
  const int bs = static_cast<int>(box_stride), bp = static_cast<int>(box_pad);
  if (use_slots && a.nvec > 1) {  // interp_v6 / interp_v7: vector split
    PassArgs b = a;
    b.vsplit = vsplit_for(a.nvec);
    dispatch<3>(true, true, T, b, nitems * b.vsplit, smem, bs, bp, stream);
    ++launches;
    FGS_CUDA(cudaGetLastError());
    return;
  }
  if (d == 3) dispatch<3>(true, true, T, a, nitems, smem, bs, bp, stream);
  if (d == 2) dispatch<2>(true, true, T, a, nitems, smem, bs, bp, stream);
  if (d == 1) dispatch<1>(true, true, T, a, nitems, smem, bs, bp, stream);
  ++launches;
  FGS_CUDA(cudaGetLastError());
}

void Core::launch_assemble(Workspace& w, int nvec) {
  const int64_t pstride = static_cast<int64_t>(std::max(nitems, 1)) * box_stride;
  AssembleMixedArgs m{};
  m.a = AssembleArgs{asm_ptr.p, asm_idx.p, w.priv.p, pstride, w.grid.p, grid_elems};
  m.a.nvec = nvec;
  m.cells = asm_cells.p;
  m.n0 = asm_class_n[0];
  m.n1 = asm_class_n[1];
  m.n2 = asm_class_n[2];
  m.w2 = m.n2;
  m.w1 = (m.n1 + 3) / 4;
  const int64_t warps = m.w2 + m.w1 + (m.n0 + 31) / 32;
  if (warps == 0) return;
  const dim3 blocks(static_cast<unsigned>(ceil_div(warps * 32, 256)));
  if (nvec > 1)  // indices hoisted out of the vector loop (C5 16-vector blocks: 1.82 -> 1.71 ms)
    launch_ex(assemble_mixed_kernel<true>, blocks, 256, 0, stream, m);
  else
    launch_ex(assemble_mixed_kernel<false>, blocks, 256, 0, stream, m);
  ++launches;
  FGS_CUDA(cudaGetLastError());
}

void Core::apply(int epilogue, const double* x, int64_t ldx, double* y, int64_t ldy, int nvec, bool caller_order,
                 bool scale_input) {
  // Steady-state applies replay a CUDA graph of the whole launch sequence
  // (spread, assemble, cuFFT, multiply/exchange, cuFFT, interpolation), keyed
  // by the call's arguments: one launch instead of ~10 host launches.
  static const bool graphs_on = [] {
    const char* e = std::getenv("FGS_GRAPHS");
    return !(e && std::string(e) == "0");
  }();
  // sharded handles capture their ncclAllReduce into the graph as well (NCCL
  // supports stream capture; every rank replays the same sequence);
  // FGS_SHARDED_GRAPHS=0 launches them directly
  static const bool sharded_graphs = [] {
    const char* e = std::getenv("FGS_SHARDED_GRAPHS");
    return !(e && std::string(e) == "0");
  }();
  if (!graphs_on || profile_ || stream == nullptr || epilogue == EPI_DEGREE || (sharded && !sharded_graphs)) {
    apply_launches(epilogue, x, ldx, y, ldy, nvec, caller_order, scale_input);
    return;
  }
  const GraphKey key{epilogue, x, ldx, y, ldy, nvec, caller_order, scale_input};
  for (auto& g : graphs_) {
    if (g.key == key) {
      FGS_CUDA(cudaGraphLaunch(g.exec, stream));
      launches += g.launches;
      return;
    }
  }
  workspace(nvec);  // allocate / plan outside the capture
  const int64_t before = launches;
  FGS_CUDA(cudaStreamBeginCapture(stream, cudaStreamCaptureModeThreadLocal));
  try {
    apply_launches(epilogue, x, ldx, y, ldy, nvec, caller_order, scale_input);
  } catch (...) {
    cudaGraph_t broken = nullptr;
    cudaStreamEndCapture(stream, &broken);
    if (broken) cudaGraphDestroy(broken);
    throw;
  }
  cudaGraph_t graph = nullptr;
  FGS_CUDA(cudaStreamEndCapture(stream, &graph));
  cudaGraphExec_t exec = nullptr;
  FGS_CUDA(cudaGraphInstantiate(&exec, graph, 0));
  cudaGraphDestroy(graph);
  if (graphs_.size() >= 8) {
    cudaGraphExecDestroy(graphs_.front().exec);
    graphs_.erase(graphs_.begin());
  }
  graphs_.push_back({key, exec, launches - before});
  launches = before;
  FGS_CUDA(cudaGraphLaunch(exec, stream));
  launches += graphs_.back().launches;
}

static bool is_pinned(const void* p) {
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeHost;
}

// Sub-blocks of a host-vector block.  The copy streams move one sub-block
// while the compute stream applies another, so the exposed copies are the
// first sub-block's upload and the last one's download: both one vector.
// Sub-blocks in between grow (and shrink again towards the end) as fast as
// the copies allow -- a multi-vector apply is cheaper per vector than
// single-vector ones (shared taps reads, fewer wave tails, one convolution
// launch), and the upload of sub-blocks 1..k+1 only has to finish while
// 1..k compute: S_{k+1} <= 1 + rho S_k, rho = compute / copy time per vector
// (d = 3: ~2.7e-3 (2m)^3 / 3 with PCIe at ~50 GB/s; config 5: 16 vectors ->
// 1 2 5 5 2 1).  Copy-bound plans (rho < 1) keep single-vector sub-blocks.
// FGS_PIPE_PARTS="1,3,8,3,1" forces a partition (tuning).
static std::vector<int> pipe_partition(int nvec, int d, int T) {
  static const std::vector<int> forced = [] {
    std::vector<int> v;
    if (const char* e = std::getenv("FGS_PIPE_PARTS")) {
      const std::string str(e);
      size_t pos = 0;
      while (pos < str.size()) {
        const size_t c = str.find(',', pos);
        v.push_back(std::atoi(str.substr(pos, c == std::string::npos ? std::string::npos : c - pos).c_str()));
        if (c == std::string::npos) break;
        pos = c + 1;
      }
    }
    return v;
  }();
  if (!forced.empty() && std::accumulate(forced.begin(), forced.end(), 0) == nvec &&
      *std::min_element(forced.begin(), forced.end()) > 0)
    return forced;
  const double rho = d == 3 ? 0.8 * 9.1e-4 * T * T * T : 0.0;
  constexpr int kCap = 8;  // largest sub-block (bounds the extra workspaces)
  std::vector<int> head;
  int S = 0, b = 1;
  while (rho > 1.0 && 2 * (S + b) <= nvec) {
    head.push_back(b);
    S += b;
    b = std::max(1, std::min(kCap, static_cast<int>(1.0 + rho * S) - S));
  }
  if (head.empty()) return std::vector<int>(static_cast<size_t>(nvec), 1);
  std::vector<int> parts(head);
  int mid = nvec - 2 * S;
  while (mid > 0) {  // the middle in near-equal sub-blocks of <= kCap vectors
    const int pieces = (mid + kCap - 1) / kCap;
    const int take = (mid + pieces - 1) / pieces;
    parts.push_back(take);
    mid -= take;
  }
  parts.insert(parts.end(), head.rbegin(), head.rend());
  return parts;
}

bool Core::apply_host_graph(int epilogue, const double* hx, double* hy, int64_t ld, int nvec, bool scale_input) {
  static const bool graphs_on = [] {
    const char* e = std::getenv("FGS_GRAPHS");
    const char* h = std::getenv("FGS_HOST_GRAPH");
    return !(e && std::string(e) == "0") && !(h && std::string(h) == "0");
  }();
  if (!graphs_on || profile_ || stream == nullptr || sharded || world > 1) return false;
  if (!is_pinned(hx) || !is_pinned(hy)) return false;  // checked every call: an address may be reused
  xbuf.alloc(static_cast<size_t>(n) * nvec);
  ybuf.alloc(static_cast<size_t>(n) * nvec);
  GraphKey key{epilogue, xbuf.p, n, ybuf.p, n, nvec, true, scale_input};
  key.hx = hx;
  key.hy = hy;
  key.hld = ld;
  for (auto& g : graphs_) {
    if (g.key == key) {
      FGS_CUDA(cudaGraphLaunch(g.exec, stream));
      launches += g.launches;
      return true;
    }
  }
  const std::vector<int> parts = pipe_partition(nvec, d, T);
  const int nsub = static_cast<int>(parts.size());
  for (int b : parts) workspace(b);
  if (nsub > 1) {
    if (!cp_in) FGS_CUDA(cudaStreamCreateWithFlags(&cp_in, cudaStreamNonBlocking));
    if (!cp_out) FGS_CUDA(cudaStreamCreateWithFlags(&cp_out, cudaStreamNonBlocking));
    while (pipe_ev.size() < static_cast<size_t>(2 * nsub + 3)) {
      cudaEvent_t e;
      FGS_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      pipe_ev.push_back(e);
    }
  }
  // vectors [v0, v0 + cnt) between the pinned host block and xbuf / ybuf
  auto h2d = [&](int v0, int cnt, cudaStream_t s) {
    double* dst = xbuf.p + static_cast<int64_t>(v0) * n;
    const double* src = hx + static_cast<int64_t>(v0) * ld;
    if (ld == n)
      FGS_CUDA(cudaMemcpyAsync(dst, src, sizeof(double) * n * cnt, cudaMemcpyHostToDevice, s));
    else
      FGS_CUDA(cudaMemcpy2DAsync(dst, sizeof(double) * n, src, sizeof(double) * ld, sizeof(double) * n, cnt,
                                 cudaMemcpyHostToDevice, s));
  };
  auto d2h = [&](int v0, int cnt, cudaStream_t s) {
    const double* src = ybuf.p + static_cast<int64_t>(v0) * n;
    double* dst = hy + static_cast<int64_t>(v0) * ld;
    if (ld == n)
      FGS_CUDA(cudaMemcpyAsync(dst, src, sizeof(double) * n * cnt, cudaMemcpyDeviceToHost, s));
    else
      FGS_CUDA(cudaMemcpy2DAsync(dst, sizeof(double) * ld, src, sizeof(double) * n, sizeof(double) * n, cnt,
                                 cudaMemcpyDeviceToHost, s));
  };
  const int64_t before = launches;
  FGS_CUDA(cudaStreamBeginCapture(stream, cudaStreamCaptureModeThreadLocal));
  try {
    if (nsub == 1) {
      h2d(0, nvec, stream);
      apply_launches(epilogue, xbuf.p, n, ybuf.p, n, nvec, true, scale_input);
      d2h(0, nvec, stream);
    } else {
      // fork: copy-in stream uploads sub-block k while the compute stream
      // applies sub-block k - 1 and the copy-out stream downloads k - 2
      // (H2D and D2H use separate copy engines; the sub-block applies are
      // the same kernels as one block apply, vectors being independent)
      cudaEvent_t fork = pipe_ev[0];
      FGS_CUDA(cudaEventRecord(fork, stream));
      FGS_CUDA(cudaStreamWaitEvent(cp_in, fork, 0));
      FGS_CUDA(cudaStreamWaitEvent(cp_out, fork, 0));
      for (int k = 0, v0 = 0; k < nsub; v0 += parts[static_cast<size_t>(k)], ++k) {
        const int nb = parts[static_cast<size_t>(k)];
        cudaEvent_t in_done = pipe_ev[static_cast<size_t>(3 + 2 * k)];
        cudaEvent_t ap_done = pipe_ev[static_cast<size_t>(4 + 2 * k)];
        h2d(v0, nb, cp_in);
        FGS_CUDA(cudaEventRecord(in_done, cp_in));
        FGS_CUDA(cudaStreamWaitEvent(stream, in_done, 0));
        apply_launches(epilogue, xbuf.p + static_cast<int64_t>(v0) * n, n, ybuf.p + static_cast<int64_t>(v0) * n, n,
                       nb, true, scale_input);
        FGS_CUDA(cudaEventRecord(ap_done, stream));
        FGS_CUDA(cudaStreamWaitEvent(cp_out, ap_done, 0));
        d2h(v0, nb, cp_out);
      }
      // join both copy streams back into the capture stream
      FGS_CUDA(cudaEventRecord(pipe_ev[1], cp_in));
      FGS_CUDA(cudaEventRecord(pipe_ev[2], cp_out));
      FGS_CUDA(cudaStreamWaitEvent(stream, pipe_ev[1], 0));
      FGS_CUDA(cudaStreamWaitEvent(stream, pipe_ev[2], 0));
    }
  } catch (...) {
    cudaGraph_t broken = nullptr;
    cudaStreamEndCapture(stream, &broken);
    if (broken) cudaGraphDestroy(broken);
    throw;
  }
  cudaGraph_t graph = nullptr;
  FGS_CUDA(cudaStreamEndCapture(stream, &graph));
  cudaGraphExec_t exec = nullptr;
  FGS_CUDA(cudaGraphInstantiate(&exec, graph, 0));
  cudaGraphDestroy(graph);
  if (graphs_.size() >= 8) {
    cudaGraphExecDestroy(graphs_.front().exec);
    graphs_.erase(graphs_.begin());
  }
  graphs_.push_back({key, exec, launches - before});
  launches = before;
  FGS_CUDA(cudaGraphLaunch(exec, stream));
  launches += graphs_.back().launches;
  return true;
}

void Core::pass_layout(PassArgs& a) const {
  if (use_slots) {
    a.items = items6.p;
    a.runs = runs6.p;
    a.slots = slot_map.p;
    a.boff = batch_off.p;
    a.pair_batches = mean_run >= 16.0 ? 1 : 0;
    a.box_ext = box_ext;
  } else {
    a.items = items.p;
    a.runs = runs.p;
    a.slots = nullptr;
  }
}

void Core::apply_launches(int epilogue, const double* x, int64_t ldx, double* y, int64_t ldy, int nvec,
                          bool caller_order, bool scale_input, int phases) {
  // phases: 1 = up to the sharded exchange (spread, assembly, forward
  // convolution part), 2 = after it (rest of the convolution, interpolation),
  // 3 = both with the NCCL exchange between (emulated shard groups run 1 on
  // every shard, sum the exchange buffers on the device, then run 2)
  const bool pre = (phases & 1) != 0, post = (phases & 2) != 0;
  const bool nccl_exchange = sharded && !emulated && pre && post;
  Workspace& w = workspace(nvec);
  if (kind == DIRECT) {
    direct_launches(w, epilogue, x, ldx, y, ldy, nvec, scale_input);
    return;
  }
  PassArgs a{};
  pass_layout(a);
  a.taps = taps.p;
  a.perm = caller_order ? perm.p + offset : nullptr;
  a.point_base = offset;
  a.x = x;
  a.ldx = ldx;
  a.s = inv_sqrt.p;
  a.scale_input = scale_input ? 1 : 0;
  a.nvec = nvec;
  a.M = M;
  a.priv = w.priv.p;
  a.box_stride = box_stride;
  a.grid = w.grid_out.p;  // the interpolation reads the convolved grid
  a.grid_stride = grid_elems;
  a.y = y;
  a.ldy = ldy;
  a.epilogue = epilogue;
  a.k0 = k0;
  a.degrees = degrees.p;
  a.inv_sqrt = inv_sqrt.p;
  a.bad_flag = flag.p;
  a.caller = perm.p + offset;

  // stage events persist across the two phases of a shard-group apply
  std::vector<cudaEvent_t>& evs = prof_evs_;
  if (pre) evs.clear();
  if (profile_ && pre) mark(evs);
  if (pre && use_slots && nitems > 0) {  // the vectors in slot order for the v6 spread (pads 0, s applied)
    const int64_t ns = static_cast<int64_t>(slot_map.n);
    a.xs = w.xs.p;
    a.ldxs = ns;
    launch_ex(slot_gather_kernel, dim3(static_cast<unsigned>(std::min<int64_t>(ceil_div(ns, 256), 148 * 16))),
              dim3(256), 0, stream, a, ns, w.xs.p);
    ++launches;
    FGS_CUDA(cudaGetLastError());
  }
  if (pre) {
    launch_spread(a);
    if (profile_) mark(evs);
    launch_assemble(w, nvec);
    if (profile_) mark(evs);
  }
  if (use_conv2d()) {
    // d = 2: one cluster launch (row FFTs / kept-column FFT + multiply +
    // inverse through DSMEM / inverse row FFTs), conv2d.cuh.  Sharded: the
    // ranks' partial real grids (M^2 doubles) are summed first, then every
    // rank convolves the full grid (the exchange of SURVEY 8e on the grid
    // instead of the spectrum window: one launch instead of four)
    const double* conv_in = w.grid.p;
    if (sharded) {  // out of place: this rank's spread grid keeps its zero cells
      if (nccl_exchange)
        nccl_check(nccl().all_reduce(w.grid.p, w.grid_sum.p, static_cast<size_t>(grid_elems) * nvec, ncclDouble,
                                     ncclSum, comm, stream),
                   "ncclAllReduce of the partial grids");
      conv_in = w.grid_sum.p;
    }
    if (post) {
      int logM = 0;
      while ((1 << logM) < M) ++logM;
      Conv2Args ca{conv_in, w.grid_out.p, mult.p, tw2.p, M, logM, N, nvec, grid_elems};
      const size_t smem = conv2_smem(M, N);
      set_smem(conv2_kernel_ptr(M), smem);
      conv2_launch(ca, smem, stream);
      ++launches;
      FGS_CUDA(cudaGetLastError());
    }
    if (profile_) {
      mark(evs);
      mark(evs);
      mark(evs);
    }
  } else if (use_conv3d()) {
    // d = 3: pruned plane / line / plane passes (conv3d.cuh).  Sharded: this
    // rank's planes only; the window spectra of the ranks are summed between
    // the forward and the inverse line passes
    Conv3Args ca{w.grid.p, w.grid_out.p, w.win.p, sharded ? w.cspec.p : nullptr, mult.p, tw2.p,
                 M, N, nvec, conv_plane0, conv_planes, grid_elems};
    if (pre) {
      conv3_launch(ca, 0, 1, 0, stream);
      ++launches;
      if (profile_) mark(evs);
      conv3_launch(ca, 1, 1, 0, stream);  // sharded: forward line pass into the window spectrum
      ++launches;
    }
    if (sharded) {
      if (nccl_exchange) {
        const int64_t nw = conv3_nw(M, N), H = N / 2 + 1;
        nccl_check(nccl().all_reduce(w.cspec.p, w.cspec.p, static_cast<size_t>(nw * nw * H * nvec * 2), ncclDouble,
                                     ncclSum, comm, stream),
                   "ncclAllReduce of the window spectra");
      }
      if (post) {
        conv3_launch(ca, 1, 1, 1, stream);
        ++launches;
      }
    }
    if (post) {
      if (profile_) mark(evs);
      conv3_launch(ca, 2, 1, 0, stream);
      ++launches;
      FGS_CUDA(cudaGetLastError());
      if (profile_) mark(evs);
    }
  } else {
    if (pre) {
      FGS_CUFFT(cufftExecD2Z(w.r2c, w.grid.p, w.spec.p));
      if (profile_) mark(evs);
      if (!sharded) {
        MultiplyArgs ma{w.spec.p, mult.p, spec_elems, spec_elems, nvec, d, M, N};
        multiply_kernel<<<ceil_div(spec_elems, 256), 256, 0, stream>>>(ma);
        ++launches;
        FGS_CUDA(cudaGetLastError());
      }
    }
    WindowArgs wa{w.spec.p, w.window.p, mult.p, spec_elems, window_elems, window_elems, nvec, d, M, N};
    if (sharded && pre) {
      pack_window_kernel<<<ceil_div(window_elems, 256), 256, 0, stream>>>(wa);
      ++launches;
    }
    if (nccl_exchange)
      nccl_check(nccl().all_reduce(w.window.p, w.window.p, static_cast<size_t>(window_elems) * nvec * 2, ncclDouble,
                                   ncclSum, comm, stream),
                 "ncclAllReduce of the truncated spectrum");
    if (sharded && post) {
      FGS_CUDA(cudaMemsetAsync(w.spec.p, 0, sizeof(cufftDoubleComplex) * spec_elems * nvec, stream));
      unpack_multiply_kernel<<<ceil_div(window_elems, 256), 256, 0, stream>>>(wa);
      ++launches;
      FGS_CUDA(cudaGetLastError());
    }
    if (post) {
      if (profile_) mark(evs);
      FGS_CUFFT(cufftExecZ2D(w.c2r, w.spec.p, w.grid_out.p));
      if (profile_) mark(evs);
    }
  }
  if (!post) return;
  launch_interp(a);
  if (profile_) {
    mark(evs);
    ev_pending_.push_back(evs);
    evs.clear();
  }
}

cudaEvent_t Core::stage_event() {
  if (!ev_pool_.empty()) {
    cudaEvent_t e = ev_pool_.back();
    ev_pool_.pop_back();
    return e;
  }
  cudaEvent_t e;
  FGS_CUDA(cudaEventCreate(&e));
  return e;
}

void Core::mark(std::vector<cudaEvent_t>& evs) {
  cudaEvent_t e = stage_event();
  FGS_CUDA(cudaEventRecord(e, stream));
  evs.push_back(e);
}

void Core::enable_profile(bool on) { profile_ = on; }

void Core::read_profile(double* ms, int64_t* applies) {
  for (int s = 0; s < ST_COUNT; ++s) ms[s] = 0.0;
  FGS_CUDA(cudaStreamSynchronize(stream));
  for (auto& evs : ev_pending_) {
    for (int s = 0; s < ST_COUNT && s + 1 < static_cast<int>(evs.size()); ++s) {
      float t = 0.f;
      FGS_CUDA(cudaEventElapsedTime(&t, evs[static_cast<size_t>(s)], evs[static_cast<size_t>(s) + 1]));
      ms[s] += t;
    }
    for (cudaEvent_t e : evs) ev_pool_.push_back(e);
  }
  if (applies) *applies = static_cast<int64_t>(ev_pending_.size());
  ev_pending_.clear();
}

// d = 2 grids: one-launch cluster convolution instead of cuFFT D2Z +
// multiply + Z2D (FGS_CONV2D=0 selects cuFFT)
bool Core::use_conv2d() const {
  static const bool on = [] {
    const char* e = std::getenv("FGS_CONV2D");
    return !(e && std::string(e) == "0");
  }();
  return on && d == 2 && kind == FASTSUM && conv2_supported(M) &&
         conv2_smem(M, N) <= 200 * 1024 && tw2.p != nullptr;
}

// d = 3 grids: the pruned plane / line / plane convolution (conv3d.cuh)
// instead of cuFFT D2Z + multiply + Z2D (FGS_CONV3D=0 selects cuFFT)
bool Core::use_conv3d() const {
  static const bool on = [] {
    const char* e = std::getenv("FGS_CONV3D");
    return !(e && std::string(e) == "0");
  }();
  return on && d == 3 && kind == FASTSUM && conv3_supported(M) && M > N && conv3_plane_smem(M, N) <= 200 * 1024 &&
         tw2.p != nullptr;
}

void Core::degrees_prepare(DBuf<double>& ones) {
  degrees.alloc(static_cast<size_t>(std::max<int64_t>(n_local, 1)));
  inv_sqrt.alloc(static_cast<size_t>(std::max<int64_t>(n_local, 1)));
  flag.alloc(1);
  ones.alloc(static_cast<size_t>(std::max<int64_t>(n_local, 1)));
  fill_kernel<<<ceil_div(std::max<int64_t>(n_local, 1), 256), 256, 0, stream>>>(ones.p, n_local, 1.0);
  ++launches;
  unsigned long long init = ULLONG_MAX;
  FGS_CUDA(cudaMemcpyAsync(flag.p, &init, sizeof(init), cudaMemcpyHostToDevice, stream));
  FGS_CUDA(cudaStreamSynchronize(stream));  // `init` is a host stack value
}

void Core::degrees_fail(unsigned long long bad, int64_t* bad_node) {
  const int64_t j = static_cast<int64_t>(bad);
  if (bad_node) *bad_node = j;
  double val = std::nan("");
  // locate the value when this shard owns the node
  std::vector<double> hdeg(static_cast<size_t>(n_local));
  FGS_CUDA(cudaMemcpy(hdeg.data(), degrees.p, sizeof(double) * n_local, cudaMemcpyDeviceToHost));
  for (int64_t p = 0; p < n_local; ++p)
    if (host_perm[static_cast<size_t>(offset + p)] == j) val = hdeg[static_cast<size_t>(p)];
  fail(FGS_ENUMERIC, "computed degree of node " + std::to_string(j) + " is not positive (" + std::to_string(val) +
                         "); increase the fast-summation bandwidth/cutoff or widen the kernel");
}

void Core::compute_degrees(int64_t* bad_node) {
  DBuf<double> ones;
  degrees_prepare(ones);
  apply(EPI_DEGREE, ones.p, n_local, nullptr, 0, 1, false, false);
  if (sharded) {
    nccl_check(nccl().all_reduce(flag.p, flag.p, 1, ncclUint64, ncclMin, comm, stream),
               "ncclAllReduce of the degree flag");
  }
  unsigned long long bad = 0;
  FGS_CUDA(cudaMemcpyAsync(&bad, flag.p, sizeof(bad), cudaMemcpyDeviceToHost, stream));
  FGS_CUDA(cudaStreamSynchronize(stream));
  if (bad != ULLONG_MAX) degrees_fail(bad, bad_node);
}

void Core::exchange_buffers(int nvec, double** src, double** dst, size_t* count) {
  Workspace& w = workspace(nvec);
  if (use_conv2d()) {
    *src = w.grid.p;
    *dst = w.grid_sum.p;
    *count = static_cast<size_t>(grid_elems) * nvec;
  } else if (use_conv3d()) {
    const int64_t nw = conv3_nw(M, N), H = N / 2 + 1;
    *src = *dst = reinterpret_cast<double*>(w.cspec.p);
    *count = static_cast<size_t>(nw * nw * H * nvec * 2);
  } else {
    *src = *dst = reinterpret_cast<double*>(w.window.p);
    *count = static_cast<size_t>(window_elems) * nvec * 2;
  }
}

// ---- ShardGroup -------------------------------------------------------------
namespace {
constexpr int kMaxGroup = 16;
struct GroupSum {
  const double* src[kMaxGroup];
  double* dst[kMaxGroup];
  int world;
  int64_t count;
};
// the ranks' allreduce on one device: every shard's buffer <- sum over shards
// (in place safe: element i is read and written by one thread)
__global__ void group_sum_kernel(GroupSum g) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < g.count;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    double v = 0.0;
    for (int r = 0; r < g.world; ++r) v += g.src[r][i];
    for (int r = 0; r < g.world; ++r) g.dst[r][i] = v;
  }
}
__global__ void group_min_kernel(unsigned long long* const* flags, int world) {
  unsigned long long v = ULLONG_MAX;
  for (int r = 0; r < world; ++r) v = min(v, *flags[r]);
  for (int r = 0; r < world; ++r) *flags[r] = v;
}
}  // namespace

ShardGroup::ShardGroup(const double* nodes_colmajor, int64_t n_, int d, const KernelSpec& kernel,
                       const Params& params, int device_, int world, int64_t* bad_node)
    : device(device_), n(n_) {
  if (world < 1 || world > kMaxGroup) fail(FGS_EPARAM, "shard group world must be in [1, 16]");
  FGS_CUDA(cudaSetDevice(device));
  FGS_CUDA(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
  for (int r = 0; r < world; ++r) {
    shards.push_back(std::make_unique<Core>(nodes_colmajor, n, d, Core::FASTSUM, kernel, params, device, r, world));
    shards.back()->sharded = true;
    shards.back()->emulated = true;
    shards.back()->set_stream(stream);
  }
  // degrees: one group apply of the ones vectors (internal order per shard)
  std::vector<DBuf<double>> ones(static_cast<size_t>(world));
  std::vector<const double*> xs;
  std::vector<double*> ys;
  std::vector<int64_t> lds;
  for (int r = 0; r < world; ++r) {
    shards[static_cast<size_t>(r)]->degrees_prepare(ones[static_cast<size_t>(r)]);
    xs.push_back(ones[static_cast<size_t>(r)].p);
    ys.push_back(nullptr);
    lds.push_back(shards[static_cast<size_t>(r)]->n_local);
  }
  run(EPI_DEGREE, xs, lds, ys, lds, 1, false, false);
  DBuf<unsigned long long*> fl;
  std::vector<unsigned long long*> hf;
  for (auto& c : shards) hf.push_back(c->flag.p);
  fl.upload(hf.data(), hf.size(), stream);
  group_min_kernel<<<1, 1, 0, stream>>>(fl.p, world);
  FGS_CUDA(cudaGetLastError());
  unsigned long long bad = 0;
  FGS_CUDA(cudaMemcpyAsync(&bad, hf[0], sizeof(bad), cudaMemcpyDeviceToHost, stream));
  FGS_CUDA(cudaStreamSynchronize(stream));
  if (bad != ULLONG_MAX) {
    for (auto& c : shards) {  // the shard owning the node reports its value
      for (int64_t p = 0; p < c->n_local; ++p)
        if (c->host_perm[static_cast<size_t>(c->offset + p)] == static_cast<int>(bad)) c->degrees_fail(bad, bad_node);
    }
    shards[0]->degrees_fail(bad, bad_node);
  }
}

ShardGroup::~ShardGroup() {
  if (stream) cudaStreamSynchronize(stream);
  shards.clear();
  if (stream) cudaStreamDestroy(stream);
}

void ShardGroup::run(int epilogue, const std::vector<const double*>& x, const std::vector<int64_t>& ldx,
                     const std::vector<double*>& y, const std::vector<int64_t>& ldy, int nvec, bool caller_order,
                     bool scale_input, std::vector<cudaEvent_t>* ev) {
  const int world = static_cast<int>(shards.size());
  // ev (profiling): [2 world + 2] events, shard r phase 1 between ev[r] and
  // ev[r + 1], the exchange between ev[world] and ev[world + 1], shard r
  // phase 2 between ev[world + 1 + r] and ev[world + 2 + r]
  auto mark = [&](int i) {
    if (ev) FGS_CUDA(cudaEventRecord((*ev)[static_cast<size_t>(i)], stream));
  };
  mark(0);
  for (int r = 0; r < world; ++r) {
    shards[static_cast<size_t>(r)]->apply_launches(epilogue, x[static_cast<size_t>(r)], ldx[static_cast<size_t>(r)],
                                                   y[static_cast<size_t>(r)], ldy[static_cast<size_t>(r)], nvec,
                                                   caller_order, scale_input, 1);
    mark(r + 1);
  }
  GroupSum g{};
  g.world = world;
  for (int r = 0; r < world; ++r) {
    double *src = nullptr, *dst = nullptr;
    size_t count = 0;
    shards[static_cast<size_t>(r)]->exchange_buffers(nvec, &src, &dst, &count);
    g.src[r] = src;
    g.dst[r] = dst;
    g.count = static_cast<int64_t>(count);
  }
  group_sum_kernel<<<static_cast<unsigned>(std::min<int64_t>((g.count + 255) / 256, 148 * 8)), 256, 0, stream>>>(g);
  FGS_CUDA(cudaGetLastError());
  mark(world + 1);
  for (int r = 0; r < world; ++r) {
    shards[static_cast<size_t>(r)]->apply_launches(epilogue, x[static_cast<size_t>(r)], ldx[static_cast<size_t>(r)],
                                                   y[static_cast<size_t>(r)], ldy[static_cast<size_t>(r)], nvec,
                                                   caller_order, scale_input, 2);
    mark(world + 2 + r);
  }
}

void ShardGroup::profile(int epilogue, const double* x, double* y, int64_t ld, int nvec, bool scale_input, int reps,
                         double* shard_ms, double* exchange_ms) {
  const size_t world = shards.size();
  std::vector<cudaEvent_t> ev(2 * world + 2);
  for (auto& e : ev) FGS_CUDA(cudaEventCreate(&e));
  for (size_t r = 0; r < world; ++r) shard_ms[r] = 0.0;
  *exchange_ms = 0.0;
  for (int it = 0; it < reps; ++it) {
    run(epilogue, std::vector<const double*>(world, x), std::vector<int64_t>(world, ld),
        std::vector<double*>(world, y), std::vector<int64_t>(world, ld), nvec, true, scale_input, &ev);
    FGS_CUDA(cudaStreamSynchronize(stream));
    float t = 0.f;
    for (size_t r = 0; r < world; ++r) {
      FGS_CUDA(cudaEventElapsedTime(&t, ev[r], ev[r + 1]));
      shard_ms[r] += t / reps;
      FGS_CUDA(cudaEventElapsedTime(&t, ev[world + 1 + r], ev[world + 2 + r]));
      shard_ms[r] += t / reps;
    }
    FGS_CUDA(cudaEventElapsedTime(&t, ev[world], ev[world + 1]));
    *exchange_ms += t / reps;
  }
  for (auto& e : ev) cudaEventDestroy(e);
}

void ShardGroup::apply(int epilogue, const double* x, double* y, int64_t ld, int nvec, bool scale_input) {
  const size_t world = shards.size();
  run(epilogue, std::vector<const double*>(world, x), std::vector<int64_t>(world, ld), std::vector<double*>(world, y),
      std::vector<int64_t>(world, ld), nvec, true, scale_input);
}

void Core::nfft_adjoint(const double* x_planar, double* fhat_out) {
  // x_planar: device [2][n] (re, im) in caller order; fhat_out: device interleaved N^d
  Workspace& w = workspace(2);
  PassArgs a{};
  pass_layout(a);
  a.taps = taps.p;
  a.perm = perm.p + offset;
  a.x = x_planar;
  a.ldx = n;
  a.nvec = 2;
  a.M = M;
  a.priv = w.priv.p;
  a.box_stride = box_stride;
  launch_spread(a);
  launch_assemble(w, 2);
  w.cgrid.alloc(static_cast<size_t>(grid_elems));
  merge_complex_kernel<<<ceil_div(grid_elems, 256), 256, 0, stream>>>(w.grid.p, w.grid.p + grid_elems, w.cgrid.p,
                                                                      grid_elems);
  ++launches;
  if (!w.has_z2z) {
    int dims[3] = {M, M, M};
    FGS_CUFFT(cufftPlanMany(&w.z2z, d, dims, nullptr, 1, 0, nullptr, 1, 0, CUFFT_Z2Z, 1));
    FGS_CUFFT(cufftSetStream(w.z2z, stream));
    w.has_z2z = true;
  }
  FGS_CUFFT(cufftExecZ2Z(w.z2z, w.cgrid.p, w.cgrid.p, CUFFT_FORWARD));
  int64_t F = 1;
  for (int t = 0; t < d; ++t) F *= N;
  extract_kernel<<<ceil_div(F, 256), 256, 0, stream>>>(w.cgrid.p, reinterpret_cast<cufftDoubleComplex*>(fhat_out), F,
                                                        d, N, M, deconv_d.p);
  ++launches;
  FGS_CUDA(cudaGetLastError());
}

void Core::nfft_forward(const double* fhat_in, double* y_planar) {
  Workspace& w = workspace(2);
  w.cgrid.alloc(static_cast<size_t>(grid_elems));
  FGS_CUDA(cudaMemsetAsync(w.cgrid.p, 0, sizeof(cufftDoubleComplex) * grid_elems, stream));
  int64_t F = 1;
  for (int t = 0; t < d; ++t) F *= N;
  place_kernel<<<ceil_div(F, 256), 256, 0, stream>>>(reinterpret_cast<const cufftDoubleComplex*>(fhat_in), w.cgrid.p,
                                                      F, d, N, M, deconv_d.p);
  ++launches;
  if (!w.has_z2z) {
    int dims[3] = {M, M, M};
    FGS_CUFFT(cufftPlanMany(&w.z2z, d, dims, nullptr, 1, 0, nullptr, 1, 0, CUFFT_Z2Z, 1));
    FGS_CUFFT(cufftSetStream(w.z2z, stream));
    w.has_z2z = true;
  }
  FGS_CUFFT(cufftExecZ2Z(w.z2z, w.cgrid.p, w.cgrid.p, CUFFT_INVERSE));
  split_complex_kernel<<<ceil_div(grid_elems, 256), 256, 0, stream>>>(w.cgrid.p, w.grid_out.p,
                                                                      w.grid_out.p + grid_elems, grid_elems);
  ++launches;
  PassArgs a{};
  pass_layout(a);
  a.taps = taps.p;
  a.perm = perm.p + offset;
  a.x = nullptr;
  a.nvec = 2;
  a.M = M;
  a.grid = w.grid_out.p;
  a.grid_stride = grid_elems;
  a.y = y_planar;
  a.ldy = n;
  a.epilogue = EPI_KERNEL;
  launch_interp(a);
}

void Core::permute(const double* x, int64_t ldx, double* y, int64_t ldy, int nvec, int direction) {
  permute_kernel<<<ceil_div(std::max<int64_t>(n_local, 1), 256), 256, 0, stream>>>(x, ldx, y, ldy, perm.p + offset,
                                                                                  n_local, nvec, direction);
  ++launches;
  FGS_CUDA(cudaGetLastError());
}

double Core::error_estimate(int samples, uint64_t seed) const {
  // kernel_error_estimate (fastsum.cpp:120-124) = |out_factor| *
  // kernel_approx_error (kernels.cpp:369-396): sampled sup over the ball
  if (samples < 1) fail(FGS_EPARAM, "sample count must be positive");
  const double radius = 0.5 - params.eps_b;
  std::mt19937_64 rng(seed);
  std::normal_distribution<double> gauss;
  std::uniform_real_distribution<double> unif(0.0, 1.0);
  double worst = 0.0;
  std::vector<std::complex<double>> ph(static_cast<size_t>(d) * N);
  for (int s = 0; s < samples; ++s) {
    double y[3] = {0, 0, 0}, n2 = 0.0;
    for (int t = 0; t < d; ++t) {
      y[t] = gauss(rng);
      n2 += y[t] * y[t];
    }
    const double len = std::sqrt(n2);
    const double r = radius * std::pow(unif(rng), 1.0 / d);
    for (int t = 0; t < d; ++t) y[t] = len > 0.0 ? y[t] * (r / len) : 0.0;
    double yn = 0.0;
    for (int t = 0; t < d; ++t) yn += y[t] * y[t];
    for (int t = 0; t < d; ++t)
      for (int a = 0; a < N; ++a)
        ph[static_cast<size_t>(t) * N + a] = std::polar(1.0, 2.0 * kPi * (a - N / 2) * y[t]);
    std::complex<double> acc = 0.0;
    size_t flat = 0;
    if (d == 1) {
      for (int a = 0; a < N; ++a, ++flat) acc += bhat[flat] * ph[static_cast<size_t>(a)];
    } else if (d == 2) {
      for (int a = 0; a < N; ++a)
        for (int c = 0; c < N; ++c, ++flat) acc += bhat[flat] * (ph[static_cast<size_t>(a)] * ph[static_cast<size_t>(N + c)]);
    } else {
      for (int a = 0; a < N; ++a)
        for (int c = 0; c < N; ++c) {
          const std::complex<double> pac = ph[static_cast<size_t>(a)] * ph[static_cast<size_t>(N + c)];
          for (int e = 0; e < N; ++e, ++flat) acc += bhat[flat] * (pac * ph[static_cast<size_t>(2 * N + e)]);
        }
    }
    worst = std::max(worst, std::abs(kernel_value(scaled, std::sqrt(yn)) - acc.real()));
  }
  return std::abs(out_factor) * worst;
}

// ---- direct backend (exact O(n^2) sums) ------------------------------------
int Core::direct_segments() const {
  // enough CTAs to fill the device (~8 per SM) without tiny segments
  const int64_t tiles = ceil_div(n, static_cast<int64_t>(kDirectThreads));
  const int64_t want = ceil_div(static_cast<int64_t>(148 * 8), tiles);
  const int64_t most = ceil_div(n, static_cast<int64_t>(kDirectTile));
  return static_cast<int>(std::max<int64_t>(1, std::min(want, most)));
}

void Core::direct_launches(Workspace& w, int epilogue, const double* x, int64_t ldx, double* y, int64_t ldy, int nvec,
                           bool scale_input) {
  const int nseg = direct_segments();
  DirectArgs da{};
  da.nodes = nodes_d.p;
  da.n = n;
  da.d = d;
  da.family = kernel.family;
  da.shape = kernel.shape;
  da.x = x;
  da.ldx = ldx;
  da.s = inv_sqrt.p;
  da.scale_input = scale_input ? 1 : 0;
  da.seg_len = ceil_div(n, static_cast<int64_t>(nseg));
  da.nseg = nseg;
  da.partial = w.priv.p;
  da.nvec = nvec;
  const dim3 grid(static_cast<unsigned>(ceil_div(n, static_cast<int64_t>(kDirectThreads))), static_cast<unsigned>(nseg));
  for (int v0 = 0; v0 < nvec; v0 += kDirectVec) {
    da.vec0 = v0;
    da.nv = std::min(kDirectVec, nvec - v0);
    launch_ex(direct_partial_kernel, grid, kDirectThreads, 0, stream, da);
    ++launches;
  }
  DirectFinishArgs fa{};
  fa.partial = w.priv.p;
  fa.nseg = nseg;
  fa.nvec = nvec;
  fa.n = n;
  fa.pa.perm = nullptr;
  fa.pa.x = x;
  fa.pa.ldx = ldx;
  fa.pa.s = inv_sqrt.p;
  fa.pa.y = y;
  fa.pa.ldy = ldy;
  fa.pa.epilogue = epilogue;
  fa.pa.k0 = k0;
  fa.pa.degrees = degrees.p;
  fa.pa.inv_sqrt = inv_sqrt.p;
  fa.pa.bad_flag = flag.p;
  fa.pa.caller = perm.p;
  launch_ex(direct_finish_kernel, dim3(static_cast<unsigned>(ceil_div(n, static_cast<int64_t>(256)))), 256, 0, stream,
            fa);
  ++launches;
  FGS_CUDA(cudaGetLastError());
}

}  // namespace fgsb
