// common.cuh -- error plumbing, plan geometry and device-side PODs shared by
// the B200 fast-summation kernels (paper_1808_04580_b200/csrc).
#pragma once

#include <cstdlib>

#include <cuda_runtime.h>
#include <cufft.h>

#include <cstdint>
#include <stdexcept>
#include <string>

#include "fgs_b200.h"

namespace fgsb {

// Typed failure carrying an fgs_status; the C ABI converts it to a return
// code + fgs_last_error() message, the C++ drop-in layer rethrows the
// matching reference exception class (errors.hpp:8-49).
struct Error : std::runtime_error {
  fgs_status code;
  Error(fgs_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void fail(fgs_status code, const std::string& msg) { throw Error(code, msg); }

#define FGS_CUDA(call)                                                                    \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess)                                                                \
      ::fgsb::fail(e_ == cudaErrorMemoryAllocation ? FGS_ERESOURCE : FGS_ECUDA,            \
                   std::string(#call) + ": " + cudaGetErrorString(e_) + " (" + __FILE__ +  \
                       ":" + std::to_string(__LINE__) + ")");                             \
  } while (0)

#define FGS_CUFFT(call)                                                              \
  do {                                                                               \
    cufftResult r_ = (call);                                                         \
    if (r_ != CUFFT_SUCCESS)                                                         \
      ::fgsb::fail(FGS_ECUDA, std::string(#call) + ": cufft error " +               \
                                  std::to_string(static_cast<int>(r_)) + " (" + __FILE__ + \
                                  ":" + std::to_string(__LINE__) + ")");             \
  } while (0)

// Programmatic dependent launch: the hot kernels of an apply (spread,
// assemble, d=2 convolution, interp) start with pdl_wait() -- which blocks
// until the preceding grid in the stream has completed and its writes are
// visible -- and then allow their own successor to be scheduled, so each
// kernel's CTAs are resident and waiting when its predecessor drains
// instead of paying the launch gap.  A no-op when launched without the
// attribute.  FGS_PDL selects the mode (see pdl_mode).
// (An explicit early trigger -- launch_dependents right after the wait --
// parked the successor's CTAs on the SMs the predecessor still needed and
// measured slower; it also cost every kernel a global flag load.)
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }

// FGS_PDL: 0 off, otherwise (default 2) PDL launches with the implicit
// trigger at grid end (validated with FGS_POISON=1 over the GPU suite).
inline int pdl_mode() {
  static const int mode = [] {
    const char* e = std::getenv("FGS_PDL");
    return e ? std::atoi(e) : 2;
  }();
  return mode;
}
inline bool pdl_on() { return pdl_mode() != 0; }

template <class... KP, class... Args>
inline void launch_ex(void (*k)(KP...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = (pdl_on() && s != nullptr) ? 1 : 0;
  FGS_CUDA(cudaLaunchKernelEx(&cfg, k, static_cast<KP>(args)...));
}

// One work item = one CTA of the spread / interp kernels: a run list of
// point cells inside one spatial tile, with the bounding box of the union of
// their (2m)^d window footprints.  `a` is the wrapped grid origin of that
// box, `ext` its extent per dimension (<= B + 2m - 1).
struct DItem {
  int run_begin, run_end;
  int a0, a1, a2;
  int e0, e1, e2;
  int p_begin, p_end;  // the item's points [p_begin, p_end) (first tap prefetch needs no run load)
};

// A run = consecutive points (in the internal order) that share the same
// first window tap u0 = ceil(v M - m) in every dimension, i.e. the same
// footprint.  `off` packs the footprint origin relative to the item box,
// 10 bits per dimension.
struct DRun {
  int pstart, pcount, off;
};

// Epilogue selector of the interpolation kernel (graphop.cpp:87-103).
enum Epilogue : int {
  EPI_KERNEL = 0,     // y = W~ x                                  apply_kernel
  EPI_WEIGHT = 1,     // y = W~ x - K0 x                           apply_weight
  EPI_NORMALIZED = 2, // y = s (W~ (s x) - K0 s x)                 apply_normalized
  EPI_LAPLACIAN = 3,  // y = x - s (W~ (s x) - K0 s x)             apply_sym_laplacian
  EPI_DEGREE = 4      // d = W~ 1 - K0;  s = d^-1/2; flag d <= 0    AdjacencyOperator ctor
};

// Arguments shared by spread and interp launches.
struct PassArgs {
  const DItem* items;
  const DRun* runs;
  const double* taps;    // [n_local][D][T] internal order
  const int* perm;       // internal -> caller index (nullable: vectors already internal)
  int64_t point_base;    // first internal index owned by this shard (perm offset)
  const double* x;       // input vectors, column j at x + j*ldx
  int64_t ldx;
  const double* s;       // D^-1/2 in internal order (nullable)
  int scale_input;       // multiply x by s before spreading
  int nvec;
  int M;
  double* priv;          // spread: per-item private boxes, item k at priv + k*box_stride
  int64_t box_stride;    // doubles per item box per vector
  const double* grid;    // interp: real grid(s), vector j at grid + j*grid_stride
  int64_t grid_stride;
  double* y;             // interp output
  int64_t ldy;
  int epilogue;
  double k0;
  double* degrees;       // EPI_DEGREE outputs (internal order)
  double* inv_sqrt;
  unsigned long long* bad_flag;  // EPI_DEGREE: min caller index with d <= 0
  const int* caller;   // internal -> caller index of this shard's slice (always set)
  const int* slots;    // v6 kernels: slot -> local internal point (-1: pad); items / runs in slots
  const int* boff;     // v6 interp: packed footprint offset of each 8-slot batch's run
  int pair_batches;    // slot layout, 2m = 16: runs long enough for interp_v7's batch pairs
  const double* xs;    // v6 spread: the vectors gathered into slot order (pads 0, s applied)
  int64_t ldxs;
  int box_ext;         // slot-layout interpolation: fixed box extent (tile B + 2m - 1), 0 = per-item strides
  int vsplit;          // slot-layout kernels: CTAs per item, each a share of the block's vectors (0/1: one)
};

// Vector split of the slot-layout kernels.  A block of nvec vectors re-reads
// every item's taps once per vector; with `vsplit` CTAs per item (consecutive
// block indices, so they are resident at the same time) each CTA takes a
// share of the vectors and the CTAs of one item stream the same taps rows
// within microseconds of one another: all but the first read hit L2 instead
// of HBM.  Narrows `a` to this CTA's vectors; returns (item, number of items).
struct ItemOfBlock {
  int item, nitems;
};
__device__ __forceinline__ ItemOfBlock vsplit_narrow(PassArgs& a) {
  const int vs = a.vsplit > 1 ? a.vsplit : 1;
  ItemOfBlock r{static_cast<int>(blockIdx.x) / vs, static_cast<int>(gridDim.x) / vs};
  if (vs > 1) {
    const int part = static_cast<int>(blockIdx.x) - r.item * vs;
    const int vper = (a.nvec + vs - 1) / vs;
    const int v0 = min(part * vper, a.nvec), v1 = min(v0 + vper, a.nvec);
    if (a.x) a.x += v0 * a.ldx;
    if (a.xs) a.xs += v0 * a.ldxs;
    if (a.y) a.y += v0 * a.ldy;
    if (a.grid) a.grid += v0 * a.grid_stride;
    if (a.priv) a.priv += static_cast<int64_t>(v0) * r.nitems * a.box_stride;
    a.nvec = v1 - v0;
  }
  return r;
}

}  // namespace fgsb
