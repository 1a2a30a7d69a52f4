// core.cuh -- device-resident plan of the fast summation (the state behind
// fgs::NfftPlan / FastsumPlan / AdjacencyOperator on one GPU or one shard).
#pragma once

#include <nccl.h>

#include <complex>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "common.cuh"
#include "hostmath.hpp"

namespace fgsb {

struct Params {
  int N = 32, m = 4, p = 4;
  double eps_b = 0.0, oversampling = 2.0;
};

// FGS_POISON=1: fill every new device buffer with 0xff bytes (NaN) -- a
// debugging aid that turns reads of never-written memory into NaNs.
inline bool poison_allocations() {
  static const bool on = [] {
    const char* e = std::getenv("FGS_POISON");
    return e && std::string(e) == "1";
  }();
  return on;
}

// RAII device buffer
template <class T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
  DBuf() = default;
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept : p(o.p), n(o.n) {
    o.p = nullptr;
    o.n = 0;
  }
  DBuf& operator=(DBuf&& o) noexcept {
    if (this != &o) {
      reset();
      p = o.p;
      n = o.n;
      o.p = nullptr;
      o.n = 0;
    }
    return *this;
  }
  ~DBuf() { reset(); }
  void reset() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  void alloc(size_t count) {
    if (count <= n && p) return;
    reset();
    if (count == 0) return;
    FGS_CUDA(cudaMalloc(&p, count * sizeof(T)));
    n = count;
    if (poison_allocations()) {  // NaN bytes: exposes reads of unwritten memory
      FGS_CUDA(cudaMemset(p, 0xff, count * sizeof(T)));
      FGS_CUDA(cudaDeviceSynchronize());  // legacy-stream memset vs the non-blocking handle streams
    }
  }
  void upload(const T* h, size_t count, cudaStream_t s) {
    alloc(count);
    if (count) FGS_CUDA(cudaMemcpyAsync(p, h, count * sizeof(T), cudaMemcpyHostToDevice, s));
  }
};

struct Workspace {
  int nvec = 0;
  // grid: the assembled spread (zeroed once; cells outside the plan's
  // footprint are never written); grid_out: the convolved grid the
  // interpolation reads; grid_sum: d = 2 sharded, the ranks' summed grids
  DBuf<double> priv, grid, grid_out, grid_sum;
  DBuf<cufftDoubleComplex> spec, cgrid, window;
  DBuf<double2> win, cspec;  // d = 3 pruned convolution: plane-pass window, sharded window spectrum
  DBuf<double> xs;           // slot layout: the block's vectors gathered into slot order
  cufftHandle r2c = 0, c2r = 0, z2z = 0;
  bool has_plans = false, has_z2z = false;
};

class Core {
 public:
  enum Kind { NFFT = 0, FASTSUM = 1, DIRECT = 2 };  // DIRECT: exact O(n^2) operator (AdjacencyBackend::Direct)

  Core(const double* nodes_colmajor, int64_t n, int d, Kind kind, const KernelSpec& kernel,
       const Params& params, int device, int rank = 0, int world = 1, const void* nccl_id = nullptr);
  ~Core();
  Core(const Core&) = delete;
  Core& operator=(const Core&) = delete;

  // geometry / plan scalars
  Kind kind;
  int d = 0, N = 0, m = 0, T = 0, M = 0, B = 0, nt = 0, ntiles = 0;
  int rot0 = 0;  // dim-0 tile rotation of the cell keys (sharded plans)
  int64_t n = 0, n_local = 0, offset = 0;
  int rank = 0, world = 1;
  double b_kb = 0.0;
  KernelSpec kernel, scaled;
  Params params;
  double rho = 1.0, out_factor = 1.0, k0 = 0.0;
  RegKernel reg;
  std::vector<std::complex<double>> bhat;  // N^d, FrequencyIndexSet order
  std::vector<double> deconv;              // N
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = true;
  ncclComm_t comm = nullptr;
  bool sharded = false;  // created through fgs_adjacency_create_sharded (owns an NCCL communicator)
  bool emulated = false; // a shard of a ShardGroup: sharded data path, exchange done by the group
  int64_t launches = 0;
  double lanczos_stats[4] = {0, 0, 0, 0};  // last run: apply ms, reorth ms, loop wall ms, iterations

  // device plan
  DBuf<int> perm;  // internal -> caller, all n points (identical on every rank)
  DBuf<double> taps;  // [n_local][d][T]
  DBuf<DItem> items;
  DBuf<DRun> runs;
  // run-aligned slot layout of the d = 3, 2m = 16 tensor kernels
  // (kernels_v6.cuh): items / runs in slot coordinates and slot -> local
  // internal point (-1: pad slot); empty when the plan does not use it
  DBuf<DItem> items6;
  DBuf<DRun> runs6;
  DBuf<int> slot_map;
  DBuf<int> batch_off;  // per 8-slot batch: its run's packed footprint offset
  std::vector<int> slot_host;  // plan-time copy (freed once the taps are built)
  bool use_slots = false;
  void pass_layout(PassArgs& a) const;
  DBuf<int> asm_ptr, asm_idx;  // grid cell -> private-box entries (CSR, item order)
  DBuf<int> asm_cells;  // nonempty cells by list-length class: > 64 | 9..64 | <= 8 entries
  int64_t asm_class_n[3] = {0, 0, 0};
  DBuf<cufftDoubleComplex> mult;  // compact Hermitian multiplier (FASTSUM)
  DBuf<double> deconv_d;
  DBuf<double2> tw2;  // d = 2 pruned-convolution twiddles
  DBuf<double> nodes_d;  // DIRECT: raw nodes [d][n], caller order
  bool use_conv2d() const;
  bool use_conv3d() const;
  // d = 3 convolution planes of this rank: [conv_plane0, conv_plane0 + conv_planes)
  // (all M unsharded; sharded: the dim-0 planes its items' boxes cover)
  int conv_plane0 = 0, conv_planes = 0;
  int nitems = 0;
  double mean_run = 0.0;  // points per run (cell piece) of this shard: picks the spread kernel
  bool tensor_spread() const;  // the DMMA spread runs (dense runs, 2m in {8, 12, 16}, d in {2, 3})
  bool tensor_interp() const;
  int64_t box_stride = 0;
  int box_ext = 0;      // slot layout: fixed interpolation box extent (tile B + 2m - 1), 0 = per-item
  int64_t box_pad = 0;  // largest item box with rows padded for the d = 3 interpolation (kernels_v5.cuh)
  int64_t grid_elems = 0, spec_elems = 0, window_elems = 0;
  std::vector<int> host_perm;

  // graph-operator state (AdjacencyOperator)
  DBuf<double> degrees, inv_sqrt;  // internal order, local slice
  DBuf<unsigned long long> flag;

  // staging buffers for host-vector calls
  DBuf<double> xbuf, ybuf;
  // host-vector graphs of multi-vector blocks: copy-in / copy-out streams
  // forked from `stream` inside the capture, and the capture's events
  cudaStream_t cp_in = nullptr, cp_out = nullptr;
  std::vector<cudaEvent_t> pipe_ev;
  // Lanczos workspace, reused across solves (lanczos.cu)
  DBuf<double> lz_basis, lz_z, lz_partial, lz_partial3, lz_hbuf, lz_scal, lz_qin;
  DBuf<double> lz_alpha, lz_nrm, lz_beta, lz_st;  // run-ahead recurrence scalars
  std::vector<cudaEvent_t> lz_events;              // per-step timing events
  char* bounce = nullptr;  // pinned staging for host_copy (bounce_threads x kBounceChunk)
  int bounce_threads = 0;
  DBuf<unsigned> lz_ticket;
  // Ritz-vector buffers kept between solves (cudaMalloc/cudaFree per solve
  // cost ~6 ms of a 10 ms C2 solve: every free synchronises the device)
  DBuf<double> lz_vecs, lz_vc, lz_S, lz_pval, lz_psigned;
  DBuf<int64_t> lz_pidx;
  DBuf<int> lz_order;                        // last-block reduction tickets (reset by their kernels)
  // start vector drawn on the device: mt19937_64 seed state, caller-order
  // uniforms, sum-of-squares partials
  DBuf<unsigned long long> lz_mt;
  DBuf<double> lz_start, lz_sq;

  void set_stream(cudaStream_t s);
  Workspace& workspace(int nvec);

  // y = op(x) for the fast-summation pipeline.  x, y device pointers; when
  // `caller_order` the vectors are full-length in caller order (perm
  // indexing), else local-slice internal order.
  void apply(int epilogue, const double* x, int64_t ldx, double* y, int64_t ldy, int nvec,
             bool caller_order, bool scale_input);
  // y_host = op(x_host) as ONE graph (H2D into xbuf, the apply, D2H from
  // ybuf) when both host buffers are pinned; false -> caller stages itself.
  // Blocks of several vectors are cut into sub-blocks whose copies overlap
  // the other sub-blocks' applies (pipe_blocks).  Does not synchronise.
  bool apply_host_graph(int epilogue, const double* hx, double* hy, int64_t ld, int nvec, bool scale_input);
  // Contiguous host <-> device copy ordered after the work queued on
  // `stream`; returns when the data has landed.  Large copies to or from
  // pageable memory go through per-thread pinned bounce buffers so the host
  // side (memcpy and first-touch page faults, the bound for fresh output
  // arrays) runs on several cores while the copy engine streams.
  void host_copy(bool to_device, void* dst, const void* src, size_t bytes);
  void compute_degrees(int64_t* bad_node);
  // the launch sequence of one apply; phases 1 / 2 split it at the sharded
  // exchange (ShardGroup), 3 = whole apply (NCCL exchange when sharded)
  void apply_launches(int epilogue, const double* x, int64_t ldx, double* y, int64_t ldy, int nvec,
                      bool caller_order, bool scale_input, int phases = 3);
  // device buffer a sharded apply exchanges between its phases, and the
  // buffer the summed exchange lands in (== src except d = 2: grid_sum)
  void exchange_buffers(int nvec, double** src, double** dst, size_t* count);
  // degree pass split for ShardGroup: prepare (ones, flag), check the flag
  void degrees_prepare(DBuf<double>& ones);
  void degrees_fail(unsigned long long bad, int64_t* bad_node);

  // complex NFFT transforms (NfftPlan), interleaved complex on device
  void nfft_adjoint(const double* x_re_im_planar, double* fhat_interleaved);
  void nfft_forward(const double* fhat_interleaved, double* y_planar);

  // permutation helpers (caller <-> internal), full length
  void permute(const double* x, int64_t ldx, double* y, int64_t ldy, int nvec, int direction);

  double error_estimate(int samples, uint64_t seed) const;

  // stage profiling: when enabled, apply() records CUDA events on the
  // handle's stream at every stage boundary; read_profile() syncs and
  // returns the summed milliseconds per stage since the last read.
  enum Stage { ST_SPREAD = 0, ST_ASSEMBLE, ST_R2C, ST_MULTIPLY, ST_C2R, ST_INTERP, ST_COUNT };
  void enable_profile(bool on);
  void read_profile(double* ms, int64_t* applies);

 private:
  std::map<int, std::unique_ptr<Workspace>> ws_;
  struct GraphKey {
    int epi;
    const double* x;
    int64_t ldx;
    double* y;
    int64_t ldy;
    int nvec;
    bool caller_order, scale;
    const double* hx = nullptr;  // host-vector graphs: pinned x / y with their leading dimension
    double* hy = nullptr;
    int64_t hld = 0;
    bool operator==(const GraphKey& o) const {
      return epi == o.epi && x == o.x && ldx == o.ldx && y == o.y && ldy == o.ldy && nvec == o.nvec &&
             caller_order == o.caller_order && scale == o.scale && hx == o.hx && hy == o.hy && hld == o.hld;
    }
  };
  struct GraphEntry {
    GraphKey key;
    cudaGraphExec_t exec;
    int64_t launches;
  };
  std::vector<GraphEntry> graphs_;
  bool profile_ = false;
  std::vector<cudaEvent_t> ev_pool_;
  std::vector<std::vector<cudaEvent_t>> ev_pending_;
  std::vector<cudaEvent_t> prof_evs_;  // the apply in flight (phase 1 -> phase 2)
  cudaEvent_t stage_event();
  void mark(std::vector<cudaEvent_t>& evs);
  void build_plan(const double* nodes_colmajor);
  void build_coefficients();
  void launch_spread(const PassArgs& a);
  void launch_interp(const PassArgs& a);
  void launch_assemble(Workspace& w, int nvec);
  int direct_segments() const;
  void direct_launches(Workspace& w, int epilogue, const double* x, int64_t ldx, double* y, int64_t ldy, int nvec,
                       bool scale_input);
  size_t smem_bytes(bool interp) const;
  int threads() const;
};

// FastsumParams validation (fastsum.cpp:25-36)
void validate_params(const Params& p);

// fp64 FMA peak of a device in TFLOP/s (peak.cu)
double measure_fp64_peak(int device);
double measure_dmma_peak(int device);

// Single-GPU emulation of the N-rank sharded path (validation of the
// multi-GPU data path on one device): `world` shards (Core rank r of world
// W: the same plan slices, slab-pruned convolutions and exchange buffers as
// the NCCL ranks) on one device and stream.  An apply runs phase 1 on every
// shard, sums the shards' exchange buffers with one device kernel (what
// ncclAllReduce computes across the ranks), then phase 2 on every shard.
// Ranks that wait on one another are never separate launches on one GPU
// (B200_PROFILING.md): the exchange is a plain kernel between the phases.
class ShardGroup {
 public:
  ShardGroup(const double* nodes_colmajor, int64_t n, int d, const KernelSpec& kernel, const Params& params,
             int device, int world, int64_t* bad_node);
  ~ShardGroup();
  ShardGroup(const ShardGroup&) = delete;
  ShardGroup& operator=(const ShardGroup&) = delete;
  // y = op(x) for full-length device vectors in caller order (column j at x + j ld)
  void apply(int epilogue, const double* x, double* y, int64_t ld, int nvec, bool scale_input);
  // `reps` applies with CUDA events around every shard's two phases and the
  // exchange: mean ms per apply of each shard (phase 1 + phase 2: what rank r
  // computes on its own GPU) and of the device-sum exchange
  void profile(int epilogue, const double* x, double* y, int64_t ld, int nvec, bool scale_input, int reps,
               double* shard_ms, double* exchange_ms);
  std::vector<std::unique_ptr<Core>> shards;
  cudaStream_t stream = nullptr;
  int device = 0;
  int64_t n = 0;

 private:
  void run(int epilogue, const std::vector<const double*>& x, const std::vector<int64_t>& ldx,
           const std::vector<double*>& y, const std::vector<int64_t>& ldy, int nvec, bool caller_order,
           bool scale_input, std::vector<cudaEvent_t>* ev = nullptr);
};

}  // namespace fgsb
