// capi.cu -- the extern "C" boundary (include/fgs_b200.h) over fgsb::Core.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "core.cuh"
#include "cg.hpp"
#include "nystrom.hpp"
#include "kmeans.hpp"
#include "fgs_b200.h"
#include "lanczos.cuh"
#include "nccl_shim.hpp"

using fgsb::Core;
using fgsb::fail;

struct fgs_nfft {
  std::unique_ptr<Core> core;
};
struct fgs_fastsum {
  std::unique_ptr<Core> core;
};
struct fgs_adjacency {
  std::unique_ptr<Core> core;
};
struct fgs_shard_group {
  std::unique_ptr<fgsb::ShardGroup> group;
};

namespace {

thread_local std::string g_err;

template <class F>
fgs_status guard(F&& f) {
  try {
    f();
    g_err.clear();
    return FGS_OK;
  } catch (const fgsb::Error& e) {
    g_err = e.what();
    return e.code;
  } catch (const std::bad_alloc&) {
    g_err = "host out of memory";
    return FGS_ERESOURCE;
  } catch (const std::exception& e) {
    g_err = e.what();
    return FGS_ECUDA;
  }
}

fgsb::Params to_params(const fgs_fastsum_params* p) {
  fgsb::Params out;
  if (p) {
    out.N = p->bandwidth;
    out.m = p->cutoff;
    out.p = p->smoothness;
    out.eps_b = p->eps_b;
    out.oversampling = p->oversampling;
  }
  return out;
}

void need(const void* p, const char* what) {
  if (!p) fail(FGS_EPARAM, std::string(what) + " must not be NULL");
}

// validate_common (nfft.cpp:33-50)
void validate_nfft_nodes(int d, int N, const double* nodes, int64_t n) {
  if (d < 1 || d > 3) fail(FGS_EPARAM, "dims must be 1, 2, or 3, got " + std::to_string(d));
  if (N < 2 || N % 2 != 0) fail(FGS_EPARAM, "bandwidth must be even and >= 2, got " + std::to_string(N));
  if (n == 0) fail(FGS_ESHAPE, "node set is empty");
  for (int64_t j = 0; j < n; ++j)
    for (int t = 0; t < d; ++t) {
      const double v = nodes[t * n + j];
      if (!(v >= -0.5 && v < 0.5))
        fail(FGS_ERANGE, "node " + std::to_string(j) + " component " + std::to_string(t) + " = " +
                             std::to_string(v) + " outside [-1/2, 1/2)");
    }
}

fgsb::KernelSpec spec_of(fgs_kernel k, double shape) {
  fgsb::KernelSpec s;
  s.family = static_cast<int>(k);
  s.shape = shape;
  return s;
}

int epilogue_of(fgs_op op, bool* scale) {
  switch (op) {
    case FGS_OP_KERNEL: *scale = false; return fgsb::EPI_KERNEL;
    case FGS_OP_WEIGHT: *scale = false; return fgsb::EPI_WEIGHT;
    case FGS_OP_NORMALIZED: *scale = true; return fgsb::EPI_NORMALIZED;
    case FGS_OP_SYM_LAPLACIAN: *scale = true; return fgsb::EPI_LAPLACIAN;
  }
  fail(FGS_EPARAM, "unknown operator");
}

// host column block (ld) -> contiguous device block
void upload_block(Core& c, fgsb::DBuf<double>& dst, const double* src, int64_t n, int nvec, int64_t ld) {
  dst.alloc(static_cast<size_t>(n) * nvec);
  if (ld == n) {
    c.host_copy(true, dst.p, src, sizeof(double) * n * nvec);
  } else {
    FGS_CUDA(cudaMemcpy2DAsync(dst.p, sizeof(double) * n, src, sizeof(double) * ld, sizeof(double) * n, nvec,
                               cudaMemcpyHostToDevice, c.stream));
  }
}
void download_block(Core& c, double* dst, const fgsb::DBuf<double>& src, int64_t n, int nvec, int64_t ld) {
  if (ld == n) {
    c.host_copy(false, dst, src.p, sizeof(double) * n * nvec);
  } else {
    FGS_CUDA(cudaMemcpy2DAsync(dst, sizeof(double) * ld, src.p, sizeof(double) * n, sizeof(double) * n, nvec,
                               cudaMemcpyDeviceToHost, c.stream));
  }
  FGS_CUDA(cudaStreamSynchronize(c.stream));
}

}  // namespace

extern "C" {

const char* fgs_last_error(void) { return g_err.c_str(); }

fgs_status fgs_fastsum_preset(int level, double eps_b, fgs_fastsum_params* out) {
  return guard([&] {  // fastsum.cpp:9-21
    need(out, "out");
    fgs_fastsum_params p{32, 4, 4, 0.0, 2.0};
    switch (level) {
      case 1: p.bandwidth = 16; p.cutoff = 2; break;
      case 2: p.bandwidth = 32; p.cutoff = 4; break;
      case 3: p.bandwidth = 64; p.cutoff = 7; break;
      default: fail(FGS_EPARAM, "preset level must be 1, 2, or 3");
    }
    p.smoothness = p.cutoff;
    p.eps_b = eps_b;
    *out = p;
  });
}

fgs_status fgs_bessel_i0(double x, double* out) {
  return guard([&] {
    need(out, "out");
    *out = fgsb::i0_series(x);
  });
}

// ---- NfftPlan --------------------------------------------------------------
fgs_status fgs_nfft_create(int dims, int bandwidth, int cutoff, const double* nodes, int64_t n, double oversampling,
                           int device, fgs_nfft_t* out) {
  return guard([&] {
    need(out, "out");
    *out = nullptr;
    if (n > 0) need(nodes, "nodes");
    validate_nfft_nodes(dims, bandwidth, nodes, n);
    fgsb::Params p;
    p.N = bandwidth;
    p.m = cutoff;
    p.oversampling = oversampling;
    auto h = std::make_unique<fgs_nfft>();
    h->core = std::make_unique<Core>(nodes, n, dims, Core::NFFT, fgsb::KernelSpec{}, p, device);
    *out = h.release();
  });
}

fgs_status fgs_nfft_info(fgs_nfft_t h, int* grid_size, int64_t* coefficient_count) {
  return guard([&] {
    need(h, "handle");
    if (grid_size) *grid_size = h->core->M;
    int64_t F = 1;
    for (int t = 0; t < h->core->d; ++t) F *= h->core->N;
    if (coefficient_count) *coefficient_count = F;
  });
}

static void nfft_forward_impl(fgs_nfft_t h, const double* fhat, int64_t len, std::vector<double>& planar) {
  Core& c = *h->core;
  int64_t F = 1;
  for (int t = 0; t < c.d; ++t) F *= c.N;
  if (len != F) fail(FGS_ESHAPE, "coefficient vector has wrong length");
  FGS_CUDA(cudaSetDevice(c.device));
  c.xbuf.upload(fhat, static_cast<size_t>(2 * F), c.stream);
  c.ybuf.alloc(static_cast<size_t>(2 * c.n));
  c.nfft_forward(c.xbuf.p, c.ybuf.p);
  planar.resize(static_cast<size_t>(2 * c.n));
  FGS_CUDA(cudaMemcpyAsync(planar.data(), c.ybuf.p, sizeof(double) * 2 * c.n, cudaMemcpyDeviceToHost, c.stream));
  FGS_CUDA(cudaStreamSynchronize(c.stream));
}

fgs_status fgs_nfft_forward(fgs_nfft_t h, const double* fhat, int64_t len, double* out) {
  return guard([&] {
    need(h, "handle");
    std::vector<double> planar;
    nfft_forward_impl(h, fhat, len, planar);
    const int64_t n = h->core->n;
    for (int64_t j = 0; j < n; ++j) {
      out[2 * j] = planar[static_cast<size_t>(j)];
      out[2 * j + 1] = planar[static_cast<size_t>(n + j)];
    }
  });
}

fgs_status fgs_nfft_forward_real(fgs_nfft_t h, const double* fhat, int64_t len, double* out) {
  return guard([&] {
    need(h, "handle");
    std::vector<double> planar;
    nfft_forward_impl(h, fhat, len, planar);
    std::copy(planar.begin(), planar.begin() + h->core->n, out);
  });
}

fgs_status fgs_nfft_adjoint(fgs_nfft_t h, const double* x, int64_t len, double* out) {
  return guard([&] {
    need(h, "handle");
    Core& c = *h->core;
    if (len != c.n) fail(FGS_ESHAPE, "input vector length does not match node count");
    FGS_CUDA(cudaSetDevice(c.device));
    std::vector<double> planar(static_cast<size_t>(2 * c.n));
    for (int64_t j = 0; j < c.n; ++j) {
      planar[static_cast<size_t>(j)] = x[2 * j];
      planar[static_cast<size_t>(c.n + j)] = x[2 * j + 1];
    }
    int64_t F = 1;
    for (int t = 0; t < c.d; ++t) F *= c.N;
    c.xbuf.upload(planar.data(), planar.size(), c.stream);
    c.ybuf.alloc(static_cast<size_t>(2 * F));
    c.nfft_adjoint(c.xbuf.p, c.ybuf.p);
    FGS_CUDA(cudaMemcpyAsync(out, c.ybuf.p, sizeof(double) * 2 * F, cudaMemcpyDeviceToHost, c.stream));
    FGS_CUDA(cudaStreamSynchronize(c.stream));
  });
}

void fgs_nfft_destroy(fgs_nfft_t h) { delete h; }

// ---- FastsumPlan -----------------------------------------------------------
fgs_status fgs_fastsum_create(const double* nodes, int64_t n, int d, fgs_kernel kernel, double shape,
                              const fgs_fastsum_params* params, int device, fgs_fastsum_t* out) {
  return guard([&] {
    need(out, "out");
    *out = nullptr;
    if (n > 0) need(nodes, "nodes");
    auto h = std::make_unique<fgs_fastsum>();
    h->core = std::make_unique<Core>(nodes, n, d, Core::FASTSUM, spec_of(kernel, shape), to_params(params), device);
    *out = h.release();
  });
}

fgs_status fgs_fastsum_apply(fgs_fastsum_t h, const double* x, int64_t len, double* y) {
  return guard([&] {
    need(h, "handle");
    Core& c = *h->core;
    if (len != c.n) fail(FGS_ESHAPE, "input vector length does not match node count");
    FGS_CUDA(cudaSetDevice(c.device));
    upload_block(c, c.xbuf, x, c.n, 1, c.n);
    c.ybuf.alloc(static_cast<size_t>(c.n));
    c.apply(fgsb::EPI_KERNEL, c.xbuf.p, c.n, c.ybuf.p, c.n, 1, true, false);
    download_block(c, y, c.ybuf, c.n, 1, c.n);
  });
}

fgs_status fgs_fastsum_info(fgs_fastsum_t h, double* rho, double* out_factor, double* k0, double* scaled_shape) {
  return guard([&] {
    need(h, "handle");
    if (rho) *rho = h->core->rho;
    if (out_factor) *out_factor = h->core->out_factor;
    if (k0) *k0 = h->core->k0;
    if (scaled_shape) *scaled_shape = h->core->scaled.shape;
  });
}

fgs_status fgs_fastsum_coefficients(fgs_fastsum_t h, double* out) {
  return guard([&] {
    need(h, "handle");
    for (size_t i = 0; i < h->core->bhat.size(); ++i) {
      out[2 * i] = h->core->bhat[i].real();
      out[2 * i + 1] = h->core->bhat[i].imag();
    }
  });
}

fgs_status fgs_fastsum_error_estimate(fgs_fastsum_t h, int samples, uint64_t seed, double* out) {
  return guard([&] {
    need(h, "handle");
    *out = h->core->error_estimate(samples, seed);
  });
}

void fgs_fastsum_destroy(fgs_fastsum_t h) { delete h; }

// ---- AdjacencyOperator -----------------------------------------------------
static fgs_status adjacency_create_impl(const double* nodes, int64_t n, int d, fgs_kernel kernel, double shape,
                                        const fgs_fastsum_params* params, int device, int rank, int world,
                                        const void* nccl_id, fgs_adjacency_t* out, int64_t* bad_node) {
  return guard([&] {
    need(out, "out");
    *out = nullptr;
    if (bad_node) *bad_node = -1;
    if (n < 2) fail(FGS_ESHAPE, "adjacency operator needs at least two nodes");  // graphop.cpp:39-42
    if (d < 1 || d > 3) fail(FGS_EPARAM, "node dimension must be 1, 2, or 3");
    need(nodes, "nodes");
    auto h = std::make_unique<fgs_adjacency>();
    h->core = std::make_unique<Core>(nodes, n, d, Core::FASTSUM, spec_of(kernel, shape), to_params(params), device,
                                     rank, world, nccl_id);
    h->core->compute_degrees(bad_node);
    *out = h.release();
  });
}

fgs_status fgs_adjacency_create(const double* nodes, int64_t n, int d, fgs_kernel kernel, double shape,
                                const fgs_fastsum_params* params, int device, fgs_adjacency_t* out,
                                int64_t* bad_node) {
  return adjacency_create_impl(nodes, n, d, kernel, shape, params, device, 0, 1, nullptr, out, bad_node);
}

fgs_status fgs_adjacency_create_direct(const double* nodes, int64_t n, int d, fgs_kernel kernel, double shape,
                                       int device, fgs_adjacency_t* out, int64_t* bad_node) {
  return guard([&] {
    need(out, "out");
    *out = nullptr;
    if (bad_node) *bad_node = -1;
    if (n < 2) fail(FGS_ESHAPE, "adjacency operator needs at least two nodes");  // graphop.cpp:39-42
    if (d < 1 || d > 3) fail(FGS_EPARAM, "node dimension must be 1, 2, or 3");
    need(nodes, "nodes");
    auto h = std::make_unique<fgs_adjacency>();
    h->core = std::make_unique<Core>(nodes, n, d, Core::DIRECT, spec_of(kernel, shape), fgsb::Params{}, device);
    h->core->compute_degrees(bad_node);
    *out = h.release();
  });
}

fgs_status fgs_nccl_unique_id(void* out128) {
  return guard([&] {
    need(out128, "out");
    ncclUniqueId id;
    fgsb::nccl_check(fgsb::nccl().get_unique_id(&id), "ncclGetUniqueId");
    static_assert(sizeof(id) == 128, "ncclUniqueId is 128 bytes");
    std::memcpy(out128, &id, sizeof(id));
  });
}

fgs_status fgs_adjacency_create_sharded(const double* nodes, int64_t n, int d, fgs_kernel kernel, double shape,
                                        const fgs_fastsum_params* params, int device, int rank, int world,
                                        const void* nccl_id, fgs_adjacency_t* out, int64_t* bad_node) {
  if (!nccl_id) {
    g_err = "nccl_id must not be NULL for a sharded handle";
    return FGS_EPARAM;
  }
  return adjacency_create_impl(nodes, n, d, kernel, shape, params, device, rank, world, nccl_id, out, bad_node);
}

fgs_status fgs_adjacency_apply(fgs_adjacency_t h, fgs_op op, const double* x, double* y, int nvec, int64_t ld) {
  return guard([&] {
    need(h, "handle");
    Core& c = *h->core;
    if (c.world > 1) fail(FGS_EPARAM, "host-vector apply needs an unsharded handle; use fgs_adjacency_apply_device");
    if (nvec < 1) fail(FGS_ESHAPE, "nvec must be >= 1");
    if (ld < c.n) fail(FGS_ESHAPE, "input length does not match operator dimension");
    need(x, "x");
    need(y, "y");
    bool scale = false;
    const int epi = epilogue_of(op, &scale);
    FGS_CUDA(cudaSetDevice(c.device));
    if (c.apply_host_graph(epi, x, y, ld, nvec, scale)) {  // pinned x / y: copies inside the graph
      FGS_CUDA(cudaStreamSynchronize(c.stream));
      return;
    }
    upload_block(c, c.xbuf, x, c.n, nvec, ld);
    c.ybuf.alloc(static_cast<size_t>(c.n) * nvec);
    c.apply(epi, c.xbuf.p, c.n, c.ybuf.p, c.n, nvec, true, scale);
    download_block(c, y, c.ybuf, c.n, nvec, ld);
  });
}

fgs_status fgs_adjacency_apply_device(fgs_adjacency_t h, fgs_op op, const double* dx, double* dy, int nvec, int64_t ld,
                                      int internal_order) {
  return guard([&] {
    need(h, "handle");
    Core& c = *h->core;
    if (nvec < 1) fail(FGS_ESHAPE, "nvec must be >= 1");
    const int64_t len = internal_order ? c.n_local : c.n;
    if (ld < len) fail(FGS_ESHAPE, "input length does not match operator dimension");
    if (!internal_order && c.world > 1) fail(FGS_EPARAM, "sharded handles take internal-order slices");
    bool scale = false;
    const int epi = epilogue_of(op, &scale);
    FGS_CUDA(cudaSetDevice(c.device));
    c.apply(epi, dx, ld, dy, ld, nvec, !internal_order, scale);
  });
}

fgs_status fgs_adjacency_degrees(fgs_adjacency_t h, double* out) {
  return guard([&] {
    need(h, "handle");
    need(out, "out");
    Core& c = *h->core;
    if (c.world > 1) fail(FGS_EPARAM, "degrees() in caller order needs an unsharded handle");
    std::vector<double> d(static_cast<size_t>(c.n));
    FGS_CUDA(cudaMemcpy(d.data(), c.degrees.p, sizeof(double) * c.n, cudaMemcpyDeviceToHost));
    for (int64_t p = 0; p < c.n; ++p) out[c.host_perm[static_cast<size_t>(p)]] = d[static_cast<size_t>(p)];
  });
}

fgs_status fgs_adjacency_info(fgs_adjacency_t h, double* rho, double* out_factor, double* k0, int64_t* n_local,
                              int64_t* offset_local) {
  return guard([&] {
    need(h, "handle");
    if (rho) *rho = h->core->rho;
    if (out_factor) *out_factor = h->core->out_factor;
    if (k0) *k0 = h->core->k0;
    if (n_local) *n_local = h->core->n_local;
    if (offset_local) *offset_local = h->core->offset;
  });
}

fgs_status fgs_adjacency_set_stream(fgs_adjacency_t h, void* stream) {
  return guard([&] {
    need(h, "handle");
    h->core->set_stream(static_cast<cudaStream_t>(stream));
  });
}

fgs_status fgs_adjacency_permute_device(fgs_adjacency_t h, const double* dx, double* dy, int nvec, int64_t ld,
                                        int direction) {
  return guard([&] {
    need(h, "handle");
    FGS_CUDA(cudaSetDevice(h->core->device));
    h->core->permute(dx, ld, dy, ld, nvec, direction);
  });
}

fgs_status fgs_adjacency_launch_count(fgs_adjacency_t h, int64_t* out) {
  return guard([&] {
    need(h, "handle");
    need(out, "out");
    *out = h->core->launches;
  });
}

fgs_status fgs_adjacency_profile(fgs_adjacency_t h, int enable) {
  return guard([&] {
    need(h, "handle");
    h->core->enable_profile(enable != 0);
  });
}

fgs_status fgs_adjacency_profile_read(fgs_adjacency_t h, double* ms6, int64_t* applies) {
  return guard([&] {
    need(h, "handle");
    need(ms6, "ms6");
    h->core->read_profile(ms6, applies);
  });
}

fgs_status fgs_adjacency_geometry(fgs_adjacency_t h, int* d, int* N, int* M, int* taps, int* items,
                                  int64_t* box_stride) {
  return guard([&] {
    need(h, "handle");
    const Core& c = *h->core;
    if (d) *d = c.d;
    if (N) *N = c.N;
    if (M) *M = c.M;
    if (taps) *taps = c.T;
    if (items) *items = c.nitems;
    if (box_stride) *box_stride = c.box_stride;
  });
}

fgs_status fgs_adjacency_plan_stats(fgs_adjacency_t h, double* mean_run, int* tensor_spread, int* tensor_interp) {
  return guard([&] {
    need(h, "handle");
    const Core& c = *h->core;
    if (mean_run) *mean_run = c.mean_run;
    if (tensor_spread) *tensor_spread = c.tensor_spread() ? 1 : 0;
    if (tensor_interp) *tensor_interp = c.tensor_interp() ? 1 : 0;
  });
}

fgs_status fgs_adjacency_plan_layout(fgs_adjacency_t h, int* slot_layout, int64_t* slots) {
  return guard([&] {
    need(h, "handle");
    const Core& c = *h->core;
    if (slot_layout) *slot_layout = c.use_slots ? 1 : 0;
    if (slots) *slots = c.use_slots ? static_cast<int64_t>(c.slot_map.n) : c.n_local;
  });
}

fgs_status fgs_measure_fp64_peak(int device, double* tflops) {
  return guard([&] {
    need(tflops, "tflops");
    *tflops = fgsb::measure_fp64_peak(device);
  });
}

fgs_status fgs_measure_dmma_peak(int device, double* tflops) {
  return guard([&] {
    need(tflops, "tflops");
    *tflops = fgsb::measure_dmma_peak(device);
  });
}

fgs_status fgs_lanczos_stats(fgs_adjacency_t h, double* out4) {
  return guard([&] {
    need(h, "handle");
    need(out4, "out4");
    for (int i = 0; i < 4; ++i) out4[i] = h->core->lanczos_stats[i];
  });
}

void fgs_adjacency_destroy(fgs_adjacency_t h) { delete h; }

// ---- single-GPU shard-group emulation of the N-rank path --------------------
fgs_status fgs_shard_group_create(const double* nodes, int64_t n, int d, fgs_kernel kernel, double shape,
                                  const fgs_fastsum_params* params, int device, int world, fgs_shard_group_t* out,
                                  int64_t* bad_node) {
  return guard([&] {
    need(out, "out");
    *out = nullptr;
    if (bad_node) *bad_node = -1;
    if (n < 2) fail(FGS_ESHAPE, "adjacency operator needs at least two nodes");  // graphop.cpp:39-42
    if (d < 1 || d > 3) fail(FGS_EPARAM, "node dimension must be 1, 2, or 3");
    need(nodes, "nodes");
    auto g = std::make_unique<fgs_shard_group>();
    g->group = std::make_unique<fgsb::ShardGroup>(nodes, n, d, spec_of(kernel, shape), to_params(params), device,
                                                  world, bad_node);
    *out = g.release();
  });
}

fgs_status fgs_shard_group_apply_device(fgs_shard_group_t g, fgs_op op, const double* dx, double* dy, int nvec,
                                        int64_t ld) {
  return guard([&] {
    need(g, "group");
    if (nvec < 1) fail(FGS_ESHAPE, "nvec must be >= 1");
    if (ld < g->group->n) fail(FGS_ESHAPE, "input length does not match operator dimension");
    need(dx, "x");
    need(dy, "y");
    bool scale = false;
    const int epi = epilogue_of(op, &scale);
    FGS_CUDA(cudaSetDevice(g->group->device));
    g->group->apply(epi, dx, dy, ld, nvec, scale);
    FGS_CUDA(cudaStreamSynchronize(g->group->stream));
  });
}

fgs_status fgs_shard_group_stats(fgs_shard_group_t g, int rank, int64_t* n_local, int* conv_plane0,
                                 int* conv_planes, int* items) {
  return guard([&] {
    need(g, "group");
    if (rank < 0 || rank >= static_cast<int>(g->group->shards.size())) fail(FGS_EPARAM, "rank out of range");
    const Core& c = *g->group->shards[static_cast<size_t>(rank)];
    if (n_local) *n_local = c.n_local;
    if (conv_plane0) *conv_plane0 = c.conv_plane0;
    if (conv_planes) *conv_planes = c.conv_planes;
    if (items) *items = c.nitems;
  });
}

fgs_status fgs_shard_group_profile(fgs_shard_group_t g, fgs_op op, const double* dx, double* dy, int nvec, int64_t ld,
                                   int reps, double* shard_ms, double* exchange_ms) {
  return guard([&] {
    need(g, "group");
    need(dx, "x");
    need(dy, "y");
    need(shard_ms, "shard_ms");
    need(exchange_ms, "exchange_ms");
    if (nvec < 1 || reps < 1) fail(FGS_ESHAPE, "nvec and reps must be >= 1");
    if (ld < g->group->n) fail(FGS_ESHAPE, "input length does not match operator dimension");
    bool scale = false;
    const int epi = epilogue_of(op, &scale);
    FGS_CUDA(cudaSetDevice(g->group->device));
    g->group->profile(epi, dx, dy, ld, nvec, scale, reps, shard_ms, exchange_ms);
  });
}

fgs_status fgs_shard_group_stage_profile(fgs_shard_group_t g, fgs_op op, const double* dx, double* dy, int nvec,
                                         int64_t ld, int reps, double* stage_ms) {
  return guard([&] {
    need(g, "group");
    need(dx, "x");
    need(dy, "y");
    need(stage_ms, "stage_ms");
    if (nvec < 1 || reps < 1) fail(FGS_ESHAPE, "nvec and reps must be >= 1");
    bool scale = false;
    const int epi = epilogue_of(op, &scale);
    FGS_CUDA(cudaSetDevice(g->group->device));
    auto& sh = g->group->shards;
    for (auto& c : sh) c->enable_profile(true);
    for (int r = 0; r < reps; ++r) g->group->apply(epi, dx, dy, ld, nvec, scale);
    for (size_t r = 0; r < sh.size(); ++r) {
      int64_t napp = 0;
      double ms[Core::ST_COUNT];
      sh[r]->read_profile(ms, &napp);
      sh[r]->enable_profile(false);
      for (int k = 0; k < Core::ST_COUNT; ++k) stage_ms[r * Core::ST_COUNT + k] = napp ? ms[k] / napp : 0.0;
    }
  });
}

void fgs_shard_group_destroy(fgs_shard_group_t g) { delete g; }

// ---- lanczos_largest -------------------------------------------------------
fgs_status fgs_lanczos_largest(fgs_adjacency_t h, int which, int k, int max_iter, double tol, uint64_t seed,
                               double* values, double* vectors, int* count, int* iterations, int* converged) {
  return guard([&] {
    need(h, "handle");
    need(values, "values");
    Core& c = *h->core;
    if (which != 0 && which != 1) fail(FGS_EPARAM, "which must be 0 (adjacency) or 1 (laplacian)");
    if (vectors && c.world > 1) fail(FGS_EPARAM, "Ritz vectors in caller order need an unsharded handle");
    FGS_CUDA(cudaSetDevice(c.device));
    fgsb::LanczosResult r = fgsb::lanczos_device(c, which, k, max_iter, tol, seed, vectors != nullptr);
    c.lanczos_stats[0] = r.apply_ms;
    c.lanczos_stats[1] = r.reorth_ms;
    c.lanczos_stats[2] = r.loop_ms;
    c.lanczos_stats[3] = r.iterations;
    const int cnt = static_cast<int>(r.values.size());
    // make_eigenpairs (spectral.cpp:105-127): stable descending sort, then
    // flip each column so its first largest-magnitude entry is positive
    std::vector<int> order(static_cast<size_t>(cnt));
    for (int i = 0; i < cnt; ++i) order[static_cast<size_t>(i)] = i;
    std::stable_sort(order.begin(), order.end(),
                     [&](int a, int b) { return r.values[static_cast<size_t>(a)] > r.values[static_cast<size_t>(b)]; });
    for (int i = 0; i < cnt; ++i) values[i] = r.values[static_cast<size_t>(order[static_cast<size_t>(i)])];
    if (vectors) {
      std::vector<int> ord(order.begin(), order.end());
      fgsb::lanczos_finish_vectors(c, r, ord, vectors);
    }
    if (count) *count = cnt;
    if (iterations) *iterations = r.iterations;
    if (converged) *converged = r.converged ? 1 : 0;
  });
}

fgs_status fgs_lanczos_largest_operator(int64_t n, fgs_operator_apply apply, void* ctx, int device, int k,
                                        int max_iter, double tol, uint64_t seed, double* values, double* vectors,
                                        int* count, int* iterations, int* converged) {
  return guard([&] {
    need(values, "values");
    fgsb::lanczos_operator(n, apply, ctx, device, k, max_iter, tol, seed, values, vectors, count, iterations,
                           converged);
  });
}

// ---- conjugate gradients (spectral.cpp:446-495) ---------------------------
static fgs_status cg_impl(Core* c, int system, double beta, const double* f, int64_t len, double tol, int max_iter,
                          double* x, int* iterations, int* status) {
  return guard([&] {
    need(c, "handle");
    need(f, "f");
    need(x, "x");
    if (len != c->n) fail(FGS_ESHAPE, "fidelity length does not match operator dimension");
    FGS_CUDA(cudaSetDevice(c->device));
    const fgsb::CgOutcome o = fgsb::cg_solve(*c, system == 0 ? fgsb::CG_SSL : fgsb::CG_KRR, beta, f, tol, max_iter, x);
    if (iterations) *iterations = o.iterations;
    if (status) *status = static_cast<int>(o.status);
  });
}

fgs_status fgs_kernel_ssl_solve(fgs_adjacency_t h, const double* f, int64_t len, double beta, double tol,
                                int max_iter, double* x, int* iterations, int* status) {
  return cg_impl(h ? h->core.get() : nullptr, 0, beta, f, len, tol, max_iter, x, iterations, status);
}

fgs_status fgs_fastsum_ridge_solve(fgs_fastsum_t h, const double* f, int64_t len, double beta, double tol,
                                   int max_iter, double* x, int* iterations, int* status) {
  return cg_impl(h ? h->core.get() : nullptr, 1, beta, f, len, tol, max_iter, x, iterations, status);
}

// ---- nystrom_gaussian (spectral.cpp:384-444) --------------------------------
fgs_status fgs_nystrom_gaussian(fgs_adjacency_t h, int k, int L, int M, uint64_t seed, double* values, double* vectors) {
  return guard([&] {
    need(h, "handle");
    need(values, "values");
    need(vectors, "vectors");
    Core& c = *h->core;
    FGS_CUDA(cudaSetDevice(c.device));
    const std::vector<double> v = fgsb::nystrom_gaussian(c, k, L, M, seed, vectors);
    std::copy(v.begin(), v.end(), values);
  });
}

// ---- k-means / spectral clustering (learn.cpp:17-167, 441-486) -----------
fgs_status fgs_kmeans(const double* points_colmajor, int64_t n, int dim, int k, int restarts, int max_iter,
                      uint64_t seed, int device, int* labels, double* centroids_colmajor, double* wcss) {
  return guard([&] {
    need(points_colmajor, "points");
    need(labels, "labels");
    fgsb::kmeans_run(points_colmajor, false, n, dim, k, restarts, max_iter, seed, device, false, labels,
                     centroids_colmajor, wcss);
  });
}

fgs_status fgs_spectral_cluster(const double* vectors_colmajor, int64_t n, int kv, int k, int restarts, int max_iter,
                                uint64_t seed, int device, int on_device, int* labels) {
  return guard([&] {
    need(vectors_colmajor, "vectors");
    need(labels, "labels");
    if (kv < k) fail(FGS_EPARAM, "need at least as many eigenvectors as clusters");
    fgsb::kmeans_run(vectors_colmajor, on_device != 0, n, kv, k, restarts, max_iter, seed, device, true, labels,
                     nullptr, nullptr);
  });
}

fgs_status fgs_misclassification_rate(const int* predicted, const int* truth, int64_t n, int permuted, double* out) {
  return guard([&] {
    need(out, "out");
    *out = 0.0;
    if (n == 0) return;
    need(predicted, "predicted");
    need(truth, "truth");
    if (!permuted) {
      int64_t wrong = 0;
      for (int64_t i = 0; i < n; ++i) wrong += predicted[i] != truth[i];
      *out = static_cast<double>(wrong) / static_cast<double>(n);
      return;
    }
    int classes = 0;
    for (int64_t i = 0; i < n; ++i) {
      if (predicted[i] < 0 || truth[i] < 0) fail(FGS_ERANGE, "labels must be nonnegative");
      classes = std::max(classes, std::max(predicted[i], truth[i]) + 1);
    }
    if (classes > 8) fail(FGS_EPARAM, "permutation matching supports at most 8 classes");
    std::vector<int64_t> cnt(static_cast<size_t>(classes) * classes, 0);
    for (int64_t i = 0; i < n; ++i) ++cnt[static_cast<size_t>(predicted[i]) * classes + truth[i]];
    std::vector<int> map(static_cast<size_t>(classes));
    for (int c = 0; c < classes; ++c) map[static_cast<size_t>(c)] = c;
    int64_t best = 0;
    do {
      int64_t matched = 0;
      for (int p = 0; p < classes; ++p) matched += cnt[static_cast<size_t>(p) * classes + map[static_cast<size_t>(p)]];
      best = std::max(best, matched);
    } while (std::next_permutation(map.begin(), map.end()));
    *out = 1.0 - static_cast<double>(best) / static_cast<double>(n);
  });
}

}  // extern "C"
