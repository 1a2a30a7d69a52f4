// ============================================================================
// ref_capi.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A plain C entry layer over the REFERENCE'S OWN hot-path code: the files
// /root/reference/proj/src/{nfft,kernels,fastsum,graphop,spectral}.cpp are
// compiled unchanged, where they lie, against the shim headers in
// oracle/shim (Eigen/FFTW stand-ins), together with this file, into
// oracle/_ref/libfgsref.so by oracle/build_ref.sh.  oracle/ref.py wraps it
// for tests/ and for bench.py's reference arm / cpu_baseline ("kind":
// "reference").  Nothing in the product links or loads it.
//
// Each entry calls the reference API exactly as its own callers do:
//   AdjacencyOperator(nodes, kernel, params, backend)   graphop.cpp:36-67
//   apply_kernel / _weight / _normalized / _sym_laplacian graphop.cpp:87-103
//   lanczos_largest(adjacency_handle | laplacian_handle) commands.cpp:171-183
//   FastsumPlan / NfftPlan / direct_apply                fastsum.cpp, nfft.cpp
// and maps the reference's exception classes (errors.hpp:8-49) onto the
// status codes of include/fgs_b200.h.
// ============================================================================
#include <cstdint>
#include <cstring>
#include <memory>
#include <string>

#include "fgs/errors.hpp"
#include "fgs/fastsum.hpp"
#include "fgs/graphop.hpp"
#include "fgs/nfft.hpp"
#include "fgs/spectral.hpp"

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    g_err.clear();
    return 0;
  } catch (const fgs::ParameterError& e) {
    g_err = e.what();
    return 1;
  } catch (const fgs::RangeError& e) {
    g_err = e.what();
    return 2;
  } catch (const fgs::ShapeError& e) {
    g_err = e.what();
    return 3;
  } catch (const fgs::NumericalError& e) {
    g_err = e.what();
    return 4;
  } catch (const fgs::ResourceError& e) {
    g_err = e.what();
    return 5;
  } catch (const std::bad_alloc&) {
    g_err = "out of memory";
    return 5;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 4;
  }
}

fgs::MatrixXd nodes_of(const double* colmajor, int64_t n, int d) {
  fgs::MatrixXd m(n, d);
  std::memcpy(m.data(), colmajor, sizeof(double) * static_cast<size_t>(n) * d);
  return m;
}

fgs::VectorXd vec_of(const double* x, int64_t n) {
  fgs::VectorXd v(n);
  std::memcpy(v.data(), x, sizeof(double) * static_cast<size_t>(n));
  return v;
}

void store(const fgs::VectorXd& v, double* out) { std::memcpy(out, v.data(), sizeof(double) * v.size()); }

fgs::KernelSpec spec_of(int family, double shape) {
  switch (family) {
    case 0: return fgs::KernelSpec::gaussian(shape);
    case 1: return fgs::KernelSpec::laplacian_rbf(shape);
    case 2: return fgs::KernelSpec::multiquadric(shape);
    case 3: return fgs::KernelSpec::inverse_multiquadric(shape);
    default: throw fgs::ParameterError("unknown kernel family");
  }
}

fgs::FastsumParams params_of(int N, int m, int p, double eps_b, double oversampling) {
  fgs::FastsumParams prm;
  prm.bandwidth = N;
  prm.cutoff = m;
  prm.smoothness = p;
  prm.eps_b = eps_b;
  prm.oversampling = oversampling;
  return prm;
}

// graphop.cpp:57-64 names the node in the message: "computed degree of node <j> ..."
int64_t node_in_message(const std::string& msg) {
  const std::string key = "node ";
  const size_t at = msg.find(key);
  if (at == std::string::npos) return -1;
  return std::strtoll(msg.c_str() + at + key.size(), nullptr, 10);
}

void store_pairs(const fgs::EigenPairs& pairs, double* values, double* vectors, int* count) {
  const int64_t c = pairs.count();
  *count = static_cast<int>(c);
  for (int64_t i = 0; i < c; ++i) values[i] = pairs.values(i);
  if (vectors)
    std::memcpy(vectors, pairs.vectors.data(), sizeof(double) * static_cast<size_t>(pairs.vectors.size()));
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

// ---- AdjacencyOperator ------------------------------------------------------
int ref_adjacency_create(const double* nodes, int64_t n, int d, int family, double shape, int N, int m, int p,
                         double eps_b, double oversampling, int direct, void** out, int64_t* bad_node) {
  *bad_node = -1;
  const int st = guarded([&] {
    auto op = std::make_unique<fgs::AdjacencyOperator>(
        nodes_of(nodes, n, d), spec_of(family, shape), params_of(N, m, p, eps_b, oversampling),
        direct ? fgs::AdjacencyBackend::Direct : fgs::AdjacencyBackend::Fastsum);
    *out = op.release();
  });
  if (st == 4) *bad_node = node_in_message(g_err);
  return st;
}

void ref_adjacency_destroy(void* h) { delete static_cast<fgs::AdjacencyOperator*>(h); }

int ref_adjacency_apply(void* h, int op, const double* x, int64_t len, double* y) {
  return guarded([&] {
    const auto& a = *static_cast<const fgs::AdjacencyOperator*>(h);
    const fgs::VectorXd xv = vec_of(x, len);
    fgs::VectorXd r;
    switch (op) {
      case 0: r = a.apply_kernel(xv); break;
      case 1: r = a.apply_weight(xv); break;
      case 2: r = a.apply_normalized(xv); break;
      case 3: r = a.apply_sym_laplacian(xv); break;
      default: throw fgs::ParameterError("unknown operator");
    }
    store(r, y);
  });
}

int ref_adjacency_degrees(void* h, double* out) {
  return guarded([&] { store(static_cast<const fgs::AdjacencyOperator*>(h)->degrees(), out); });
}

int ref_adjacency_info(void* h, double* rho, double* out_factor, double* k0) {
  return guarded([&] {
    const auto& a = *static_cast<const fgs::AdjacencyOperator*>(h);
    *k0 = a.kernel_zero();
    *rho = a.plan() ? a.plan()->scaling() : 1.0;
    *out_factor = a.plan() ? a.plan()->output_factor() : 1.0;
  });
}

// lanczos_largest(adjacency_handle(op) | laplacian_handle(op), k, opts, &info)
// as solve_pairs does (commands.cpp:171-183); vectors n x count column-major
int ref_lanczos_adjacency(void* h, int which, int k, int max_iter, double tol, uint64_t seed, double* values,
                          double* vectors, int* count, int* iterations, int* converged) {
  return guarded([&] {
    const auto& a = *static_cast<const fgs::AdjacencyOperator*>(h);
    fgs::LanczosOptions opts;
    opts.max_iter = max_iter;
    opts.tol = tol;
    opts.seed = seed;
    fgs::LanczosInfo info;
    const fgs::SymmetricOperatorHandle handle = which == 0 ? fgs::adjacency_handle(a) : fgs::laplacian_handle(a);
    const fgs::EigenPairs pairs = fgs::lanczos_largest(handle, k, opts, &info);
    store_pairs(pairs, values, vectors, count);
    *iterations = info.iterations;
    *converged = info.converged ? 1 : 0;
  });
}

// lanczos_largest(dense_handle(A)) -- the reference's dense test operators
// (test_spectral.cpp:84-140)
int ref_lanczos_dense(const double* A, int64_t n, int k, int max_iter, double tol, uint64_t seed, double* values,
                      double* vectors, int* count, int* iterations, int* converged) {
  return guarded([&] {
    fgs::MatrixXd m(n, n);
    std::memcpy(m.data(), A, sizeof(double) * static_cast<size_t>(n * n));
    fgs::LanczosOptions opts;
    opts.max_iter = max_iter;
    opts.tol = tol;
    opts.seed = seed;
    fgs::LanczosInfo info;
    const fgs::EigenPairs pairs = fgs::lanczos_largest(fgs::dense_handle(std::move(m)), k, opts, &info);
    store_pairs(pairs, values, vectors, count);
    *iterations = info.iterations;
    *converged = info.converged ? 1 : 0;
  });
}

// ---- FastsumPlan --------------------------------------------------------------
int ref_fastsum_create(const double* nodes, int64_t n, int d, int family, double shape, int N, int m, int p,
                       double eps_b, double oversampling, void** out) {
  return guarded([&] {
    *out = new fgs::FastsumPlan(nodes_of(nodes, n, d), spec_of(family, shape),
                                params_of(N, m, p, eps_b, oversampling));
  });
}

void ref_fastsum_destroy(void* h) { delete static_cast<fgs::FastsumPlan*>(h); }

int ref_fastsum_apply(void* h, const double* x, int64_t len, double* y) {
  return guarded([&] { store(static_cast<const fgs::FastsumPlan*>(h)->apply(vec_of(x, len)), y); });
}

int ref_fastsum_info(void* h, double* rho, double* out_factor, double* k0, double* scaled_shape) {
  return guarded([&] {
    const auto& f = *static_cast<const fgs::FastsumPlan*>(h);
    *rho = f.scaling();
    *out_factor = f.output_factor();
    *k0 = f.kernel_zero();
    *scaled_shape = f.scaled_kernel().shape;
  });
}

// b-hat in FrequencyIndexSet order, interleaved complex
int ref_fastsum_coefficients(void* h, double* out) {
  return guarded([&] {
    const auto& c = static_cast<const fgs::FastsumPlan*>(h)->coefficients().values;
    std::memcpy(out, c.data(), sizeof(double) * 2 * static_cast<size_t>(c.size()));
  });
}

// ---- NfftPlan ------------------------------------------------------------------
int ref_nfft_create(int d, int N, int m, const double* nodes, int64_t n, double oversampling, void** out) {
  return guarded([&] { *out = new fgs::NfftPlan(d, N, m, nodes_of(nodes, n, d), oversampling); });
}

void ref_nfft_destroy(void* h) { delete static_cast<fgs::NfftPlan*>(h); }

int ref_nfft_info(void* h, int* M, int64_t* coefficients) {
  return guarded([&] {
    const auto& p = *static_cast<const fgs::NfftPlan*>(h);
    *M = p.grid_size();
    *coefficients = static_cast<int64_t>(p.coefficient_count());
  });
}

int ref_nfft_forward(void* h, const double* fhat, int64_t len, double* out) {
  return guarded([&] {
    fgs::VectorXcd f(len);
    std::memcpy(f.data(), fhat, sizeof(double) * 2 * static_cast<size_t>(len));
    const fgs::VectorXcd r = static_cast<const fgs::NfftPlan*>(h)->forward(f);
    std::memcpy(out, r.data(), sizeof(double) * 2 * static_cast<size_t>(r.size()));
  });
}

int ref_nfft_adjoint(void* h, const double* x, int64_t len, double* out) {
  return guarded([&] {
    fgs::VectorXcd v(len);
    std::memcpy(v.data(), x, sizeof(double) * 2 * static_cast<size_t>(len));
    const fgs::VectorXcd r = static_cast<const fgs::NfftPlan*>(h)->adjoint(v);
    std::memcpy(out, r.data(), sizeof(double) * 2 * static_cast<size_t>(r.size()));
  });
}

int ref_nfft_forward_real(void* h, const double* fhat, int64_t len, double* out) {
  return guarded([&] {
    fgs::VectorXcd f(len);
    std::memcpy(f.data(), fhat, sizeof(double) * 2 * static_cast<size_t>(len));
    store(static_cast<const fgs::NfftPlan*>(h)->forward_real(f), out);
  });
}

// ---- direct_apply (fastsum.cpp:126-139) -----------------------------------------
int ref_direct_apply(const double* nodes, int64_t n, int d, int family, double shape, const double* x, double* y) {
  return guarded([&] { store(fgs::direct_apply(nodes_of(nodes, n, d), spec_of(family, shape), vec_of(x, n)), y); });
}

}  // extern "C"
