// nystrom.cu -- nystrom_gaussian (spectral.cpp:384-444): the sketch-based
// Nystrom approximation of A = D^-1/2 W D^-1/2 from 2L applications of the
// fast operator.
//
//   probes  Omega (n x L) ~ N(0,1) from std::mt19937_64(seed), column by
//           column (the reference's draw order)
//   sketch  S = A Omega                       L block applies (ours)
//   QR      S = Q R                           cuSOLVER geqrf / orgqr
//   B1      = A Q                             L block applies (ours)
//   B2      = sym(Q^T B1)                     cuBLAS gemm, L x L
//   eig(B2) -> top M (sigma, U_M), all M must be positive
//   QR      B1 U_M = Qh Rh                    cuBLAS gemm + cuSOLVER
//   middle  = sym(Rh diag(1/sigma) Rh^T)      host, M x M
//   eig(middle) -> top k (values, W_k);  vectors = Qh W_k   (cuBLAS gemm)
//   make_eigenpairs: descending, first-max-entry sign   (device, lanczos.cu)
//
// All n-sized data stays in HBM in the handle's internal order (a row
// permutation does not change the QR's column space or R up to signs, and
// the final pairs are invariant to those signs).  The L x L / M x M
// symmetric eigenproblems run on the host with cyclic Jacobi (ascending, as
// Eigen's SelfAdjointEigenSolver).
#include <cublas_v2.h>
#include <cuda_runtime.h>
#include <cusolverDn.h>

#include <algorithm>
#include <cmath>
#include <random>
#include <vector>

#include "common.cuh"
#include "core.cuh"
#include "lanczos.cuh"
#include "nystrom.hpp"

namespace fgsb {
namespace {

#define FGS_CUBLAS(call)                                                                        \
  do {                                                                                          \
    cublasStatus_t s_ = (call);                                                                 \
    if (s_ != CUBLAS_STATUS_SUCCESS) fail(FGS_ECUDA, std::string(#call) + ": cublas error " + std::to_string(s_)); \
  } while (0)
#define FGS_CUSOLVER(call)                                                                      \
  do {                                                                                          \
    cusolverStatus_t s_ = (call);                                                               \
    if (s_ != CUSOLVER_STATUS_SUCCESS)                                                          \
      fail(FGS_ECUDA, std::string(#call) + ": cusolver error " + std::to_string(s_));           \
  } while (0)

struct Handles {
  cublasHandle_t blas = nullptr;
  cusolverDnHandle_t solver = nullptr;
  ~Handles() {
    if (blas) cublasDestroy(blas);
    if (solver) cusolverDnDestroy(solver);
  }
};

// Thin Householder QR of the n x c column-major A (in place -> Q); R (c x c,
// upper, column-major) to r_host when non-null.
void thin_qr(Handles& h, cudaStream_t st, double* A, int64_t n, int c, std::vector<double>* r_host) {
  DBuf<double> tau;
  tau.alloc(static_cast<size_t>(c));
  DBuf<int> info;
  info.alloc(1);
  int lw1 = 0, lw2 = 0;
  FGS_CUSOLVER(cusolverDnDgeqrf_bufferSize(h.solver, static_cast<int>(n), c, A, static_cast<int>(n), &lw1));
  FGS_CUSOLVER(cusolverDnDorgqr_bufferSize(h.solver, static_cast<int>(n), c, c, A, static_cast<int>(n), tau.p, &lw2));
  DBuf<double> work;
  work.alloc(static_cast<size_t>(std::max(lw1, lw2)) + 1);
  FGS_CUSOLVER(cusolverDnDgeqrf(h.solver, static_cast<int>(n), c, A, static_cast<int>(n), tau.p, work.p,
                                std::max(lw1, lw2), info.p));
  if (r_host) {
    std::vector<double> full(static_cast<size_t>(c) * c);
    FGS_CUDA(cudaMemcpy2DAsync(full.data(), sizeof(double) * c, A, sizeof(double) * n, sizeof(double) * c, c,
                               cudaMemcpyDeviceToHost, st));
    FGS_CUDA(cudaStreamSynchronize(st));
    r_host->assign(static_cast<size_t>(c) * c, 0.0);
    for (int j = 0; j < c; ++j)
      for (int i = 0; i <= j; ++i) (*r_host)[static_cast<size_t>(j) * c + i] = full[static_cast<size_t>(j) * c + i];
  }
  FGS_CUSOLVER(cusolverDnDorgqr(h.solver, static_cast<int>(n), c, c, A, static_cast<int>(n), tau.p, work.p,
                                std::max(lw1, lw2), info.p));
  int hinfo = 0;
  FGS_CUDA(cudaMemcpyAsync(&hinfo, info.p, sizeof(int), cudaMemcpyDeviceToHost, st));
  FGS_CUDA(cudaStreamSynchronize(st));
  if (hinfo != 0) fail(FGS_ENUMERIC, "QR factorisation failed (info " + std::to_string(hinfo) + ")");
}

// y (n x L) = A x (n x L) in chunks of <= 16 vectors through the graph-cached apply
void block_apply(Core& c, const double* x, double* y, int L) {
  for (int v0 = 0; v0 < L; v0 += 16) {
    const int nv = std::min(16, L - v0);
    c.apply(EPI_NORMALIZED, x + static_cast<int64_t>(v0) * c.n_local, c.n_local, y + static_cast<int64_t>(v0) * c.n_local,
            c.n_local, nv, false, true);
  }
}

}  // namespace

// cyclic Jacobi for a symmetric s x s column-major matrix: ascending
// eigenvalues, eigenvectors as columns of vecs
void symmetric_eigen(int s, std::vector<double> a, std::vector<double>& vals, std::vector<double>& vecs) {
  vecs.assign(static_cast<size_t>(s) * s, 0.0);
  for (int i = 0; i < s; ++i) vecs[static_cast<size_t>(i) * s + i] = 1.0;
  auto A = [&](int i, int j) -> double& { return a[static_cast<size_t>(j) * s + i]; };
  auto V = [&](int i, int j) -> double& { return vecs[static_cast<size_t>(j) * s + i]; };
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0, scale = 0.0;
    for (int j = 0; j < s; ++j)
      for (int i = 0; i < s; ++i) (i == j ? scale : off) += A(i, j) * A(i, j);
    if (off <= 1e-30 * std::max(scale, 1e-300)) break;
    for (int p = 0; p < s - 1; ++p)
      for (int q = p + 1; q < s; ++q) {
        const double apq = A(p, q);
        if (apq == 0.0) continue;
        const double theta = (A(q, q) - A(p, p)) / (2.0 * apq);
        const double t = (theta >= 0.0 ? 1.0 : -1.0) / (std::abs(theta) + std::sqrt(theta * theta + 1.0));
        const double c = 1.0 / std::sqrt(t * t + 1.0), sn = t * c;
        for (int k = 0; k < s; ++k) {  // A <- A G (columns p, q)
          const double akp = A(k, p), akq = A(k, q);
          A(k, p) = c * akp - sn * akq;
          A(k, q) = sn * akp + c * akq;
        }
        for (int k = 0; k < s; ++k) {  // A <- G^T A (rows p, q)
          const double apk = A(p, k), aqk = A(q, k);
          A(p, k) = c * apk - sn * aqk;
          A(q, k) = sn * apk + c * aqk;
        }
        for (int k = 0; k < s; ++k) {
          const double vkp = V(k, p), vkq = V(k, q);
          V(k, p) = c * vkp - sn * vkq;
          V(k, q) = sn * vkp + c * vkq;
        }
      }
  }
  std::vector<int> order(static_cast<size_t>(s));
  for (int i = 0; i < s; ++i) order[static_cast<size_t>(i)] = i;
  std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return A(x, x) < A(y, y); });
  vals.resize(static_cast<size_t>(s));
  std::vector<double> sorted(static_cast<size_t>(s) * s);
  for (int j = 0; j < s; ++j) {
    const int o = order[static_cast<size_t>(j)];
    vals[static_cast<size_t>(j)] = A(o, o);
    for (int i = 0; i < s; ++i) sorted[static_cast<size_t>(j) * s + i] = V(i, o);
  }
  vecs.swap(sorted);
}

std::vector<double> nystrom_gaussian(Core& c, int k, int L, int M, uint64_t seed, double* vectors_host) {
  const int64_t n = c.n;
  if (c.world > 1) fail(FGS_EPARAM, "nystrom_gaussian needs an unsharded handle");
  if (k < 1 || M < k || L < M || L > n) fail(FGS_EPARAM, "need 1 <= k <= M <= L <= n");
  cudaStream_t st = c.stream;
  Handles h;
  FGS_CUBLAS(cublasCreate(&h.blas));
  FGS_CUBLAS(cublasSetStream(h.blas, st));
  FGS_CUSOLVER(cusolverDnCreate(&h.solver));
  FGS_CUSOLVER(cusolverDnSetStream(h.solver, st));

  // probes, caller order, column by column (spectral.cpp:394-397)
  std::vector<double> probes(static_cast<size_t>(n) * L);
  {
    std::mt19937_64 rng(seed);
    std::normal_distribution<double> gauss;
    for (int col = 0; col < L; ++col)
      for (int64_t r = 0; r < n; ++r) probes[static_cast<size_t>(col) * n + r] = gauss(rng);
  }
  DBuf<double> omega_c, omega, sketch, b1;
  omega_c.upload(probes.data(), probes.size(), st);
  omega.alloc(static_cast<size_t>(n) * L);
  c.permute(omega_c.p, n, omega.p, n, L, 0);  // caller -> internal
  omega_c.reset();
  sketch.alloc(static_cast<size_t>(n) * L);
  block_apply(c, omega.p, sketch.p, L);
  omega.reset();
  thin_qr(h, st, sketch.p, n, L, nullptr);  // sketch -> Q (range)
  b1.alloc(static_cast<size_t>(n) * L);
  block_apply(c, sketch.p, b1.p, L);
  // B2 = Q^T B1, symmetrised
  DBuf<double> b2d;
  b2d.alloc(static_cast<size_t>(L) * L);
  const double one = 1.0, zero = 0.0;
  FGS_CUBLAS(cublasDgemm(h.blas, CUBLAS_OP_T, CUBLAS_OP_N, L, L, static_cast<int>(n), &one, sketch.p,
                         static_cast<int>(n), b1.p, static_cast<int>(n), &zero, b2d.p, L));
  std::vector<double> b2(static_cast<size_t>(L) * L);
  FGS_CUDA(cudaMemcpyAsync(b2.data(), b2d.p, sizeof(double) * L * L, cudaMemcpyDeviceToHost, st));
  FGS_CUDA(cudaStreamSynchronize(st));
  for (int j = 0; j < L; ++j)
    for (int i = 0; i < j; ++i) {
      const double s = 0.5 * (b2[static_cast<size_t>(j) * L + i] + b2[static_cast<size_t>(i) * L + j]);
      b2[static_cast<size_t>(j) * L + i] = s;
      b2[static_cast<size_t>(i) * L + j] = s;
    }
  std::vector<double> ev, evec;
  symmetric_eigen(L, b2, ev, evec);
  int positives = 0;
  for (double v : ev) positives += v > 0.0;
  if (positives < M)
    fail(FGS_ENUMERIC, "sketch captured fewer than the requested number of positive eigenvalues; increase the "
                       "sketch size");
  std::vector<double> sigma(static_cast<size_t>(M)), um(static_cast<size_t>(L) * M);
  for (int i = 0; i < M; ++i) {
    sigma[static_cast<size_t>(i)] = ev[static_cast<size_t>(L - 1 - i)];
    for (int r = 0; r < L; ++r) um[static_cast<size_t>(i) * L + r] = evec[static_cast<size_t>(L - 1 - i) * L + r];
  }
  // B1 U_M -> QR
  DBuf<double> umd, bu;
  umd.upload(um.data(), um.size(), st);
  bu.alloc(static_cast<size_t>(n) * M);
  FGS_CUBLAS(cublasDgemm(h.blas, CUBLAS_OP_N, CUBLAS_OP_N, static_cast<int>(n), M, L, &one, b1.p, static_cast<int>(n),
                         umd.p, L, &zero, bu.p, static_cast<int>(n)));
  b1.reset();
  sketch.reset();
  std::vector<double> rh;
  thin_qr(h, st, bu.p, n, M, &rh);
  // middle = sym(Rh diag(1/sigma) Rh^T)
  std::vector<double> mid(static_cast<size_t>(M) * M, 0.0);
  for (int i = 0; i < M; ++i)
    for (int j = 0; j < M; ++j) {
      double s = 0.0;
      for (int t = 0; t < M; ++t)
        s += rh[static_cast<size_t>(t) * M + i] / sigma[static_cast<size_t>(t)] * rh[static_cast<size_t>(t) * M + j];
      mid[static_cast<size_t>(j) * M + i] = s;
    }
  for (int j = 0; j < M; ++j)
    for (int i = 0; i < j; ++i) {
      const double s = 0.5 * (mid[static_cast<size_t>(j) * M + i] + mid[static_cast<size_t>(i) * M + j]);
      mid[static_cast<size_t>(j) * M + i] = s;
      mid[static_cast<size_t>(i) * M + j] = s;
    }
  std::vector<double> mv, mvec;
  symmetric_eigen(M, mid, mv, mvec);
  std::vector<double> values(static_cast<size_t>(k)), wk(static_cast<size_t>(M) * k);
  for (int i = 0; i < k; ++i) {
    values[static_cast<size_t>(i)] = mv[static_cast<size_t>(M - 1 - i)];
    for (int r = 0; r < M; ++r) wk[static_cast<size_t>(i) * M + r] = mvec[static_cast<size_t>(M - 1 - i) * M + r];
  }
  DBuf<double> wkd;
  wkd.upload(wk.data(), wk.size(), st);
  LanczosResult res;
  res.vectors_dev.alloc(static_cast<size_t>(n) * k);
  FGS_CUBLAS(cublasDgemm(h.blas, CUBLAS_OP_N, CUBLAS_OP_N, static_cast<int>(n), k, M, &one, bu.p, static_cast<int>(n),
                         wkd.p, M, &zero, res.vectors_dev.p, static_cast<int>(n)));
  // make_eigenpairs (spectral.cpp:105-127): values already descending; the
  // first-max-entry sign and the caller order on the device
  std::vector<int> order(static_cast<size_t>(k));
  for (int i = 0; i < k; ++i) order[static_cast<size_t>(i)] = i;
  lanczos_finish_vectors(c, res, order, vectors_host);
  return values;
}

}  // namespace fgsb
