/*
 * fgs_b200.h -- C ABI of the B200-native NFFT fast-summation graph operator.
 *
 * Drop-in boundary for the reference's hot path (/root/reference/proj):
 *   fgs::NfftPlan          nfft.hpp:59-94      -> fgs_nfft_*
 *   fgs::FastsumPlan       fastsum.hpp:34-67   -> fgs_fastsum_*
 *   fgs::AdjacencyOperator graphop.hpp:45-97   -> fgs_adjacency_*
 *   fgs::lanczos_largest   spectral.hpp:68-70  -> fgs_lanczos_largest
 * Plain pointers and sizes only.  Matrices are column-major (Eigen's
 * default, the layout of the reference's `MatrixXd nodes`); complex vectors
 * are interleaved (re, im) doubles; every host vector is in the caller's
 * point order (any internal spatial permutation is applied and removed
 * inside the handle).  Every call returns an fgs_status whose nonzero values
 * map 1:1 onto the reference's exception classes (errors.hpp:8-49), with the
 * message available from fgs_last_error() (thread-local).
 *
 * Threading (nfft.hpp:57-58 / fastsum.hpp:55-56 promise concurrent apply on
 * one plan but share plan-owned scratch, nfft.cpp:150-153): here each handle
 * owns its device workspaces and ONE CUDA stream; calls on one handle are
 * serialised in stream order.  Use one handle per host thread for
 * concurrency.
 */
#ifndef FGS_B200_H
#define FGS_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  FGS_OK = 0,
  FGS_EPARAM = 1,    /* fgs::ParameterError  (errors.hpp:8-11)  */
  FGS_ERANGE = 2,    /* fgs::RangeError      (errors.hpp:14-17) */
  FGS_ESHAPE = 3,    /* fgs::ShapeError      (errors.hpp:20-23) */
  FGS_ENUMERIC = 4,  /* fgs::NumericalError  (errors.hpp:27-30) */
  FGS_ERESOURCE = 5, /* fgs::ResourceError   (errors.hpp:45-48) */
  FGS_ECUDA = 6,     /* CUDA / cuFFT runtime failure (no reference analogue) */
  FGS_ENCCL = 7      /* NCCL failure (no reference analogue) */
} fgs_status;

/* kernels.hpp:20-25 */
typedef enum {
  FGS_GAUSSIAN = 0,
  FGS_LAPLACIAN_RBF = 1,
  FGS_MULTIQUADRIC = 2,
  FGS_INV_MULTIQUADRIC = 3
} fgs_kernel;

/* graphop.hpp:71-81 */
typedef enum {
  FGS_OP_KERNEL = 0,        /* (W + K(0) I) x      apply_kernel        */
  FGS_OP_WEIGHT = 1,        /* W x                 apply_weight        */
  FGS_OP_NORMALIZED = 2,    /* D^-1/2 W D^-1/2 x   apply_normalized    */
  FGS_OP_SYM_LAPLACIAN = 3  /* x - A x             apply_sym_laplacian */
} fgs_op;

/* fastsum.hpp:13-23 (FastsumParams) */
typedef struct {
  int bandwidth;      /* N, even                      default 32 */
  int cutoff;         /* m, window half-support        default 4  */
  int smoothness;     /* p, boundary blend order       default 4  */
  double eps_b;       /* blend width, 0 = truncate     default 0  */
  double oversampling;/* grid oversampling sigma       default 2  */
} fgs_fastsum_params;

typedef struct fgs_nfft* fgs_nfft_t;
typedef struct fgs_fastsum* fgs_fastsum_t;
typedef struct fgs_adjacency* fgs_adjacency_t;

/* ---- library ------------------------------------------------------------ */
const char* fgs_last_error(void);
/* FastsumParams::preset (fastsum.cpp:9-21): level 1..3 */
fgs_status fgs_fastsum_preset(int level, double eps_b, fgs_fastsum_params* out);
fgs_status fgs_bessel_i0(double x, double* out); /* nfft.cpp:60-69 */

/* ---- NfftPlan (nfft.hpp:59-94, nfft.cpp:328-438) ------------------------ */
fgs_status fgs_nfft_create(int dims, int bandwidth, int cutoff, const double* nodes_colmajor,
                           int64_t n, double oversampling, int device, fgs_nfft_t* out);
fgs_status fgs_nfft_info(fgs_nfft_t h, int* grid_size, int64_t* coefficient_count);
/* result_j ~= sum_{l in I_N} fhat_l exp(+2 pi i l.v_j)       nfft.cpp:402-413 */
fgs_status fgs_nfft_forward(fgs_nfft_t h, const double* fhat, int64_t len, double* out);
/* result_l ~= sum_j x_j exp(-2 pi i l.v_j)                   nfft.cpp:415-427 */
fgs_status fgs_nfft_adjoint(fgs_nfft_t h, const double* x, int64_t len, double* out);
/* Re(forward(fhat))                                           nfft.cpp:429-438 */
fgs_status fgs_nfft_forward_real(fgs_nfft_t h, const double* fhat, int64_t len, double* out);
void fgs_nfft_destroy(fgs_nfft_t h);

/* ---- FastsumPlan (fastsum.hpp:34-67, fastsum.cpp:69-124) ----------------- */
fgs_status fgs_fastsum_create(const double* nodes_colmajor, int64_t n, int d, fgs_kernel kernel,
                              double shape, const fgs_fastsum_params* params, int device,
                              fgs_fastsum_t* out);
/* y_j ~= sum_i K(v_j - v_i) x_i (diagonal K(0) included)    fastsum.cpp:111-118 */
fgs_status fgs_fastsum_apply(fgs_fastsum_t h, const double* x, int64_t len, double* y);
/* rho, output factor, K(0) of the requested kernel, rescaled shape (fastsum.hpp:50-52) */
fgs_status fgs_fastsum_info(fgs_fastsum_t h, double* rho, double* out_factor, double* k0,
                            double* scaled_shape);
/* bhat in FrequencyIndexSet order, interleaved complex, N^d entries (kernels.cpp:266-335) */
fgs_status fgs_fastsum_coefficients(fgs_fastsum_t h, double* out);
/* kernel_error_estimate (fastsum.cpp:120-124, kernels.cpp:369-396) */
fgs_status fgs_fastsum_error_estimate(fgs_fastsum_t h, int samples, uint64_t seed, double* out);
void fgs_fastsum_destroy(fgs_fastsum_t h);

/* ---- AdjacencyOperator (graphop.hpp:45-97, graphop.cpp:36-103) ----------- */
/* On a nonpositive approximate degree returns FGS_ENUMERIC and writes the
 * first offending node (caller order) to *bad_node (graphop.cpp:57-64). */
fgs_status fgs_adjacency_create(const double* nodes_colmajor, int64_t n, int d, fgs_kernel kernel,
                                double shape, const fgs_fastsum_params* params, int device,
                                fgs_adjacency_t* out, int64_t* bad_node);
/* AdjacencyBackend::Direct (graphop.hpp:19-22, graphop.cpp:29-34): the exact
 * O(n^2) operator W~x = sum_i K(||v_j - v_i||) x_i on raw (unscaled) nodes
 * (fastsum.cpp:126-139 direct_apply), also the recompute-mode dense
 * reference (spectral.cpp:497-554).  Same apply/degrees/Lanczos calls. */
fgs_status fgs_adjacency_create_direct(const double* nodes_colmajor, int64_t n, int d, fgs_kernel kernel,
                                       double shape, int device, fgs_adjacency_t* out, int64_t* bad_node);
/* Multi-GPU: one process per GPU.  Every rank passes the SAME nodes; rank r
 * owns the r-th contiguous slice of the internal spatial order.  nccl_id is
 * the 128-byte ncclUniqueId from fgs_nccl_unique_id() on rank 0, broadcast
 * by the caller. */
fgs_status fgs_nccl_unique_id(void* out128);
fgs_status fgs_adjacency_create_sharded(const double* nodes_colmajor, int64_t n, int d,
                                        fgs_kernel kernel, double shape,
                                        const fgs_fastsum_params* params, int device, int rank,
                                        int world, const void* nccl_id, fgs_adjacency_t* out,
                                        int64_t* bad_node);
/* Host vectors, caller order.  nvec >= 1 column vectors with leading
 * dimension ld >= n (block apply). */
fgs_status fgs_adjacency_apply(fgs_adjacency_t h, fgs_op op, const double* x, double* y,
                               int nvec, int64_t ld);
/* Device-resident vectors.  `internal_order` != 0: vectors are in the
 * handle's internal spatial order (no permutation), as used by the
 * device-resident Lanczos; 0: caller order.  On a sharded handle the device
 * vectors hold this rank's slice (internal order only). */
fgs_status fgs_adjacency_apply_device(fgs_adjacency_t h, fgs_op op, const double* dx, double* dy,
                                      int nvec, int64_t ld, int internal_order);
/* Node degrees d_j = sum_{i != j} K(v_j - v_i), caller order (graphop.hpp:69) */
fgs_status fgs_adjacency_degrees(fgs_adjacency_t h, double* out);
fgs_status fgs_adjacency_info(fgs_adjacency_t h, double* rho, double* out_factor, double* k0,
                              int64_t* n_local, int64_t* offset_local);
/* Run subsequent work of this handle on `stream` (a cudaStream_t). */
fgs_status fgs_adjacency_set_stream(fgs_adjacency_t h, void* stream);
/* Permute between caller order and internal order on the device
 * (direction 0: caller -> internal, 1: internal -> caller). */
fgs_status fgs_adjacency_permute_device(fgs_adjacency_t h, const double* dx, double* dy, int nvec,
                                        int64_t ld, int direction);
/* Stage profiling (instrumentation): when enabled, every apply records CUDA
 * events on the handle's stream between its stages.  fgs_adjacency_profile_read
 * synchronises and returns the summed device milliseconds per stage since the
 * previous read -- ms[6] = {spread, assemble, fft r2c, spectral multiply (+
 * exchange), fft c2r, interpolation} -- and the number of applies covered. */
fgs_status fgs_adjacency_profile(fgs_adjacency_t h, int enable);
fgs_status fgs_adjacency_profile_read(fgs_adjacency_t h, double* ms6, int64_t* applies);
/* Plan geometry: grid M, taps per dim 2m, work items, tile edge, internal
 * nonempty cells are implied; used by bench.py for algorithmic byte/flop
 * counts. */
fgs_status fgs_adjacency_geometry(fgs_adjacency_t h, int* d, int* N, int* M, int* taps, int* items,
                                  int64_t* box_stride);
/* Which spread / interpolation kernels the plan runs (instrumentation for
 * the parity tests): points per run (nonempty cell piece), and 1 when the
 * fp64 tensor-core (DMMA) spread / interpolation is used, 0 for the scalar
 * kernels. */
fgs_status fgs_adjacency_plan_stats(fgs_adjacency_t h, double* mean_run, int* tensor_spread, int* tensor_interp);
/* 1 when the plan uses the run-aligned slot layout (d = 3, 2m = 16 dense
 * plans: every footprint run starts on a multiple of 8 slots), and the
 * number of slots (points + pad slots); 0 / the point count otherwise. */
fgs_status fgs_adjacency_plan_layout(fgs_adjacency_t h, int* slot_layout, int64_t* slots);
/* fp64 FMA-pipe peak of `device` in TFLOP/s (independent DFMA chains, CUDA
 * events), the denominator of the spread/interp roofline. */
fgs_status fgs_measure_fp64_peak(int device, double* tflops);
/* fp64 tensor-core (DMMA m8n8k4) peak in TFLOP/s, same method. */
fgs_status fgs_measure_dmma_peak(int device, double* tflops);
/* Kernel launches issued by this handle since creation (instrumentation). */
fgs_status fgs_adjacency_launch_count(fgs_adjacency_t h, int64_t* out);
void fgs_adjacency_destroy(fgs_adjacency_t h);

/* ---- single-GPU emulation of the N-rank sharded path ---------------------
 * `world` shards of one operator (the plan slices, slab-pruned convolutions
 * and exchange buffers that fgs_adjacency_create_sharded ranks 0..world-1
 * build) on one device; every apply runs phase 1 on each shard, sums the
 * shards' exchange buffers with a device kernel in place of ncclAllReduce,
 * then phase 2.  Validation of the multi-GPU data path where fewer GPUs than
 * ranks exist (no kernels that wait on one another share the GPU).  No
 * reference counterpart: the reference is serial (README.md:85-91). */
typedef struct fgs_shard_group* fgs_shard_group_t;
fgs_status fgs_shard_group_create(const double* nodes_colmajor, int64_t n, int d, fgs_kernel kernel, double shape,
                                  const fgs_fastsum_params* params, int device, int world, fgs_shard_group_t* out,
                                  int64_t* bad_node);
/* y = op(x), full-length device vectors in caller order, column j at x + j ld */
fgs_status fgs_shard_group_apply_device(fgs_shard_group_t g, fgs_op op, const double* dx, double* dy, int nvec,
                                        int64_t ld);
/* shard `rank`: points owned, first dim-0 plane and plane count of its
 * pruned convolution (M planes when unpruned), work items */
fgs_status fgs_shard_group_stats(fgs_shard_group_t g, int rank, int64_t* n_local, int* conv_plane0,
                                 int* conv_planes, int* items);
/* `reps` applies timed with CUDA events around each shard's two phases:
 * shard_ms[world] = mean ms per apply of shard r (what rank r computes on
 * its own GPU), exchange_ms = the device-sum exchange on one GPU (not an
 * NVLink figure) */
fgs_status fgs_shard_group_profile(fgs_shard_group_t g, fgs_op op, const double* dx, double* dy, int nvec, int64_t ld,
                                   int reps, double* shard_ms, double* exchange_ms);
/* per-shard stage times of `reps` applies (CUDA events between the launches,
 * as fgs_adjacency_profile_read): stage_ms[world][6] = spread (+ slot
 * gather), assembly, forward plane pass, line passes (+ the exchange and the
 * other shards' phase-1 work that runs between them on one GPU), inverse
 * plane pass, interpolation; mean ms per apply */
fgs_status fgs_shard_group_stage_profile(fgs_shard_group_t g, fgs_op op, const double* dx, double* dy, int nvec,
                                         int64_t ld, int reps, double* stage_ms);
void fgs_shard_group_destroy(fgs_shard_group_t g);

/* ---- lanczos_largest (spectral.hpp:68-70, spectral.cpp:141-256) ---------
 * Device-resident Lanczos with full two-pass reorthogonalisation on the
 * operator `which` (0: A = apply_normalized as adjacency_handle does,
 * spectral.cpp:91-96; 1: L_s = apply_sym_laplacian, laplacian_handle).
 * Returns the `count` <= k largest Ritz pairs, descending, sign-normalised
 * (make_eigenpairs, spectral.cpp:105-127); vectors column-major n x count in
 * caller order (may be NULL to skip the Ritz vectors). */
fgs_status fgs_lanczos_largest(fgs_adjacency_t h, int which, int k, int max_iter, double tol,
                               uint64_t seed, double* values, double* vectors, int* count,
                               int* iterations, int* converged);

/* lanczos_largest over a generic symmetric operator: the reference's
 * SymmetricOperatorHandle {dimension, std::function apply} (spectral.hpp:
 * 18-30; dense_handle, user operators).  `apply(ctx, x, y, n)` writes y = A x
 * for host vectors of length n and returns 0 (nonzero aborts with
 * FGS_ENUMERIC).  The recurrence and both Gram-Schmidt passes run on
 * `device` (basis in HBM); q_m and A q_m cross to/from the host once per
 * step.  Same outputs as fgs_lanczos_largest (values descending, vectors
 * n x count column-major, sign-normalised; vectors may be NULL). */
typedef int (*fgs_operator_apply)(void* ctx, const double* x, double* y, int64_t n);
fgs_status fgs_lanczos_largest_operator(int64_t n, fgs_operator_apply apply, void* ctx, int device, int k,
                                        int max_iter, double tol, uint64_t seed, double* values, double* vectors,
                                        int* count, int* iterations, int* converged);

/* Device milliseconds of the last fgs_lanczos_largest on this handle spent in
 * operator applies and in reorthogonalisation, the host wall time of its
 * iteration loop, and its iteration count (instrumentation). */
fgs_status fgs_lanczos_stats(fgs_adjacency_t h, double* out4);

/* ---- synthetic workloads of BASELINE.json (seeded mt19937_64) ----------- */
/* config 1..5: writes n x d column-major nodes; returns n, d, sigma, N, m, p, k */
fgs_status fgs_workload_info(int config, int64_t* n, int* d, double* sigma, int* N, int* m, int* p,
                             int* k);
fgs_status fgs_workload_generate(int config, uint64_t seed, double* nodes_colmajor);
/* the same generator with n_points points instead of the config's n (0: the
 * config's n; config 3's image is fixed-size) -- BASELINE config 5's weak
 * scaling at 1.25M points per GPU */
fgs_status fgs_workload_generate_n(int config, uint64_t seed, int64_t n_points, double* nodes_colmajor);
fgs_status fgs_workload_vectors(int64_t n, int nvec, uint64_t seed, double* out);

/* ---- conjugate gradients (spectral.hpp:120-140, spectral.cpp:446-495) ---- */
/* status: 0 converged, 1 max iterations, 2 indefinite (CgStatus).  f, x in
 * caller order, length n.  Convergence on the true relative residual
 * ||f - Ax|| <= tol ||f||, as the reference. */
/* kernel_ssl_solve (learn.cpp:364-381): (I + beta L_s) x = f; beta = 0 -> x = f */
fgs_status fgs_kernel_ssl_solve(fgs_adjacency_t h, const double* f, int64_t len, double beta, double tol,
                                int max_iter, double* x, int* iterations, int* status);
/* krr_fit's system (learn.cpp:403-430): (W~ + beta I) alpha = f on a FastsumPlan */
fgs_status fgs_fastsum_ridge_solve(fgs_fastsum_t h, const double* f, int64_t len, double beta, double tol,
                                   int max_iter, double* x, int* iterations, int* status);

/* ---- Nystrom (spectral.hpp:81-86, spectral.cpp:384-444) ------------------ */
/* nystrom_gaussian(adjacency_handle(op), {k, L, M, seed}): k approximate
 * eigenpairs of A from a Gaussian sketch of L columns (2L fast applies) with
 * inversion rank M; 1 <= k <= M <= L <= n.  values[k] descending, vectors
 * n x k column-major (caller order, first-max-entry positive).  Fewer than M
 * positive sketch eigenvalues -> FGS_ENUMERIC. */
fgs_status fgs_nystrom_gaussian(fgs_adjacency_t h, int k, int L, int M, uint64_t seed, double* values,
                                double* vectors);

/* ---- k-means / spectral clustering (learn.hpp, learn.cpp:17-167) --------- */
/* kmeans(points, k, {restarts, max_iter, seed}) (learn.cpp:140-155): points
 * column-major n x dim; labels[n]; centroids k x dim column-major and wcss
 * may be NULL.  k-means++ seeding from std::mt19937_64(seed) shared across
 * restarts, Lloyd iterations on the device, best run by strict wcss. */
fgs_status fgs_kmeans(const double* points_colmajor, int64_t n, int dim, int k, int restarts, int max_iter,
                      uint64_t seed, int device, int* labels, double* centroids_colmajor, double* wcss);
/* spectral_cluster(pairs, k, opts) (learn.cpp:157-167): unit-normalised rows
 * of the n x kv eigenvector block (host, or device memory when on_device),
 * then kmeans.  kv < k -> FGS_EPARAM. */
fgs_status fgs_spectral_cluster(const double* vectors_colmajor, int64_t n, int kv, int k, int restarts, int max_iter,
                                uint64_t seed, int device, int on_device, int* labels);
/* misclassification_rate / _permuted (learn.cpp:441-486), host-side */
fgs_status fgs_misclassification_rate(const int* predicted, const int* truth, int64_t n, int permuted, double* out);

#ifdef __cplusplus
}
#endif

#endif /* FGS_B200_H */
