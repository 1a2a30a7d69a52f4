"""ctypes front-end of the CPU oracle -- TEST INFRASTRUCTURE ONLY.

Wraps ``oracle/liboracle.so`` (built from ``oracle/fgs_oracle.cpp`` by
``oracle/build_oracle.sh``), a serial restatement of the reference's hot path
(``/root/reference/proj/src/{nfft,kernels,fastsum,graphop,spectral}.cpp``).
Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU baseline /
reference arm may import this module, and only as the checker.  The product
package ``paper_1808_04580_b200`` never imports it.

Parity pin: ``tests/test_ref_pin.py`` requires it to reproduce, bit for bit,
the reference's own sources compiled against shim Eigen/FFTW headers
(``oracle/_ref``, wrapped by ``oracle/ref.py``); ``tests/test_oracle_*.py``
run the reference's known-answer tests (test_nfft.cpp, test_kernels.cpp,
test_fastsum.cpp, test_graphop.cpp, test_spectral.cpp, acceptance.cpp) and
check its FFT against numpy.fft.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")

GAUSSIAN, LAPLACIAN_RBF, MULTIQUADRIC, INV_MULTIQUADRIC = 0, 1, 2, 3
OP_KERNEL, OP_WEIGHT, OP_NORMALIZED, OP_SYM_LAPLACIAN = 0, 1, 2, 3


class OracleError(Exception):
    """Raised with the reference exception class name as ``kind``."""

    KINDS = {1: "ParameterError", 2: "RangeError", 3: "ShapeError",
             4: "NumericalError", 5: "ResourceError"}

    def __init__(self, code: int, msg: str):
        super().__init__(f"{self.KINDS.get(code, code)}: {msg}")
        self.code = code
        self.kind = self.KINDS.get(code, str(code))
        self.msg = msg


def build() -> str:
    """Compile the oracle if its shared object is missing or stale."""
    srcs = [os.path.join(_HERE, "fgs_oracle.cpp"),
            os.path.join(_HERE, "..", "paper_1808_04580_b200", "csrc", "workload.cpp")]
    if (not os.path.exists(_SO)) or os.path.getmtime(_SO) < max(os.path.getmtime(s) for s in srcs if os.path.exists(s)):
        subprocess.check_call(["bash", os.path.join(_HERE, "build_oracle.sh")])
    return _SO


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_SO):
            build()
        _lib = C.CDLL(_SO)
        _lib.orc_last_error.restype = C.c_char_p
        _lib.orc_bessel_i0.restype = C.c_double
        _lib.orc_bessel_i0.argtypes = [C.c_double]
        _lib.orc_std_bessel_i0.restype = C.c_double
        _lib.orc_std_bessel_i0.argtypes = [C.c_double]
    return _lib


_D = C.POINTER(C.c_double)
_I = C.POINTER(C.c_int)


def _dp(a: np.ndarray):
    return a.ctypes.data_as(_D)


def _check(status: int):
    if status != 0:
        raise OracleError(status, lib().orc_last_error().decode())


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _nodes_colmajor(nodes) -> tuple[np.ndarray, int, int]:
    nodes = np.asarray(nodes, dtype=np.float64)
    if nodes.ndim == 1:
        nodes = nodes[:, None]
    n, d = nodes.shape
    return np.asfortranarray(nodes).ravel(order="F").copy(), n, d


def _cplx_in(v) -> np.ndarray:
    v = np.ascontiguousarray(v, dtype=np.complex128)
    return v.view(np.float64)


def set_threads(threads: int) -> int:
    """Host threads of the oracle's NFFT loops (1 = the serial reference
    order, pinned bitwise to oracle/_ref); returns the previous setting."""
    return lib().orc_set_threads(int(threads))


class threads:
    """with orc.threads(n): ... -- temporarily parallel oracle NFFT loops."""

    def __init__(self, n):
        self.n = n

    def __enter__(self):
        self.old = set_threads(self.n)
        return self

    def __exit__(self, *exc):
        set_threads(self.old)


def bessel_i0(x: float) -> float:
    return lib().orc_bessel_i0(C.c_double(x))


def std_bessel_i0(x: float) -> float:
    return lib().orc_std_bessel_i0(C.c_double(x))


def fft(data, d: int, M: int, sign: int) -> np.ndarray:
    buf = np.ascontiguousarray(data, dtype=np.complex128).reshape(-1).copy()
    _check(lib().orc_fft(_dp(buf.view(np.float64)), d, M, sign))
    return buf


def freq_component(d, N, flat, dim) -> int:
    out = C.c_int()
    _check(lib().orc_freq_component(d, N, C.c_int64(flat), dim, C.byref(out)))
    return out.value


def direct_ndft(d, N, nodes, fhat) -> np.ndarray:
    nd, n, dd = _nodes_colmajor(nodes)
    out = np.zeros(n, np.complex128)
    f = _cplx_in(fhat)
    _check(lib().orc_direct_ndft(d, N, _dp(nd), C.c_int64(n), _dp(f), _dp(out.view(np.float64))))
    return out


def direct_adjoint_ndft(d, N, nodes, x) -> np.ndarray:
    nd, n, dd = _nodes_colmajor(nodes)
    out = np.zeros(N ** d, np.complex128)
    xv = _cplx_in(x)
    _check(lib().orc_direct_adjoint_ndft(d, N, _dp(nd), C.c_int64(n), _dp(xv), _dp(out.view(np.float64))))
    return out


class NfftPlan:
    """Mirror of ``fgs::NfftPlan`` (nfft.hpp:59-94) over the oracle."""

    def __init__(self, dims, bandwidth, cutoff, nodes, oversampling=2.0):
        nd, n, d = _nodes_colmajor(nodes)
        h = C.c_void_p()
        _check(lib().orc_nfft_create(dims, bandwidth, cutoff, _dp(nd), C.c_int64(n),
                                     C.c_double(oversampling), C.byref(h)))
        self._h = h
        self.n = n
        self.d = dims
        M = C.c_int()
        cnt = C.c_int64()
        _check(lib().orc_nfft_info(h, C.byref(M), C.byref(cnt)))
        self.grid_size = M.value
        self.coefficient_count = cnt.value
        self.cutoff = cutoff

    def __del__(self):
        if getattr(self, "_h", None):
            lib().orc_nfft_destroy(self._h)
            self._h = None

    def forward(self, fhat) -> np.ndarray:
        f = _cplx_in(fhat)
        out = np.zeros(self.n, np.complex128)
        _check(lib().orc_nfft_forward(self._h, _dp(f), C.c_int64(f.size // 2), _dp(out.view(np.float64))))
        return out

    def adjoint(self, x) -> np.ndarray:
        xv = _cplx_in(x)
        out = np.zeros(self.coefficient_count, np.complex128)
        _check(lib().orc_nfft_adjoint(self._h, _dp(xv), C.c_int64(xv.size // 2), _dp(out.view(np.float64))))
        return out

    def forward_real(self, fhat) -> np.ndarray:
        f = _cplx_in(fhat)
        out = np.zeros(self.n, np.float64)
        _check(lib().orc_nfft_forward_real(self._h, _dp(f), C.c_int64(f.size // 2), _dp(out)))
        return out

    def taps(self):
        T = 2 * self.cutoff
        w = np.zeros(self.n * self.d * T)
        idx = np.zeros(self.n * self.d * T, np.int32)
        _check(lib().orc_nfft_taps(self._h, _dp(w), idx.ctypes.data_as(_I)))
        return w.reshape(self.n, self.d, T), idx.reshape(self.n, self.d, T)


def eval_kernel(family, shape, r) -> float:
    out = C.c_double()
    _check(lib().orc_eval_kernel(family, C.c_double(shape), C.c_double(r), C.byref(out)))
    return out.value


def kernel_radial_derivatives(family, shape, r0, count) -> np.ndarray:
    out = np.zeros(count)
    _check(lib().orc_kernel_radial_derivatives(family, C.c_double(shape), C.c_double(r0), count, _dp(out)))
    return out


def two_point_taylor(family, shape, eps_b, p):
    center, scale = C.c_double(), C.c_double()
    coeffs = np.zeros(2 * p + 2)
    cnt = C.c_int()
    _check(lib().orc_two_point_taylor(family, C.c_double(shape), C.c_double(eps_b), p, C.byref(center),
                                      C.byref(scale), _dp(coeffs), C.byref(cnt)))
    return center.value, scale.value, coeffs[:cnt.value].copy()


def regularized_value(family, shape, eps_b, p, r) -> np.ndarray:
    r = _f64(np.atleast_1d(r))
    out = np.zeros_like(r)
    _check(lib().orc_regularized_value(family, C.c_double(shape), C.c_double(eps_b), p, _dp(r),
                                       C.c_int64(r.size), _dp(out)))
    return out


def kernel_coefficients(family, shape, eps_b, p, d, N) -> np.ndarray:
    out = np.zeros(N ** d, np.complex128)
    _check(lib().orc_kernel_coefficients(family, C.c_double(shape), C.c_double(eps_b), p, d, N,
                                         _dp(out.view(np.float64))))
    return out


def trig_polynomial_value(coeffs, d, N, y) -> complex:
    c = _cplx_in(coeffs)
    yv = _f64(y)
    out = np.zeros(2)
    _check(lib().orc_trig_polynomial_value(_dp(c), d, N, _dp(yv), _dp(out)))
    return complex(out[0], out[1])


class FastsumPlan:
    """Mirror of ``fgs::FastsumPlan`` (fastsum.hpp:34-67) over the oracle."""

    def __init__(self, nodes, family, shape, N=32, m=4, p=4, eps_b=0.0, oversampling=2.0):
        nd, n, d = _nodes_colmajor(nodes)
        h = C.c_void_p()
        _check(lib().orc_fastsum_create(_dp(nd), C.c_int64(n), d, family, C.c_double(shape), N, m, p,
                                        C.c_double(eps_b), C.c_double(oversampling), C.byref(h)))
        self._h = h
        self.n, self.d, self.N = n, d, N
        rho, of, k0, ss = C.c_double(), C.c_double(), C.c_double(), C.c_double()
        _check(lib().orc_fastsum_info(h, C.byref(rho), C.byref(of), C.byref(k0), C.byref(ss)))
        self.scaling, self.output_factor, self.kernel_zero, self.scaled_shape = rho.value, of.value, k0.value, ss.value

    def __del__(self):
        if getattr(self, "_h", None):
            lib().orc_fastsum_destroy(self._h)
            self._h = None

    def apply(self, x) -> np.ndarray:
        xv = _f64(x)
        y = np.zeros(xv.size)
        _check(lib().orc_fastsum_apply(self._h, _dp(xv), C.c_int64(xv.size), _dp(y)))
        return y

    def coefficients(self) -> np.ndarray:
        out = np.zeros(self.N ** self.d, np.complex128)
        _check(lib().orc_fastsum_coefficients(self._h, _dp(out.view(np.float64))))
        return out

    def kernel_error_estimate(self, samples, seed) -> float:
        out = C.c_double()
        _check(lib().orc_fastsum_error_estimate(self._h, samples, C.c_uint64(seed), C.byref(out)))
        return out.value


def direct_apply(nodes, family, shape, x) -> np.ndarray:
    nd, n, d = _nodes_colmajor(nodes)
    xv = _f64(x)
    y = np.zeros(n)
    _check(lib().orc_direct_apply(_dp(nd), C.c_int64(n), d, family, C.c_double(shape), _dp(xv), _dp(y)))
    return y


class AdjacencyOperator:
    """Mirror of ``fgs::AdjacencyOperator`` (graphop.hpp:45-97) over the oracle."""

    def __init__(self, nodes, family, shape, N=32, m=4, p=4, eps_b=0.0, oversampling=2.0, direct=False):
        nd, n, d = _nodes_colmajor(nodes)
        h = C.c_void_p()
        bad = C.c_int64(-1)
        st = lib().orc_adjacency_create(_dp(nd), C.c_int64(n), d, family, C.c_double(shape), N, m, p,
                                        C.c_double(eps_b), C.c_double(oversampling), int(direct),
                                        C.byref(h), C.byref(bad))
        self.bad_node = bad.value
        _check(st)
        self._h = h
        self.n = n

    def __del__(self):
        if getattr(self, "_h", None):
            lib().orc_adjacency_destroy(self._h)
            self._h = None

    def _apply(self, op, x):
        xv = _f64(x)
        y = np.zeros(xv.size)
        _check(lib().orc_adjacency_apply(self._h, op, _dp(xv), C.c_int64(xv.size), _dp(y)))
        return y

    def apply_kernel(self, x):
        return self._apply(OP_KERNEL, x)

    def apply_weight(self, x):
        return self._apply(OP_WEIGHT, x)

    def apply_normalized(self, x):
        return self._apply(OP_NORMALIZED, x)

    def apply_sym_laplacian(self, x):
        return self._apply(OP_SYM_LAPLACIAN, x)

    def degrees(self) -> np.ndarray:
        out = np.zeros(self.n)
        _check(lib().orc_adjacency_degrees(self._h, _dp(out)))
        return out

    def lanczos_largest(self, k, max_iter=1000, tol=1e-12, seed=1, which=0):
        return _lanczos(lib().orc_lanczos_adjacency, (self._h, which), self.n, k, max_iter, tol, seed)


def _lanczos(fn, head, n, k, max_iter, tol, seed):
    values = np.zeros(k)
    vectors = np.zeros(n * k)
    cnt, it, conv = C.c_int(), C.c_int(), C.c_int()
    _check(fn(*head, k, max_iter, C.c_double(tol), C.c_uint64(seed), _dp(values), _dp(vectors),
              C.byref(cnt), C.byref(it), C.byref(conv)))
    c = cnt.value
    return values[:c].copy(), vectors[: n * c].reshape(c, n).T.copy(), it.value, bool(conv.value)


def lanczos_dense(A, k, max_iter=1000, tol=1e-12, seed=1):
    A = np.asfortranarray(np.asarray(A, dtype=np.float64))
    n = A.shape[0]
    flat = A.ravel(order="F").copy()
    return _lanczos(lib().orc_lanczos_dense, (_dp(flat), C.c_int64(n)), n, k, max_iter, tol, seed)


def tridiag_eig(diag, sub):
    diag = _f64(diag)
    sub = _f64(sub) if len(sub) else np.zeros(1)
    m = diag.size
    vals = np.zeros(m)
    vecs = np.zeros(m * m)
    _check(lib().orc_tridiag_eig(m, _dp(diag), _dp(sub), _dp(vals), _dp(vecs)))
    return vals, vecs.reshape(m, m).T.copy()


def make_eigenpairs(values, vectors):
    values = _f64(values)
    vectors = np.asfortranarray(np.asarray(vectors, dtype=np.float64))
    n, k = vectors.shape
    ov = np.zeros(k)
    ovec = np.zeros(n * k)
    flat = vectors.ravel(order="F").copy()
    _check(lib().orc_make_eigenpairs(_dp(values), _dp(flat), C.c_int64(n), k, _dp(ov), _dp(ovec)))
    return ov, ovec.reshape(k, n).T.copy()


# ---- reference-test input generators (same std::mt19937_64 streams) -------
def random_nodes(n, d, seed) -> np.ndarray:
    out = np.zeros(n * d)
    lib().orc_random_nodes(C.c_int64(n), d, C.c_uint64(seed), _dp(out))
    return out.reshape(d, n).T.copy()


def random_coeffs(count, seed) -> np.ndarray:
    out = np.zeros(2 * count)
    lib().orc_random_coeffs(C.c_int64(count), C.c_uint64(seed), _dp(out))
    return out.view(np.complex128).copy()


def random_cloud(n, d, extent, seed) -> np.ndarray:
    out = np.zeros(n * d)
    lib().orc_random_cloud(C.c_int64(n), d, C.c_double(extent), C.c_uint64(seed), _dp(out))
    return out.reshape(d, n).T.copy()


def random_vector(n, seed) -> np.ndarray:
    out = np.zeros(n)
    lib().orc_random_vector(C.c_int64(n), C.c_uint64(seed), _dp(out))
    return out


# ---- k-means / spectral clustering (learn.cpp:17-167, 441-486) -------------
def kmeans(points, k, restarts=10, max_iter=100, seed=1):
    """-> (labels int32[n], centroids [k][dim], wcss)."""
    pts = np.asarray(points, dtype=np.float64)
    pts = pts[:, None] if pts.ndim == 1 else pts
    n, dim = pts.shape
    col = np.asfortranarray(pts)
    labels = np.zeros(n, dtype=np.int32)
    cen = np.zeros(k * dim) if k > 0 else np.zeros(1)
    w = C.c_double()
    _check(lib().orc_kmeans(_dp(col), C.c_int64(n), int(dim), int(k), int(restarts), int(max_iter),
                            C.c_uint64(seed), labels.ctypes.data_as(C.POINTER(C.c_int)), _dp(cen), C.byref(w)))
    return labels, cen[:k * dim].reshape(dim, k).T.copy(), w.value


def spectral_cluster(vectors, k, restarts=10, max_iter=100, seed=1):
    v = np.asfortranarray(np.asarray(vectors, dtype=np.float64))
    n, kv = v.shape
    labels = np.zeros(n, dtype=np.int32)
    _check(lib().orc_spectral_cluster(_dp(v), C.c_int64(n), int(kv), int(k), int(restarts), int(max_iter),
                                      C.c_uint64(seed), labels.ctypes.data_as(C.POINTER(C.c_int))))
    return labels


def misclassification_rate(pred, truth, permuted=False):
    p = np.ascontiguousarray(pred, dtype=np.int32)
    t = np.ascontiguousarray(truth, dtype=np.int32)
    if p.shape != t.shape:
        raise OracleError(3, "label vectors differ in length")
    out = C.c_double()
    _check(lib().orc_misclassification(p.ctypes.data_as(C.POINTER(C.c_int)), t.ctypes.data_as(C.POINTER(C.c_int)),
                                       C.c_int64(p.size), int(permuted), C.byref(out)))
    return out.value


def blobs(counts, centers, spread, seed):
    """test_learn.cpp:23-39 -> (points [n][dim], labels)."""
    cts = np.ascontiguousarray(counts, dtype=np.int32)
    cen = np.ascontiguousarray(centers, dtype=np.float64)
    n, dim = int(cts.sum()), cen.shape[1]
    out = np.zeros(n * dim)
    labels = np.zeros(n, dtype=np.int32)
    lib().orc_blobs(cts.ctypes.data_as(C.POINTER(C.c_int)), len(cts), _dp(cen), int(dim), C.c_double(spread),
                    C.c_uint64(seed), _dp(out), labels.ctypes.data_as(C.POINTER(C.c_int)))
    return out.reshape(dim, n).T.copy(), labels


# ---- conjugate gradients (spectral.cpp:446-495) ------------------------------
def _cg(fn, h, f, beta, tol, max_iter):
    fv = _f64(f)
    x = np.zeros_like(fv)
    it, st = C.c_int(), C.c_int()
    _check(fn(h, _dp(fv), C.c_int64(fv.size), C.c_double(beta), C.c_double(tol), int(max_iter), _dp(x),
              C.byref(it), C.byref(st)))
    return x, it.value, st.value


def kernel_ssl_solve(adj, f, beta, tol=1e-8, max_iter=1000):
    """learn.cpp:364-381 -> (x, iterations, status 0/1/2)."""
    return _cg(lib().orc_kernel_ssl_solve, adj._h, f, beta, tol, max_iter)


def fastsum_ridge_solve(plan, f, beta, tol=1e-8, max_iter=1000):
    """(W~ + beta I) alpha = f, krr_fit's system (learn.cpp:403-430)."""
    return _cg(lib().orc_fastsum_ridge_solve, plan._h, f, beta, tol, max_iter)


# ---- nystrom_gaussian (spectral.cpp:384-444) ----------------------------------
def _nystrom(fn, head, n, k, L, M, seed):
    vals = np.zeros(k)
    vecs = np.zeros(n * k)
    _check(fn(*head, int(k), int(L), int(M), C.c_uint64(seed), _dp(vals), _dp(vecs)))
    return vals, vecs.reshape(k, n).T.copy()


def nystrom_dense(A, k, L, M, seed=1):
    A = np.asfortranarray(np.asarray(A, dtype=np.float64))
    n = A.shape[0]
    flat = A.ravel(order="F").copy()
    return _nystrom(lib().orc_nystrom_dense, (_dp(flat), C.c_int64(n)), n, k, L, M, seed)


def nystrom_adjacency(adj, n, k, L, M, seed=1):
    return _nystrom(lib().orc_nystrom_adjacency, (adj._h,), n, k, L, M, seed)


# ---- seeded BASELINE workloads (the same generator the product exports) ----
def workload_info(config: int) -> dict:
    n, d, N, m, p, k = C.c_int64(), C.c_int(), C.c_int(), C.c_int(), C.c_int(), C.c_int()
    sigma = C.c_double()
    _check(lib().fgs_workload_info(int(config), C.byref(n), C.byref(d), C.byref(sigma), C.byref(N), C.byref(m),
                                   C.byref(p), C.byref(k)))
    return dict(n=n.value, d=d.value, sigma=sigma.value, N=N.value, m=m.value, p=p.value, k=k.value)


def workload_nodes(config: int, seed: int = 2024, n: int = 0) -> np.ndarray:
    info = workload_info(config)
    npts = n or info["n"]
    out = np.zeros(npts * info["d"])
    _check(lib().fgs_workload_generate_n(int(config), C.c_uint64(seed), C.c_int64(n), _dp(out)))
    return out.reshape(info["d"], npts).T.copy()


def workload_vectors(n: int, nvec: int, seed: int) -> np.ndarray:
    out = np.zeros(n * nvec)
    _check(lib().fgs_workload_vectors(C.c_int64(n), int(nvec), C.c_uint64(seed), _dp(out)))
    return out.reshape(nvec, n).T if nvec > 1 else out
