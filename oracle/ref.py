"""ctypes front-end of oracle/_ref/libfgsref.so -- TEST INFRASTRUCTURE ONLY.

``libfgsref.so`` is the reference's OWN hot-path code
(/root/reference/proj/src/{nfft,kernels,fastsum,graphop,spectral}.cpp,
compiled unchanged against the Eigen/FFTW shim headers in oracle/shim by
oracle/build_ref.sh) behind the C layer oracle/ref_capi.cpp.  It is the root
of trust of the parity tests: tests/test_ref_pin.py pins the oracle
restatement (oracle.py) to it, and bench.py times it as the reference arm /
cpu_baseline (``"kind": "reference"``).  The classes mirror oracle.py's
(same constructor arguments and methods), so either can stand in for the
other.  Only tests/, __graft_entry__ and bench.py may import this module.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "_ref", "libfgsref.so")

OP_KERNEL, OP_WEIGHT, OP_NORMALIZED, OP_SYM_LAPLACIAN = 0, 1, 2, 3
KINDS = {1: "ParameterError", 2: "RangeError", 3: "ShapeError", 4: "NumericalError", 5: "ResourceError"}


class RefError(Exception):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{KINDS.get(code, code)}: {msg}")
        self.code = code
        self.kind = KINDS.get(code, str(code))
        self.msg = msg


def available() -> bool:
    return os.path.exists(_SO)


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise ImportError(f"{_SO} is missing: run oracle/build_ref.sh (needs /root/reference)")
        _lib = C.CDLL(_SO)
        _lib.ref_last_error.restype = C.c_char_p
    return _lib


_D = C.POINTER(C.c_double)


def _dp(a):
    return a.ctypes.data_as(_D)


def _check(st):
    if st != 0:
        raise RefError(st, lib().ref_last_error().decode())


def _nodes(nodes):
    a = np.asarray(nodes, dtype=np.float64)
    if a.ndim == 1:
        a = a[:, None]
    return np.asfortranarray(a).ravel(order="F").copy(), a.shape[0], a.shape[1]


def _f64(x):
    return np.ascontiguousarray(x, dtype=np.float64)


def _cplx(v):
    return np.ascontiguousarray(np.asarray(v, dtype=np.complex128)).view(np.float64).copy()


def _pairs(fn, head, n, k, max_iter, tol, seed):
    values = np.zeros(k)
    vectors = np.zeros(n * k)
    cnt, it, conv = C.c_int(), C.c_int(), C.c_int()
    _check(fn(*head, int(k), int(max_iter), C.c_double(tol), C.c_uint64(seed), _dp(values), _dp(vectors),
              C.byref(cnt), C.byref(it), C.byref(conv)))
    c = cnt.value
    return values[:c].copy(), vectors[: n * c].reshape(c, n).T.copy(), it.value, bool(conv.value)


class AdjacencyOperator:
    """fgs::AdjacencyOperator (graphop.hpp:45-97), the reference binary."""

    def __init__(self, nodes, family, shape, N=32, m=4, p=4, eps_b=0.0, oversampling=2.0, direct=False):
        nd, n, d = _nodes(nodes)
        h = C.c_void_p()
        bad = C.c_int64(-1)
        st = lib().ref_adjacency_create(_dp(nd), C.c_int64(n), d, family, C.c_double(shape), N, m, p,
                                        C.c_double(eps_b), C.c_double(oversampling), int(direct), C.byref(h),
                                        C.byref(bad))
        self.bad_node = bad.value
        _check(st)
        self._h = h
        self.n = n
        rho, of, k0 = C.c_double(), C.c_double(), C.c_double()
        _check(lib().ref_adjacency_info(h, C.byref(rho), C.byref(of), C.byref(k0)))
        self.scaling, self.output_factor, self.kernel_zero = rho.value, of.value, k0.value

    def __del__(self):
        if getattr(self, "_h", None):
            lib().ref_adjacency_destroy(self._h)
            self._h = None

    def _apply(self, op, x):
        xv = _f64(x)
        y = np.zeros(xv.size)
        _check(lib().ref_adjacency_apply(self._h, op, _dp(xv), C.c_int64(xv.size), _dp(y)))
        return y

    def apply_kernel(self, x):
        return self._apply(OP_KERNEL, x)

    def apply_weight(self, x):
        return self._apply(OP_WEIGHT, x)

    def apply_normalized(self, x):
        return self._apply(OP_NORMALIZED, x)

    def apply_sym_laplacian(self, x):
        return self._apply(OP_SYM_LAPLACIAN, x)

    def degrees(self):
        out = np.zeros(self.n)
        _check(lib().ref_adjacency_degrees(self._h, _dp(out)))
        return out

    def lanczos_largest(self, k, max_iter=1000, tol=1e-12, seed=1, which=0):
        """lanczos_largest(adjacency_handle(op) (which=0) | laplacian_handle(op))
        -> (values, vectors n x count, iterations, converged)."""
        return _pairs(lib().ref_lanczos_adjacency, (self._h, int(which)), self.n, k, max_iter, tol, seed)


def lanczos_dense(A, k, max_iter=1000, tol=1e-12, seed=1):
    A = np.asfortranarray(np.asarray(A, dtype=np.float64))
    n = A.shape[0]
    flat = A.ravel(order="F").copy()
    return _pairs(lib().ref_lanczos_dense, (_dp(flat), C.c_int64(n)), n, k, max_iter, tol, seed)


class FastsumPlan:
    """fgs::FastsumPlan (fastsum.hpp:34-67), the reference binary."""

    def __init__(self, nodes, family, shape, N=32, m=4, p=4, eps_b=0.0, oversampling=2.0):
        nd, n, d = _nodes(nodes)
        h = C.c_void_p()
        _check(lib().ref_fastsum_create(_dp(nd), C.c_int64(n), d, family, C.c_double(shape), N, m, p,
                                        C.c_double(eps_b), C.c_double(oversampling), C.byref(h)))
        self._h = h
        self.n, self.d, self.N = n, d, N
        rho, of, k0, ss = C.c_double(), C.c_double(), C.c_double(), C.c_double()
        _check(lib().ref_fastsum_info(h, C.byref(rho), C.byref(of), C.byref(k0), C.byref(ss)))
        self.scaling, self.output_factor, self.kernel_zero, self.scaled_shape = rho.value, of.value, k0.value, ss.value

    def __del__(self):
        if getattr(self, "_h", None):
            lib().ref_fastsum_destroy(self._h)
            self._h = None

    def apply(self, x):
        xv = _f64(x)
        y = np.zeros(xv.size)
        _check(lib().ref_fastsum_apply(self._h, _dp(xv), C.c_int64(xv.size), _dp(y)))
        return y

    def coefficients(self):
        out = np.zeros(self.N ** self.d, np.complex128)
        _check(lib().ref_fastsum_coefficients(self._h, _dp(out.view(np.float64))))
        return out


class NfftPlan:
    """fgs::NfftPlan (nfft.hpp:59-94), the reference binary."""

    def __init__(self, dims, bandwidth, cutoff, nodes, oversampling=2.0):
        nd, n, d = _nodes(nodes)
        h = C.c_void_p()
        _check(lib().ref_nfft_create(dims, bandwidth, cutoff, _dp(nd), C.c_int64(n), C.c_double(oversampling),
                                     C.byref(h)))
        self._h = h
        self.n = n
        M, cnt = C.c_int(), C.c_int64()
        _check(lib().ref_nfft_info(h, C.byref(M), C.byref(cnt)))
        self.grid_size, self.coefficient_count = M.value, cnt.value

    def __del__(self):
        if getattr(self, "_h", None):
            lib().ref_nfft_destroy(self._h)
            self._h = None

    def forward(self, fhat):
        f = _cplx(fhat)
        out = np.zeros(self.n, np.complex128)
        _check(lib().ref_nfft_forward(self._h, _dp(f), C.c_int64(f.size // 2), _dp(out.view(np.float64))))
        return out

    def adjoint(self, x):
        xv = _cplx(x)
        out = np.zeros(self.coefficient_count, np.complex128)
        _check(lib().ref_nfft_adjoint(self._h, _dp(xv), C.c_int64(xv.size // 2), _dp(out.view(np.float64))))
        return out

    def forward_real(self, fhat):
        f = _cplx(fhat)
        out = np.zeros(self.n)
        _check(lib().ref_nfft_forward_real(self._h, _dp(f), C.c_int64(f.size // 2), _dp(out)))
        return out


def direct_apply(nodes, family, shape, x):
    nd, n, d = _nodes(nodes)
    xv = _f64(x)
    y = np.zeros(n)
    _check(lib().ref_direct_apply(_dp(nd), C.c_int64(n), d, family, C.c_double(shape), _dp(xv), _dp(y)))
    return y
