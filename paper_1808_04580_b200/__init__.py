"""paper_1808_04580_b200 -- B200-native NFFT fast-summation graph operator.

Python mirror of the reference's hot-path interface (/root/reference/proj,
namespace ``fgs``) over the C ABI in ``include/fgs_b200.h``:

=======================  ==========================  ===========================
reference                this module                 C ABI
=======================  ==========================  ===========================
fgs::NfftPlan            NfftPlan                    fgs_nfft_*
fgs::FastsumParams       FastsumParams               fgs_fastsum_params
fgs::KernelSpec          KernelSpec                  fgs_kernel + shape
fgs::FastsumPlan         FastsumPlan                 fgs_fastsum_*
fgs::AdjacencyOperator   AdjacencyOperator           fgs_adjacency_*
fgs::lanczos_largest     lanczos_largest             fgs_lanczos_largest
fgs::make_eigenpairs,    EigenPairs,                 (host)
adjacency_to_laplacian   adjacency_to_laplacian
errors.hpp exceptions    ParameterError, ...         fgs_status codes
=======================  ==========================  ===========================

All compute runs in ``libfgs_b200.so`` (hand-written sm_100a CUDA + cuFFT);
there is no CPU fallback: importing works anywhere, but constructing a plan
without a CUDA device raises ``CudaError``.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libfgs_b200.so")


# ---- errors (errors.hpp:8-49) -------------------------------------------
class FgsError(Exception):
    """Base of the reference's exception hierarchy mirror."""


class ParameterError(FgsError, ValueError):
    pass


class RangeError(FgsError, ValueError):
    pass


class ShapeError(FgsError, ValueError):
    pass


class NumericalError(FgsError, RuntimeError):
    def __init__(self, msg, bad_node=-1):
        super().__init__(msg)
        self.bad_node = bad_node


class ResourceError(FgsError, RuntimeError):
    pass


class CudaError(FgsError, RuntimeError):
    pass


class NcclError(FgsError, RuntimeError):
    pass


_ERRORS = {1: ParameterError, 2: RangeError, 3: ShapeError, 4: NumericalError, 5: ResourceError,
           6: CudaError, 7: NcclError}

GAUSSIAN, LAPLACIAN_RBF, MULTIQUADRIC, INV_MULTIQUADRIC = 0, 1, 2, 3
OP_KERNEL, OP_WEIGHT, OP_NORMALIZED, OP_SYM_LAPLACIAN = 0, 1, 2, 3

_lib = None


class _Params(C.Structure):
    _fields_ = [("bandwidth", C.c_int), ("cutoff", C.c_int), ("smoothness", C.c_int),
                ("eps_b", C.c_double), ("oversampling", C.c_double)]


def lib():
    """Load libfgs_b200.so (fails loudly if the extension is not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_1808_04580_b200.build` "
                              "(or __graft_entry__.build())")
        L = C.CDLL(LIB_PATH)
        L.fgs_last_error.restype = C.c_char_p
        _lib = L
    return _lib


def _check(status, bad_node=-1):
    if status != 0:
        msg = lib().fgs_last_error().decode()
        cls = _ERRORS.get(status, FgsError)
        if cls is NumericalError:
            raise NumericalError(msg, bad_node)
        raise cls(msg)


_D = C.POINTER(C.c_double)


def _dp(a):
    return a.ctypes.data_as(_D)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _nodes(nodes):
    a = np.asarray(nodes, dtype=np.float64)
    if a.ndim == 1:
        a = a[:, None]
    n, d = a.shape
    return np.asfortranarray(a).ravel(order="F").copy(), n, d


# ---- parameters (fastsum.hpp:13-23, kernels.hpp:27-35) ------------------
@dataclass
class FastsumParams:
    bandwidth: int = 32
    cutoff: int = 4
    smoothness: int = 4
    eps_b: float = 0.0
    oversampling: float = 2.0

    @staticmethod
    def preset(level: int, eps_b: float = 0.0) -> "FastsumParams":
        p = _Params()
        _check(lib().fgs_fastsum_preset(int(level), C.c_double(eps_b), C.byref(p)))
        return FastsumParams(p.bandwidth, p.cutoff, p.smoothness, p.eps_b, p.oversampling)

    def _c(self):
        return _Params(self.bandwidth, self.cutoff, self.smoothness, self.eps_b, self.oversampling)


@dataclass
class KernelSpec:
    family: int = GAUSSIAN
    shape: float = 1.0

    @staticmethod
    def gaussian(sigma):
        return KernelSpec(GAUSSIAN, sigma)

    @staticmethod
    def laplacian_rbf(sigma):
        return KernelSpec(LAPLACIAN_RBF, sigma)

    @staticmethod
    def multiquadric(c):
        return KernelSpec(MULTIQUADRIC, c)

    @staticmethod
    def inverse_multiquadric(c):
        return KernelSpec(INV_MULTIQUADRIC, c)


def bessel_i0(x: float) -> float:
    out = C.c_double()
    _check(lib().fgs_bessel_i0(C.c_double(x), C.byref(out)))
    return out.value


# ---- NfftPlan (nfft.hpp:59-94) ------------------------------------------
class NfftPlan:
    def __init__(self, dims, bandwidth, cutoff, nodes, oversampling=2.0, device=0):
        nd, n, d = _nodes(nodes)
        h = C.c_void_p()
        _check(lib().fgs_nfft_create(int(dims), int(bandwidth), int(cutoff), _dp(nd), C.c_int64(n),
                                     C.c_double(oversampling), int(device), C.byref(h)))
        self._h = h
        self._n = n
        M = C.c_int()
        F = C.c_int64()
        _check(lib().fgs_nfft_info(h, C.byref(M), C.byref(F)))
        self._M, self._F = M.value, F.value
        self._d, self._N, self._m = dims, bandwidth, cutoff

    def __del__(self):
        if getattr(self, "_h", None):
            try:
                lib().fgs_nfft_destroy(self._h)
            except Exception:  # noqa: BLE001 - interpreter teardown: module globals already gone
                pass
            self._h = None

    def dims(self):
        return self._d

    def bandwidth(self):
        return self._N

    def cutoff(self):
        return self._m

    def node_count(self):
        return self._n

    def coefficient_count(self):
        return self._F

    def grid_size(self):
        return self._M

    def forward(self, fhat) -> np.ndarray:
        f = np.ascontiguousarray(fhat, dtype=np.complex128)
        out = np.zeros(self._n, np.complex128)
        _check(lib().fgs_nfft_forward(self._h, _dp(f.view(np.float64)), C.c_int64(f.size),
                                      _dp(out.view(np.float64))))
        return out

    def adjoint(self, x) -> np.ndarray:
        xv = np.ascontiguousarray(x, dtype=np.complex128)
        out = np.zeros(self._F, np.complex128)
        _check(lib().fgs_nfft_adjoint(self._h, _dp(xv.view(np.float64)), C.c_int64(xv.size),
                                      _dp(out.view(np.float64))))
        return out

    def forward_real(self, fhat) -> np.ndarray:
        f = np.ascontiguousarray(fhat, dtype=np.complex128)
        out = np.zeros(self._n)
        _check(lib().fgs_nfft_forward_real(self._h, _dp(f.view(np.float64)), C.c_int64(f.size), _dp(out)))
        return out


# ---- FastsumPlan (fastsum.hpp:34-67) ------------------------------------
class FastsumPlan:
    def __init__(self, nodes, kernel: KernelSpec, params: FastsumParams = None, device=0):
        params = params or FastsumParams()
        nd, n, d = _nodes(nodes)
        h = C.c_void_p()
        cp = params._c()
        _check(lib().fgs_fastsum_create(_dp(nd), C.c_int64(n), int(d), int(kernel.family),
                                        C.c_double(kernel.shape), C.byref(cp), int(device), C.byref(h)))
        self._h = h
        self._n, self._d = n, d
        self._params = params
        self._kernel = kernel
        rho, of, k0, ss = C.c_double(), C.c_double(), C.c_double(), C.c_double()
        _check(lib().fgs_fastsum_info(h, C.byref(rho), C.byref(of), C.byref(k0), C.byref(ss)))
        self._rho, self._of, self._k0, self._ss = rho.value, of.value, k0.value, ss.value

    def __del__(self):
        if getattr(self, "_h", None):
            try:
                lib().fgs_fastsum_destroy(self._h)
            except Exception:  # noqa: BLE001 - interpreter teardown: module globals already gone
                pass
            self._h = None

    def size(self):
        return self._n

    def dims(self):
        return self._d

    def params(self):
        return self._params

    def kernel(self):
        return self._kernel

    def scaled_kernel(self):
        return KernelSpec(self._kernel.family, self._ss)

    def scaling(self):
        return self._rho

    def output_factor(self):
        return self._of

    def kernel_zero(self):
        return self._k0

    def coefficients(self) -> np.ndarray:
        out = np.zeros(self._params.bandwidth ** self._d, np.complex128)
        _check(lib().fgs_fastsum_coefficients(self._h, _dp(out.view(np.float64))))
        return out

    def apply(self, x) -> np.ndarray:
        xv = _f64(x)
        y = np.zeros(xv.size)
        _check(lib().fgs_fastsum_apply(self._h, _dp(xv), C.c_int64(xv.size), _dp(y)))
        return y

    def kernel_error_estimate(self, sample_count, seed) -> float:
        out = C.c_double()
        _check(lib().fgs_fastsum_error_estimate(self._h, int(sample_count), C.c_uint64(seed), C.byref(out)))
        return out.value


# ---- AdjacencyOperator (graphop.hpp:45-97) ------------------------------
BACKEND_FASTSUM, BACKEND_DIRECT = "fastsum", "direct"  # AdjacencyBackend (graphop.hpp:19-22)


class AdjacencyOperator:
    """graphop.hpp:45-97.  backend "fastsum" (default) or "direct" (the exact
    O(n^2) sum, graphop.cpp:29-34)."""

    def __init__(self, nodes, kernel: KernelSpec, params: FastsumParams = None, device=0,
                 rank=0, world=1, nccl_id: bytes = None, backend: str = BACKEND_FASTSUM):
        params = params or FastsumParams()
        nd, n, d = _nodes(nodes)
        h = C.c_void_p()
        bad = C.c_int64(-1)
        cp = params._c()
        self.backend = backend
        if backend == BACKEND_DIRECT:
            if world > 1 or nccl_id is not None:
                raise ParameterError("the direct backend is single-device")
            st = lib().fgs_adjacency_create_direct(_dp(nd), C.c_int64(n), int(d), int(kernel.family),
                                                   C.c_double(kernel.shape), int(device), C.byref(h),
                                                   C.byref(bad))
        elif backend != BACKEND_FASTSUM:
            raise ParameterError(f"unknown adjacency backend {backend!r}")
        elif world > 1 or nccl_id is not None:
            idbuf = C.create_string_buffer(bytes(nccl_id), 128)
            st = lib().fgs_adjacency_create_sharded(_dp(nd), C.c_int64(n), int(d), int(kernel.family),
                                                    C.c_double(kernel.shape), C.byref(cp), int(device),
                                                    int(rank), int(world), idbuf, C.byref(h), C.byref(bad))
        else:
            st = lib().fgs_adjacency_create(_dp(nd), C.c_int64(n), int(d), int(kernel.family),
                                            C.c_double(kernel.shape), C.byref(cp), int(device), C.byref(h),
                                            C.byref(bad))
        _check(st, bad.value)
        self._h = h
        self._n, self._d = n, d
        self._kernel, self._params = kernel, params
        rho, of, k0 = C.c_double(), C.c_double(), C.c_double()
        nl, off = C.c_int64(), C.c_int64()
        _check(lib().fgs_adjacency_info(h, C.byref(rho), C.byref(of), C.byref(k0), C.byref(nl), C.byref(off)))
        self._k0 = k0.value
        self.n_local, self.offset = nl.value, off.value
        self.world = world

    def __del__(self):
        if getattr(self, "_h", None):
            try:
                lib().fgs_adjacency_destroy(self._h)
            except Exception:  # noqa: BLE001 - interpreter teardown: module globals already gone
                pass
            self._h = None

    @property
    def handle(self):
        return self._h

    def size(self):
        return self._n

    def dims(self):
        return self._d

    def kernel(self):
        return self._kernel

    def kernel_zero(self):
        return self._k0

    def degrees(self) -> np.ndarray:
        out = np.zeros(self._n)
        _check(lib().fgs_adjacency_degrees(self._h, _dp(out)))
        return out

    def _apply(self, op, x):
        xv = np.asarray(x, dtype=np.float64)
        block = xv.ndim == 2
        xm = np.asfortranarray(xv if block else xv[:, None])
        if xm.shape[0] != self._n:
            raise ShapeError("input length does not match operator dimension")
        ym = np.zeros_like(xm, order="F")
        _check(lib().fgs_adjacency_apply(self._h, int(op), _dp(xm), _dp(ym), int(xm.shape[1]),
                                         C.c_int64(self._n)))
        return ym if block else ym[:, 0].copy()

    def apply_kernel(self, x):
        return self._apply(OP_KERNEL, x)

    def apply_weight(self, x):
        return self._apply(OP_WEIGHT, x)

    def apply_normalized(self, x):
        return self._apply(OP_NORMALIZED, x)

    def apply_sym_laplacian(self, x):
        return self._apply(OP_SYM_LAPLACIAN, x)

    def apply_device(self, op, dx_ptr: int, dy_ptr: int, nvec=1, ld=None, internal_order=True):
        ld = ld if ld is not None else (self.n_local if internal_order else self._n)
        _check(lib().fgs_adjacency_apply_device(self._h, int(op), C.c_void_p(dx_ptr), C.c_void_p(dy_ptr),
                                                int(nvec), C.c_int64(ld), int(bool(internal_order))))

    def permute_device(self, dx_ptr: int, dy_ptr: int, nvec=1, ld=None, direction=0):
        ld = ld if ld is not None else self._n
        _check(lib().fgs_adjacency_permute_device(self._h, C.c_void_p(dx_ptr), C.c_void_p(dy_ptr), int(nvec),
                                                  C.c_int64(ld), int(direction)))

    def set_stream(self, stream_ptr: int):
        _check(lib().fgs_adjacency_set_stream(self._h, C.c_void_p(stream_ptr)))

    def profile(self, enable: bool):
        _check(lib().fgs_adjacency_profile(self._h, int(bool(enable))))

    def profile_read(self):
        """(ms per stage summed since last read, applies covered); stages =
        spread, assemble, r2c, multiply, c2r, interp."""
        ms = np.zeros(6)
        n = C.c_int64()
        _check(lib().fgs_adjacency_profile_read(self._h, _dp(ms), C.byref(n)))
        return ms, n.value

    def geometry(self) -> dict:
        d, N, M, T, items = C.c_int(), C.c_int(), C.c_int(), C.c_int(), C.c_int()
        bs = C.c_int64()
        _check(lib().fgs_adjacency_geometry(self._h, C.byref(d), C.byref(N), C.byref(M), C.byref(T),
                                            C.byref(items), C.byref(bs)))
        return dict(d=d.value, N=N.value, M=M.value, taps=T.value, items=items.value, box_stride=bs.value)

    def plan_stats(self) -> dict:
        """mean points per run and whether the DMMA spread / interpolation run."""
        mr, ts, ti = C.c_double(), C.c_int(), C.c_int()
        _check(lib().fgs_adjacency_plan_stats(self._h, C.byref(mr), C.byref(ts), C.byref(ti)))
        sl, ns = C.c_int(), C.c_int64()
        _check(lib().fgs_adjacency_plan_layout(self._h, C.byref(sl), C.byref(ns)))
        return dict(mean_run=mr.value, tensor_spread=bool(ts.value), tensor_interp=bool(ti.value),
                    slot_layout=bool(sl.value), slots=ns.value)

    def lanczos_stats(self) -> dict:
        out = np.zeros(4)
        _check(lib().fgs_lanczos_stats(self._h, _dp(out)))
        return dict(apply_ms=out[0], reorth_ms=out[1], loop_ms=out[2], iterations=int(out[3]))

    def launch_count(self) -> int:
        out = C.c_int64()
        _check(lib().fgs_adjacency_launch_count(self._h, C.byref(out)))
        return out.value


STAGES = ("spread", "assemble", "fft_r2c", "multiply", "fft_c2r", "interp")


def measure_fp64_peak(device=0) -> float:
    out = C.c_double()
    _check(lib().fgs_measure_fp64_peak(int(device), C.byref(out)))
    return out.value


def measure_dmma_peak(device=0) -> float:
    """fp64 tensor-core (DMMA m8n8k4) peak of `device` in TFLOP/s."""
    out = C.c_double()
    _check(lib().fgs_measure_dmma_peak(int(device), C.byref(out)))
    return out.value


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(lib().fgs_nccl_unique_id(buf))
    return buf.raw


# ---- spectral (spectral.hpp:33-70) --------------------------------------
class ShardGroup:
    """Single-GPU emulation of the N-rank sharded path (fgs_shard_group_*):
    `world` shards of one operator on one device, the ranks' exchange summed
    by a device kernel between the two apply phases.  Validates the
    multi-GPU data path (plan slices, slab-pruned convolutions, exchange
    layout) where fewer GPUs than ranks exist."""

    def __init__(self, nodes, kernel: KernelSpec, params: FastsumParams = None, device=0, world=2):
        params = params or FastsumParams()
        nd, n, d = _nodes(nodes)
        h = C.c_void_p()
        bad = C.c_int64(-1)
        cp = params._c()
        st = lib().fgs_shard_group_create(_dp(nd), C.c_int64(n), int(d), int(kernel.family),
                                          C.c_double(kernel.shape), C.byref(cp), int(device), int(world),
                                          C.byref(h), C.byref(bad))
        _check(st, bad.value)
        self._h = h
        self._n, self.world = n, world

    def __del__(self):
        if getattr(self, "_h", None):
            try:
                lib().fgs_shard_group_destroy(self._h)
            except Exception:  # noqa: BLE001 - interpreter teardown: module globals already gone
                pass
            self._h = None

    def apply_device(self, op, dx_ptr: int, dy_ptr: int, nvec=1, ld=None):
        """y = op(x) for full-length device vectors in caller order."""
        ld = ld if ld is not None else self._n
        _check(lib().fgs_shard_group_apply_device(self._h, int(op), C.c_void_p(dx_ptr), C.c_void_p(dy_ptr),
                                                  int(nvec), C.c_int64(ld)))

    def profile(self, op, dx_ptr: int, dy_ptr: int, nvec=1, ld=None, reps=3):
        """(per-shard ms per apply, exchange ms): CUDA events around each
        shard's phases -- what rank r computes on its own GPU."""
        ld = ld if ld is not None else self._n
        ms = np.zeros(self.world)
        ex = C.c_double()
        _check(lib().fgs_shard_group_profile(self._h, int(op), C.c_void_p(dx_ptr), C.c_void_p(dy_ptr), int(nvec),
                                             C.c_int64(ld), int(reps), _dp(ms), C.byref(ex)))
        return ms, ex.value

    def stage_profile(self, op, dx_ptr: int, dy_ptr: int, nvec=1, ld=None, reps=3):
        """[world][6] mean ms per apply: spread, assembly, forward planes,
        lines (+ exchange and the other shards' work between), inverse
        planes, interpolation."""
        ld = ld if ld is not None else self._n
        ms = np.zeros((self.world, 6))
        _check(lib().fgs_shard_group_stage_profile(self._h, int(op), C.c_void_p(dx_ptr), C.c_void_p(dy_ptr),
                                                   int(nvec), C.c_int64(ld), int(reps), _dp(ms)))
        return ms

    def stats(self, rank: int) -> dict:
        nl, p0, pn, it = C.c_int64(), C.c_int(), C.c_int(), C.c_int()
        _check(lib().fgs_shard_group_stats(self._h, int(rank), C.byref(nl), C.byref(p0), C.byref(pn), C.byref(it)))
        return dict(n_local=nl.value, conv_plane0=p0.value, conv_planes=pn.value, items=it.value)


@dataclass
class LanczosOptions:
    max_iter: int = 1000
    tol: float = 1e-12
    seed: int = 1


@dataclass
class LanczosInfo:
    iterations: int = 0
    converged: bool = False


@dataclass
class EigenPairs:
    values: np.ndarray
    vectors: np.ndarray

    def count(self):
        return self.values.size


def lanczos_largest(op: AdjacencyOperator, k: int, opts: LanczosOptions = None, info: LanczosInfo = None,
                    which: int = 0, want_vectors: bool = True) -> EigenPairs:
    """k largest Ritz pairs of A = D^-1/2 W D^-1/2 (which=0, adjacency_handle)
    or of L_s (which=1, laplacian_handle), device-resident Lanczos."""
    opts = opts or LanczosOptions()
    n = op.size()
    values = np.zeros(max(k, 1))
    vectors = np.empty((n, max(k, 1)), order="F") if want_vectors else None  # fully written by the library
    cnt, it, conv = C.c_int(), C.c_int(), C.c_int()
    _check(lib().fgs_lanczos_largest(op.handle, int(which), int(k), int(opts.max_iter), C.c_double(opts.tol),
                                     C.c_uint64(opts.seed), _dp(values),
                                     _dp(vectors) if want_vectors else None,
                                     C.byref(cnt), C.byref(it), C.byref(conv)))
    if info is not None:
        info.iterations, info.converged = it.value, bool(conv.value)
    c = cnt.value
    vecs = None
    if want_vectors:
        vecs = vectors if c == vectors.shape[1] else vectors[:, :c].copy()
    return EigenPairs(values[:c].copy(), vecs)


def adjacency_to_laplacian(pairs: EigenPairs) -> EigenPairs:
    """spectral.cpp:129-139: lambda_L = 1 - lambda_A, ascending."""
    k = pairs.count()
    vals = np.array([1.0 - pairs.values[k - 1 - i] for i in range(k)])
    vecs = None if pairs.vectors is None else pairs.vectors[:, ::-1].copy()
    return EigenPairs(vals, vecs)


# ---- Nystrom (spectral.hpp:81-86, spectral.cpp:384-444) -------------------
@dataclass
class NystromOptions:
    k: int = 10
    L: int = 100
    M: int = 10
    seed: int = 1


def nystrom_gaussian(op: AdjacencyOperator, opts: NystromOptions = None) -> EigenPairs:
    """k approximate eigenpairs of A from a Gaussian sketch (2L fast applies,
    as block applies on the device)."""
    opts = opts or NystromOptions()
    n = op.size()
    vals = np.zeros(max(opts.k, 1))
    vecs = np.zeros((n, max(opts.k, 1)), order="F")
    _check(lib().fgs_nystrom_gaussian(op.handle, int(opts.k), int(opts.L), int(opts.M), C.c_uint64(opts.seed),
                                      _dp(vals), _dp(vecs)))
    return EigenPairs(vals[:opts.k].copy(), vecs[:, :opts.k].copy())


# ---- conjugate gradients and its consumers (spectral.hpp:120-140) ---------
CG_CONVERGED, CG_MAX_ITERATIONS, CG_INDEFINITE = 0, 1, 2  # CgStatus


@dataclass
class CgResult:
    x: np.ndarray
    iterations: int = 0
    status: int = CG_MAX_ITERATIONS

    def converged(self) -> bool:
        return self.status == CG_CONVERGED


def _cg_call(fn, h, f, beta, tol, max_iter, n):
    fv = np.ascontiguousarray(f, dtype=np.float64)
    if fv.size != n:
        raise ShapeError("fidelity length does not match operator dimension")
    x = np.zeros(n)
    it, st = C.c_int(), C.c_int()
    _check(fn(h, _dp(fv), C.c_int64(fv.size), C.c_double(beta), C.c_double(tol), int(max_iter), _dp(x),
              C.byref(it), C.byref(st)))
    return CgResult(x, it.value, st.value)


def kernel_ssl_solve(op: AdjacencyOperator, f, beta: float, tol: float = 1e-4, max_iter: int = 1000) -> CgResult:
    """learn.cpp:364-381: (I + beta L_s) x = f by CG on the device."""
    return _cg_call(lib().fgs_kernel_ssl_solve, op.handle, f, beta, tol, max_iter, op.size())


def kernel_ssl_truncated(pairs: "EigenPairs", f, beta: float) -> np.ndarray:
    """learn.cpp:383-394: the same system solved in a truncated eigenbasis
    of A (O(n k) host arithmetic on the Lanczos output)."""
    if not beta >= 0.0:
        raise ParameterError("beta must be nonnegative")
    fv = np.asarray(f, dtype=np.float64)
    V, lam = pairs.vectors, pairs.values
    if V is not None and V.shape[1] > 0 and V.shape[0] != fv.size:
        raise ShapeError("fidelity length does not match eigenvectors")
    coords = V.T @ fv
    inside = coords / (1.0 + beta * (1.0 - lam))
    return V @ inside + (fv - V @ coords) / (1.0 + beta)


@dataclass
class RidgeModel:
    train_nodes: np.ndarray
    kernel: KernelSpec
    params: FastsumParams
    beta: float
    alpha: np.ndarray
    cg_iterations: int
    cg_tol: float


def krr_fit(train_nodes, kernel: KernelSpec, beta: float, f, params: FastsumParams = None, tol: float = 1e-6,
            max_iter: int = 1000, device: int = 0) -> RidgeModel:
    """learn.cpp:403-430: (W~ + beta I) alpha = f by CG on a device FastsumPlan."""
    if not beta > 0.0:
        raise ParameterError("beta must be positive")
    params = params or FastsumParams()
    X = np.asarray(train_nodes, dtype=np.float64)
    X = X[:, None] if X.ndim == 1 else X
    if np.asarray(f).size != X.shape[0]:
        raise ShapeError("target length does not match training node count")
    plan = FastsumPlan(X, kernel, params, device)
    cg = _cg_call(lib().fgs_fastsum_ridge_solve, plan._h, f, beta, tol, max_iter, X.shape[0])
    if cg.status == CG_INDEFINITE:
        raise NumericalError("regularized Gram operator is indefinite for this kernel; solve dense regularized "
                             "normal equations instead")
    return RidgeModel(X.copy(), kernel, params, beta, cg.x, cg.iterations, tol)


def krr_predict(model: RidgeModel, query_nodes, device: int = 0) -> np.ndarray:
    """learn.cpp:432-445: one fast summation over train + query nodes."""
    Q = np.asarray(query_nodes, dtype=np.float64)
    Q = Q[:, None] if Q.ndim == 1 else Q
    if Q.shape[1] != model.train_nodes.shape[1]:
        raise ShapeError("query dimension does not match training dimension")
    allx = np.concatenate([model.train_nodes, Q])
    plan = FastsumPlan(allx, model.kernel, model.params, device)
    masked = np.zeros(allx.shape[0])
    masked[:model.train_nodes.shape[0]] = model.alpha
    return plan.apply(masked)[model.train_nodes.shape[0]:]


# ---- k-means / spectral clustering (learn.hpp, learn.cpp:17-167) ----------
@dataclass
class KMeansOptions:
    restarts: int = 10
    max_iter: int = 100
    seed: int = 1


@dataclass
class KMeansResult:
    labels: np.ndarray     # int32 [n]
    centroids: np.ndarray  # [k][dim]
    wcss: float


def _ip(a):
    return a.ctypes.data_as(C.POINTER(C.c_int))


def kmeans(points, k: int, opts: KMeansOptions = None, device: int = 0) -> KMeansResult:
    """learn.cpp:140-155 on the device (k-means++ seeding, Lloyd, restarts)."""
    opts = opts or KMeansOptions()
    pts = np.asarray(points, dtype=np.float64)
    pts = pts[:, None] if pts.ndim == 1 else pts
    n, dim = pts.shape
    col = np.asfortranarray(pts)
    labels = np.zeros(n, dtype=np.int32)
    cen = np.zeros(max(k, 1) * dim)
    w = C.c_double()
    _check(lib().fgs_kmeans(_dp(col), C.c_int64(n), int(dim), int(k), int(opts.restarts), int(opts.max_iter),
                            C.c_uint64(opts.seed), int(device), _ip(labels), _dp(cen), C.byref(w)))
    return KMeansResult(labels, cen[:k * dim].reshape(dim, k).T.copy(), w.value)


def spectral_cluster(pairs, k_clusters: int, opts: KMeansOptions = None, device: int = 0) -> np.ndarray:
    """learn.cpp:157-167: unit rows of the eigenvectors, then k-means.
    ``pairs`` is an EigenPairs or an n x kv array."""
    opts = opts or KMeansOptions()
    vecs = pairs.vectors if isinstance(pairs, EigenPairs) else pairs
    v = np.asfortranarray(np.asarray(vecs, dtype=np.float64))
    n, kv = v.shape
    labels = np.zeros(n, dtype=np.int32)
    _check(lib().fgs_spectral_cluster(_dp(v), C.c_int64(n), int(kv), int(k_clusters), int(opts.restarts),
                                      int(opts.max_iter), C.c_uint64(opts.seed), int(device), 0, _ip(labels)))
    return labels


def misclassification_rate(predicted, truth) -> float:
    """learn.cpp:441-450."""
    return _misclass(predicted, truth, 0)


def misclassification_rate_permuted(predicted, truth) -> float:
    """learn.cpp:452-486 (best relabeling, at most 8 classes)."""
    return _misclass(predicted, truth, 1)


def _misclass(predicted, truth, permuted):
    p = np.ascontiguousarray(predicted, dtype=np.int32)
    t = np.ascontiguousarray(truth, dtype=np.int32)
    if p.shape != t.shape:
        raise ShapeError("label vectors differ in length")
    out = C.c_double()
    _check(lib().fgs_misclassification_rate(_ip(p), _ip(t), C.c_int64(p.size), int(permuted), C.byref(out)))
    return out.value


# ---- synthetic BASELINE workloads ----------------------------------------
def workload_info(config: int) -> dict:
    n, d, N, m, p, k = C.c_int64(), C.c_int(), C.c_int(), C.c_int(), C.c_int(), C.c_int()
    sigma = C.c_double()
    _check(lib().fgs_workload_info(int(config), C.byref(n), C.byref(d), C.byref(sigma), C.byref(N), C.byref(m),
                                   C.byref(p), C.byref(k)))
    return dict(n=n.value, d=d.value, sigma=sigma.value, N=N.value, m=m.value, p=p.value, k=k.value)


def workload_nodes(config: int, seed: int = 2024, n: int = 0) -> np.ndarray:
    """Seeded synthetic nodes of BASELINE config 1..5 (n > 0: that many
    points from the same generator, e.g. config 5's weak scaling)."""
    info = workload_info(config)
    npts = n or info["n"]
    out = np.zeros(npts * info["d"])
    _check(lib().fgs_workload_generate_n(int(config), C.c_uint64(seed), C.c_int64(n), _dp(out)))
    return out.reshape(info["d"], npts).T.copy()


def workload_vectors(n: int, nvec: int, seed: int) -> np.ndarray:
    out = np.zeros(n * nvec)
    _check(lib().fgs_workload_vectors(C.c_int64(n), int(nvec), C.c_uint64(seed), _dp(out)))
    # column-major (n, nvec): vector j contiguous, the layout the C ABI takes
    return out.reshape(nvec, n).T if nvec > 1 else out
