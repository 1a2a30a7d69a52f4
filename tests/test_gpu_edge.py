"""Edge cases of the device path against the CPU oracle: coincident and
duplicated points, d = 1, eps_b > 0 blends, every kernel family, non-power-
of-two grids, large cutoffs (runtime-2m kernels), NaN / out-of-range nodes,
block vectors with ld > n through the raw C ABI, caller-order device apply."""
import ctypes as C

import numpy as np
import pytest

import paper_1808_04580_b200 as fgs

pytestmark = pytest.mark.gpu


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def _pair(orc, X, fam, shape, N, m, p=None, eps_b=0.0, os_=2.0):
    p = p or min(m, 8)
    op = fgs.AdjacencyOperator(X, fgs.KernelSpec(fam, shape), fgs.FastsumParams(N, m, p, eps_b, os_))
    ref = orc.AdjacencyOperator(X, fam, shape, N=N, m=m, p=p, eps_b=eps_b, oversampling=os_)
    return op, ref


def _check_ops(op, ref, n, seed=1, tol=1e-10):
    x = np.random.default_rng(seed).standard_normal(n)
    assert rel(op.degrees(), ref.degrees()) <= tol
    for name in ("apply_kernel", "apply_weight", "apply_normalized", "apply_sym_laplacian"):
        assert rel(getattr(op, name)(x), getattr(ref, name)(x)) <= tol, name


def test_duplicated_points(orc):
    rng = np.random.default_rng(2)
    base = rng.uniform(-0.2, 0.2, (300, 3))
    X = np.concatenate([base, base[:100], np.zeros((50, 3))])  # exact duplicates + a 50-fold point
    op, ref = _pair(orc, X, 0, 0.3, 32, 4)
    _check_ops(op, ref, X.shape[0])


@pytest.mark.parametrize("fam,shape", [(0, 0.7), (1, 1.0), (2, 0.5), (3, 0.5)])
def test_one_dimensional_every_family(orc, fam, shape):
    X = np.random.default_rng(3).uniform(-1, 1, (800, 1))
    op, ref = _pair(orc, X, fam, shape, 64, 6)
    _check_ops(op, ref, 800)


def test_blend_eps_b_positive_3d(orc):
    X = np.random.default_rng(4).uniform(-1, 1, (1500, 3))
    op, ref = _pair(orc, X, 0, 1.0, 64, 7, p=7, eps_b=0.125)  # preset 3 with a blend (test_graphop tight)
    _check_ops(op, ref, 1500)


def test_non_power_of_two_grid(orc):
    X = np.random.default_rng(5).uniform(-0.3, 0.3, (700, 2))
    op, ref = _pair(orc, X, 0, 0.4, 10, 3, os_=1.7)  # M = 2 ceil(8.5) = 18
    _check_ops(op, ref, 700)


@pytest.mark.parametrize("d,m", [(2, 10), (3, 9)])
def test_large_cutoff_runtime_kernels(orc, d, m):
    X = np.random.default_rng(6).uniform(-0.2, 0.2, (600, d))
    op, ref = _pair(orc, X, 0, 0.3, 16, m, p=8)
    _check_ops(op, ref, 600)


@pytest.mark.parametrize("d", [2, 3])
def test_block_vectors_dense_paths(orc, d):
    X = np.random.default_rng(7).uniform(-0.1, 0.1, (4000, d))  # dense cells -> tensor-core kernels
    N, m = (64, 6) if d == 2 else (32, 8)
    op, ref = _pair(orc, X, 0, 0.05, N, m)
    B = np.random.default_rng(8).standard_normal((4000, 3))
    Y = op.apply_sym_laplacian(B)
    for j in range(3):
        assert rel(Y[:, j], ref.apply_sym_laplacian(B[:, j])) <= 1e-10


def test_nan_and_out_of_range_nodes_raise_range_error(orc):
    X = np.random.default_rng(9).uniform(-0.2, 0.2, (50, 2))
    X[7, 1] = np.nan
    with pytest.raises(fgs.RangeError):
        fgs.AdjacencyOperator(X, fgs.KernelSpec.gaussian(1.0))
    Y = np.random.default_rng(9).uniform(-0.4, 0.4, (50, 2))
    with pytest.raises(fgs.RangeError):
        fgs.NfftPlan(2, 8, 4, Y + 0.2)


def test_block_apply_with_leading_dimension_through_c_abi(orc):
    X = np.random.default_rng(10).uniform(-0.2, 0.2, (500, 3))
    op, ref = _pair(orc, X, 0, 0.3, 32, 4)
    n, ld, nvec = 500, 512, 2
    xb = np.zeros(ld * nvec)
    xv = np.random.default_rng(11).standard_normal((nvec, n))
    for j in range(nvec):
        xb[j * ld:j * ld + n] = xv[j]
    yb = np.full(ld * nvec, 7.0)
    dp = lambda a: a.ctypes.data_as(C.POINTER(C.c_double))  # noqa: E731
    st = fgs.lib().fgs_adjacency_apply(op.handle, fgs.OP_NORMALIZED, dp(xb), dp(yb), nvec, C.c_int64(ld))
    assert st == 0
    for j in range(nvec):
        assert rel(yb[j * ld:j * ld + n], ref.apply_normalized(xv[j])) <= 1e-10
        assert np.all(yb[j * ld + n:(j + 1) * ld] == 7.0)  # padding untouched


def test_device_apply_caller_order(orc):
    import torch
    X = np.random.default_rng(12).uniform(-0.2, 0.2, (900, 2))
    op, ref = _pair(orc, X, 0, 0.1, 32, 4)
    x = np.random.default_rng(13).standard_normal(900)
    dx = torch.from_numpy(x).cuda()
    dy = torch.empty_like(dx)
    op.apply_device(fgs.OP_SYM_LAPLACIAN, dx.data_ptr(), dy.data_ptr(), internal_order=False)
    torch.cuda.synchronize()
    assert rel(dy.cpu().numpy(), ref.apply_sym_laplacian(x)) <= 1e-10
    # internal order round trip
    di = torch.empty_like(dx)
    op.permute_device(dx.data_ptr(), di.data_ptr(), direction=0)
    dyi = torch.empty_like(dx)
    op.apply_device(fgs.OP_SYM_LAPLACIAN, di.data_ptr(), dyi.data_ptr(), internal_order=True)
    back = torch.empty_like(dx)
    op.permute_device(dyi.data_ptr(), back.data_ptr(), direction=1)
    torch.cuda.synchronize()
    assert np.array_equal(back.cpu().numpy(), dy.cpu().numpy())


def test_sharded_exchange_path_with_one_rank(orc):
    # The N>1 data path (truncated-spectrum window pack -> ncclAllReduce ->
    # unpack-multiply, NCCL-reduced Lanczos dots, ncclMin degree flag) run
    # with a single-rank communicator must reproduce the unsharded operator.
    import torch
    X = fgs.workload_nodes(1, seed=2024)[:6000]
    info = fgs.workload_info(1)
    params = fgs.FastsumParams(info["N"], info["m"], info["p"])
    kern = fgs.KernelSpec.gaussian(info["sigma"])
    plain = fgs.AdjacencyOperator(X, kern, params)
    shard = fgs.AdjacencyOperator(X, kern, params, rank=0, world=1, nccl_id=fgs.nccl_unique_id())
    assert shard.n_local == X.shape[0] and shard.offset == 0
    x = np.random.default_rng(14).standard_normal(X.shape[0])
    dx = torch.from_numpy(x).cuda()
    di = torch.empty_like(dx)
    shard.permute_device(dx.data_ptr(), di.data_ptr(), direction=0)
    dy = torch.empty_like(dx)
    shard.apply_device(fgs.OP_SYM_LAPLACIAN, di.data_ptr(), dy.data_ptr(), internal_order=True)
    back = torch.empty_like(dx)
    shard.permute_device(dy.data_ptr(), back.data_ptr(), direction=1)
    torch.cuda.synchronize()
    assert rel(back.cpu().numpy(), plain.apply_sym_laplacian(x)) <= 1e-12
    a = fgs.lanczos_largest(plain, 4, fgs.LanczosOptions(tol=1e-10))
    b = fgs.lanczos_largest(shard, 4, fgs.LanczosOptions(tol=1e-10))
    assert np.max(np.abs(a.values - b.values)) <= 1e-12


def test_pinned_host_block_pipelined_graph(orc):
    # Pinned host blocks of several vectors run as one graph whose sub-block
    # H2D / apply / D2H overlap on three streams (Core::apply_host_graph):
    # every column equals the same vector applied alone from device memory
    # (bitwise: the kernels are the same, vectors are independent) and the
    # oracle; the padding of the leading dimension stays untouched.
    import torch
    X = np.random.default_rng(14).uniform(-0.1, 0.1, (5000, 3))
    op, ref = _pair(orc, X, 0, 0.05, 32, 8)
    n, ld, nvec = 5000, 5003, 16
    xv = np.random.default_rng(15).standard_normal((nvec, n))
    hx = torch.zeros(nvec * ld, dtype=torch.float64).pin_memory()
    for j in range(nvec):
        hx[j * ld:j * ld + n] = torch.from_numpy(xv[j])
    hy = torch.full((nvec * ld,), 7.0, dtype=torch.float64).pin_memory()
    dp = lambda t: C.cast(t.data_ptr(), C.POINTER(C.c_double))  # noqa: E731
    for _ in range(2):  # capture, then replay of the cached graph
        st = fgs.lib().fgs_adjacency_apply(op.handle, fgs.OP_SYM_LAPLACIAN, dp(hx), dp(hy), nvec, C.c_int64(ld))
        assert st == 0, fgs.lib().fgs_last_error()
    y = hy.numpy()
    for j in range(nvec):
        dx = torch.from_numpy(xv[j]).cuda()
        dy = torch.empty_like(dx)
        op.apply_device(fgs.OP_SYM_LAPLACIAN, dx.data_ptr(), dy.data_ptr(), internal_order=False)
        torch.cuda.synchronize()
        assert np.array_equal(y[j * ld:j * ld + n], dy.cpu().numpy())
        assert np.all(y[j * ld + n:(j + 1) * ld] == 7.0)
    for j in (0, nvec - 1):
        assert rel(y[j * ld:j * ld + n], ref.apply_sym_laplacian(xv[j])) <= 1e-10
