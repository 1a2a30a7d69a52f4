"""The N-rank sharded data path on one GPU (fgs_shard_group_*).

`world` shards of one operator -- each with rank r's plan slice, its
slab-pruned convolution planes and its exchange buffers, exactly what
fgs_adjacency_create_sharded builds on rank r -- run phase 1 of an apply,
their exchange buffers are summed on the device (what ncclAllReduce computes
across the ranks: the d = 3 window spectra, the d = 2 partial grids, the
cuFFT path's truncated spectrum), then phase 2.  The result must equal the
unsharded operator to rounding (the spread contributions are summed in a
different order), so the multi-GPU decomposition is validated on the GPU
kernels themselves, not only on the CPU restatement (tests/test_sharding.py).
Ranks that wait on one another never share the GPU as separate launches
(B200_PROFILING.md), so this is how the pool's single GPU exercises N > 1.
"""
import numpy as np
import pytest

import paper_1808_04580_b200 as fgs

pytestmark = pytest.mark.gpu


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def _pair(X, sigma, N, m, p, world):
    params = fgs.FastsumParams(N, m, p, 0.0)
    kern = fgs.KernelSpec.gaussian(sigma)
    return fgs.AdjacencyOperator(X, kern, params), fgs.ShardGroup(X, kern, params, world=world)


def _compare(plain, grp, n, ops=(fgs.OP_SYM_LAPLACIAN,), nvec=2, tol=1e-12):
    import torch
    x = torch.from_numpy(np.ascontiguousarray(fgs.workload_vectors(n, nvec, 5).T)).cuda()  # [nvec][n]
    for op in ops:
        y1 = torch.empty_like(x)
        y2 = torch.full_like(x, np.nan)
        plain.apply_device(op, x.data_ptr(), y1.data_ptr(), nvec=nvec, ld=n, internal_order=False)
        grp.apply_device(op, x.data_ptr(), y2.data_ptr(), nvec=nvec, ld=n)
        torch.cuda.synchronize()
        a, b = y2.cpu().numpy(), y1.cpu().numpy()
        for j in range(nvec):
            assert rel(a[j], b[j]) <= tol, (op, j, rel(a[j], b[j]))


@pytest.mark.parametrize("config,n_max,world", [(1, 0, 2), (1, 0, 4), (2, 0, 2), (2, 0, 8), (3, 0, 2),
                                                (4, 400_000, 4), (5, 2_000_000, 2)])
def test_shard_group_equals_unsharded(config, n_max, world):
    info = fgs.workload_info(config)
    X = fgs.workload_nodes(config, seed=2024)
    if n_max:
        X = X[:n_max]
    n = X.shape[0]
    plain, grp = _pair(X, info["sigma"], info["N"], info["m"], info["p"], world)
    ops = (fgs.OP_SYM_LAPLACIAN, fgs.OP_KERNEL) if config in (1, 2) else (fgs.OP_SYM_LAPLACIAN,)
    _compare(plain, grp, n, ops)
    stats = [grp.stats(r) for r in range(world)]
    assert sum(s["n_local"] for s in stats) == n  # the slices partition the points
    M = 2 * info["N"]
    if info["d"] == 3:
        # slab-pruned convolutions: every shard transforms only the dim-0
        # planes its boxes cover (the internal order is slab-major in dim 0)
        assert all(s["conv_planes"] <= M for s in stats)
        assert min(s["conv_planes"] for s in stats) < M, stats


def test_shard_group_cufft_path_and_normalized_op():
    # d = 1: no hand-written convolution, the sharded cuFFT path (window pack
    # -> exchange -> unpack-multiply)
    X = np.random.default_rng(3).uniform(-0.2, 0.2, (30_000, 1))
    plain, grp = _pair(X, 0.05, 64, 6, 6, 3)
    _compare(plain, grp, X.shape[0], (fgs.OP_SYM_LAPLACIAN, fgs.OP_NORMALIZED, fgs.OP_WEIGHT))


def test_shard_group_reports_nonpositive_degree():
    # the degree check of the group (ncclMin of the flag on the ranks) names
    # the same node as the unsharded operator (test_graphop.cpp:236-263 setup)
    hits = 0
    for seed in range(20):
        X = np.random.default_rng(100 + seed).uniform(-0.5, 0.5, (40, 2)) * 0.99
        params = fgs.FastsumParams.preset(1)
        kern = fgs.KernelSpec.gaussian(0.05)
        try:
            fgs.AdjacencyOperator(X, kern, params)
            continue
        except fgs.NumericalError as e:
            want = e.bad_node
        with pytest.raises(fgs.NumericalError) as err:
            fgs.ShardGroup(X, kern, params, world=2)
        assert err.value.bad_node == want
        hits += 1
    assert hits > 0
