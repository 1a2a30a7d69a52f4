"""Multi-process (gloo, world_size 2) test of the sharded matvec decomposition
used by the N>1 path: each rank spreads its contiguous slice of
the spatially sorted points, the truncated spectra are summed with an
allreduce, each rank multiplies by b-hat and interpolates its own targets.
The result must equal the unsharded fast summation (fastsum.cpp:111-118) --
checked with the CPU oracle standing in for the device kernels.  CPU only."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _internal_order(X, M, m, B):
    """(tile, cell) sort of the first window tap, as point_keys_kernel."""
    u0 = np.mod(np.ceil(X * M - m).astype(np.int64), M)
    nt = -(-M // B)
    tile = np.zeros(len(X), np.int64)
    cell = np.zeros(len(X), np.int64)
    for t in range(X.shape[1]):
        tile = tile * nt + u0[:, t] // B
        cell = cell * B + u0[:, t] % B
    key = tile * B ** X.shape[1] + cell
    return np.argsort(key, kind="stable")


def _worker(rank, world, port, result):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle as orc
    rng = np.random.default_rng(3)
    n, d, N, m, sigma = 600, 2, 16, 4, 0.08
    X = rng.uniform(-0.2, 0.2, (n, d))
    x = rng.standard_normal(n)
    full = orc.FastsumPlan(X, 0, sigma, N=N, m=m, p=m)
    want = full.apply(x)
    bhat = full.coefficients()
    # sharding: contiguous slices of the internal spatial order
    Xs = full.scaling * X  # fastsum.cpp:79-91 rescaling, as every rank computes it
    order = _internal_order(Xs, 2 * N, m, 8)
    lo, hi = n * rank // world, n * (rank + 1) // world
    mine = order[lo:hi]
    plan = orc.NfftPlan(d, N, m, Xs[mine])
    spec = plan.adjoint(x[mine].astype(np.complex128))  # partial truncated spectrum
    t = torch.from_numpy(np.ascontiguousarray(spec).view(np.float64).copy())
    dist.all_reduce(t)  # the one exchange per matvec
    total = t.numpy().view(np.complex128)
    y_mine = plan.forward_real(total * bhat)
    err = np.max(np.abs(y_mine - want[mine])) / np.max(np.abs(want))
    result[rank] = err
    dist.destroy_process_group()


def test_sharded_spectrum_exchange_equals_unsharded_fastsum():
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    result = mgr.dict()
    mp.spawn(_worker, args=(world, port, result), nprocs=world, join=True)
    assert len(result) == world
    for r in range(world):
        assert result[r] <= 1e-12, result[r]


def test_internal_order_is_a_permutation_with_contiguous_cells():
    rng = np.random.default_rng(0)
    X = rng.uniform(-0.25, 0.25, (2000, 3))
    order = _internal_order(X, 64, 4, 4)
    assert np.array_equal(np.sort(order), np.arange(2000))
    u0 = np.mod(np.ceil(X[order] * 64 - 4).astype(np.int64), 64)
    keys = [tuple(r) for r in u0]
    # every cell's points are contiguous in the internal order
    seen, last = set(), None
    for k in keys:
        if k != last:
            assert k not in seen
            seen.add(k)
            last = k
