"""GPU parity of the Direct backend (graphop.hpp:19-22, graphop.cpp:29-34):
the exact O(n^2) operator W~x = sum_i K(||v_j - v_i||) x_i on the raw nodes
(fastsum.cpp:126-139 direct_apply), checked against the CPU oracle's direct
AdjacencyOperator on the same seeded inputs.  The device sums run in a fixed
segment order (not the oracle's single serial loop), so agreement is to
rounding: relative l2 <= 1e-12."""
import numpy as np
import pytest

import paper_1808_04580_b200 as fgs

pytestmark = pytest.mark.gpu

TOL = 1e-12

FAMILIES = [(fgs.GAUSSIAN, 0.6), (fgs.LAPLACIAN_RBF, 0.8), (fgs.MULTIQUADRIC, 0.5), (fgs.INV_MULTIQUADRIC, 0.5)]


def rel_l2(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def _spec(family, shape):
    return fgs.KernelSpec(family, shape)


@pytest.mark.parametrize("d", [1, 2, 3])
@pytest.mark.parametrize("fam", range(4))
def test_direct_backend_matches_oracle(orc, d, fam):
    family, shape = FAMILIES[fam]
    n = 1500 + 7 * d
    X = orc.random_cloud(n, d, 2.0, 40 + d)  # raw nodes: no [-1/2, 1/2) requirement on this backend
    op = fgs.AdjacencyOperator(X, _spec(family, shape), backend=fgs.BACKEND_DIRECT)
    ref = orc.AdjacencyOperator(X, family, shape, direct=True)
    x = orc.random_vector(n, 9)
    assert rel_l2(op.degrees(), ref.degrees()) <= TOL
    for name in ("apply_kernel", "apply_weight", "apply_normalized", "apply_sym_laplacian"):
        assert rel_l2(getattr(op, name)(x), getattr(ref, name)(x)) <= TOL, name
    # direct_apply (fastsum.cpp:126-139) is apply_kernel
    assert rel_l2(op.apply_kernel(x), orc.direct_apply(X, family, shape, x)) <= TOL


def test_direct_block_apply_and_determinism(orc):
    X = orc.random_cloud(2100, 3, 1.0, 5)
    op = fgs.AdjacencyOperator(X, fgs.KernelSpec.gaussian(0.4), backend=fgs.BACKEND_DIRECT)
    B = np.stack([orc.random_vector(2100, s) for s in range(6)], axis=1)  # crosses the 4-vector pass
    Y = op.apply_normalized(B)
    for j in range(6):
        assert np.array_equal(Y[:, j], op.apply_normalized(B[:, j]))
    assert np.array_equal(op.apply_sym_laplacian(B), op.apply_sym_laplacian(B))


def test_direct_lanczos_matches_oracle(orc):
    X = orc.random_cloud(1200, 2, 1.0, 77)
    op = fgs.AdjacencyOperator(X, fgs.KernelSpec.gaussian(0.3), backend=fgs.BACKEND_DIRECT)
    ref = orc.AdjacencyOperator(X, 0, 0.3, direct=True)
    pairs = fgs.lanczos_largest(op, 6, fgs.LanczosOptions(tol=1e-10))
    rv, rV, _, conv = ref.lanczos_largest(6, tol=1e-10)
    assert conv
    assert np.max(np.abs(pairs.values - rv) / np.abs(rv)) <= 1e-8
    AV = op.apply_normalized(pairs.vectors)
    assert np.max(np.linalg.norm(AV - pairs.vectors * pairs.values, axis=0)) <= 1e-7


def test_fastsum_eigenvalues_close_to_direct(orc):
    # the reference's acceptance metric max_eigenvalue_error (commands.cpp:222-249)
    X = orc.random_cloud(3000, 3, 0.4, 3)
    k = fgs.KernelSpec.gaussian(0.35)
    fast = fgs.AdjacencyOperator(X, k, fgs.FastsumParams(32, 4, 4, 0.0))
    exact = fgs.AdjacencyOperator(X, k, backend=fgs.BACKEND_DIRECT)
    a = fgs.lanczos_largest(fast, 5, fgs.LanczosOptions(tol=1e-10))
    b = fgs.lanczos_largest(exact, 5, fgs.LanczosOptions(tol=1e-10))
    assert np.max(np.abs(a.values - b.values)) <= 1e-4


def test_direct_nonpositive_degree_names_node(orc):
    # graphop.cpp:57-64: exp underflow leaves node 0 without neighbours
    X = np.array([[0.0], [1000.0], [1000.5]])
    with pytest.raises(fgs.NumericalError) as e:
        fgs.AdjacencyOperator(X, fgs.KernelSpec.gaussian(0.01), backend=fgs.BACKEND_DIRECT)
    assert e.value.bad_node == 0


def test_block_residuals_after_lanczos_fast_and_direct(orc):
    # regression: fast-op Lanczos, then block applies (nvec = 6) on the fast
    # and on a freshly created direct handle must read back fully written
    # results (stale-memory columns were once observed with PDL launches)
    rng = np.random.default_rng(4)
    t = rng.uniform(0, 1, 2000)
    X = np.stack([2 * t * np.cos(6 * t), 2 * t * np.sin(6 * t), 10 * t], 1) + rng.normal(0, 0.2, (2000, 3))
    k = fgs.KernelSpec.gaussian(3.5)
    op = fgs.AdjacencyOperator(X, k, fgs.FastsumParams.preset(2))
    pairs = fgs.lanczos_largest(op, 6, fgs.LanczosOptions(tol=1e-12, seed=1))
    for _ in range(3):
        r = np.linalg.norm(op.apply_normalized(pairs.vectors) - pairs.vectors * pairs.values, axis=0)
        assert np.max(r) <= 1e-10
        ex = fgs.AdjacencyOperator(X, k, backend=fgs.BACKEND_DIRECT)
        r = np.linalg.norm(ex.apply_normalized(pairs.vectors) - pairs.vectors * pairs.values, axis=0)
        assert np.max(r) <= 1e-5
        del ex


def test_lanczos_breakdown_restart_matches_oracle(orc):
    # A = three 2x2 swap blocks (three far-apart pairs of coincident nodes):
    # the Krylov space is exhausted after 2 steps, so k = 4 forces the
    # reference's random restart (spectral.cpp:225-238) -- on the device the
    # run-ahead recurrence must roll back to the breakdown step
    X = np.array([[0.0, 0.0], [0.0, 0.0], [5.0, 0.0], [5.0, 0.0], [0.0, 5.0], [0.0, 5.0]])
    op = fgs.AdjacencyOperator(X, fgs.KernelSpec.gaussian(0.1), backend=fgs.BACKEND_DIRECT)
    ref = orc.AdjacencyOperator(X, 0, 0.1, direct=True)
    li = fgs.LanczosInfo()
    pairs = fgs.lanczos_largest(op, 4, fgs.LanczosOptions(tol=1e-10, seed=3), li)
    rv, rV, rit, rconv = ref.lanczos_largest(4, tol=1e-10, seed=3)
    assert np.allclose(pairs.values, rv, atol=1e-12) and np.allclose(np.abs(pairs.values), 1.0, atol=1e-12)
    assert li.iterations == rit
    res = np.linalg.norm(op.apply_normalized(pairs.vectors) - pairs.vectors * pairs.values, axis=0)
    assert np.max(res) <= 1e-10
