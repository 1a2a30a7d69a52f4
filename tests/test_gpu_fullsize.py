"""Full BASELINE sizes on the GPU.

C3 (480k points) and C4 (2M points): one L_s apply against the CPU oracle at
the full size (rel-l2 <= 1e-10, the north-star tolerance).  C5 (10M points,
16-vector blocks) is beyond the oracle's reach, so it is checked through the
size-independent identities of the operator:
  * Perron: A (D^1/2 1) = D^1/2 1 to rounding (the degrees come from the
    same fast operator, graphop.cpp:55-56);
  * symmetry: x^T (A y) = y^T (A x) (spread is the adjoint of the
    interpolation, the multiplier is Hermitian-symmetrised);
  * linearity, block apply == column-wise applies, bitwise determinism."""
import numpy as np
import pytest

import paper_1808_04580_b200 as fgs

pytestmark = pytest.mark.gpu


def rel_l2(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def _op(config):
    info = fgs.workload_info(config)
    X = fgs.workload_nodes(config, seed=2024)
    params = fgs.FastsumParams(info["N"], info["m"], info["p"], 0.0)
    return X, info, params, fgs.AdjacencyOperator(X, fgs.KernelSpec.gaussian(info["sigma"]), params)


@pytest.mark.parametrize("config", [3, 4])
def test_full_size_apply_matches_oracle(orc, config):
    X, info, params, op = _op(config)
    assert X.shape[0] == info["n"]
    ref = orc.AdjacencyOperator(X, 0, info["sigma"], N=info["N"], m=info["m"], p=info["p"])
    x = fgs.workload_vectors(X.shape[0], 1, 99)
    assert rel_l2(op.degrees(), ref.degrees()) <= 1e-10
    assert rel_l2(op.apply_sym_laplacian(x), ref.apply_sym_laplacian(x)) <= 1e-10


def test_config5_full_size_identities():
    X, info, params, op = _op(5)
    n = X.shape[0]
    assert n == 10_000_000
    d = op.degrees()
    assert np.all(d > 0)
    sq = np.sqrt(d)
    # Perron identity of the normalized adjacency
    assert rel_l2(op.apply_normalized(sq), sq) <= 1e-12
    # 16-vector block (the config-5 workload) == column-wise, bitwise repeatable
    B = fgs.workload_vectors(n, 16, 7)
    Y = op.apply_sym_laplacian(B)
    assert np.array_equal(Y, op.apply_sym_laplacian(B))
    for j in (0, 7, 15):
        assert rel_l2(op.apply_sym_laplacian(B[:, j]), Y[:, j]) <= 1e-14
    # symmetry and linearity
    x, y = B[:, 0], B[:, 1]
    Ax, Ay = op.apply_normalized(x), op.apply_normalized(y)
    assert abs(x @ Ay - y @ Ax) <= 1e-12 * np.linalg.norm(x) * np.linalg.norm(Ay)
    z = op.apply_normalized(2.5 * x - 0.75 * y)
    assert rel_l2(z, 2.5 * Ax - 0.75 * Ay) <= 1e-12
    # L_s = I - A
    assert rel_l2(Y[:, 0], x - Ax) <= 1e-13


def test_config4_lanczos_full_size_residuals():
    # the headline eigen-workload (k = 20 at 2M points): converged pairs with
    # small residuals through the same operator, A-space sign convention
    X, info, params, op = _op(4)
    li = fgs.LanczosInfo()
    pairs = fgs.lanczos_largest(op, info["k"], fgs.LanczosOptions(tol=1e-8), li)
    assert li.converged and pairs.count() == info["k"]
    assert abs(pairs.values[0] - 1.0) <= 1e-10
    res = np.linalg.norm(op.apply_normalized(pairs.vectors) - pairs.vectors * pairs.values, axis=0)
    assert np.max(res) <= 1e-6
    G = pairs.vectors.T @ pairs.vectors
    assert np.max(np.abs(G - np.eye(info["k"]))) <= 1e-8
