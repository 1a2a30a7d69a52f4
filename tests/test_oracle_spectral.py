"""Pins the CPU oracle's Lanczos / tridiagonal / eigen-pair conventions
against the reference's known-answer tests (proj/tests/test_spectral.cpp,
acceptance.cpp perron-identity).  CPU only."""
import numpy as np
import pytest

from conftest import approx


def with_spectrum(spectrum, seed):
    rng = np.random.default_rng(seed)
    n = len(spectrum)
    q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    return q @ np.diag(spectrum) @ q.T


def test_tridiagonal_solver_matches_numpy(orc):
    rng = np.random.default_rng(1)
    for m in (1, 2, 5, 40, 150):
        d = rng.standard_normal(m)
        e = np.abs(rng.standard_normal(m - 1))
        vals, vecs = orc.tridiag_eig(d, e)
        T = np.diag(d) + np.diag(e, 1) + np.diag(e, -1)
        ref = np.linalg.eigvalsh(T)
        assert np.max(np.abs(vals - ref)) <= 1e-12 * max(1.0, np.max(np.abs(ref)))
        assert np.max(np.abs(T @ vecs - vecs * vals)) <= 1e-12 * max(1.0, np.max(np.abs(ref)))
        assert np.max(np.abs(vecs.T @ vecs - np.eye(m))) <= 1e-12


def test_eigenpair_container_conventions(orc):
    # test_spectral.cpp:62-82
    values = np.array([1.0, 3.0, 2.0])
    vectors = np.eye(4)[:, :3].copy()
    vectors[0, 1] = 0.0
    vectors[1, 1] = -1.0
    v, V = orc.make_eigenpairs(values, vectors)
    assert list(v) == [3.0, 2.0, 1.0]
    assert V[1, 0] == 1.0 and V[2, 1] == 1.0 and V[0, 2] == 1.0


def test_diagonal_operator_yields_exact_dominant_pairs(orc):
    # test_spectral.cpp:84-97
    vals, vecs, it, conv = orc.lanczos_dense(np.diag([5.0, 4, 3, 2, 1]), 2)
    assert conv
    assert approx(vals[0], 5.0, 1e-10) and approx(vals[1], 4.0, 1e-10)
    assert approx(abs(vecs[0, 0]), 1.0, 1e-10) and approx(abs(vecs[1, 1]), 1.0, 1e-10)
    assert vecs[0, 0] > 0 and vecs[1, 1] > 0


def test_two_dimensional_swap_operator_terminates_exactly(orc):
    # test_spectral.cpp:99-110
    S = np.array([[0.0, 1.0], [1.0, 0.0]])
    vals, vecs, it, conv = orc.lanczos_dense(S, 2)
    assert conv and it == 2
    assert approx(vals[0], 1.0, 1e-12) and approx(vals[1], -1.0, 1e-12)
    assert np.max(np.linalg.norm(S @ vecs - vecs * vals, axis=0)) <= 1e-12


def test_orthonormal_basis_and_residuals_on_synthetic_spectrum(orc):
    # test_spectral.cpp:112-123
    spectrum = 10.0 / (1.0 + np.arange(30))
    A = with_spectrum(spectrum, 5)
    vals, vecs, it, conv = orc.lanczos_dense(A, 6)
    assert np.max(np.abs(vecs.T @ vecs - np.eye(6))) <= 1e-8
    assert np.max(np.linalg.norm(A @ vecs - vecs * vals, axis=0)) <= 1e-9
    for i in range(6):
        assert approx(vals[i], spectrum[i], 1e-10)


def test_shift_invariance_of_the_iteration(orc):
    # test_spectral.cpp:125-140
    spectrum = 5.0 * 0.8 ** np.arange(25)
    A = with_spectrum(spectrum, 9)
    base = orc.lanczos_dense(A, 4, seed=31)
    moved = orc.lanczos_dense(A + 2.75 * np.eye(25), 4, seed=31)
    for i in range(4):
        assert approx(moved[0][i] - base[0][i], 2.75, 1e-10)
        assert np.linalg.norm(moved[1][:, i] - base[1][:, i]) <= 1e-6


def test_agreement_between_iterative_and_dense_ground_truth_on_a_graph(orc):
    # test_spectral.cpp:175-188
    n = 150
    nodes = orc.random_cloud(n, 2, 1.5, 41)
    D = np.linalg.norm(nodes[:, None] - nodes[None], axis=-1)
    W = np.exp(-D ** 2 / 1.5 ** 2)
    np.fill_diagonal(W, 0.0)
    rs = W.sum(1)
    A = W / np.sqrt(np.outer(rs, rs))
    ref = np.sort(np.linalg.eigvalsh(A))[::-1][:5]
    vals, vecs, it, conv = orc.lanczos_dense(A, 5)
    for i in range(5):
        assert approx(vals[i], ref[i], 1e-10)
    assert np.max(np.linalg.norm(A @ vecs - vecs * vals, axis=0)) <= 1e-10
    assert approx(ref[0], 1.0, 1e-10)


def test_lanczos_on_adjacency_matches_dense_of_same_operator(orc):
    # Lanczos through the fast operator equals Lanczos through the same
    # operator materialised column by column (operator-level parity).
    n = 160
    nodes = orc.random_cloud(n, 2, 1.0, 5)
    op = orc.AdjacencyOperator(nodes, 0, 1.0, N=32, m=4, p=4)
    vals, vecs, it, conv = op.lanczos_largest(5, tol=1e-10)
    Amat = np.stack([op.apply_normalized(e) for e in np.eye(n)], 1)
    Asym = 0.5 * (Amat + Amat.T)
    ref = np.sort(np.linalg.eigvalsh(Asym))[::-1][:5]
    assert conv
    assert np.max(np.abs(vals - ref)) <= 1e-8
    assert np.max(np.linalg.norm(Amat @ vecs - vecs * vals, axis=0)) <= 1e-8


def test_perron_identity(orc):
    # acceptance.cpp:379-391 on a seeded cloud (the spiral generator is an
    # external dataset; a uniform cloud stands in)
    nodes = orc.random_cloud(400, 2, 5.0, 18)
    op = orc.AdjacencyOperator(nodes, 0, 3.5, N=64, m=7, p=7)
    vals, vecs, it, conv = op.lanczos_largest(1)
    direction = np.sqrt(op.degrees())
    direction /= np.linalg.norm(direction)
    assert abs(vals[0] - 1.0) <= 1e-8
    assert np.linalg.norm(op.apply_normalized(direction) - direction) <= 1e-8


# ---- nystrom_gaussian (test_spectral.cpp:265-316) ----------------------------
def _signed_top(A, k):
    w, V = np.linalg.eigh(A)
    out = []
    for i in range(k):
        v = V[:, -1 - i]
        out.append(v if v[np.argmax(np.abs(v))] > 0 else -v)
    return w[::-1][:k], np.stack(out, 1)


def test_gaussian_sketch_recovers_low_rank_operator(orc):
    spectrum = np.zeros(40)
    spectrum[:3] = [3.0, 2.0, 1.0]
    A = with_spectrum(spectrum, 83)
    vals, vecs = orc.nystrom_dense(A, 3, 6, 3, seed=5)
    ev, V = _signed_top(A, 3)
    for i in range(3):
        assert approx(vals[i], ev[i], 1e-8)
        assert np.linalg.norm(vecs[:, i] - V[:, i]) <= 1e-6
    assert np.max(np.abs(vecs.T @ vecs - np.eye(3))) <= 1e-8


def test_gaussian_sketch_deterministic_and_rank_deficiency(orc):
    A = with_spectrum(0.7 ** np.arange(30), 91)
    a = orc.nystrom_dense(A, 4, 12, 6, seed=17)
    b = orc.nystrom_dense(A, 4, 12, 6, seed=17)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    with pytest.raises(orc.OracleError) as e:
        orc.nystrom_dense(np.zeros((20, 20)), 2, 6, 3)
    assert e.value.kind == "NumericalError"
    for args in ((0, 6, 3), (4, 6, 3), (2, 6, 7), (2, 30, 3)):
        with pytest.raises(orc.OracleError) as e:
            orc.nystrom_dense(np.eye(20), *args)
        assert e.value.kind == "ParameterError"


def test_householder_qr_and_dense_eig_helpers(orc):
    # full sketch (L = n) of a full-rank operator reproduces its top pairs
    rng = np.random.default_rng(3)
    A = with_spectrum(np.linspace(2.0, 0.1, 25), 4)
    vals, vecs = orc.nystrom_dense(A, 5, 25, 25, seed=2)
    ev, V = _signed_top(A, 5)
    assert np.max(np.abs(vals - ev)) <= 1e-10
    assert np.max(np.abs(vecs - V)) <= 1e-8
