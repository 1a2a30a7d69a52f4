"""Oracle pin for k-means / spectral clustering (learn.cpp:17-167) and the
label metrics (learn.cpp:441-486): the reference's own test_learn.cpp cases,
restated.  CPU only."""
import numpy as np
import pytest

from conftest import approx


def test_kmeans_degenerate_extremes(orc):
    # test_learn.cpp:43-55
    pts = orc.random_cloud(12, 2, 1.0, 3)
    _, _, w = orc.kmeans(pts, 12)
    assert abs(w) <= 1e-12
    _, cen, _ = orc.kmeans(pts, 1)
    assert np.linalg.norm(cen[0] - pts.mean(0)) <= 1e-12
    for k in (0, 13):
        with pytest.raises(orc.OracleError) as e:
            orc.kmeans(pts, k)
        assert e.value.kind == "ParameterError"


def test_kmeans_optimal_two_pair_split(orc):
    # test_learn.cpp:57-69
    pts = np.array([[0.0, 0.0], [0.1, 0.0], [10.0, 0.0], [10.1, 0.0]])
    lab, _, w = orc.kmeans(pts, 2)
    assert lab[0] == lab[1] and lab[2] == lab[3] and lab[0] != lab[2]
    assert approx(w, 2.0 * 2.0 * 0.05 * 0.05, 1e-12)
    lab2, _, _ = orc.kmeans(pts, 2)
    assert np.array_equal(lab, lab2)


def test_indicator_eigenvectors_give_exact_block_recovery(orc):
    # test_learn.cpp:71-84
    n = 10
    V = np.zeros((n, 2))
    V[:5, 0] = 1.0 / np.sqrt(5.0)
    V[5:, 1] = 1.0 / np.sqrt(5.0)
    lab = orc.spectral_cluster(V, 2)
    assert np.all(lab[:5] == lab[0]) and np.all(lab[5:] == lab[5]) and lab[0] != lab[5]
    with pytest.raises(orc.OracleError) as e:
        orc.spectral_cluster(V, 3)
    assert e.value.kind == "ParameterError"


def _dense_adjacency(X, sigma):
    D = np.linalg.norm(X[:, None] - X[None], axis=-1)
    W = np.exp(-(D * D) / sigma ** 2)
    np.fill_diagonal(W, 0.0)
    rs = W.sum(1)
    return W / np.sqrt(np.outer(rs, rs))


def test_two_separated_blobs_cluster_perfectly_through_the_graph(orc):
    # test_learn.cpp:86-95 (dense_reference_eig of 400 points, top 2 pairs)
    X, truth = orc.blobs([200, 200], [[0.0, 0.0], [6.0, 0.0]], 0.5, 7)
    vals, vecs, _, conv = orc.lanczos_dense(_dense_adjacency(X, 1.0), 2, tol=1e-13, seed=12345)
    assert conv
    lab = orc.spectral_cluster(vecs, 2)
    assert orc.misclassification_rate(lab, truth, permuted=True) == 0.0


def test_misclassification_metrics(orc):
    # test_learn.cpp:97-119
    a = [0, 1, 0, 1]
    assert orc.misclassification_rate(a, a) == 0.0
    sw = [1, 0, 1, 0]
    assert orc.misclassification_rate(a, sw) == 1.0
    assert orc.misclassification_rate(a, sw, permuted=True) == 0.0
    assert orc.misclassification_rate(a, [0, 1, 1, 0]) == 0.5
    rng = np.random.default_rng(11)
    x, y = rng.integers(0, 4, 200), rng.integers(0, 4, 200)
    assert orc.misclassification_rate(x, y, permuted=True) <= orc.misclassification_rate(x, y)
    with pytest.raises(orc.OracleError) as e:
        orc.misclassification_rate([9], [9], permuted=True)
    assert e.value.kind == "ParameterError"
    with pytest.raises(orc.OracleError) as e:
        orc.misclassification_rate(a, [0])
    assert e.value.kind == "ShapeError"


def test_kmeans_empty_cluster_reseed_and_duplicates(orc):
    # learn.cpp:50-62 (all distances zero) and 108-124 (empty cluster re-seed)
    pts = np.zeros((6, 2))
    lab, cen, w = orc.kmeans(pts, 3)
    assert w == 0.0 and lab.min() >= 0 and lab.max() < 3
    rng = np.random.default_rng(5)
    pts = np.concatenate([rng.normal(0, 0.01, (50, 2)), rng.normal(5, 0.01, (3, 2))])
    lab, cen, w = orc.kmeans(pts, 4, restarts=3)
    assert len(set(lab.tolist())) == 4
