"""GPU k-means / spectral clustering (learn.cpp:17-167) against the oracle.

Labels are integers: the bar is exact equality with the oracle on the same
seeded inputs (same mt19937_64 stream, same k-means++ picks, same Lloyd
trajectory).  Centroids and wcss are sums whose order differs from the
serial oracle only by the fixed chunking (kmeans.cu), so they agree to
rounding (1e-12 relative)."""
import numpy as np
import pytest

import paper_1808_04580_b200 as fgs

pytestmark = pytest.mark.gpu


def _blob_cloud(orc, n_per, k, dim, spread, seed):
    rng = np.random.default_rng(seed)
    centers = rng.uniform(-4, 4, (k, dim))
    return orc.blobs([n_per] * k, centers, spread, seed)


@pytest.mark.parametrize("case", [(400, 5, 3, 0.6, 1), (2000, 4, 4, 1.5, 2), (700, 8, 2, 2.5, 3)])
def test_kmeans_matches_oracle(orc, case):
    n_per, k, dim, spread, seed = case
    X, _ = _blob_cloud(orc, n_per, k, dim, spread, seed)
    got = fgs.kmeans(X, k, fgs.KMeansOptions(restarts=4, max_iter=100, seed=seed))
    lab, cen, w = orc.kmeans(X, k, restarts=4, max_iter=100, seed=seed)
    assert np.array_equal(got.labels, lab)
    assert np.max(np.abs(got.centroids - cen)) <= 1e-12 * np.max(np.abs(cen))
    assert abs(got.wcss - w) <= 1e-12 * abs(w)


def test_kmeans_reference_cases():
    # test_learn.cpp:43-69
    pts = np.array([[0.0, 0.0], [0.1, 0.0], [10.0, 0.0], [10.1, 0.0]])
    r = fgs.kmeans(pts, 2)
    assert r.labels[0] == r.labels[1] and r.labels[2] == r.labels[3] and r.labels[0] != r.labels[2]
    assert abs(r.wcss - 2.0 * 2.0 * 0.05 * 0.05) <= 1e-12 * 0.01
    assert np.array_equal(fgs.kmeans(pts, 2).labels, r.labels)
    one = fgs.kmeans(pts, 1)
    assert np.linalg.norm(one.centroids[0] - pts.mean(0)) <= 1e-12
    assert fgs.kmeans(pts, 4).wcss <= 1e-24
    for k in (0, 5):
        with pytest.raises(fgs.ParameterError):
            fgs.kmeans(pts, k)


def test_kmeans_degenerate_and_empty_clusters_match_oracle(orc):
    # all-zero distances (learn.cpp:50-62) and empty-cluster re-seeding (108-124)
    z = np.zeros((9, 2))
    got = fgs.kmeans(z, 3)
    lab, _, w = orc.kmeans(z, 3)
    assert np.array_equal(got.labels, lab) and got.wcss == w == 0.0
    rng = np.random.default_rng(5)
    X = np.concatenate([rng.normal(0, 0.01, (50, 2)), rng.normal(5, 0.01, (3, 2))])
    got = fgs.kmeans(X, 4, fgs.KMeansOptions(restarts=3))
    lab, cen, w = orc.kmeans(X, 4, restarts=3)
    assert np.array_equal(got.labels, lab)


def test_spectral_cluster_matches_oracle_on_device_eigenvectors(orc):
    # the C3 "labels" step: Lanczos eigenvectors -> unit rows -> k-means
    centers = [[3.0, 0.0, 0.0], [-3.0, 0.0, 0.0], [0.0, 3.0, 0.0], [0.0, -3.0, 0.0]]
    X, truth = orc.blobs([1500] * 4, centers, 0.4, 11)
    X = X / (4.0 * np.max(np.linalg.norm(X, axis=1)))
    op = fgs.AdjacencyOperator(X, fgs.KernelSpec.gaussian(0.08), fgs.FastsumParams(32, 4, 4, 0.0))
    pairs = fgs.lanczos_largest(op, 4, fgs.LanczosOptions(tol=1e-10))
    got = fgs.spectral_cluster(pairs, 4)
    want = orc.spectral_cluster(pairs.vectors, 4)
    assert np.array_equal(got, want)
    assert fgs.misclassification_rate_permuted(got, truth) <= 0.01
    with pytest.raises(fgs.ParameterError):
        fgs.spectral_cluster(pairs, 5)


def test_kmeans_large_matches_oracle(orc):
    rng = np.random.default_rng(8)
    X = np.concatenate([rng.normal(c, 0.3, (25000, 4)) for c in range(4)])
    got = fgs.kmeans(X, 4, fgs.KMeansOptions(restarts=2, seed=3))
    lab, cen, w = orc.kmeans(X, 4, restarts=2, seed=3)
    assert np.array_equal(got.labels, lab)
    assert abs(got.wcss - w) <= 1e-12 * w


def test_misclassification_metrics():
    a = [0, 1, 0, 1]
    assert fgs.misclassification_rate(a, a) == 0.0
    assert fgs.misclassification_rate(a, [1, 0, 1, 0]) == 1.0
    assert fgs.misclassification_rate_permuted(a, [1, 0, 1, 0]) == 0.0
    with pytest.raises(fgs.ParameterError):
        fgs.misclassification_rate_permuted([9], [9])
    with pytest.raises(fgs.ShapeError):
        fgs.misclassification_rate(a, [0])
