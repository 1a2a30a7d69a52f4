"""Oracle pin for cg_solve and its consumers (spectral.cpp:446-495,
learn.cpp:364-445): the reference's test_learn.cpp SSL / ridge cases,
restated on the CPU oracle."""
import numpy as np
import pytest


def test_laplacian_regularized_solve_meets_residual_contract(orc):
    # test_learn.cpp:215-239
    X = orc.random_cloud(200, 2, 1.5, 51)
    op = orc.AdjacencyOperator(X, 0, 1.0, N=32, m=4, p=4)
    f = orc.random_vector(200, 52)
    x, it, st = orc.kernel_ssl_solve(op, f, 0.0)
    assert st == 0 and np.max(np.abs(x - f)) == 0.0
    beta = 50.0
    x, it, st = orc.kernel_ssl_solve(op, f, beta, 1e-6, 1000)
    assert st == 0
    r = f - (x + beta * op.apply_sym_laplacian(x))
    assert np.linalg.norm(r) <= 1e-6 * np.linalg.norm(f)
    x, it, st = orc.kernel_ssl_solve(op, f, beta, 1e-12, 1)
    assert st != 0 and it == 1


def test_huge_regularization_pulls_onto_stationary_direction(orc):
    # test_learn.cpp:241-256
    X = orc.random_cloud(200, 2, 1.2, 61)
    op = orc.AdjacencyOperator(X, 0, 1.0, N=32, m=4, p=4)
    f = orc.random_vector(200, 62)
    x, it, st = orc.kernel_ssl_solve(op, f, 1e8, 1e-10, 5000)
    assert st == 0
    perron = np.sqrt(op.degrees())
    assert abs(x @ perron) / (np.linalg.norm(x) * np.linalg.norm(perron)) >= 0.99


def test_ridge_single_point_and_explicit_sum(orc):
    # test_learn.cpp:296-328
    plan = orc.FastsumPlan(np.array([[0.3, -0.4]]), 0, 1.0, N=64, m=7, p=7)
    a, it, st = orc.fastsum_ridge_solve(plan, [2.0], 0.5, 1e-12, 50)
    assert st == 0 and abs(a[0] - 2.0 / 1.5) <= 1e-8 * (2.0 / 1.5)
    train, query = orc.random_cloud(40, 2, 1.0, 81), orc.random_cloud(15, 2, 1.0, 82)
    f = orc.random_vector(40, 83)
    plan = orc.FastsumPlan(train, 0, 0.8, N=64, m=7, p=7, eps_b=0.125)
    alpha, it, st = orc.fastsum_ridge_solve(plan, f, 1e-2, 1e-10, 500)
    assert st == 0
    allx = np.concatenate([train, query])
    pred = orc.FastsumPlan(allx, 0, 0.8, N=64, m=7, p=7, eps_b=0.125).apply(np.concatenate([alpha, np.zeros(15)]))[40:]
    D = np.linalg.norm(train[:, None] - query[None], axis=-1)
    direct = (np.exp(-D ** 2 / 0.64) * alpha[:, None]).sum(0)
    assert np.max(np.abs(pred - direct) / np.abs(direct)) <= 1e-7


def test_indefinite_gram_is_flagged(orc):
    # test_learn.cpp:350-363 (multiquadric Gram is indefinite)
    train = orc.random_cloud(30, 2, 1.0, 95)
    f = np.where(np.arange(30) % 2 == 0, 1.0, -1.0)
    plan = orc.FastsumPlan(train, 2, 1.0, N=32, m=4, p=4)
    _, _, st = orc.fastsum_ridge_solve(plan, f, 1e-6, 1e-10, 200)
    assert st == 2
    plan = orc.FastsumPlan(train, 3, 1.0, N=64, m=7, p=7, eps_b=0.125)
    a, _, st = orc.fastsum_ridge_solve(plan, f, 1e-3, 1e-10, 500)
    assert st == 0 and np.all(np.isfinite(a))


def test_cg_rejects_bad_configuration(orc):
    X = orc.random_cloud(20, 2, 1.0, 1)
    op = orc.AdjacencyOperator(X, 0, 1.0, N=32, m=4, p=4)
    for args in ((-1.0, 1e-6, 10), (1.0, 0.0, 10), (1.0, 1e-6, 0)):
        with pytest.raises(orc.OracleError) as e:
            orc.kernel_ssl_solve(op, np.ones(20), *args)
        assert e.value.kind == "ParameterError"
