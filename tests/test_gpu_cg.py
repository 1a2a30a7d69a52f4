"""GPU conjugate gradients (cg.cu) against the oracle's cg_solve restatement
and the reference's SSL / ridge contracts (learn.cpp:364-445).  The device
dot products are fixed-order block sums, the oracle's serial, so iterates
agree to rounding; solutions are compared at the solver tolerance."""
import numpy as np
import pytest

import paper_1808_04580_b200 as fgs

pytestmark = pytest.mark.gpu


def test_kernel_ssl_matches_oracle_and_contract(orc):
    X = orc.random_cloud(200, 2, 1.5, 51)
    op = fgs.AdjacencyOperator(X, fgs.KernelSpec.gaussian(1.0), fgs.FastsumParams.preset(2))
    ref = orc.AdjacencyOperator(X, 0, 1.0, N=32, m=4, p=4)
    f = orc.random_vector(200, 52)
    z = fgs.kernel_ssl_solve(op, f, 0.0)
    assert z.converged() and np.array_equal(z.x, f)
    beta = 50.0
    r = fgs.kernel_ssl_solve(op, f, beta, 1e-10, 1000)
    x, it, st = orc.kernel_ssl_solve(ref, f, beta, 1e-10, 1000)
    assert r.converged() and st == 0 and abs(r.iterations - it) <= 1
    assert np.linalg.norm(r.x - x) <= 1e-8 * np.linalg.norm(x)
    res = f - (r.x + beta * op.apply_sym_laplacian(r.x))
    assert np.linalg.norm(res) <= 1e-10 * np.linalg.norm(f)
    capped = fgs.kernel_ssl_solve(op, f, beta, 1e-12, 1)
    assert not capped.converged() and capped.iterations == 1


def test_kernel_ssl_large_and_deterministic(orc):
    X = fgs.workload_nodes(1, 2024)
    op = fgs.AdjacencyOperator(X, fgs.KernelSpec.gaussian(0.35), fgs.FastsumParams(32, 4, 4, 0.0))
    ref = orc.AdjacencyOperator(X, 0, 0.35, N=32, m=4, p=4)
    f = orc.random_vector(X.shape[0], 7)
    a = fgs.kernel_ssl_solve(op, f, 1e3, 1e-8, 2000)
    b = fgs.kernel_ssl_solve(op, f, 1e3, 1e-8, 2000)
    assert a.converged() and np.array_equal(a.x, b.x) and a.iterations == b.iterations
    x, it, st = orc.kernel_ssl_solve(ref, f, 1e3, 1e-8, 2000)
    assert st == 0 and abs(a.iterations - it) <= 2
    assert np.linalg.norm(a.x - x) <= 1e-6 * np.linalg.norm(x)


def test_truncated_solver_matches_cg_on_direct_full_basis(orc):
    # test_learn.cpp:258-294 on the device: full Lanczos basis of the exact
    # operator, truncated closed form == CG
    X = orc.random_cloud(80, 2, 1.2, 71)
    g = fgs.KernelSpec.gaussian(1.0)
    f = orc.random_vector(80, 72)
    op = fgs.AdjacencyOperator(X, g, backend=fgs.BACKEND_DIRECT)
    full = fgs.lanczos_largest(op, 80, fgs.LanczosOptions(tol=1e-13, seed=12345))
    assert np.max(np.abs(fgs.kernel_ssl_truncated(full, f, 0.0) - f)) <= 1e-12
    solved = fgs.kernel_ssl_solve(op, f, 30.0, 1e-10, 2000)
    assert solved.converged()
    assert np.max(np.abs(fgs.kernel_ssl_truncated(full, f, 30.0) - solved.x)) <= 1e-8


def test_krr_matches_oracle_and_reference_cases(orc):
    # test_learn.cpp:296-363
    m = fgs.krr_fit(np.array([[0.3, -0.4]]), fgs.KernelSpec.gaussian(1.0), 0.5, [2.0], fgs.FastsumParams.preset(3),
                    1e-12, 50)
    assert abs(m.alpha[0] - 2.0 / 1.5) <= 1e-8 * (2.0 / 1.5)
    assert abs(fgs.krr_predict(m, np.array([[0.3, -0.4]]))[0] - 2.0 / 1.5) <= 1e-7 * (2.0 / 1.5)
    train, query = orc.random_cloud(40, 2, 1.0, 81), orc.random_cloud(15, 2, 1.0, 82)
    f = orc.random_vector(40, 83)
    g = fgs.KernelSpec.gaussian(0.8)
    p3 = fgs.FastsumParams.preset(3, 0.125)
    model = fgs.krr_fit(train, g, 1e-2, f, p3, 1e-10, 500)
    plan = orc.FastsumPlan(train, 0, 0.8, N=p3.bandwidth, m=p3.cutoff, p=p3.smoothness, eps_b=0.125)
    alpha, it, st = orc.fastsum_ridge_solve(plan, f, 1e-2, 1e-10, 500)
    assert st == 0 and np.linalg.norm(model.alpha - alpha) <= 1e-8 * np.linalg.norm(alpha)
    pred = fgs.krr_predict(model, query)
    D = np.linalg.norm(train[:, None] - query[None], axis=-1)
    direct = (np.exp(-D ** 2 / 0.64) * model.alpha[:, None]).sum(0)
    assert np.max(np.abs(pred - direct) / np.abs(direct)) <= 1e-7
    t2 = orc.random_cloud(30, 2, 1.0, 95)
    f2 = np.where(np.arange(30) % 2 == 0, 1.0, -1.0)
    with pytest.raises(fgs.NumericalError):
        fgs.krr_fit(t2, fgs.KernelSpec.multiquadric(1.0), 1e-6, f2, fgs.FastsumParams.preset(2), 1e-10, 200)
    ok = fgs.krr_fit(t2, fgs.KernelSpec.inverse_multiquadric(1.0), 1e-3, f2, p3, 1e-10, 500)
    assert np.all(np.isfinite(ok.alpha))
