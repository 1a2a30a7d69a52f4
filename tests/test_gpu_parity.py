"""GPU parity: the B200 path (libfgs_b200.so through the C ABI) against the
CPU oracle restating the reference (oracle/), on the same seeded inputs.

Tolerances (BASELINE.json north_star): matvec relative l2 <= 1e-10; the
NfftPlan transforms additionally keep the reference's own 1e-12 * ||in||_1
budgets against the direct NDFT (test_nfft.cpp:91-111)."""
import numpy as np
import pytest

import paper_1808_04580_b200 as fgs

pytestmark = pytest.mark.gpu

MATVEC_TOL = 1e-10


def rel_l2(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


# ---- NfftPlan --------------------------------------------------------------
@pytest.mark.parametrize("d", [1, 2, 3])
@pytest.mark.parametrize("N", [2, 4, 16])
def test_nfft_matches_direct_and_oracle(orc, d, N):
    # test_nfft.cpp:91-111 on the device path
    n = 64 if d == 3 else 256
    nodes = orc.random_nodes(n, d, 100 * d + N)
    plan = fgs.NfftPlan(d, N, 8, nodes)
    ref = orc.NfftPlan(d, N, 8, nodes)
    fhat = orc.random_coeffs(plan.coefficient_count(), 7)
    fast = plan.forward(fhat)
    assert np.max(np.abs(fast - orc.direct_ndft(d, N, nodes, fhat))) <= 1e-12 * np.sum(np.abs(fhat))
    assert rel_l2(fast, ref.forward(fhat)) <= 1e-13
    x = orc.random_coeffs(n, 13)
    adj = plan.adjoint(x)
    assert np.max(np.abs(adj - orc.direct_adjoint_ndft(d, N, nodes, x))) <= 1e-12 * np.sum(np.abs(x))
    assert rel_l2(adj, ref.adjoint(x)) <= 1e-13


@pytest.mark.parametrize("m", [2, 4, 6])
def test_nfft_small_cutoffs_match_oracle(orc, m):
    nodes = orc.random_nodes(500, 3, 5 + m)
    plan, ref = fgs.NfftPlan(3, 16, m, nodes), orc.NfftPlan(3, 16, m, nodes)
    f = orc.random_coeffs(16 ** 3, 3)
    assert rel_l2(plan.forward(f), ref.forward(f)) <= 1e-13
    x = orc.random_coeffs(500, 4)
    assert rel_l2(plan.adjoint(x), ref.adjoint(x)) <= 1e-13


def test_nfft_transpose_pair_and_real_part(orc):
    # test_nfft.cpp:113-126, 172-191
    nodes = orc.random_nodes(120, 2, 21)
    plan = fgs.NfftPlan(2, 16, 4, nodes)
    fhat = orc.random_coeffs(plan.coefficient_count(), 3)
    x = orc.random_coeffs(120, 5)
    lhs = np.vdot(x, plan.forward(fhat))
    rhs = np.vdot(plan.adjoint(x), fhat)
    assert abs(lhs - rhs) <= 1e-10 * (abs(lhs) + abs(rhs))
    p1 = fgs.NfftPlan(1, 8, 8, orc.random_nodes(40, 1, 55))
    assert np.array_equal(p1.forward_real(fhat[:8]), p1.forward(fhat[:8]).real)


def test_nfft_rejects_invalid_inputs(orc):
    # test_nfft.cpp:193-208
    good = orc.random_nodes(4, 2, 1)
    with pytest.raises(fgs.ParameterError):
        fgs.NfftPlan(2, 7, 4, good)
    with pytest.raises(fgs.ParameterError):
        fgs.NfftPlan(2, 8, 0, good)
    with pytest.raises(fgs.ParameterError):
        fgs.NfftPlan(2, 8, 4, good, 0.5)
    bad = good.copy()
    bad[1, 0] = 0.5
    with pytest.raises(fgs.RangeError):
        fgs.NfftPlan(2, 8, 4, bad)
    plan = fgs.NfftPlan(2, 8, 4, good)
    with pytest.raises(fgs.ShapeError):
        plan.forward(np.zeros(63, np.complex128))
    with pytest.raises(fgs.ShapeError):
        plan.adjoint(np.zeros(3, np.complex128))


# ---- FastsumPlan ------------------------------------------------------------
FAMILIES = [(0, 1.5), (1, 2.0), (2, 1.2), (3, 0.9)]


@pytest.mark.parametrize("d", [1, 2, 3])
@pytest.mark.parametrize("fam,shape", FAMILIES)
def test_fastsum_matches_oracle_every_family(orc, d, fam, shape):
    # test_fastsum.cpp:93-109 inputs, tight params (eps_b > 0, p = 8)
    n = 220
    nodes = orc.random_cloud(n, d, 2.0, 17 * d)
    x = orc.random_vector(n, 23)
    params = fgs.FastsumParams(64, 8, 8, 8.0 / 64.0)
    plan = fgs.FastsumPlan(nodes, fgs.KernelSpec(fam, shape), params)
    ref = orc.FastsumPlan(nodes, fam, shape, N=64, m=8, p=8, eps_b=8.0 / 64.0)
    assert plan.scaling() == ref.scaling and plan.output_factor() == ref.output_factor
    c_dev, c_ref = plan.coefficients(), ref.coefficients()
    assert np.max(np.abs(c_dev - c_ref)) <= 1e-14 * np.max(np.abs(c_ref))
    assert rel_l2(plan.apply(x), ref.apply(x)) <= MATVEC_TOL
    exact = orc.direct_apply(nodes, fam, shape, x)
    budget = np.sum(np.abs(x)) * (10.0 * plan.kernel_error_estimate(300, 11) + 1e-10)
    assert np.max(np.abs(plan.apply(x) - exact)) <= budget


def test_fastsum_is_deterministic_and_linear(orc):
    # test_fastsum.cpp:130-145: repeated applies are bitwise identical
    nodes = orc.random_cloud(5000, 3, 1.0, 7)
    plan = fgs.FastsumPlan(nodes, fgs.KernelSpec.gaussian(1.0), fgs.FastsumParams.preset(2))
    x, y = orc.random_vector(5000, 1), orc.random_vector(5000, 2)
    once, twice = plan.apply(x), plan.apply(x)
    assert np.array_equal(once, twice)
    combined = plan.apply(2 * x - 3 * y)
    split = 2 * plan.apply(x) - 3 * plan.apply(y)
    assert np.max(np.abs(combined - split)) <= 1e-12 * np.max(np.abs(split))


def test_fastsum_rejects_invalid_configurations(orc):
    nodes = orc.random_cloud(5, 2, 1.0, 1)
    with pytest.raises(fgs.ParameterError):
        fgs.FastsumPlan(nodes, fgs.KernelSpec.gaussian(1.0), fgs.FastsumParams(31, 4, 4))
    with pytest.raises(fgs.ParameterError):
        fgs.FastsumPlan(nodes, fgs.KernelSpec.gaussian(1.0), fgs.FastsumParams(32, 4, 4, 0.5))
    plan = fgs.FastsumPlan(nodes, fgs.KernelSpec.gaussian(1.0), fgs.FastsumParams.preset(2))
    with pytest.raises(fgs.ShapeError):
        plan.apply(np.zeros(4))
    with pytest.raises(fgs.ShapeError):
        fgs.FastsumPlan(np.zeros((0, 2)), fgs.KernelSpec.gaussian(1.0))


# ---- AdjacencyOperator on the BASELINE workloads ---------------------------
def _config_case(config, n_max):
    info = fgs.workload_info(config)
    X = fgs.workload_nodes(config, seed=2024)
    if X.shape[0] > n_max:
        X = X[np.random.default_rng(config).choice(X.shape[0], n_max, replace=False)]
    params = fgs.FastsumParams(info["N"], info["m"], info["p"], 0.0)
    return X, info, params


@pytest.mark.parametrize("config,n_max", [(1, 20000), (2, 100000), (3, 120000), (4, 150000), (5, 40000)])
def test_adjacency_matches_oracle_on_baseline_configs(orc, config, n_max):
    X, info, params = _config_case(config, n_max)
    op = fgs.AdjacencyOperator(X, fgs.KernelSpec.gaussian(info["sigma"]), params)
    ref = orc.AdjacencyOperator(X, 0, info["sigma"], N=info["N"], m=info["m"], p=info["p"])
    assert rel_l2(op.degrees(), ref.degrees()) <= MATVEC_TOL
    x = fgs.workload_vectors(X.shape[0], 1, 99)
    for name in ("apply_kernel", "apply_weight", "apply_normalized", "apply_sym_laplacian"):
        got, want = getattr(op, name)(x), getattr(ref, name)(x)
        assert rel_l2(got, want) <= MATVEC_TOL, name


def test_block_apply_equals_columnwise(orc):
    X, info, params = _config_case(1, 8000)
    op = fgs.AdjacencyOperator(X, fgs.KernelSpec.gaussian(info["sigma"]), params)
    B = fgs.workload_vectors(X.shape[0], 4, 5)
    Y = op.apply_sym_laplacian(B)
    for j in range(4):
        assert np.array_equal(Y[:, j], op.apply_sym_laplacian(B[:, j].copy()))


def test_graph_operator_identities(orc):
    # test_graphop.cpp:60-73, 98-127 on the device
    P3 = fgs.FastsumParams.preset(3, 0.125)
    op = fgs.AdjacencyOperator(np.array([[0.0, 0.0], [0.6, 0.8]]), fgs.KernelSpec.gaussian(1.0), P3)
    assert np.allclose(op.degrees(), np.exp(-1.0), rtol=1e-9)
    y = op.apply_normalized([1.0, 0.0])
    assert abs(y[0]) <= 1e-9 and abs(y[1] - 1.0) <= 2e-9
    op = fgs.AdjacencyOperator(np.zeros((12, 2)), fgs.KernelSpec.gaussian(1.0), P3)
    assert np.max(np.abs(op.degrees() - 11.0)) <= 1e-9
    nodes = orc.random_cloud(600, 2, 2.0, 21)
    op = fgs.AdjacencyOperator(nodes, fgs.KernelSpec.gaussian(2.0), P3)
    fixed = np.sqrt(op.degrees())
    assert np.max(np.abs(op.apply_normalized(fixed) - fixed)) <= 1e-8 * np.max(fixed)
    assert np.max(np.abs(op.apply_sym_laplacian(fixed))) <= 1e-8 * np.max(fixed)


def test_failed_degrees_name_the_node(orc):
    # test_graphop.cpp:236-263 -- same node as the oracle names
    with pytest.raises(fgs.ShapeError):
        fgs.AdjacencyOperator(np.zeros((1, 2)), fgs.KernelSpec.gaussian(1.0))
    hits = 0
    for seed in range(20):
        cloud = orc.random_cloud(40, 2, 1.0, 100 + seed)
        try:
            orc.AdjacencyOperator(cloud, 0, 0.05, N=16, m=2, p=2)
            continue
        except orc.OracleError as e:
            want = int(e.msg.split("node ")[1].split()[0])
        with pytest.raises(fgs.NumericalError) as err:
            fgs.AdjacencyOperator(cloud, fgs.KernelSpec.gaussian(0.05), fgs.FastsumParams.preset(1))
        assert err.value.bad_node == want
        assert "degree" in str(err.value) and str(want) in str(err.value)
        hits += 1
    assert hits > 0


# ---- lanczos_largest --------------------------------------------------------
def _subspace_sin(U, V):
    """sine of the largest principal angle between span(U) and span(V)."""
    Qu, _ = np.linalg.qr(U)
    Qv, _ = np.linalg.qr(V)
    s = np.linalg.svd(Qu.T @ Qv, compute_uv=False)
    return np.sqrt(max(0.0, 1.0 - np.min(s) ** 2))


def test_lanczos_matches_oracle_on_config1(orc):
    X, info, params = _config_case(1, 20000)
    op = fgs.AdjacencyOperator(X, fgs.KernelSpec.gaussian(info["sigma"]), params)
    ref = orc.AdjacencyOperator(X, 0, info["sigma"], N=info["N"], m=info["m"], p=info["p"])
    k, tol = info["k"], 1e-8
    li = fgs.LanczosInfo()
    pairs = fgs.lanczos_largest(op, k, fgs.LanczosOptions(tol=tol), li)
    rv, rV, rit, rconv = ref.lanczos_largest(k, tol=tol)
    assert li.converged and rconv
    # eigenvalues in A-space (|theta| ~ 1 at the top; SURVEY §8a hazard v)
    assert np.max(np.abs(pairs.values - rv) / np.abs(rv)) <= 1e-8
    # eigenvectors by whole near-degenerate clusters (hazard vi)
    vals = rv
    groups, start = [], 0
    for i in range(1, k + 1):
        if i == k or abs(vals[i] - vals[i - 1]) > 1e-3 * abs(vals[0]):
            groups.append(list(range(start, i)))
            start = i
    for g in groups:
        assert _subspace_sin(pairs.vectors[:, g], rV[:, g]) <= 1e-6
    # residuals through the device operator
    AV = op.apply_normalized(pairs.vectors)
    assert np.max(np.linalg.norm(AV - pairs.vectors * pairs.values, axis=0)) <= 1e-6
    # conventions: descending, sign of the largest-magnitude entry positive
    assert np.all(np.diff(pairs.values) <= 0)
    for j in range(k):
        col = pairs.vectors[:, j]
        assert col[np.argmax(np.abs(col))] > 0
    # adjacency_to_laplacian: values 1 - lambda_A(k-1-i) (spectral.cpp:129-139,
    # test_spectral.cpp:76-81), so the Perron pair (L-eigenvalue ~0) is last
    lap = fgs.adjacency_to_laplacian(pairs)
    assert abs(lap.values[-1]) <= 1e-8
    assert np.array_equal(lap.values, 1.0 - pairs.values[::-1])
    assert np.array_equal(lap.vectors[:, 0], pairs.vectors[:, -1])


@pytest.mark.parametrize("n,seed", [(155, 1), (157, 7), (20000, 1), (20000, 12345678901234)])
def test_lanczos_start_vector_drawn_on_device(orc, n, seed):
    # one step, one pair: the Ritz vector is the normalised start vector
    # (spectral.cpp:152-156: mt19937_64(seed), uniform(-1, 1)), which the
    # device draws itself -- it must be the reference's draw sequence
    X, info, params = _config_case(1, n)
    op = fgs.AdjacencyOperator(X, fgs.KernelSpec.gaussian(info["sigma"]), params)
    ref = orc.AdjacencyOperator(X, 0, info["sigma"], N=info["N"], m=info["m"], p=info["p"])
    li = fgs.LanczosInfo()
    pairs = fgs.lanczos_largest(op, 1, fgs.LanczosOptions(max_iter=1, tol=1e-8, seed=seed), li)
    rv, rV, rit, _ = ref.lanczos_largest(1, max_iter=1, tol=1e-8, seed=seed)
    assert li.iterations == rit == 1
    # same draws; the norm is summed in another order (a tree on the device,
    # the reference's serial loop: ~sqrt(n) ulps apart)
    assert np.max(np.abs(pairs.vectors[:, 0] - rV[:, 0])) <= 1e-14 * np.max(np.abs(rV[:, 0]))
    assert abs(pairs.values[0] - rv[0]) <= 1e-12 * abs(rv[0])


def test_lanczos_laplacian_handle_and_reproducibility(orc):
    X, info, params = _config_case(2, 20000)
    op = fgs.AdjacencyOperator(X, fgs.KernelSpec.gaussian(info["sigma"]), params)
    a = fgs.lanczos_largest(op, 4, fgs.LanczosOptions(tol=1e-10))
    b = fgs.lanczos_largest(op, 4, fgs.LanczosOptions(tol=1e-10))
    assert np.array_equal(a.values, b.values) and np.array_equal(a.vectors, b.vectors)
    ref = orc.AdjacencyOperator(X, 0, info["sigma"], N=info["N"], m=info["m"], p=info["p"])
    lv, lV, it, conv = ref.lanczos_largest(3, tol=1e-10, which=1)
    lp = fgs.lanczos_largest(op, 3, fgs.LanczosOptions(tol=1e-10), which=1)
    assert np.max(np.abs(lp.values - lv)) <= 1e-8 * np.max(np.abs(lv))


@pytest.mark.parametrize("eigen", [False, True])
def test_cpp_dropin_program_passes(eigen):
    # the reference's test cases and its CLI's solve_pairs call site
    # (commands.cpp:171-188, verbatim) written against include/fgs/b200.hpp;
    # eigen=True: the header's Eigen-typed mode
    import subprocess
    import __graft_entry__ as g
    exe = g.build_cpp_dropin_test(eigen=eigen)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr


def test_ritz_vectors_sign_convention_is_race_free():
    # colsign_kernel scales each column in place over many blocks; the sign
    # must come from the pre-scaling argmax entry (a partial flip of a column
    # once slipped through when blocks re-read the entry mid-scaling)
    X = fgs.workload_nodes(2, 2024)[:60000]
    op = fgs.AdjacencyOperator(X, fgs.KernelSpec.gaussian(0.05), fgs.FastsumParams(64, 6, 6, 0.0))
    for _ in range(4):
        pairs = fgs.lanczos_largest(op, 6, fgs.LanczosOptions(tol=1e-10))
        AV = op.apply_normalized(pairs.vectors)
        assert np.max(np.linalg.norm(AV - pairs.vectors * pairs.values, axis=0)) <= 1e-7
        for j in range(6):
            col = pairs.vectors[:, j]
            assert col[np.argmax(np.abs(col))] > 0
