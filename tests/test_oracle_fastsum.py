"""Pins the CPU oracle's kernels / fastsum / graph-operator restatement
against the reference's known-answer tests (proj/tests/test_kernels.cpp,
test_fastsum.cpp, test_graphop.cpp, acceptance.cpp).  CPU only."""
import numpy as np
import pytest

from conftest import approx

G, LRBF, MQ, IMQ = 0, 1, 2, 3
CATALOG = [(G, 1.0), (G, 3.5), (LRBF, 2.0), (MQ, 1.5), (IMQ, 0.8)]


def test_kernel_values_match_closed_forms(orc):
    # test_kernels.cpp:32-44
    assert orc.eval_kernel(G, 3.5, 3.5) == pytest.approx(np.exp(-1.0), rel=1e-14)
    assert orc.eval_kernel(LRBF, 2.0, 2.0) == pytest.approx(np.exp(-1.0), rel=1e-14)
    assert orc.eval_kernel(MQ, 4.0, 3.0) == pytest.approx(5.0, rel=1e-15)
    assert orc.eval_kernel(IMQ, 2.0, 0.0) == pytest.approx(0.5, rel=1e-15)
    with pytest.raises(orc.OracleError) as e:
        orc.eval_kernel(G, 0.0, 1.0)
    assert e.value.kind == "ParameterError"
    with pytest.raises(orc.OracleError) as e:
        orc.eval_kernel(G, 1.0, -0.1)
    assert e.value.kind == "RangeError"


def test_radial_derivatives_agree_with_finite_differences(orc):
    # test_kernels.cpp:46-57
    for fam, shape in CATALOG:
        for r in (0.1, 0.37, 1.0, 2.3):
            der = orc.kernel_radial_derivatives(fam, shape, r, 8)
            for j in range(7):
                h = 1e-5
                lo = orc.kernel_radial_derivatives(fam, shape, r - h, j + 1)
                hi = orc.kernel_radial_derivatives(fam, shape, r + h, j + 1)
                fd = (hi[j] - lo[j]) / (2 * h)
                scale = max(abs(der[j + 1]), abs(der[j]), 1.0)
                assert abs(der[j + 1] - fd) <= 1e-5 * scale


def _poly_deriv(center, scale, coeffs, r, order):
    c = np.array(coeffs, float)
    for _ in range(order):
        if c.size == 1:
            return 0.0
        c = c[1:] * np.arange(1, c.size)
    s = (r - center) / scale
    return np.polyval(c[::-1], s) / scale ** order


def test_blend_conditions_hold_across_catalog(orc):
    # test_kernels.cpp:59-117 (value + derivative matching, flat tail)
    center, scale, c = orc.two_point_taylor(G, 1.0, 0.125, 1)
    assert len(c) == 1 and c[0] == pytest.approx(orc.eval_kernel(G, 1.0, 0.375), rel=1e-15)
    for fam, shape in CATALOG:
        for p in (2, 4, 8):
            eps_b = 0.1
            a = 0.5 - eps_b
            center, scale, c = orc.two_point_taylor(fam, shape, eps_b, p)
            assert len(c) - 1 <= 2 * p - 1
            der = orc.kernel_radial_derivatives(fam, shape, a, p)
            for i in range(p):
                noise = sum(abs(c[k]) * np.prod([k - q for q in range(i)]) for k in range(i, len(c)))
                noise = noise / scale ** i * 1e-13
                tol = 1e-8 * max(abs(der[i]), 1.0) + noise
                assert abs(_poly_deriv(center, scale, c, a, i) - der[i]) <= tol
            assert abs(_poly_deriv(center, scale, c, 0.5, 1)) <= 1e-10 * max(abs(der[0]) / eps_b, 1.0)


def test_regularized_kernel_branches(orc):
    # test_kernels.cpp:119-139
    v = orc.regularized_value(G, 1.0, 0.125, 4, [0.2, 0.375 - 1e-12, 0.375 + 1e-12, 0.6, 0.86, 0.51])
    assert v[0] == pytest.approx(orc.eval_kernel(G, 1.0, 0.2), rel=1e-15)
    assert abs(v[1] - v[2]) <= 1e-9
    assert v[4] == v[5]
    v0 = orc.regularized_value(G, 0.2, 0.0, 4, [0.3, 0.7])
    assert v0[0] == pytest.approx(orc.eval_kernel(G, 0.2, 0.3), rel=1e-15)
    assert v0[1] == pytest.approx(orc.eval_kernel(G, 0.2, 0.5), rel=1e-15)


@pytest.mark.parametrize("d", [1, 2])
def test_coefficients_interpolate_regularized_kernel_on_grid(orc, d):
    # test_kernels.cpp:141-166
    N = 32 if d == 1 else 16
    coeffs = orc.kernel_coefficients(G, 0.25, 2.0 / N, 2, d, N)
    assert np.max(np.abs(coeffs.imag)) <= 1e-12 * np.max(np.abs(coeffs))
    rng = np.random.default_rng(3)
    for _ in range(20):
        y = (rng.integers(0, N, size=d) - N / 2) / N
        val = orc.trig_polynomial_value(coeffs, d, N, y)
        ref = orc.regularized_value(G, 0.25, 2.0 / N, 2, [np.linalg.norm(y)])[0]
        assert abs(val.real - ref) <= 1e-12
        assert abs(val.imag) <= 1e-12


def test_coefficients_match_quadratic_cost_transform_1d(orc):
    # test_kernels.cpp:168-183
    N = 16
    coeffs = orc.kernel_coefficients(IMQ, 0.6, 0.125, 3, 1, N)
    j = np.arange(N) - N // 2
    vals = orc.regularized_value(IMQ, 0.6, 0.125, 3, np.abs(j / N))
    for a in range(N):
        l = a - N // 2
        acc = np.sum(vals * np.exp(-2j * np.pi * j * l / N)) / N
        assert abs(coeffs[a] - acc) <= 1e-13


def test_coefficients_match_numpy_fft_3d(orc):
    # independent witness of kernels.cpp:266-335 with numpy's FFT
    d, N = 3, 8
    coeffs = orc.kernel_coefficients(G, 0.3, 0.0, 4, d, N)
    j = (np.arange(N) - N // 2) / N
    Y = np.stack(np.meshgrid(j, j, j, indexing="ij"), -1)
    samples = np.exp(-np.minimum(np.linalg.norm(Y, axis=-1), 0.5) ** 2 / 0.09)
    l = np.arange(N) - N // 2
    ref = np.fft.fftn(samples)[np.ix_(l % N, l % N, l % N)]
    L = np.add.outer(np.add.outer(l, l), l)
    ref = ref * np.where(L % 2 == 0, 1.0, -1.0) / N ** d
    assert np.max(np.abs(coeffs - ref.ravel())) <= 1e-14


def test_presets_and_rescaling(orc):
    # test_fastsum.cpp:57-67
    nodes = np.array([[0.0, 0.0, 10.0], [0.0, 0.0, -10.0]])
    plan = orc.FastsumPlan(nodes, G, 3.5, N=16, m=2, p=2)
    assert plan.scaling == pytest.approx(1 / 40, rel=1e-14)
    small = orc.random_cloud(10, 2, 0.05, 3)
    assert orc.FastsumPlan(small, G, 1.0, N=16, m=2, p=2).scaling == 1.0


TIGHT = dict(N=64, m=8, p=8, eps_b=8.0 / 64.0)


def test_single_and_two_nodes(orc):
    # test_fastsum.cpp:69-91
    plan = orc.FastsumPlan(np.array([[0.3, -0.2]]), G, 1.0, **TIGHT)
    budget = 2.5 * (10.0 * plan.kernel_error_estimate(200, 5) + 1e-10)
    assert abs(plan.apply([2.5])[0] - 2.5 * plan.kernel_zero) <= budget
    nodes = np.array([[0.0, 0.0], [0.6, 0.8]])
    plan = orc.FastsumPlan(nodes, G, 1.0, **TIGHT)
    out = plan.apply([1.0, 0.0])
    budget = 10.0 * plan.kernel_error_estimate(200, 5) + 1e-10
    assert abs(out[0] - 1.0) <= budget
    assert abs(out[1] - np.exp(-1.0)) <= budget


@pytest.mark.parametrize("d", [1, 2, 3])
def test_plan_matches_quadratic_cost_oracle_for_every_family(orc, d):
    # test_fastsum.cpp:93-109
    n = 220
    nodes = orc.random_cloud(n, d, 2.0, 17 * d)
    x = orc.random_vector(n, 23)
    for fam, shape in [(G, 1.5), (LRBF, 2.0), (MQ, 1.2), (IMQ, 0.9)]:
        plan = orc.FastsumPlan(nodes, fam, shape, **TIGHT)
        fast = plan.apply(x)
        exact = orc.direct_apply(nodes, fam, shape, x)
        budget = np.sum(np.abs(x)) * (10.0 * plan.kernel_error_estimate(300, 11) + 1e-10)
        assert np.max(np.abs(fast - exact)) <= budget


def test_application_is_deterministic_and_linear(orc):
    # test_fastsum.cpp:130-145
    nodes = orc.random_cloud(130, 2, 1.0, 7)
    plan = orc.FastsumPlan(nodes, G, 1.0, N=32, m=4, p=4)
    x, y = orc.random_vector(130, 1), orc.random_vector(130, 2)
    assert np.max(np.abs(plan.apply(x) - plan.apply(x))) == 0.0
    combined = plan.apply(2 * x - 3 * y)
    split = 2 * plan.apply(x) - 3 * plan.apply(y)
    assert np.max(np.abs(combined - split)) <= 1e-12 * np.max(np.abs(split))


def test_accuracy_ladder_improves_strictly(orc):
    # test_fastsum.cpp:177-192
    n = 260
    nodes = orc.random_cloud(n, 3, 5.0, 99)
    x = orc.random_vector(n, 100)
    exact = orc.direct_apply(nodes, G, 3.5, x)
    prev = np.inf
    for N, m in [(16, 2), (32, 4), (64, 7)]:
        plan = orc.FastsumPlan(nodes, G, 3.5, N=N, m=m, p=m)
        err = np.max(np.abs(plan.apply(x) - exact)) / np.sum(np.abs(x))
        assert err < prev
        prev = err
    assert prev <= 1e-10


def test_invalid_configurations_are_rejected(orc):
    # test_fastsum.cpp:194-209
    nodes = orc.random_cloud(5, 2, 1.0, 1)
    for kw in [dict(N=31, m=4, p=4), dict(N=32, m=4, p=4, eps_b=0.5)]:
        with pytest.raises(orc.OracleError) as e:
            orc.FastsumPlan(nodes, G, 1.0, **kw)
        assert e.value.kind == "ParameterError"
    plan = orc.FastsumPlan(nodes, G, 1.0)
    with pytest.raises(orc.OracleError) as e:
        plan.apply(np.zeros(4))
    assert e.value.kind == "ShapeError"


# ---- graph operator (test_graphop.cpp) -------------------------------------
P3 = dict(N=64, m=7, p=7, eps_b=0.125)


def test_two_nodes_give_the_swap_adjacency(orc):
    # test_graphop.cpp:60-73
    op = orc.AdjacencyOperator(np.array([[0.0, 0.0], [0.6, 0.8]]), G, 1.0, **P3)
    deg = op.degrees()
    assert approx(deg[0], np.exp(-1.0), 1e-9) and approx(deg[1], np.exp(-1.0), 1e-9)
    y = op.apply_normalized([1.0, 0.0])
    assert abs(y[0]) <= 1e-9 and approx(y[1], 1.0, 1e-9)


def test_direct_backend_reproduces_dense_products(orc):
    # test_graphop.cpp:75-96
    n = 120
    nodes = orc.random_cloud(n, 2, 1.5, 11)
    op = orc.AdjacencyOperator(nodes, G, 1.0, N=16, m=2, p=2, direct=True)
    D = np.linalg.norm(nodes[:, None] - nodes[None], axis=-1)
    W = np.exp(-D ** 2)
    np.fill_diagonal(W, 0.0)
    rs = W.sum(1)
    assert np.max(np.abs(op.degrees() - rs)) <= 1e-12 * rs.max()
    x = orc.random_vector(n, 12)
    assert np.max(np.abs(op.apply_weight(x) - W @ x)) <= 1e-11 * np.max(np.abs(W @ x))
    A = W / np.sqrt(np.outer(rs, rs))
    assert np.max(np.abs(op.apply_normalized(x) - A @ x)) <= 1e-11 * np.max(np.abs(x))


def test_coincident_nodes_have_degree_n_minus_1(orc):
    # test_graphop.cpp:98-107
    for direct in (False, True):
        op = orc.AdjacencyOperator(np.zeros((12, 2)), G, 1.0, direct=direct, **P3)
        assert np.max(np.abs(op.degrees() - 11.0)) <= 1e-9


def test_square_root_degree_vector_is_fixed_point(orc):
    # test_graphop.cpp:109-127
    n = 600
    nodes = orc.random_cloud(n, 2, 2.0, 21)
    op = orc.AdjacencyOperator(nodes, G, 2.0, **P3)
    fixed = np.sqrt(op.degrees())
    assert np.max(np.abs(op.apply_normalized(fixed) - fixed)) <= 1e-8 * np.max(np.abs(fixed))
    assert np.max(np.abs(op.apply_sym_laplacian(fixed))) <= 1e-8 * np.max(np.abs(fixed))
    x = orc.random_vector(n, 22)
    x -= x @ fixed / (fixed @ fixed) * fixed
    x /= np.linalg.norm(x)
    assert x @ op.apply_sym_laplacian(x) >= -1e-10


def test_failed_degrees_name_the_node(orc):
    # test_graphop.cpp:236-263
    with pytest.raises(orc.OracleError) as e:
        orc.AdjacencyOperator(np.zeros((1, 2)), G, 1.0, N=16, m=2, p=2)
    assert e.value.kind == "ShapeError"
    failures = 0
    for seed in range(20):
        cloud = orc.random_cloud(40, 2, 1.0, 100 + seed)
        try:
            orc.AdjacencyOperator(cloud, G, 0.05, N=16, m=2, p=2)
        except orc.OracleError as err:
            assert err.kind == "NumericalError"
            assert "degree" in err.msg and any(ch.isdigit() for ch in err.msg)
            failures += 1
            break
    assert failures > 0
