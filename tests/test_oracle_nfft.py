"""Pins the CPU oracle's NFFT restatement against the reference's own
known-answer tests (proj/tests/test_nfft.cpp, acceptance.cpp:218-252) and its
FFT against numpy.fft.  CPU only."""
import numpy as np
import pytest


def test_fft_matches_numpy(orc):
    rng = np.random.default_rng(0)
    for d, M in [(1, 64), (2, 16), (3, 8), (1, 12), (2, 6)]:
        x = rng.standard_normal(M ** d) + 1j * rng.standard_normal(M ** d)
        fwd = orc.fft(x, d, M, -1)
        bwd = orc.fft(x, d, M, +1)
        shape = (M,) * d
        ref_f = np.fft.fftn(x.reshape(shape)).ravel()
        ref_b = np.fft.ifftn(x.reshape(shape)).ravel() * M ** d
        assert np.max(np.abs(fwd - ref_f)) <= 1e-12 * np.max(np.abs(ref_f))
        assert np.max(np.abs(bwd - ref_b)) <= 1e-12 * np.max(np.abs(ref_b))


def test_frequency_index_set_enumerates_the_centered_cube(orc):
    # test_nfft.cpp:40-55
    assert orc.freq_component(1, 2, 0, 0) == -1
    assert orc.freq_component(1, 2, 1, 0) == 0
    assert orc.freq_component(3, 4, 0, 0) == -2
    assert orc.freq_component(3, 4, 0, 2) == -2
    assert orc.freq_component(3, 4, 1, 2) == -1
    assert orc.freq_component(3, 4, 16, 0) == -1
    assert orc.freq_component(3, 4, 63, 0) == 1
    assert orc.freq_component(3, 4, 63, 2) == 1


def test_direct_transform_reproduces_a_pure_exponential(orc):
    # test_nfft.cpp:57-72
    d, N = 2, 4
    nodes = orc.random_nodes(7, d, 11)
    for f in (0, 5, 15):
        fhat = np.zeros(N ** d, np.complex128)
        fhat[f] = 1.0
        out = orc.direct_ndft(d, N, nodes, fhat)
        comps = [orc.freq_component(d, N, f, t) for t in range(d)]
        expect = np.exp(2j * np.pi * (nodes @ np.array(comps, float)))
        assert np.max(np.abs(out - expect)) < 1e-14


def test_adjoint_oracle_at_the_origin_sums_plainly(orc):
    # test_nfft.cpp:74-81
    out = orc.direct_adjoint_ndft(1, 8, np.zeros((1, 1)), np.array([1.0 + 0j]))
    assert np.max(np.abs(out - 1.0)) < 1e-15


@pytest.mark.parametrize("x", [0.0, 0.3, 1.0, 4.0, 12.5, 25.0, 40.0])
def test_bessel_series_matches_standard_library(orc, x):
    # test_nfft.cpp:83-89 (std::cyl_bessel_i), plus scipy as a second witness
    import scipy.special
    mine = orc.bessel_i0(x)
    assert abs(mine - orc.std_bessel_i0(x)) <= 1e-12 * orc.std_bessel_i0(x)
    assert abs(mine - scipy.special.i0(x)) <= 1e-12 * scipy.special.i0(x)


@pytest.mark.parametrize("d", [1, 2, 3])
@pytest.mark.parametrize("N", [2, 4, 16])
def test_plan_matches_direct_transform_at_full_cutoff(orc, d, N):
    # test_nfft.cpp:91-111 (m = 8, budget 1e-12 * ||in||_1)
    n = 64 if d == 3 else 256
    nodes = orc.random_nodes(n, d, 100 * d + N)
    plan = orc.NfftPlan(d, N, 8, nodes)
    fhat = orc.random_coeffs(plan.coefficient_count, 7)
    fast = plan.forward(fhat)
    exact = orc.direct_ndft(d, N, nodes, fhat)
    assert np.max(np.abs(fast - exact)) <= 1e-12 * np.sum(np.abs(fhat))
    x = orc.random_coeffs(n, 13)
    fast_adj = plan.adjoint(x)
    exact_adj = orc.direct_adjoint_ndft(d, N, nodes, x)
    assert np.max(np.abs(fast_adj - exact_adj)) <= 1e-12 * np.sum(np.abs(x))


def test_forward_and_adjoint_are_exact_transposes(orc):
    # test_nfft.cpp:113-126
    d, N, n = 2, 16, 120
    nodes = orc.random_nodes(n, d, 21)
    plan = orc.NfftPlan(d, N, 4, nodes)
    fhat = orc.random_coeffs(plan.coefficient_count, 3)
    x = orc.random_coeffs(n, 5)
    lhs = np.vdot(x, plan.forward(fhat))
    rhs = np.vdot(plan.adjoint(x), fhat)
    assert abs(lhs - rhs) <= 1e-10 * (abs(lhs) + abs(rhs) + 1e-300)


def test_plan_is_linear_up_to_rounding(orc):
    # test_nfft.cpp:128-139
    nodes = orc.random_nodes(50, 1, 31)
    plan = orc.NfftPlan(1, 32, 6, nodes)
    f = orc.random_coeffs(plan.coefficient_count, 1)
    g = orc.random_coeffs(plan.coefficient_count, 2)
    a, b = complex(1.7, -0.3), complex(-0.2, 2.5)
    combined = plan.forward(a * f + b * g)
    split = a * plan.forward(f) + b * plan.forward(g)
    assert np.max(np.abs(combined - split)) <= 1e-12 * np.max(np.abs(combined))


def test_accuracy_improves_monotonically_with_cutoff(orc):
    # test_nfft.cpp:141-153
    d, N, n = 2, 16, 100
    nodes = orc.random_nodes(n, d, 77)
    fhat = orc.random_coeffs(N ** d, 9)
    exact = orc.direct_ndft(d, N, nodes, fhat)
    prev = np.inf
    for m in (2, 4, 8):
        err = np.max(np.abs(orc.NfftPlan(d, N, m, nodes).forward(fhat) - exact))
        assert err < prev
        prev = err


def test_equispaced_nodes_reduce_to_inverse_dft(orc):
    # test_nfft.cpp:155-170
    N = 16
    nodes = (np.arange(N) - N / 2)[:, None] / N
    plan = orc.NfftPlan(1, N, 8, nodes)
    fhat = orc.random_coeffs(N, 4)
    fast = plan.forward(fhat)
    l = np.arange(N) - N // 2
    for j in range(N):
        acc = np.sum(fhat * np.exp(2j * np.pi * l * nodes[j, 0]))
        assert abs(fast[j] - acc) <= 1e-12 * np.sum(np.abs(fhat))


def test_real_part_convenience_honors_conjugate_symmetry(orc):
    # test_nfft.cpp:172-191
    N, n = 8, 40
    nodes = orc.random_nodes(n, 1, 55)
    plan = orc.NfftPlan(1, N, 8, nodes)
    rng = np.random.default_rng(8)
    fhat = np.zeros(N, np.complex128)
    for l in range(1, N // 2):
        c = complex(rng.standard_normal(), rng.standard_normal())
        fhat[N // 2 + l] = c
        fhat[N // 2 - l] = np.conj(c)
    fhat[N // 2] = rng.standard_normal()
    re = plan.forward_real(fhat)
    full = plan.forward(fhat)
    assert np.max(np.abs(re - full.real)) == 0.0
    assert np.max(np.abs(full.imag)) <= 1e-10 * np.max(np.abs(full.real))


def test_invalid_inputs_are_rejected(orc):
    # test_nfft.cpp:193-208
    good = orc.random_nodes(4, 2, 1)
    with pytest.raises(orc.OracleError) as e:
        orc.NfftPlan(4, 8, 4, np.zeros((2, 4)))
    assert e.value.kind == "ParameterError"
    for args, kind in [((2, 7, 4, good), "ParameterError"), ((2, 8, 0, good), "ParameterError")]:
        with pytest.raises(orc.OracleError) as e:
            orc.NfftPlan(*args)
        assert e.value.kind == kind
    with pytest.raises(orc.OracleError) as e:
        orc.NfftPlan(2, 8, 4, good, 0.5)
    assert e.value.kind == "ParameterError"
    bad = good.copy()
    bad[1, 0] = 0.5
    with pytest.raises(orc.OracleError) as e:
        orc.NfftPlan(2, 8, 4, bad)
    assert e.value.kind == "RangeError"
    plan = orc.NfftPlan(2, 8, 4, good)
    with pytest.raises(orc.OracleError) as e:
        plan.forward(np.zeros(63, np.complex128))
    assert e.value.kind == "ShapeError"
    with pytest.raises(orc.OracleError) as e:
        plan.adjoint(np.zeros(3, np.complex128))
    assert e.value.kind == "ShapeError"


def test_acceptance_nfft_oracle_agreement(orc):
    # acceptance.cpp:218-252: d in 1..3, N in {4, 8, 16}, m = 8
    worst_f = worst_a = worst_p = 0.0
    for d in (1, 2, 3):
        for N in (4, 8, 16):
            n = 128 if d == 3 else 256
            nodes = orc.random_nodes(n, d, 100 * d + N)
            plan = orc.NfftPlan(d, N, 8, nodes)
            fhat = orc.random_coeffs(plan.coefficient_count, 7)
            x = orc.random_coeffs(n, 13)
            fwd = plan.forward(fhat)
            adj = plan.adjoint(x)
            worst_f = max(worst_f, np.max(np.abs(fwd - orc.direct_ndft(d, N, nodes, fhat))) / np.sum(np.abs(fhat)))
            worst_a = max(worst_a, np.max(np.abs(adj - orc.direct_adjoint_ndft(d, N, nodes, x))) / np.sum(np.abs(x)))
            lhs, rhs = np.vdot(x, fwd), np.vdot(adj, fhat)
            worst_p = max(worst_p, abs(lhs - rhs) / (abs(lhs) + abs(rhs) + 1e-300))
    assert worst_f <= 1e-12 and worst_a <= 1e-12 and worst_p <= 1e-10
