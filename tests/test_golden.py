"""Golden fixtures (tests/golden/golden.npz, made by tests/golden/make_golden.py
from the pinned CPU oracle): the oracle must reproduce them exactly (CPU), and
the B200 path must match them at the north-star tolerances (GPU)."""
import os

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "golden.npz")


@pytest.fixture(scope="module")
def gold():
    return dict(np.load(GOLD))


def test_oracle_reproduces_golden_fixtures(orc, gold):
    for d in (1, 2, 3):
        for m in (4, 8):
            key = f"nfft_d{d}_m{m}"
            plan = orc.NfftPlan(d, 8, m, gold[key + "_nodes"])
            assert np.array_equal(plan.forward(gold[key + "_fhat"]), gold[key + "_forward"])
            assert np.array_equal(plan.adjoint(gold[key + "_x"]), gold[key + "_adjoint"])
    for d in (3, 2):
        key = f"graph_d{d}"
        sigma, N, m = gold[key + "_params"]
        op = orc.AdjacencyOperator(gold[key + "_nodes"], 0, sigma, N=int(N), m=int(m), p=int(m))
        assert np.array_equal(op.apply_normalized(gold[key + "_x"]), gold[key + "_normalized"])
        assert np.array_equal(op.degrees(), gold[key + "_degrees"])


@pytest.mark.gpu
def test_b200_matches_golden_fixtures(gold):
    import paper_1808_04580_b200 as fgs

    def rel(a, b):
        return np.linalg.norm(a - b) / np.linalg.norm(b)

    for d in (1, 2, 3):
        for m in (4, 8):
            key = f"nfft_d{d}_m{m}"
            plan = fgs.NfftPlan(d, 8, m, gold[key + "_nodes"])
            assert rel(plan.forward(gold[key + "_fhat"]), gold[key + "_forward"]) <= 1e-13
            assert rel(plan.adjoint(gold[key + "_x"]), gold[key + "_adjoint"]) <= 1e-13
    for d in (3, 2):
        key = f"graph_d{d}"
        sigma, N, m = gold[key + "_params"]
        op = fgs.AdjacencyOperator(gold[key + "_nodes"], fgs.KernelSpec.gaussian(sigma),
                                   fgs.FastsumParams(int(N), int(m), int(m)))
        assert rel(op.degrees(), gold[key + "_degrees"]) <= 1e-10
        assert rel(op.apply_normalized(gold[key + "_x"]), gold[key + "_normalized"]) <= 1e-10
        assert rel(op.apply_sym_laplacian(gold[key + "_x"]), gold[key + "_laplacian"]) <= 1e-10
        pairs = fgs.lanczos_largest(op, 4, fgs.LanczosOptions(tol=1e-10))
        assert np.max(np.abs(pairs.values - gold[key + "_lanczos_values"])) <= 1e-8
