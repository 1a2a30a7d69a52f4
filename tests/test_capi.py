"""CPU-side checks of the product boundary: the C-ABI library builds, loads
and exports every symbol include/fgs_b200.h declares; host-only entry points
(presets, I0 series, workload generators) behave; and without a GPU the
product fails loudly instead of falling back to the CPU."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import paper_1808_04580_b200 as fgs

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    src = open(os.path.join(ROOT, "include", "fgs_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(fgs_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = fgs.lib()
    names = _declared_symbols()
    assert len(names) >= 30
    missing = [s for s in names if not hasattr(lib, s)]
    assert not missing, missing


def test_library_is_built_for_sm_100a():
    out = os.popen(f"/usr/local/cuda/bin/cuobjdump --list-elf {fgs.LIB_PATH} 2>&1").read()
    assert "sm_100a" in out


def test_presets_follow_the_documented_ladder():
    # test_fastsum.cpp:42-55
    p1 = fgs.FastsumParams.preset(1)
    assert (p1.bandwidth, p1.cutoff, p1.smoothness) == (16, 2, 2)
    p2 = fgs.FastsumParams.preset(2, 0.125)
    assert (p2.bandwidth, p2.cutoff, p2.eps_b) == (32, 4, 0.125)
    assert fgs.FastsumParams.preset(3).cutoff == 7
    with pytest.raises(fgs.ParameterError):
        fgs.FastsumParams.preset(0)


def test_bessel_series_matches_oracle(orc):
    for x in (0.0, 0.3, 1.0, 4.0, 12.5, 25.0, 40.0):
        assert fgs.bessel_i0(x) == orc.bessel_i0(x)


@pytest.mark.parametrize("config", [1, 2, 3, 4])
def test_workload_generators_match_baseline_shapes(config):
    info = fgs.workload_info(config)
    expect = {1: (20000, 3), 2: (100000, 2), 3: (480000, 3), 4: (2000000, 3)}[config]
    assert (info["n"], info["d"]) == expect
    X = fgs.workload_nodes(config, seed=7)
    assert X.shape == expect
    r = np.linalg.norm(X, axis=1)
    if config == 1:
        assert r.max() <= 0.2
    if config == 3:
        assert X.min() >= 0 and X.max() <= 255 and np.all(X == np.round(X))
    if config == 4:
        assert abs(r.max() - 0.25) < 1e-12
    # seeded: identical on regeneration
    assert np.array_equal(X, fgs.workload_nodes(config, seed=7))


def test_workload_vectors_are_seeded_normal():
    v = fgs.workload_vectors(10000, 3, 5)
    assert v.shape == (10000, 3)
    assert abs(v.mean()) < 0.05 and abs(v.std() - 1) < 0.05
    assert np.array_equal(v, fgs.workload_vectors(10000, 3, 5))


def test_no_gpu_means_a_loud_failure_not_a_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    nodes = np.random.default_rng(0).uniform(-0.2, 0.2, (50, 2))
    with pytest.raises((fgs.CudaError, fgs.ResourceError)):
        fgs.FastsumPlan(nodes, fgs.KernelSpec.gaussian(1.0))


def test_cpp_dropin_layer_compiles_against_the_header():
    import __graft_entry__ as g
    exe = g.build_cpp_dropin_test()
    assert os.path.exists(exe)


@pytest.mark.parametrize("eigen", [False, True])
def test_cpp_dropin_header_builds(eigen):
    # include/fgs/b200.hpp with the reference's solve_pairs call site
    # (commands.cpp:171-188) compiles and links, in its plain and its
    # Eigen-typed mode (the latter against oracle/shim's Eigen stand-in)
    import __graft_entry__ as g
    exe = g.build_cpp_dropin_test(eigen=eigen)
    assert os.path.exists(exe)
