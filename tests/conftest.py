"""Shared pytest setup: repo root on sys.path, the `gpu` marker, and helpers."""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running CPU oracle case")


@pytest.fixture(scope="session")
def orc():
    from oracle import oracle as o
    o.build()
    return o


def approx(a, b, eps):
    """doctest::Approx semantics: |a-b| < eps * (scale(=1) + max(|a|, |b|))."""
    return abs(a - b) < eps * (1.0 + max(abs(a), abs(b)))
